// Internal: the handle behind the C-ABI (include/pbdr_gpu.h) and the engine
// entry points the native slab driver (pbdr_slab.cu) builds on. Not installed.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "pbdr_gpu.h"
#include "pbdr_internal.h"
#include "pbdr_kernels.cuh"

namespace pbdr_engine {
struct SlabDriver;
void slab_driver_destroy(SlabDriver* d);
}  // namespace pbdr_engine

using pbdr_dev::BodyProgram;
using pbdr_dev::DevError;

struct pbdr_handle {
  int device = 0;
  int sm_count = 0;
  cudaStream_t stream = nullptr;
  int64_t n = 0;
  int32_t nb = 0;
  std::vector<int64_t> slot_to_particle;

  float4* pos[2] = {nullptr, nullptr};
  float4* vel = nullptr;
  float4* rest = nullptr;
  float4* init = nullptr;
  int* body_of = nullptr;
  int* body_scene = nullptr;
  BodyProgram* programs = nullptr;
  float2* body_mass = nullptr;
  int4* body_desc = nullptr;
  int4* warp_desc = nullptr;
  int4* cta_desc = nullptr;
  float4* anchor = nullptr;
  float4* rquat = nullptr;
  float4* mom_acc = nullptr;
  float4* wcom = nullptr;    // torque programs: per-body com and alpha
  float4* walpha = nullptr;
  bool has_torque = false;
  bool has_programs = false;  // any body with a ForceProgram
  bool pairs_possible = true; // some scene holds two or more bodies
  bool coop_iters = true;     // one-wave scenes with pairs: cooperative multi-iteration launch
  float4* sorted_pos = nullptr;  // X~ in sorted (cell-key) order, for the neighbour search
  uint8_t* near_flag = nullptr;  // near-filter test per particle (count pass -> write pass)
  float4* obb_q = nullptr;       // oriented near-filter boxes per body (null: PBDR_OBB=0)
  float4* obb_c = nullptr;
  float4* obb_lo = nullptr;
  float4* obb_hi = nullptr;
  bool single_scene = false;     // every body in scene 0
  int2* scene_range = nullptr;  // per body (first body, bodies) of its scene when scenes are contiguous
                                // runs of <= PBDR_PARTNER_CAP bodies (k_scene_partners), else null
  int scene_cluster = 0;      // batched scenes of equal tile count C <= 8: one C-CTA cluster per scene
                              // runs all iterations of a substep in one launch (0: not applicable)
  bool cluster_iters = true;  // use scene_cluster when available (PBDR_CLUSTER_ITERS=0 disables)
  bool fuse_integrate = true; // scene clusters integrate the next substep (PBDR_FUSE_INTEGRATE=0 disables)
  bool split_iso = true;      // isolated tiles iterate in one launch (PBDR_SPLIT_ISOLATED=0 disables)
  int* iso_list = nullptr;    // [ctas] isolated tiles of the current substep
  int* contact_list = nullptr;  // [ctas] the other tiles
  int* tile_counts = nullptr;   // [2] sizes of the two lists (device)
  int4* list_cd[2] = {nullptr, nullptr};  // tile / warp descriptors copied in list order (isolated,
  int4* list_wd[2] = {nullptr, nullptr};  // contact) by k_classify_tiles; PBDR_COMPACT_DESC=0 disables
  bool broadphase = true;     // body-box filter before the hash grid (PBDR_BROADPHASE=0 disables)
  int kp = 4;                 // tile shape: particles per lane (pbdr_choose_kp)
  int launch_kp = 4;          // instantiation the tiles run on (kp, or 7 for one-warp bodies at kp 8)
  bool kp7 = true;            // PBDR_KP7=0 keeps the KP = 8 instantiation
  int per_substep = 0;
  int debug_iter = 0;  // iteration index for the replay hook
  uint32_t* keys[2] = {nullptr, nullptr};
  uint32_t* vals[2] = {nullptr, nullptr};
  void* sort_temp = nullptr;
  uint4* cells = nullptr;
  // broadphase-filtered particle list
  uint32_t* key_all = nullptr;
  uint32_t* body_near = nullptr;   // [2 * nb]: near particles per body, scan offsets
  uint32_t* scan_tiles = nullptr;  // [2 * tiles]: tile totals, tile offsets
  long long* near_count = nullptr;  // [0] current, [1] previous substep
  int* near_list = nullptr;
  int near_blocks = 0;
  // body broadphase
  uint32_t* box_min = nullptr;
  uint32_t* box_max = nullptr;
  uint32_t* bkeys[2] = {nullptr, nullptr};
  uint32_t* bvals[2] = {nullptr, nullptr};
  void* bsort_temp = nullptr;
  uint2* bcells = nullptr;
  int* npartners = nullptr;
  int* partners = nullptr;
  unsigned* oversize = nullptr;
  int bhash_bits = 10;
  int bpasses = 2;
  uint32_t bmask = 0;
  float inv_cell_b = 0, max_extent = 0, inflate = 0;
  long long* timing = nullptr;      // set only while an instrumented launch is enqueued
  long long* timing_buf = nullptr;  // per-CTA phase clocks (debug hook only)
  int* ncand = nullptr;
  int* cand_j = nullptr;
  float* cand_rr = nullptr;
  DevError* err = nullptr;
  long long* counter = nullptr;
  int* tile_ctr = nullptr;  // iteration kernel: dynamic tile claims (self-resetting)
  int* big_list = nullptr;  // bodies larger than one CTA (ascending ids)
  double* stats = nullptr;
  double* xfer = nullptr;        // fp64 staging of pbdr_gpu_read/write_particles (6 n, lazy)
  int* slot_particle = nullptr;  // device copy of slot_to_particle (lazy)
  std::vector<void*> allocations;
  size_t device_bytes = 0;

  int cur = 0;         // pos buffer holding the current state
  int sorted_buf = 0;  // keys/vals buffer holding the last sorted pairs
  int ctas = 0;
  int hash_bits = 10;
  pbdr_key_layout key_layout{};  // bucket keys (pbdr_choose_key_layout)
  int passes = 2;
  uint32_t mask = 0;
  float dt = 0, inv_dt = 0, gravity = 0, relax = 1, h = 0, inv_h = 0, h2 = 0;
  double dt_d = 0;
  int iters = 10, substeps = 10;
  int incremental = 1, linfix = 1, angfix = 1;
  pbdr_dev::Planes planes{};

  // Iteration CTA packing (cta_desc / warp_desc / body_desc triples). `full` is
  // the create-time packing of every body; in slab mode `iter` packs the owned
  // bodies and `active` the owned + ghost bodies (torque prepass).
  struct Packing {
    int4* cta = nullptr;
    int4* warp = nullptr;
    int4* body = nullptr;
    int ctas = 0;
    int* big = nullptr;  // bodies larger than one CTA (one cluster each)
    int nbig = 0;
  };
  Packing pk_full, pk_iter, pk_active;
  std::vector<int64_t> h_bstart;  // host copy: first slot of each body
  std::vector<int> h_bcount;      // host copy: particles of each body
  std::vector<int> h_bscene;      // host copy: scene of each body
  int big_cluster = 0;            // CTAs per cluster of the big-body kernel (0: no big body)
  int big_warps = 0;              // warps per CTA of the big-body kernel

  // Slab mode (x-slab decomposition of one scene, pbdr_gpu_set_roles).
  bool slab = false;
  uint8_t* role = nullptr;     // [nb] 0 inactive, 1 ghost, 2 owned
  int* active_list = nullptr;  // [nb] ascending ids of owned + ghost bodies
  int n_active = 0;
  int64_t p_lo = 0, p_hi = 0;  // slot range covering the active bodies
  Packing slab_iter, slab_active;  // device storage (capacity nb CTAs)
  int stage_iter = 0;

  // Trajectory emission: per frame, per owned body, the 13-double
  // sample of pbdr_body_stats into a device ring drained by the host.
  double* traj = nullptr;
  int64_t traj_cap = 0;      // frames the ring holds
  int64_t traj_pending = 0;  // frames written since the last drain
  std::vector<double> traj_t;  // time stamp of each pending frame

  // x-slab decomposition driven natively (pbdr_gpu_slab_*, csrc/pbdr_slab.cu):
  // host copy of the owned-body tile descriptors of the current roles.
  std::vector<int4> h_iter_cdesc;
  pbdr_engine::SlabDriver* slab_driver = nullptr;

  cudaGraphExec_t graph[2] = {nullptr, nullptr};
  int graph_end[2] = {0, 0};
  int64_t substeps_done = 0;
  int64_t launches_per_frame = 0;
};


namespace pbdr_engine {
// Wrappers over the engine's internal stages (pbdr_engine.cu).
int cuda_fail(cudaError_t e, const char* what);
int device_alloc(pbdr_handle* h, void** ptr, size_t bytes);
void enqueue_substep(pbdr_handle* h);  // integrate, hash grid, candidates
// One iteration over the tiles of a device-side list (or every tile: list =
// count = null). Does not flip the position buffers: the caller does, once per
// iteration (h->cur ^= 1), so that several lists can run the same iteration.
void enqueue_iteration_tiles(pbdr_handle* h, int iter_index, const int* list, const int* count);
void enqueue_body_stats(pbdr_handle* h, double* out);
int check_errors(pbdr_handle* h);
}  // namespace pbdr_engine
