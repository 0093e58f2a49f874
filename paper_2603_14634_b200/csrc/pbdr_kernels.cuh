// Device kernels of the PBD-R substep loop (sm_100a). See pbdr_kernels.cu.
#pragma once
#include <string>

#include <cuda_runtime.h>
#include <stdint.h>

#include "pbdr_pinned.h"

namespace pbdr_dev {

struct Planes {
  int count;
  float p[PBDR_MAX_PLANES][3];
  float n[PBDR_MAX_PLANES][3];
  float mu[PBDR_MAX_PLANES];
};

// Device error record: bits (atomicOr), first body (atomicMin), first substep
// (atomicMin), null axis of the first rank-deficient body.
struct DevError {
  unsigned bits;
  int body;
  long long substep;
  double axis[3];
};

struct BodyProgram {  // ForceProgram (scene.hpp:53-61), fp32 force/torque + window
  float fx, fy, fz;
  int flags;  // bit0: has program, bit1: gravity exempt, bit2: nonzero torque
  float tx, ty, tz;
  int pad;
  double t_start, t_stop;
};

// distribute_wrench (body.cpp:126-150) on the device: per body with a torque
// program, the com c and inertia I of X at the substep start (anchored fp32
// tree sums, parallel axis) and alpha = pinv(I) tau; integrate then adds
// alpha x (x - c) to the acceleration.
struct WrenchArgs {
  const float4* pos;
  const float4* vel;  // .w = mass
  const float4* anchor;
  const int4* cta_desc;
  const int4* warp_desc;
  const float2* body_mass;
  const int4* body_desc;
  const BodyProgram* programs;
  float4* wcom;    // per body: com (xyz)
  float4* walpha;  // per body: alpha (xyz)
  DevError* err;
  const long long* substep_counter;
  const int* big_list;  // k_body_wrench_big: one CTA per listed body
};

struct IntegrateArgs {
  float4* pos;         // in: X (substep start), out: X~ (predicted)
  float4* vel;         // in: V, out: V~
  float4* init;        // out: X_init
  const int* body_of;
  const int* body_scene;
  const BodyProgram* programs;  // per body
  const float2* body_mass;      // (M, 1/M)
  uint32_t* key_all;  // [n] cell key of every particle (slot order)
  const float4* wcom;    // torque programs: per-body com and alpha (or null)
  const float4* walpha;
  uint32_t* box_min;  // per body 3 x order-preserving uint of the min corner of X~
  uint32_t* box_max;
  const long long* substep_counter;
  const uint8_t* role;  // slab mode: per-body role (0 inactive, 1 ghost, 2 owned), else null
  int has_programs;     // 0: no body has a ForceProgram (gravity only)
  int64_t p0;           // first slot of the launch range (slab mode: active range)
  int64_t n;            // end of the launch range
  float dt, gravity, inv_h;
  double dt_d;
  uint32_t mask;
  pbdr_key_layout layout;  // bucket keys (pbdr_cell_key)
};

// Body broadphase (acceleration only; the candidate set is unchanged): a
// particle can have a candidate only inside the h-inflated box of another body
// of its scene, and only such body pairs are partners.
struct BroadArgs {
  const uint32_t* box_min;
  const uint32_t* box_max;
  const int* body_scene;
  uint32_t* bkeys;     // [nb] coarse-cell key of each body's box centre
  uint32_t* bvals;     // [nb] body index
  const uint32_t* sorted_bkeys;
  const uint32_t* sorted_bvals;
  uint2* bcells;       // coarse bucket -> (start, end) in the sorted body array
  int* npartners;      // [nb], -1 = overflow (search every particle of the body)
  int* partners;       // [nb * PBDR_PARTNER_CAP]
  unsigned* oversize;  // set when a body box exceeds max_extent (disables the skip)
  const int* list;     // slab mode: the active bodies (ascending), else null (all bodies)
  const int2* scene_range;  // per body: (first body, bodies) of its scene (k_scene_partners)
  int nb;              // bodies in the list (all bodies when list is null)
  float inv_cell;      // 1 / coarse cell
  float max_extent;    // coarse cell - inflation: the largest box the grid guarantees
  float inflate;       // h, slightly enlarged
  uint32_t mask;
};

// Broadphase filter: only particles inside the h-inflated box of a partner
// body can have contact candidates (see k_near_flag); they are compacted, in
// slot order, into the list that the hash grid is built from.
struct NearArgs {
  const float4* pos;  // X~
  const int4* body_desc;  // (first slot, n, ...) per body (whole-scene packing)
  const uint32_t* box_min;
  const uint32_t* box_max;
  const int* npartners;
  const int* partners;
  const uint32_t* key_all;
  const int* list;        // slab mode: active bodies (ascending), else null (all bodies)
  int nbl;                // bodies to process
  uint32_t* body_near;    // [nbl] near particles per body
  uint32_t* body_off;     // [nbl] exclusive offsets within the scan tile
  uint32_t* tile_sum;     // [ceil(nbl / 4096)] scan tile totals
  uint32_t* tile_off;     // [ceil(nbl / 4096)] scan tile offsets
  long long* count;       // total near particles (device)
  uint32_t* keys_c;       // compacted keys  (sort input)
  uint32_t* vals_c;       // compacted slots (sort input)
  int* near_list;         // compacted slots (slot order)
  const uint8_t* role;    // slab mode: inactive bodies' particles are never near
  int all_near;           // broadphase off: every active particle is near
  float inflate;
  // Oriented boxes (optional, null = axis-aligned test only): per body the
  // frame (unit quaternion from the warm-start rotation, centre = anchor) and
  // the bounds of its X~ in that frame, built by k_body_obb for every body
  // with partners; a particle is near only if it is also inside a partner's
  // h-inflated oriented box.
  const float4* rquat;    // warm-start rotation per body (0 = none: identity frame)
  const float4* anchor;
  float4* obb_q;          // [nb] unit quaternion of the frame
  float4* obb_c;          // [nb] centre
  float4* obb_lo;         // [nb] bounds in the frame
  float4* obb_hi;
  uint8_t* near_flag;     // [n] per particle of bodies with partners: the count kernel's test result
};

struct RangesArgs {
  const uint32_t* keys;  // sorted
  const uint32_t* vals;  // sorted slots
  const long long* count;    // number of sorted entries (device)
  long long* prev_count;     // saved for the next substep's table clear
  const int* body_of;
  uint4* cells;  // per bucket (start, end, first body, last body); start = ~0 when empty
  const float4* pos;     // X~
  float4* sorted_pos;    // X~ of every sorted entry, its body's index in .w (int bits)
  long long* substep_counter;
  int64_t n;
};

struct NeighbourArgs {
  const float4* pos;  // X~
  const int* near_list;
  const long long* count;
  const float4* rest;
  const int* body_of;
  const int* body_scene;
  const uint4* cells;
  const uint32_t* sorted_vals;
  const float4* sorted_pos;  // X~ of the sorted entries, body in .w (k_cell_ranges)
  int single_scene;          // every body in scene 0: no scene test per entry
  int* ncand;
  int* cand_j;     // slot-major: [k * n + i]
  float* cand_rr;  // slot-major
  DevError* err;
  const long long* substep_counter;
  int64_t n;
  float inv_h, h2;
  uint32_t mask;
  pbdr_key_layout layout;
};

struct IterArgs {
  const float4* pos_in;  // X_i snapshot (also gathered for neighbours)
  float4* pos_out;       // X_{i+1}
  float4* vel;           // V_i -> V_{i+1} (own particles only)
  const float4* rest;    // (q0, radius)
  const float4* init;    // X_init
  const int* ncand;
  const int* cand_j;
  const float* cand_rr;
  float4* anchor;        // per body (xyz)
  float4* rquat;         // per body warm-start rotation (w, x, y, z), 0 = none
  const int4* cta_desc;  // per CTA: (first slot, slot count, first body, body count)
  const int4* warp_desc; // per CTA warp: (body, warp in body, body start, n | W << 16); body -1 = idle
  const int4* body_desc; // (start, n, W, first warp in CTA)
  const float2* body_mass;
  DevError* err;
  const long long* substep_counter;
  int64_t n;
  Planes planes;
  float dt, inv_dt, relax;
  int incremental, linfix, angfix;
  int per_substep;    // MomentumFrequency::kPerSubstep
  int iter_index;     // iteration within the substep
  int n_iters;        // iterations run by this launch (> 1: scenes without pairs, or one-wave cooperative)
  int multi_pairs;    // n_iters > 1 with contact pairs: 1 = cooperative launch, grid barrier per
                      // iteration; 2 = one cluster per batched scene, cluster barrier per iteration
  int cluster;        // multi_pairs == 2: CTAs (tiles) per scene cluster
  const int* tile_list;   // optional: claim c processes tile tile_list[c] ...
  const int* tile_count;  // ... of a device-side count (isolated / contact tiles), else null
  int fuse_integrate; // multi-iteration launch: the final writeback also integrates the next
                      // substep (writes X~, V~, X_init, cell keys, body boxes) with `ia`
  IntegrateArgs ia;
  float4* pos_b[2];   // multi_pairs: the two position buffers (pos_in, pos_out) alternated per iteration
  int last_iter;      // iteration_index == solver_iterations - 1
  float4* mom_acc;    // per body (P, L) accumulators for kPerSubstep
  long long* timing;  // optional per-CTA phase clocks (debug), else null
  int ntiles;         // packed CTAs (tiles) of this launch; set by launch_iteration
  int* tile_ctr;      // [2] tile claim counter and finished-CTA counter (self-resetting, zero at create)
  const int* big_list;  // bodies of more than one CTA (k_iteration_big, one cluster each)
};

struct ClassifyArgs {
  const int4* cta_desc;   // tiles of the iteration packing
  const int* npartners;   // per body (-1: overflow, searched in full)
  int* iso_list;          // tiles whose bodies all have no partner
  int* contact_list;      // the other tiles
  const int4* warp_desc;  // descriptors of the packing, copied in list order:
  int4* iso_cd;           // iso_cd[c] = cta_desc[iso_list[c]], iso_wd[8 c + w] likewise, so the
  int4* iso_wd;           // iteration kernel reads a claim's descriptors without the list
  int4* contact_cd;       // indirection (one dependent load less at every tile start)
  int4* contact_wd;
  int* counts;            // [2] sizes of the two lists (zeroed before the launch)
  int ntiles;
};

struct StatsArgs {
  const float4* pos;
  const float4* vel;
  const float4* rest;
  const float4* anchor;
  const int4* cta_desc;
  const int4* warp_desc;
  const int4* body_desc;
  const float2* body_mass;
  double* out;  // 13 doubles per body: com[3], quat[4], P[3], L[3]
  const int* big_list;  // k_body_stats_big: one CTA per listed body
};

void launch_integrate(const IntegrateArgs& a, cudaStream_t s);
void launch_body_keys(const BroadArgs& a, cudaStream_t s);
void launch_body_ranges(const BroadArgs& a, cudaStream_t s);
void launch_body_partners(const BroadArgs& a, cudaStream_t s);
void launch_scene_partners(const BroadArgs& a, cudaStream_t s);
void launch_classify_tiles(const ClassifyArgs& a, cudaStream_t s);  // batched scenes (scene_range)
void launch_gather4(float4* dst, const float4* src, const int* idx, int64_t count, cudaStream_t s);
void launch_scatter4(float4* dst, const float4* src, const int* idx, int64_t count, cudaStream_t s);
void launch_near(const NearArgs& a, cudaStream_t s);
void launch_tick(long long* substep_counter, cudaStream_t s);
void launch_particles_in(float4* pos, float4* vel, const double* x, const double* v, const int* slot_particle,
                         int64_t n, cudaStream_t s);
void launch_particles_out(const float4* pos, const float4* vel, double* x, double* v, const int* slot_particle,
                          int64_t n, cudaStream_t s);
void launch_anchor_reset(float4* anchor, const int4* body_desc, const float4* pos, int nb, cudaStream_t s);
void launch_ncand_clear(int* ncand, const int* prev_near, const long long* prev_count, int64_t n_max,
                        cudaStream_t s);
void launch_cell_clear(uint4* cells, const uint32_t* prev_keys, const long long* prev_count, int64_t n_max,
                       cudaStream_t s);
void launch_ranges(const RangesArgs& a, cudaStream_t s);
void launch_neighbours(const NeighbourArgs& a, cudaStream_t s);
size_t iteration_smem_bytes(int kp);
cudaError_t prepare_iteration_kernel();
std::string checked_failure();  // checked build: the device check that failed, else empty
void launch_iteration(const IterArgs& a, int ctas, int kp, cudaStream_t s);
int iteration_coop_capacity(int kp);  // CTAs a cooperative multi-iteration launch may use
int iteration_scene_clusters(int kp, int cluster);  // resident scene clusters of `cluster` CTAs (0: none)
void launch_stats(const StatsArgs& a, int ctas, int kp, cudaStream_t s);
void launch_wrench(const WrenchArgs& a, int ctas, int kp, cudaStream_t s);

// Bodies larger than one iteration CTA (pbdr_body_warps(n, 8) > 8 warps, up to
// PBDR_MAX_BODY_PARTICLES_BIG particles): one thread-block cluster of
// `cluster` CTAs per body (k_iteration_big), and one looping CTA per body for
// the per-frame statistics and the torque prepass.
int big_cluster_size(int max_warps);              // CTAs per cluster for bodies of up to max_warps warps
int big_cta_warps(int max_warps, int cluster);    // warps per CTA (spread evenly over the cluster)
cudaError_t big_cluster_check(int cluster, int warps);  // cudaSuccess if such clusters can be resident
void launch_iteration_big(const IterArgs& a, int nbig, int cluster, int warps, cudaStream_t s);
void launch_stats_big(const StatsArgs& a, int nbig, cudaStream_t s);
void launch_wrench_big(const WrenchArgs& a, int nbig, cudaStream_t s);

}  // namespace pbdr_dev
