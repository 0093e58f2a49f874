// Host orchestration + C-ABI implementation (include/pbdr_gpu.h).
//
// Replaces the missing reference solver (proj/src/solver.cpp, CMakeLists.txt:20)
// behind the scene/step API of proj/include/pbdr/scene.hpp:17-82. One handle =
// one scene on one device and one stream. Device state is float4 SoA in
// body-major order (bodies own contiguous particle ranges); a frame is captured
// once into a CUDA graph and replayed.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "pbdr_gpu.h"
#include "pbdr_internal.h"
#include "pbdr_kernels.cuh"
#include "pbdr_pinned.h"
#include "pbdr_sort.cuh"

#include "pbdr_handle.h"

namespace {

using pbdr_host::set_config_error;
using pbdr_host::set_error;

int cuda_fail(cudaError_t e, const char* what) {
  return set_error(PBDR_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e) + pbdr_dev::checked_failure());
}

#define PBDR_CUDA(call)                                   \
  do {                                                    \
    cudaError_t e_ = (call);                              \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);   \
  } while (0)

template <typename T>
int dalloc(pbdr_handle* h, T** ptr, size_t count) {
  void* p = nullptr;
  const size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc");
  h->allocations.push_back(p);
  h->device_bytes += bytes;
  *ptr = static_cast<T*>(p);
  return PBDR_OK;
}

void release(pbdr_handle* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->slab_driver) pbdr_engine::slab_driver_destroy(h->slab_driver);
  for (auto& g : h->graph)
    if (g) cudaGraphExecDestroy(g);
  for (void* p : h->allocations) cudaFree(p);
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
}

struct EventHook final : pbdr_dev::LaunchHook {
  cudaStream_t stream;
  float ms[PBDR_KCLASS_COUNT] = {0};
  int64_t launches[PBDR_KCLASS_COUNT] = {0};
  cudaEvent_t a = nullptr, b = nullptr;
  int cls = 0;
  explicit EventHook(cudaStream_t s) : stream(s) {
    cudaEventCreate(&a);
    cudaEventCreate(&b);
  }
  ~EventHook() override {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
  void before(int c) override {
    cls = c;
    cudaEventRecord(a, stream);
  }
  void after(int c, int nl) override {
    cudaEventRecord(b, stream);
    cudaEventSynchronize(b);
    float t = 0;
    cudaEventElapsedTime(&t, a, b);
    ms[c] += t;
    launches[c] += nl;
  }
};

// Enqueues one substep (integrate .. iterations) on h->stream.
// Batched scenes of few bodies find partners per scene (no body sort).
bool scene_partners(const pbdr_handle* h) { return h->scene_range != nullptr && !h->slab; }

void reset_boxes(pbdr_handle* h) {
  cudaMemsetAsync(h->box_min, 0xFF, sizeof(uint32_t) * 3 * h->nb, h->stream);
  cudaMemsetAsync(h->box_max, 0x00, sizeof(uint32_t) * 3 * h->nb, h->stream);
}

pbdr_dev::IntegrateArgs integrate_args(const pbdr_handle* h) {
  using namespace pbdr_dev;
  IntegrateArgs ia{};
  ia.pos = h->pos[h->cur];
  ia.vel = h->vel;
  ia.init = h->init;
  ia.body_of = h->body_of;
  ia.body_scene = h->body_scene;
  ia.programs = h->programs;
  ia.body_mass = h->body_mass;
  ia.key_all = h->key_all;
  ia.wcom = h->wcom;
  ia.walpha = h->walpha;
  ia.box_min = h->box_min;
  ia.box_max = h->box_max;
  ia.substep_counter = h->counter;
  ia.role = h->slab ? h->role : nullptr;
  ia.has_programs = h->has_programs ? 1 : 0;
  ia.p0 = h->p_lo;
  ia.n = h->p_hi;
  ia.dt = h->dt;
  ia.gravity = h->gravity;
  ia.inv_h = h->inv_h;
  ia.dt_d = h->dt_d;
  ia.mask = h->mask;
  ia.layout = h->key_layout;
  return ia;
}

// `integrated`: the previous substep's scene-cluster launch already ran this
// substep's integrate (and reset and filled the body boxes).
void enqueue_substep(pbdr_handle* h, pbdr_dev::LaunchHook* hook, bool integrated = false) {
  using namespace pbdr_dev;
  const IntegrateArgs ia = integrate_args(h);
  const bool pairs = h->pairs_possible || h->slab;
  if (pairs) {
    if (hook) hook->before(kHookMemset);
    if (!integrated) reset_boxes(h);
    cudaMemsetAsync(h->oversize, 0x00, sizeof(unsigned), h->stream);
    if (!scene_partners(h))
      cudaMemsetAsync(h->bcells, 0xFF, sizeof(uint2) * (size_t(1) << h->bhash_bits), h->stream);
    if (hook) hook->after(kHookMemset, (integrated ? 1 : 3) + (scene_partners(h) ? 0 : 1));
    // Reset only the buckets the previous substep filled.
    if (hook) hook->before(kHookRanges);
    launch_cell_clear(h->cells, h->keys[h->sorted_buf], h->near_count + 1, h->n, h->stream);
    launch_ncand_clear(h->ncand, h->near_list, h->near_count + 1, h->n, h->stream);
    if (hook) hook->after(kHookRanges);
  }
  if (h->has_torque) {
    WrenchArgs wa{};
    wa.pos = h->pos[h->cur];
    wa.vel = h->vel;
    wa.anchor = h->anchor;
    wa.cta_desc = h->pk_active.cta;
    wa.warp_desc = h->pk_active.warp;
    wa.body_mass = h->body_mass;
    wa.body_desc = h->pk_active.body;
    wa.programs = h->programs;
    wa.wcom = h->wcom;
    wa.walpha = h->walpha;
    wa.err = h->err;
    wa.substep_counter = h->counter;
    if (hook) hook->before(kHookIntegrate);
    wa.big_list = h->pk_active.big;
    if (h->pk_active.ctas > 0) launch_wrench(wa, h->pk_active.ctas, h->launch_kp, h->stream);
    if (h->pk_active.nbig > 0) launch_wrench_big(wa, h->pk_active.nbig, h->stream);
    if (hook) hook->after(kHookIntegrate, (h->pk_active.ctas > 0 ? 1 : 0) + (h->pk_active.nbig > 0 ? 1 : 0));
  }
  if (!integrated) {
    if (hook) hook->before(kHookIntegrate);
    launch_integrate(ia, h->stream);
    if (hook) hook->after(kHookIntegrate);
  }

  if (!pairs) {
    // Every scene holds a single body: no particle can have a contact
    // candidate (candidates are other bodies of the same scene), so the hash
    // grid is skipped; candidate counts stay 0 from creation. Only the substep
    // counter advances, as k_cell_ranges would.
    if (hook) hook->before(kHookRanges);
    launch_tick(h->counter, h->stream);
    if (hook) hook->after(kHookRanges);
    return;
  }

  // Body broadphase: partner bodies (box overlap within h) for the skip test.
  BroadArgs ba{};
  ba.box_min = h->box_min;
  ba.box_max = h->box_max;
  ba.body_scene = h->body_scene;
  ba.bkeys = h->bkeys[0];
  ba.bvals = h->bvals[0];
  ba.bcells = h->bcells;
  ba.npartners = h->npartners;
  ba.partners = h->partners;
  ba.oversize = h->oversize;
  ba.list = h->slab ? h->active_list : nullptr;
  ba.nb = h->slab ? h->n_active : h->nb;
  ba.inv_cell = h->inv_cell_b;
  ba.max_extent = h->max_extent;
  ba.inflate = h->inflate;
  ba.mask = h->bmask;
  ba.scene_range = h->scene_range;
  if (h->broadphase && scene_partners(h)) {
    if (hook) hook->before(kHookBroadphase);
    launch_scene_partners(ba, h->stream);
    if (hook) hook->after(kHookBroadphase);
  } else if (h->broadphase) {
    if (hook) hook->before(kHookBroadphase);
    launch_body_keys(ba, h->stream);
    if (hook) hook->after(kHookBroadphase);
    const int bsb = sort_pairs(h->bkeys, h->bvals, ba.nb, h->bhash_bits, h->bsort_temp, h->sm_count,
                               h->stream, hook);
    ba.sorted_bkeys = h->bkeys[bsb];
    ba.sorted_bvals = h->bvals[bsb];
    if (hook) hook->before(kHookBroadphase);
    launch_body_ranges(ba, h->stream);
    launch_body_partners(ba, h->stream);
    if (hook) hook->after(kHookBroadphase, 2);
  }

  // Broadphase filter: compact the near particles (slot order) into the sort input.
  NearArgs nr{};
  nr.pos = h->pos[h->cur];
  nr.body_desc = h->pk_full.body;
  nr.box_min = h->box_min;
  nr.box_max = h->box_max;
  nr.npartners = h->npartners;
  nr.partners = h->partners;
  nr.key_all = h->key_all;
  nr.list = h->slab ? h->active_list : nullptr;
  nr.nbl = h->slab ? h->n_active : h->nb;
  nr.body_near = h->body_near;
  nr.body_off = h->body_near + h->nb;
  nr.tile_sum = h->scan_tiles;
  nr.tile_off = h->scan_tiles + (h->nb + 4095) / 4096 + 1;
  nr.count = h->near_count;
  nr.keys_c = h->keys[0];
  nr.vals_c = h->vals[0];
  nr.near_list = h->near_list;
  nr.role = h->slab ? h->role : nullptr;
  nr.all_near = h->broadphase ? 0 : 1;
  nr.inflate = h->inflate;
  nr.near_flag = h->near_flag;
  // Oriented boxes pay off in large piles; batched small scenes keep the
  // axis-aligned test (their per-scene partners are few and contacts sparse).
  const bool obb = h->obb_q && !scene_partners(h);
  if (obb) {
    nr.rquat = h->rquat;
    nr.anchor = h->anchor;
    nr.obb_q = h->obb_q;
    nr.obb_c = h->obb_c;
    nr.obb_lo = h->obb_lo;
    nr.obb_hi = h->obb_hi;
  }
  if (hook) hook->before(kHookBroadphase);
  launch_near(nr, h->stream);
  if (hook) hook->after(kHookBroadphase, ((obb && h->broadphase) ? 5 : 4) + ((nr.nbl > 0 && nr.nbl < (1 << 16)) ? 1 : 0));

  const int sb = sort_pairs(h->keys, h->vals, h->n, h->hash_bits, h->sort_temp, h->sm_count,
                            h->stream, hook, h->near_count);
  h->sorted_buf = sb;

  RangesArgs ra{};
  ra.keys = h->keys[sb];
  ra.vals = h->vals[sb];
  ra.count = h->near_count;
  ra.prev_count = h->near_count + 1;
  ra.body_of = h->body_of;
  ra.cells = h->cells;
  ra.pos = h->pos[h->cur];
  ra.sorted_pos = h->sorted_pos;
  ra.substep_counter = h->counter;
  ra.n = h->n;
  if (hook) hook->before(kHookRanges);
  launch_ranges(ra, h->stream);
  if (hook) hook->after(kHookRanges);

  NeighbourArgs na{};
  na.pos = h->pos[h->cur];
  na.near_list = h->near_list;
  na.count = h->near_count;
  na.rest = h->rest;
  na.body_of = h->body_of;
  na.body_scene = h->body_scene;
  na.cells = h->cells;
  na.sorted_vals = h->vals[sb];
  na.sorted_pos = h->sorted_pos;
  na.single_scene = h->single_scene ? 1 : 0;
  na.ncand = h->ncand;
  na.cand_j = h->cand_j;
  na.cand_rr = h->cand_rr;
  na.err = h->err;
  na.substep_counter = h->counter;
  na.n = h->n;
  na.inv_h = h->inv_h;
  na.h2 = h->h2;
  na.mask = h->mask;
  na.layout = h->key_layout;
  if (hook) hook->before(kHookNeighbours);
  launch_neighbours(na, h->stream);
  if (hook) hook->after(kHookNeighbours);
}

// Batched scenes iterate in one launch per substep, one cluster per scene.
bool use_scene_clusters(const pbdr_handle* h) {
  return h->scene_cluster > 0 && h->cluster_iters && !h->slab && !h->timing;
}

// `list`/`count`: iterate only the tiles of a device-side list (the contact
// tiles of this substep) instead of every tile.
void enqueue_iteration(pbdr_handle* h, int iter_index, pbdr_dev::LaunchHook* hook, int n_iters = 1,
                       bool fuse_integrate = false, const int* list = nullptr, const int* count = nullptr) {
  using namespace pbdr_dev;
  IterArgs it{};
  it.tile_list = list;
  it.tile_count = count;
  it.pos_in = h->pos[h->cur];
  it.pos_out = h->pos[h->cur ^ 1];
  it.vel = h->vel;
  it.rest = h->rest;
  it.init = h->init;
  it.ncand = h->ncand;
  it.cand_j = h->cand_j;
  it.cand_rr = h->cand_rr;
  it.anchor = h->anchor;
  it.rquat = h->rquat;
  it.per_substep = h->per_substep;
  it.iter_index = iter_index;
  it.n_iters = n_iters;
  const bool isolated = n_iters > 1 && list != nullptr;  // enqueue_isolated
  it.multi_pairs = (n_iters > 1 && h->pairs_possible && !isolated) ? (use_scene_clusters(h) ? 2 : 1) : 0;
  if (isolated) it.pos_out = h->pos[h->cur ^ (n_iters & 1)];
  it.cluster = it.multi_pairs == 2 ? h->scene_cluster : 1;
  it.fuse_integrate = fuse_integrate ? 1 : 0;
  if (fuse_integrate) it.ia = integrate_args(h);
  it.pos_b[0] = h->pos[h->cur];
  it.pos_b[1] = h->pos[h->cur ^ 1];
  it.last_iter = iter_index + n_iters - 1 == h->iters - 1;
  it.mom_acc = h->mom_acc;
  it.cta_desc = h->pk_iter.cta;
  it.warp_desc = h->pk_iter.warp;
  // The isolated / contact lists of this substep come with their descriptors
  // copied in list order: claim c reads entry c directly.
  for (int l = 0; l < 2; ++l)
    if (list != nullptr && list == (l == 0 ? h->iso_list : h->contact_list) && h->list_cd[l] != nullptr &&
        !h->timing) {
      it.cta_desc = h->list_cd[l];
      it.warp_desc = h->list_wd[l];
      it.tile_list = nullptr;
    }
  it.body_desc = h->pk_iter.body;
  it.body_mass = h->body_mass;
  it.err = h->err;
  it.substep_counter = h->counter;
  it.n = h->n;
  it.planes = h->planes;
  it.dt = h->dt;
  it.inv_dt = h->inv_dt;
  it.relax = h->relax;
  it.incremental = h->incremental;
  it.linfix = h->linfix;
  it.angfix = h->angfix;
  it.timing = h->timing;
  it.tile_ctr = h->tile_ctr;
  it.big_list = h->pk_iter.big;
  if (hook) hook->before(kHookIteration);
  if (h->pk_iter.ctas > 0) launch_iteration(it, h->pk_iter.ctas, h->launch_kp, h->stream);
  // Bodies larger than one CTA: one cluster each, same iteration semantics
  // (they read pos_in and write pos_out / vel of their own slots only).
  const bool big = h->pk_iter.nbig > 0 && !isolated;
  if (big) launch_iteration_big(it, h->pk_iter.nbig, h->big_cluster, h->big_warps, h->stream);
  if (hook) hook->after(kHookIteration, (h->pk_iter.ctas > 0 ? 1 : 0) + (big ? 1 : 0));
  h->cur ^= 1;
}

// Isolated tiles (no body with a partner this substep) iterate all of the
// substep's iterations in one launch, state in shared memory; the contact
// tiles then iterate launch by launch. Both write only their own slots and no
// contact tile gathers a particle of an isolated one (pairs are symmetric),
// so the split changes no result. The isolated launch leaves its final state
// in the buffer the contact launches end in (they flip it per iteration).
void enqueue_isolated(pbdr_handle* h, pbdr_dev::LaunchHook* hook, bool fuse_integrate) {
  using namespace pbdr_dev;
  if (hook) hook->before(kHookMemset);
  cudaMemsetAsync(h->tile_counts, 0, 2 * sizeof(int), h->stream);
  if (hook) hook->after(kHookMemset);
  ClassifyArgs ca{};
  ca.cta_desc = h->pk_iter.cta;
  ca.npartners = h->npartners;
  ca.iso_list = h->iso_list;
  ca.contact_list = h->contact_list;
  ca.counts = h->tile_counts;
  ca.ntiles = h->pk_iter.ctas;
  ca.warp_desc = h->pk_iter.warp;
  ca.iso_cd = h->list_cd[0];
  ca.iso_wd = h->list_wd[0];
  ca.contact_cd = h->list_cd[1];
  ca.contact_wd = h->list_wd[1];
  if (hook) hook->before(kHookBroadphase);
  launch_classify_tiles(ca, h->stream);
  if (hook) hook->after(kHookBroadphase);
  const int cur = h->cur;
  enqueue_iteration(h, 0, hook, h->iters, fuse_integrate, h->iso_list, h->tile_counts);
  h->cur = cur;
}

bool split_isolated(const pbdr_handle* h) {
  return h->split_iso && !h->slab && h->pairs_possible && h->broadphase && h->pk_iter.ctas > 0 &&
         h->iso_list != nullptr;
}

// The launch that ends a substep also integrates the next substep of the same
// call (its final writeback has X and V in hand). Torque programs need the
// k_body_wrench prepass between the substeps; cluster bodies have their own
// launch; slab ranks integrate ghosts too.
bool fuse_next_integrate(const pbdr_handle* h) {
  return h->fuse_integrate && !h->has_torque && !h->slab && h->pairs_possible && h->pk_iter.nbig == 0 &&
         h->pk_iter.ctas > 0;
}

bool fused_iterations(const pbdr_handle* h) {
  return !h->slab && (!h->pairs_possible || use_scene_clusters(h) ||
                      (h->pk_iter.ctas <= pbdr_dev::iteration_coop_capacity(h->launch_kp) && h->coop_iters &&
                       h->pk_iter.nbig == 0));
}

void enqueue_substeps(pbdr_handle* h, int64_t count, pbdr_dev::LaunchHook* hook) {
  // Without candidate pairs a body's iterations only read its own particles:
  // one launch runs all of them (state kept in shared memory). With pairs, a
  // scene whose tiles fit in one wave does the same in a cooperative launch
  // with a grid barrier between iterations (small latency-bound scenes) --
  // unless it has bodies larger than one CTA, whose cluster launch is separate.
  const bool fused_iters = fused_iterations(h);
  bool integrated = false;
  for (int64_t s = 0; s < count; ++s) {
    enqueue_substep(h, hook, integrated);
    // The substep's last launch integrates the next substep of this call in
    // its final writeback (never across calls: a call leaves X, not X~).
    const bool fuse = fuse_next_integrate(h) && s + 1 < count;
    if (fuse) {
      if (hook) hook->before(pbdr_dev::kHookMemset);
      reset_boxes(h);  // after this substep's broadphase consumed them
      if (hook) hook->after(pbdr_dev::kHookMemset, 2);
    }
    if (fused_iters) {
      enqueue_iteration(h, 0, hook, h->iters, fuse);
    } else if (split_isolated(h)) {
      enqueue_isolated(h, hook, fuse);
      for (int i = 0; i < h->iters; ++i)
        enqueue_iteration(h, i, hook, 1, fuse && i + 1 == h->iters, h->contact_list, h->tile_counts + 1);
    } else {
      for (int i = 0; i < h->iters; ++i) enqueue_iteration(h, i, hook, 1, fuse && i + 1 == h->iters);
    }
    integrated = fuse;
  }
}

// Reads the device error record; maps it to a status (errors.hpp classes).
int check_errors(pbdr_handle* h) {
  cudaError_t e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return cuda_fail(e, "kernel execution");
  DevError de{};
  e = cudaMemcpy(&de, h->err, sizeof de, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "error readback");
  if (de.bits == 0u) return PBDR_OK;
  // Errors are recorded after the substep counter advanced (cell_ranges).
  const int64_t substep = de.substep - 1;
  const int64_t frame = substep / std::max(1, h->substeps);
  // Causes before consequences: a non-finite state also makes the polar
  // degenerate, so it is reported as the SimulationError it is.
  if (de.bits & PBDR_DEVERR_NONFINITE)
    return pbdr_host::set_sim_error("non-finite body sums", frame, de.body, nullptr, PBDR_ERR_SIMULATION);
  if (de.bits & PBDR_DEVERR_NBR_OVERFLOW)
    return pbdr_host::set_sim_error("contact candidates exceed capacity " +
                                        std::to_string(PBDR_NBR_CAP) + " per particle",
                                    frame, de.body, nullptr, PBDR_ERR_SIMULATION);
  if (de.bits & PBDR_DEVERR_RANK_DEFICIENT)
    return pbdr_host::set_sim_error("angular momentum fix: dL along a singular inertia axis",
                                    frame, de.body, de.axis, PBDR_ERR_RANK_DEFICIENT);
  if (de.bits & PBDR_DEVERR_DEGENERATE)
    return pbdr_host::set_sim_error("shape matching: polar decomposition of a degenerate moment",
                                    frame, de.body, nullptr, PBDR_ERR_DEGENERATE);
  return pbdr_host::set_sim_error("non-finite body sums", frame, de.body, nullptr,
                                  PBDR_ERR_SIMULATION);
}

int reset_errors(pbdr_handle* h) {
  DevError de{};
  de.bits = 0u;
  de.body = 0x7FFFFFFF;
  de.substep = 0x7FFFFFFFFFFFFFFFll;
  PBDR_CUDA(cudaMemcpyAsync(h->err, &de, sizeof de, cudaMemcpyHostToDevice, h->stream));
  PBDR_CUDA(cudaStreamSynchronize(h->stream));
  return PBDR_OK;
}

int build_graph(pbdr_handle* h, int parity) {
  const int saved = h->cur;
  h->cur = parity;
  PBDR_CUDA(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
  enqueue_substeps(h, h->substeps, nullptr);
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(h->stream, &g);
  h->graph_end[parity] = h->cur;
  h->cur = saved;
  if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
  e = cudaGraphInstantiate(&h->graph[parity], g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate");
  return PBDR_OK;
}

// Packs bodies (ascending ids) into 8-warp CTAs: a body of n particles takes
// W = ceil(n/(32 kp)) warps; consecutive ids (slot-contiguous in the body-major
// layout) of one scene share a CTA while its warps last (a tile never spans
// two batched scenes, so a scene is a run of whole tiles). Bodies of more than 8 warps go to
// `big` (one CTA cluster each). bdesc[b] = (first slot, n, W, first warp in the
// CTA; 0 for big bodies) is written for the listed bodies only.
void pack_bodies(const std::vector<int>& list, const std::vector<int64_t>& bstart, const std::vector<int>& bcount,
                 const std::vector<int>& bscene, int kp, std::vector<int4>& cdesc, std::vector<int4>& wdesc,
                 std::vector<int4>& bdesc, std::vector<int>& big) {
  cdesc.clear();
  wdesc.clear();
  big.clear();
  int used = 0, prev = -2;
  auto close = [&] {
    for (; used < PBDR_CTA_WARPS && used > 0; ++used) wdesc.push_back(make_int4(-1, 0, 0, 1 << 16));
    used = 0;
  };
  for (const int b : list) {
    const int cnt = bcount[b];
    const int first_slot = static_cast<int>(bstart[b]);
    const int W = pbdr_body_warps(cnt, kp);
    if (W > PBDR_CTA_WARPS) {
      bdesc[b] = make_int4(first_slot, cnt, W, 0);
      big.push_back(b);
      continue;
    }
    if (used + W > PBDR_CTA_WARPS || (used > 0 && (b != prev + 1 || bscene[b] != bscene[prev]))) close();
    if (used == 0) cdesc.push_back(make_int4(first_slot, 0, b, 0));
    cdesc.back().y += cnt;
    cdesc.back().w += 1;
    bdesc[b] = make_int4(first_slot, cnt, W, used);
    for (int u = 0; u < W; ++u) wdesc.push_back(make_int4(b, u, first_slot, cnt | (W << 16)));
    used += W;
    prev = b;
  }
  close();
}

int validate(const pbdr_scene_desc* d, const pbdr_solver_cfg* c) {
  if (!d || !c) return set_config_error("scene", "null descriptor");
  if (c->precision != PBDR_PRECISION_SINGLE)
    return set_config_error("precision",
                            "the B200 path computes in single precision (kSingle); "
                            "kDouble has no device implementation and there is no CPU fallback");
  if (!(c->frame_rate > 0.0) || !std::isfinite(c->frame_rate))
    return set_config_error("frame_rate", "must be > 0");
  if (c->substeps < 1) return set_config_error("substeps", "must be >= 1");
  if (c->solver_iterations < 1) return set_config_error("solver_iterations", "must be >= 1");
  if (!std::isfinite(c->gravity)) return set_config_error("gravity", "must be finite");
  if (c->momentum_frequency != PBDR_MOMENTUM_PER_ITERATION &&
      c->momentum_frequency != PBDR_MOMENTUM_PER_SUBSTEP)
    return set_config_error("momentum_frequency", "unknown value");
  if (c->velocity_update != PBDR_VELOCITY_LEGACY && c->velocity_update != PBDR_VELOCITY_INCREMENTAL)
    return set_config_error("velocity_update", "unknown mode");
  if (d->num_particles <= 0) return set_config_error("particles", "scene has no particles");
  if (d->num_particles >= (int64_t(1) << 31) - 1)
    return set_config_error("particles", "more than 2^31-2 particles per device");
  if (d->num_bodies <= 0) return set_config_error("bodies", "scene has no bodies");
  if (d->num_bodies > 4 * 1024 * 1024)  // near-filter body scan: <= 1024 tiles of 4096
    return set_config_error("bodies", "more than 4,194,304 bodies per device");
  if (!(d->contact_relaxation >= 0.0)) return set_config_error("contact_relaxation", "must be >= 0");
  const int planes = (d->has_ground ? 1 : 0) + std::max(0, d->num_walls);
  if (planes > PBDR_MAX_PLANES) return set_config_error("walls", "at most 8 planes (ground + walls)");
  return PBDR_OK;
}

}  // namespace

extern "C" {

int pbdr_gpu_create(const pbdr_scene_desc* d, const pbdr_solver_cfg* c, int device,
                    pbdr_handle** out) {
  if (!out) return set_error(PBDR_ERR_GENERIC, "null output handle");
  *out = nullptr;
  pbdr_host::clear_error();
  int st = validate(d, c);
  if (st != PBDR_OK) return st;

  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return set_error(PBDR_ERR_CUDA, "no CUDA device available (the PBD-R path has no CPU fallback)");
  if (device < 0 || device >= ndev) return set_config_error("device", "out of range");
  PBDR_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop{};
  PBDR_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10 || prop.minor != 0)
    return set_error(PBDR_ERR_CUDA, "this build targets sm_100a (B200); device is sm_" +
                                        std::to_string(prop.major) + std::to_string(prop.minor));

  pbdr_handle* h = new pbdr_handle();
  h->device = device;
  h->sm_count = prop.multiProcessorCount;
  h->n = d->num_particles;
  h->nb = d->num_bodies;
  const int64_t n = h->n;
  const int32_t nb = h->nb;

  // ---- Body-major layout (host) ---------------------------------------------
  std::vector<float4> pos(n), vel(n), rest(n);
  std::vector<int> body_of(n), scene(nb, 0);
  std::vector<BodyProgram> prog(nb);
  std::vector<float2> mass(nb);
  std::vector<float4> anchor(nb);
  std::vector<int4> bdesc(nb);
  std::vector<int4> wdesc;
  std::vector<int4> cdesc;
  std::vector<int> big;
  std::vector<char> seen(n, 0);
  h->slot_to_particle.resize(n);
  h->h_bstart.assign(nb, 0);
  h->h_bcount.assign(nb, 0);
  h->h_bscene.assign(nb, 0);
  double rmax = 0.0;
  int64_t slot = 0;
  for (int32_t b = 0; b < nb; ++b) {
    const int64_t k0 = d->body_offsets[b], k1 = d->body_offsets[b + 1];
    const int64_t cnt = k1 - k0;
    if (cnt <= 0) {
      release(h);
      return set_config_error("bodies.particle_indices", "empty body " + std::to_string(b));
    }
    if (cnt > PBDR_MAX_BODY_PARTICLES_BIG) {
      release(h);
      return set_config_error("bodies.particle_indices",
                              "body " + std::to_string(b) + " has " + std::to_string(cnt) +
                                  " particles; a body is processed by at most one " +
                                  std::to_string(PBDR_MAX_CLUSTER_CTAS) + "-CTA cluster (" +
                                  std::to_string(PBDR_MAX_BODY_PARTICLES_BIG) + " particles)");
    }
    const int64_t first_slot = slot;
    for (int64_t k = k0; k < k1; ++k, ++slot) {
      const int64_t i = d->body_indices[k];
      if (i < 0 || i >= n || seen[i]) {
        release(h);
        return set_config_error("bodies.particle_indices", "particle missing or in two bodies");
      }
      seen[i] = 1;
      if (!(d->inv_mass[i] > 0.0)) {
        release(h);
        return set_error(PBDR_ERR_GENERIC, "pinned particles are not supported in rigid bodies");
      }
      h->slot_to_particle[slot] = i;
      pos[slot] = make_float4(static_cast<float>(d->position[3 * i]), static_cast<float>(d->position[3 * i + 1]),
                              static_cast<float>(d->position[3 * i + 2]), static_cast<float>(d->inv_mass[i]));
      vel[slot] = make_float4(static_cast<float>(d->velocity[3 * i]), static_cast<float>(d->velocity[3 * i + 1]),
                              static_cast<float>(d->velocity[3 * i + 2]),
                              static_cast<float>(1.0 / d->inv_mass[i]));
      rest[slot] = make_float4(static_cast<float>(d->rest_offsets[3 * k]),
                               static_cast<float>(d->rest_offsets[3 * k + 1]),
                               static_cast<float>(d->rest_offsets[3 * k + 2]),
                               static_cast<float>(d->radius[i]));
      body_of[slot] = b;
      rmax = std::max(rmax, d->radius[i]);
    }
    h->h_bstart[b] = first_slot;
    h->h_bcount[b] = static_cast<int>(cnt);
    mass[b] = make_float2(static_cast<float>(d->total_mass[b]), static_cast<float>(1.0 / d->total_mass[b]));
    anchor[b] = make_float4(pos[first_slot].x, pos[first_slot].y, pos[first_slot].z, 0.0f);
    scene[b] = d->body_scene ? d->body_scene[b] : 0;
    h->h_bscene[b] = scene[b];
    BodyProgram bp{};
    if (d->programs) {
      const pbdr_force_program& p = d->programs[b];
      bp.fx = static_cast<float>(p.force[0]);
      bp.fy = static_cast<float>(p.force[1]);
      bp.fz = static_cast<float>(p.force[2]);
      bp.tx = static_cast<float>(p.torque[0]);
      bp.ty = static_cast<float>(p.torque[1]);
      bp.tz = static_cast<float>(p.torque[2]);
      const bool torque = p.torque[0] != 0.0 || p.torque[1] != 0.0 || p.torque[2] != 0.0;
      bp.flags = 1 | (p.gravity_exempt ? 2 : 0) | (torque ? 4 : 0);
      h->has_programs = true;
      h->has_torque = h->has_torque || torque;
      bp.t_start = p.t_start;
      bp.t_stop = p.t_stop;
    }
    prog[b] = bp;
  }
  if (slot != n) {
    release(h);
    return set_config_error("bodies.particle_indices", "every particle must belong to one body");
  }
  {
    std::vector<int> all(nb);
    for (int32_t b = 0; b < nb; ++b) all[b] = b;
    int max_body = 0;
    for (int32_t b = 0; b < nb; ++b) max_body = std::max(max_body, h->h_bcount[b]);
    h->kp = pbdr_choose_kp(n, nb, max_body, d->tile_kp);
    if (const char* e = std::getenv("PBDR_KP7")) h->kp7 = std::atoi(e) != 0;
    // Bodies of at most 7 * 32 particles at KP = 8 each take one warp whose
    // lanes hold at most 7 particles: the KP = 7 instantiation runs the same
    // tiles with the same trees (W = 1 either way) without the empty eighth
    // row (fewer registers and instructions). The tile shape reported and
    // used by the oracle stays 8.
    h->launch_kp = (h->kp == 8 && max_body <= 7 * 32 && h->kp7) ? 7 : h->kp;
    pack_bodies(all, h->h_bstart, h->h_bcount, h->h_bscene, h->kp, cdesc, wdesc, bdesc, big);
    if (!big.empty()) {
      const int wmax = pbdr_body_warps(max_body, h->kp);
      h->big_cluster = pbdr_dev::big_cluster_size(wmax);
      h->big_warps = pbdr_dev::big_cta_warps(wmax, h->big_cluster);
    }
  }
  h->ctas = static_cast<int>(wdesc.size() / PBDR_CTA_WARPS);
  h->p_lo = 0;
  h->p_hi = n;

  // ---- Parameters ----------------------------------------------------------
  h->substeps = c->substeps;
  h->iters = c->solver_iterations;
  h->dt_d = 1.0 / (c->frame_rate * c->substeps);
  h->dt = static_cast<float>(h->dt_d);
  h->inv_dt = static_cast<float>(c->frame_rate * c->substeps);
  h->gravity = static_cast<float>(c->gravity);
  h->relax = static_cast<float>(d->contact_relaxation);
  h->incremental = c->velocity_update == PBDR_VELOCITY_INCREMENTAL;
  h->linfix = c->linear_momentum_fix != 0;
  h->angfix = c->angular_momentum_fix != 0;
  h->per_substep = c->momentum_frequency == PBDR_MOMENTUM_PER_SUBSTEP;
  h->h = static_cast<float>(2.0 * rmax);
  h->inv_h = 1.0f / h->h;
  h->h2 = h->h * h->h;
  h->bhash_bits = pbdr_hash_bits(nb);
  h->bpasses = (h->bhash_bits + 7) / 8;
  h->bmask = static_cast<uint32_t>((uint64_t(1) << h->bhash_bits) - 1u);
  {
    float qmax = 0.0f;
    for (int64_t k = 0; k < n; ++k)
      qmax = std::max(qmax, std::sqrt(rest[k].x * rest[k].x + rest[k].y * rest[k].y + rest[k].z * rest[k].z));
    h->inflate = 1.01f * h->h;
    h->max_extent = 2.2f * qmax + 2.0f * h->h;
    h->inv_cell_b = 1.0f / (h->max_extent + 2.0f * h->h);
  }
  {
    // Bucket keys: spatially ordered for single scenes that fit (pinned
    // pbdr_choose_key_layout, from the fp32 positions the oracle also starts from).
    bool single = true;
    for (int32_t b = 0; b < nb && single; ++b) single = scene[b] == 0;
    int32_t cmin[3] = {INT32_MAX, INT32_MAX, INT32_MAX}, cmax[3] = {INT32_MIN, INT32_MIN, INT32_MIN};
    for (int64_t k = 0; k < n; ++k) {
      const int32_t c[3] = {pbdr_cell_coord(pos[k].x, h->inv_h), pbdr_cell_coord(pos[k].y, h->inv_h),
                            pbdr_cell_coord(pos[k].z, h->inv_h)};
      for (int a = 0; a < 3; ++a) {
        cmin[a] = std::min(cmin[a], c[a]);
        cmax[a] = std::max(cmax[a], c[a]);
      }
    }
    h->key_layout = pbdr_choose_key_layout(single ? 1 : 0, cmin, cmax, n);
    if (const char* e = std::getenv("PBDR_LINEAR_KEYS"))
      if (std::atoi(e) == 0) h->key_layout = pbdr_choose_key_layout(0, cmin, cmax, n);
  }
  h->hash_bits = h->key_layout.bits;
  h->passes = (h->hash_bits + 7) / 8;
  h->mask = static_cast<uint32_t>((uint64_t(1) << h->hash_bits) - 1u);
  auto add_plane = [&](const pbdr_plane& p) {
    const int k = h->planes.count++;
    for (int c2 = 0; c2 < 3; ++c2) {
      h->planes.p[k][c2] = static_cast<float>(p.point[c2]);
      h->planes.n[k][c2] = static_cast<float>(p.normal[c2]);
    }
    h->planes.mu[k] = static_cast<float>(p.friction);
  };
  if (d->has_ground) add_plane(d->ground);
  for (int w = 0; w < d->num_walls; ++w) add_plane(d->walls[w]);

  // ---- Device buffers ------------------------------------------------------
  const size_t T = size_t(1) << h->hash_bits;
  int rc = PBDR_OK;
  rc |= dalloc(h, &h->pos[0], n);
  rc |= dalloc(h, &h->pos[1], n);
  rc |= dalloc(h, &h->vel, n);
  rc |= dalloc(h, &h->rest, n);
  rc |= dalloc(h, &h->init, n);
  rc |= dalloc(h, &h->body_of, n);
  rc |= dalloc(h, &h->body_scene, nb);
  rc |= dalloc(h, &h->programs, nb);
  rc |= dalloc(h, &h->body_mass, nb);
  rc |= dalloc(h, &h->body_desc, nb);
  rc |= dalloc(h, &h->warp_desc, wdesc.size());
  rc |= dalloc(h, &h->cta_desc, cdesc.size());
  rc |= dalloc(h, &h->anchor, nb);
  rc |= dalloc(h, &h->rquat, nb);
  rc |= dalloc(h, &h->mom_acc, 2 * static_cast<size_t>(nb));
  rc |= dalloc(h, &h->wcom, nb);
  rc |= dalloc(h, &h->walpha, nb);
  rc |= dalloc(h, &h->keys[0], n);
  rc |= dalloc(h, &h->keys[1], n);
  rc |= dalloc(h, &h->vals[0], n);
  rc |= dalloc(h, &h->vals[1], n);
  {
    char* tmp = nullptr;
    rc |= dalloc(h, &tmp, pbdr_dev::sort_temp_bytes(n, h->passes));
    h->sort_temp = tmp;
  }
  rc |= dalloc(h, &h->cells, T);
  h->near_blocks = static_cast<int>((n + 255) / 256);
  rc |= dalloc(h, &h->key_all, n);
  rc |= dalloc(h, &h->body_near, 2 * static_cast<size_t>(nb));
  rc |= dalloc(h, &h->scan_tiles, 2 * (static_cast<size_t>(nb + 4095) / 4096 + 1));
  rc |= dalloc(h, &h->near_count, 2);
  rc |= dalloc(h, &h->near_list, n);
  rc |= dalloc(h, &h->box_min, 3 * static_cast<size_t>(nb));
  rc |= dalloc(h, &h->box_max, 3 * static_cast<size_t>(nb));
  rc |= dalloc(h, &h->bkeys[0], nb);
  rc |= dalloc(h, &h->bkeys[1], nb);
  rc |= dalloc(h, &h->bvals[0], nb);
  rc |= dalloc(h, &h->bvals[1], nb);
  {
    char* tmp = nullptr;
    rc |= dalloc(h, &tmp, pbdr_dev::sort_temp_bytes(nb, h->bpasses));
    h->bsort_temp = tmp;
  }
  rc |= dalloc(h, &h->bcells, size_t(1) << h->bhash_bits);
  rc |= dalloc(h, &h->npartners, nb);
  rc |= dalloc(h, &h->partners, static_cast<size_t>(nb) * PBDR_PARTNER_CAP);
  rc |= dalloc(h, &h->oversize, 1);
  rc |= dalloc(h, &h->sorted_pos, n);
  rc |= dalloc(h, &h->near_flag, n);
  {
    const char* e = std::getenv("PBDR_OBB");
    if (!e || std::atoi(e) != 0) {
      rc |= dalloc(h, &h->obb_q, nb);
      rc |= dalloc(h, &h->obb_c, nb);
      rc |= dalloc(h, &h->obb_lo, nb);
      rc |= dalloc(h, &h->obb_hi, nb);
    }
  }
  rc |= dalloc(h, &h->ncand, n);
  rc |= dalloc(h, &h->cand_j, static_cast<size_t>(n) * PBDR_NBR_CAP);
  rc |= dalloc(h, &h->cand_rr, static_cast<size_t>(n) * PBDR_NBR_CAP);
  rc |= dalloc(h, &h->err, 1);
  rc |= dalloc(h, &h->counter, 1);
  rc |= dalloc(h, &h->tile_ctr, 2);
  rc |= dalloc(h, &h->stats, static_cast<size_t>(nb) * 13);
  if (!big.empty()) rc |= dalloc(h, &h->big_list, big.size());
  if (rc != PBDR_OK) {
    const int code = pbdr_last_error_payload(nullptr, nullptr, nullptr);
    release(h);
    return code ? code : PBDR_ERR_CUDA;
  }
  e = pbdr_dev::prepare_iteration_kernel();
  if (e != cudaSuccess) {
    release(h);
    return cuda_fail(e, "cudaFuncSetAttribute(k_iteration)");
  }
  if (h->big_cluster > 0) {
    e = pbdr_dev::big_cluster_check(h->big_cluster, h->big_warps);
    if (e != cudaSuccess) {
      release(h);
      return set_config_error("bodies.particle_indices",
                              "clusters of " + std::to_string(h->big_cluster) +
                                  " iteration CTAs cannot be resident on this device (" +
                                  cudaGetErrorString(e) + ")");
    }
  }
  e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    release(h);
    return cuda_fail(e, "cudaStreamCreate");
  }
#define UP(dst, src, count)                                                                   \
  e = cudaMemcpy(dst, src, sizeof(*(src)) * (count), cudaMemcpyHostToDevice);                 \
  if (e != cudaSuccess) {                                                                     \
    release(h);                                                                               \
    return cuda_fail(e, "upload " #dst);                                                      \
  }
  UP(h->pos[0], pos.data(), n);
  UP(h->vel, vel.data(), n);
  UP(h->rest, rest.data(), n);
  UP(h->body_of, body_of.data(), n);
  UP(h->body_scene, scene.data(), nb);
  UP(h->programs, prog.data(), nb);
  UP(h->body_mass, mass.data(), nb);
  UP(h->body_desc, bdesc.data(), nb);
  UP(h->warp_desc, wdesc.data(), wdesc.size());
  UP(h->cta_desc, cdesc.data(), cdesc.size());
  UP(h->anchor, anchor.data(), nb);
  if (!big.empty()) UP(h->big_list, big.data(), big.size());
#undef UP
  {
    cudaError_t m = cudaMemset(h->init, 0, sizeof(float4) * n);
    if (m == cudaSuccess) m = cudaMemset(h->counter, 0, sizeof(long long));
    if (m == cudaSuccess) m = cudaMemset(h->tile_ctr, 0, 2 * sizeof(int));
    if (m == cudaSuccess) m = cudaMemset(h->ncand, 0, sizeof(int) * n);
    if (m == cudaSuccess) m = cudaMemset(h->cells, 0xFF, sizeof(uint4) * T);
    if (m == cudaSuccess) m = cudaMemset(h->near_count, 0, sizeof(long long) * 2);
    if (m == cudaSuccess) m = cudaMemset(h->rquat, 0, sizeof(float4) * nb);
    if (m != cudaSuccess) {
      release(h);
      return cuda_fail(m, "initialise device buffers");
    }
  }
  h->pk_full = {h->cta_desc, h->warp_desc, h->body_desc, h->ctas, h->big_list, static_cast<int>(big.size())};
  {
    // Contact candidates need two bodies of one scene (pinned P4).
    std::vector<int> per_scene;
    h->single_scene = true;
    for (int32_t b = 0; b < nb; ++b) h->single_scene = h->single_scene && scene[b] == 0;
    h->pairs_possible = false;
    for (int32_t b = 0; b < nb && !h->pairs_possible; ++b) {
      const int sc = scene[b];
      if (sc < 0) continue;
      if (static_cast<size_t>(sc) >= per_scene.size()) per_scene.resize(static_cast<size_t>(sc) + 1, 0);
      h->pairs_possible = ++per_scene[sc] > 1;
    }
  }
  if (const char* e = std::getenv("PBDR_BROADPHASE")) h->broadphase = std::atoi(e) != 0;
  if (const char* e = std::getenv("PBDR_COOP_ITERS")) h->coop_iters = std::atoi(e) != 0;
  if (const char* e = std::getenv("PBDR_CLUSTER_ITERS")) h->cluster_iters = std::atoi(e) != 0;
  if (const char* e = std::getenv("PBDR_FUSE_INTEGRATE")) h->fuse_integrate = std::atoi(e) != 0;
  if (const char* e = std::getenv("PBDR_SPLIT_ISOLATED")) h->split_iso = std::atoi(e) != 0;
  if (h->ctas > 0) {
    int rc2 = dalloc(h, &h->iso_list, static_cast<size_t>(h->ctas));
    rc2 |= dalloc(h, &h->contact_list, static_cast<size_t>(h->ctas));
    rc2 |= dalloc(h, &h->tile_counts, 2);
    bool compact = true;
    if (const char* e = std::getenv("PBDR_COMPACT_DESC")) compact = std::atoi(e) != 0;
    for (int l = 0; l < 2 && compact; ++l) {
      rc2 |= dalloc(h, &h->list_cd[l], static_cast<size_t>(h->ctas));
      rc2 |= dalloc(h, &h->list_wd[l], static_cast<size_t>(h->ctas) * PBDR_CTA_WARPS);
    }
    if (rc2 != PBDR_OK) {
      const int code = pbdr_last_error_payload(nullptr, nullptr, nullptr);
      release(h);
      return code ? code : PBDR_ERR_CUDA;
    }
  }
  if (h->pairs_possible && d->body_scene) {
    // Scenes as contiguous body runs of <= PBDR_PARTNER_CAP bodies: partners
    // are found per scene (k_scene_partners) instead of on the coarse grid.
    std::vector<int2> rng(nb);
    std::vector<char> seen;
    bool ok = true;
    for (int32_t b = 0; b < nb && ok;) {
      const int sc = scene[b];
      int32_t e = b;
      while (e < nb && scene[e] == sc) ++e;
      ok = sc >= 0 && e - b <= PBDR_PARTNER_CAP;
      if (ok) {
        if (static_cast<size_t>(sc) >= seen.size()) seen.resize(static_cast<size_t>(sc) + 1, 0);
        ok = !seen[sc];
        seen[sc] = 1;
      }
      for (int32_t i = b; i < e; ++i) rng[i] = make_int2(b, e - b);
      b = e;
    }
    if (ok) {
      void* p = nullptr;
      if (cudaMalloc(&p, sizeof(int2) * nb) == cudaSuccess) {
        h->allocations.push_back(p);
        h->scene_range = static_cast<int2*>(p);
        cudaMemcpy(h->scene_range, rng.data(), sizeof(int2) * nb, cudaMemcpyHostToDevice);
        h->device_bytes += sizeof(int2) * nb;
      }
    }
  }
  if (const char* e = std::getenv("PBDR_SCENE_PARTNERS"))
    if (std::atoi(e) == 0) h->scene_range = nullptr;
  if (h->pairs_possible && big.empty() && h->ctas > 0) {
    // Batched scenes as runs of whole tiles, every scene the same number C of
    // tiles (C <= 8, a portable cluster) and no scene in two runs: candidates
    // pair bodies of one scene only (P4), so a C-CTA cluster holds every
    // particle a scene's iterations read.
    std::vector<int> run_of_scene;
    int C = 0, run = 0;
    bool ok = true;
    for (int t = 0; t < h->ctas && ok; ++t) {
      const int b0 = cdesc[t].z, b1 = cdesc[t].z + cdesc[t].w - 1;
      const int sc = scene[b0];
      ok = sc >= 0 && scene[b1] == sc;
      if (!ok) break;
      if (t > 0 && scene[cdesc[t - 1].z] == sc) {
        ++run;
      } else {
        if (t > 0) ok = C == 0 ? (C = run, true) : run == C;
        run = 1;
        if (static_cast<size_t>(sc) >= run_of_scene.size()) run_of_scene.resize(static_cast<size_t>(sc) + 1, 0);
        ok = ok && run_of_scene[sc]++ == 0;
      }
    }
    if (ok) ok = C == 0 ? (C = run, true) : run == C;
    if (ok && C >= 1 && C <= 8 && h->ctas % C == 0 && pbdr_dev::iteration_scene_clusters(h->launch_kp, C) > 0)
      h->scene_cluster = C;
  }
  h->pk_iter = h->pk_active = h->pk_full;
  if (reset_errors(h) != PBDR_OK) {
    const int code = pbdr_last_error_payload(nullptr, nullptr, nullptr);
    release(h);
    return code;
  }
  // Per substep: 4 memsets + cell clear + [wrench] + integrate + body keys +
  // body sort (memset, histogram, scan, passes) + body ranges + partners +
  // near flag / scan / compact + particle sort (memset, histogram, scan,
  // passes) + cell ranges + neighbours + iterations.
  // Bodies larger than one CTA add their own launches (cluster iteration,
  // looping torque prepass); a scene of only such bodies has no tile launch.
  const int tile_l = h->ctas > 0 ? 1 : 0, big_l = big.empty() ? 0 : 1;
  const int torque_l = h->has_torque ? tile_l + big_l : 0;
  h->launches_per_frame = static_cast<int64_t>(h->substeps) *
                          ((scene_partners(h) ? 3 + 1 : 4 + 1 + (3 + h->bpasses) + 2) + 2 + torque_l + 1 +
                           (h->obb_q && h->broadphase && !scene_partners(h) ? 5 : 4) +
                           (3 + h->passes) + 1 + 1 +
                           static_cast<int64_t>(fused_iterations(h) ? 1 : h->iters) * (tile_l + big_l));
  if (fuse_next_integrate(h)) h->launches_per_frame -= h->substeps - 1;  // integrate inside the cluster launch
  if (h->pairs_possible && !fused_iterations(h) && split_isolated(h))
    h->launches_per_frame += static_cast<int64_t>(h->substeps) * 3;  // counts memset, classify, isolated launch
  if (!h->pairs_possible)  // single-body scenes: integrate + counter tick + all iterations in one launch
    h->launches_per_frame = static_cast<int64_t>(h->substeps) * (torque_l + 1 + 1 + tile_l + big_l);
  *out = h;
  return PBDR_OK;
}

void pbdr_gpu_destroy(pbdr_handle* h) { release(h); }

int pbdr_gpu_step(pbdr_handle* h, int64_t substeps) {
  if (!h) return set_error(PBDR_ERR_GENERIC, "null handle");
  pbdr_host::clear_error();
  PBDR_CUDA(cudaSetDevice(h->device));
  enqueue_substeps(h, substeps, nullptr);
  PBDR_CUDA(cudaGetLastError());
  h->substeps_done += substeps;
  return check_errors(h);
}

static void enqueue_stats(pbdr_handle* h, double* out) {
  pbdr_dev::StatsArgs sa{};
  sa.pos = h->pos[h->cur];
  sa.vel = h->vel;
  sa.rest = h->rest;
  sa.anchor = h->anchor;
  sa.cta_desc = h->pk_iter.cta;
  sa.warp_desc = h->pk_iter.warp;
  sa.body_desc = h->pk_iter.body;
  sa.body_mass = h->body_mass;
  sa.out = out;
  sa.big_list = h->pk_iter.big;
  if (h->pk_iter.ctas > 0) pbdr_dev::launch_stats(sa, h->pk_iter.ctas, h->launch_kp, h->stream);
  if (h->pk_iter.nbig > 0) pbdr_dev::launch_stats_big(sa, h->pk_iter.nbig, h->stream);
}

static int step_frames_async(pbdr_handle* h, int64_t frames) {
  for (int64_t f = 0; f < frames; ++f) {
    const int parity = h->cur;
    if (!h->graph[parity]) {
      const int rc = build_graph(h, parity);
      if (rc != PBDR_OK) return rc;
    }
    if (h->traj && h->traj_pending == h->traj_cap)
      return set_error(PBDR_ERR_GENERIC, "trajectory ring full: drain it (pbdr_gpu_trajectory_drain)");
    PBDR_CUDA(cudaGraphLaunch(h->graph[parity], h->stream));
    h->cur = h->graph_end[parity];
    h->substeps_done += h->substeps;
    if (h->traj) {
      enqueue_stats(h, h->traj + h->traj_pending * static_cast<int64_t>(h->nb) * 13);
      h->traj_t.push_back(static_cast<double>(h->substeps_done) * h->dt_d);
      ++h->traj_pending;
    }
  }
  return PBDR_OK;
}

int pbdr_gpu_step_frames(pbdr_handle* h, int64_t frames) {
  if (!h) return set_error(PBDR_ERR_GENERIC, "null handle");
  pbdr_host::clear_error();
  PBDR_CUDA(cudaSetDevice(h->device));
  const int rc = step_frames_async(h, frames);
  if (rc != PBDR_OK) return rc;
  return check_errors(h);
}

int pbdr_gpu_time_frames(pbdr_handle* h, int64_t frames, float* ms) {
  if (!h || !ms) return set_error(PBDR_ERR_GENERIC, "null argument");
  PBDR_CUDA(cudaSetDevice(h->device));
  // Build graphs outside the timed region.
  for (int p = 0; p < 2; ++p)
    if (!h->graph[p]) {
      const int rc = build_graph(h, p);
      if (rc != PBDR_OK) return rc;
    }
  cudaEvent_t a, b;
  PBDR_CUDA(cudaEventCreate(&a));
  PBDR_CUDA(cudaEventCreate(&b));
  PBDR_CUDA(cudaStreamSynchronize(h->stream));
  PBDR_CUDA(cudaEventRecord(a, h->stream));
  int rc = step_frames_async(h, frames);
  PBDR_CUDA(cudaEventRecord(b, h->stream));
  PBDR_CUDA(cudaEventSynchronize(b));
  PBDR_CUDA(cudaEventElapsedTime(ms, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (rc != PBDR_OK) return rc;
  return check_errors(h);
}

int pbdr_gpu_profile_frames(pbdr_handle* h, int64_t frames, float* ms, int64_t* launches) {
  if (!h || !ms || !launches) return set_error(PBDR_ERR_GENERIC, "null argument");
  PBDR_CUDA(cudaSetDevice(h->device));
  EventHook hook(h->stream);
  enqueue_substeps(h, frames * h->substeps, &hook);
  h->substeps_done += frames * h->substeps;
  for (int k = 0; k < PBDR_KCLASS_COUNT; ++k) {
    ms[k] = hook.ms[k];
    launches[k] = hook.launches[k];
  }
  return check_errors(h);
}

int pbdr_gpu_read_f32(pbdr_handle* h, float* pos4, float* vel4) {
  if (!h) return set_error(PBDR_ERR_GENERIC, "null handle");
  PBDR_CUDA(cudaSetDevice(h->device));
  if (pos4)
    PBDR_CUDA(cudaMemcpyAsync(pos4, h->pos[h->cur], sizeof(float4) * h->n, cudaMemcpyDeviceToHost, h->stream));
  if (vel4)
    PBDR_CUDA(cudaMemcpyAsync(vel4, h->vel, sizeof(float4) * h->n, cudaMemcpyDeviceToHost, h->stream));
  PBDR_CUDA(cudaStreamSynchronize(h->stream));
  return PBDR_OK;
}

int pbdr_gpu_write_f32(pbdr_handle* h, const float* pos4, const float* vel4) {
  if (!h) return set_error(PBDR_ERR_GENERIC, "null handle");
  PBDR_CUDA(cudaSetDevice(h->device));
  if (pos4)
    PBDR_CUDA(cudaMemcpyAsync(h->pos[h->cur], pos4, sizeof(float4) * h->n, cudaMemcpyHostToDevice, h->stream));
  if (vel4)
    PBDR_CUDA(cudaMemcpyAsync(h->vel, vel4, sizeof(float4) * h->n, cudaMemcpyHostToDevice, h->stream));
  PBDR_CUDA(cudaStreamSynchronize(h->stream));
  return PBDR_OK;
}

// Asynchronous variants (pinned host memory; completion and device errors at
// pbdr_gpu_sync): separate handles on separate streams overlap their host
// transfers with each other's compute.
int pbdr_gpu_write_f32_async(pbdr_handle* h, const float* pos4, const float* vel4) {
  if (!h) return set_error(PBDR_ERR_GENERIC, "null handle");
  PBDR_CUDA(cudaSetDevice(h->device));
  if (pos4)
    PBDR_CUDA(cudaMemcpyAsync(h->pos[h->cur], pos4, sizeof(float4) * h->n, cudaMemcpyHostToDevice, h->stream));
  if (vel4)
    PBDR_CUDA(cudaMemcpyAsync(h->vel, vel4, sizeof(float4) * h->n, cudaMemcpyHostToDevice, h->stream));
  return PBDR_OK;
}

int pbdr_gpu_read_f32_async(pbdr_handle* h, float* pos4, float* vel4) {
  if (!h) return set_error(PBDR_ERR_GENERIC, "null handle");
  PBDR_CUDA(cudaSetDevice(h->device));
  if (pos4)
    PBDR_CUDA(cudaMemcpyAsync(pos4, h->pos[h->cur], sizeof(float4) * h->n, cudaMemcpyDeviceToHost, h->stream));
  if (vel4)
    PBDR_CUDA(cudaMemcpyAsync(vel4, h->vel, sizeof(float4) * h->n, cudaMemcpyDeviceToHost, h->stream));
  return PBDR_OK;
}

int pbdr_gpu_step_frames_async(pbdr_handle* h, int64_t frames) {
  if (!h) return set_error(PBDR_ERR_GENERIC, "null handle");
  pbdr_host::clear_error();
  PBDR_CUDA(cudaSetDevice(h->device));
  return step_frames_async(h, frames);
}

// The reference-shaped transfer (fp64, the caller's particle order): the
// host arrays are staged in HBM and converted and permuted by a kernel
// (k_particles_in / _out), so no host loop and no device round trip.
static int ensure_xfer(pbdr_handle* h) {
  if (h->xfer) return PBDR_OK;
  int rc = dalloc(h, &h->xfer, 6 * static_cast<size_t>(h->n));
  if (rc == PBDR_OK) rc = dalloc(h, &h->slot_particle, static_cast<size_t>(h->n));
  if (rc != PBDR_OK) return rc;
  std::vector<int> sp(h->n);
  for (int64_t s = 0; s < h->n; ++s) sp[s] = static_cast<int>(h->slot_to_particle[s]);
  PBDR_CUDA(cudaMemcpy(h->slot_particle, sp.data(), sizeof(int) * h->n, cudaMemcpyHostToDevice));
  return PBDR_OK;
}

int pbdr_gpu_read_particles(pbdr_handle* h, double* position, double* velocity) {
  if (!h) return set_error(PBDR_ERR_GENERIC, "null handle");
  PBDR_CUDA(cudaSetDevice(h->device));
  const int rc = ensure_xfer(h);
  if (rc != PBDR_OK) return rc;
  const size_t bytes = sizeof(double) * 3 * h->n;
  double* xd = position ? h->xfer : nullptr;
  double* vd = velocity ? h->xfer + 3 * h->n : nullptr;
  pbdr_dev::launch_particles_out(h->pos[h->cur], h->vel, xd, vd, h->slot_particle, h->n, h->stream);
  PBDR_CUDA(cudaGetLastError());
  if (position) PBDR_CUDA(cudaMemcpyAsync(position, xd, bytes, cudaMemcpyDeviceToHost, h->stream));
  if (velocity) PBDR_CUDA(cudaMemcpyAsync(velocity, vd, bytes, cudaMemcpyDeviceToHost, h->stream));
  PBDR_CUDA(cudaStreamSynchronize(h->stream));
  return PBDR_OK;
}

int pbdr_gpu_write_particles(pbdr_handle* h, const double* position, const double* velocity) {
  if (!h) return set_error(PBDR_ERR_GENERIC, "null handle");
  PBDR_CUDA(cudaSetDevice(h->device));
  const int rc = ensure_xfer(h);
  if (rc != PBDR_OK) return rc;
  const size_t bytes = sizeof(double) * 3 * h->n;
  double* xd = position ? h->xfer : nullptr;
  double* vd = velocity ? h->xfer + 3 * h->n : nullptr;
  // Everything on the handle's stream, after the work already queued there.
  if (position) PBDR_CUDA(cudaMemcpyAsync(xd, position, bytes, cudaMemcpyHostToDevice, h->stream));
  if (velocity) PBDR_CUDA(cudaMemcpyAsync(vd, velocity, bytes, cudaMemcpyHostToDevice, h->stream));
  pbdr_dev::launch_particles_in(h->pos[h->cur], h->vel, xd, vd, h->slot_particle, h->n, h->stream);
  PBDR_CUDA(cudaGetLastError());
  if (position) {
    // New positions: the warm-start rotations are dropped (the next polar
    // starts cold) and each body's anchor moves to its first slot, exactly as
    // a handle created from this state would have them.
    PBDR_CUDA(cudaMemsetAsync(h->rquat, 0, sizeof(float4) * h->nb, h->stream));
    pbdr_dev::launch_anchor_reset(h->anchor, h->pk_full.body, h->pos[h->cur], h->nb, h->stream);
    PBDR_CUDA(cudaGetLastError());
  }
  PBDR_CUDA(cudaStreamSynchronize(h->stream));
  return PBDR_OK;
}

// Simulation time as a substep index t / dt (ForceProgram windows,
// scene.hpp:60, and the frame index of SimulationError, errors.hpp:39-44).
int pbdr_gpu_set_time(pbdr_handle* h, int64_t substep) {
  if (!h) return set_error(PBDR_ERR_GENERIC, "null handle");
  if (substep < 0) return set_config_error("time", "must be >= 0");
  PBDR_CUDA(cudaSetDevice(h->device));
  const long long c = substep;
  PBDR_CUDA(cudaMemcpyAsync(h->counter, &c, sizeof c, cudaMemcpyHostToDevice, h->stream));
  PBDR_CUDA(cudaStreamSynchronize(h->stream));
  h->substeps_done = substep;
  return PBDR_OK;
}

int pbdr_gpu_get_time(pbdr_handle* h, int64_t* substep) {
  if (!h || !substep) return set_error(PBDR_ERR_GENERIC, "null argument");
  PBDR_CUDA(cudaSetDevice(h->device));
  long long c = 0;
  PBDR_CUDA(cudaStreamSynchronize(h->stream));
  PBDR_CUDA(cudaMemcpy(&c, h->counter, sizeof c, cudaMemcpyDeviceToHost));
  *substep = c;
  return PBDR_OK;
}

int pbdr_gpu_read_bodies(pbdr_handle* h, pbdr_body_stats* out) {
  if (!h || !out) return set_error(PBDR_ERR_GENERIC, "null argument");
  static_assert(sizeof(pbdr_body_stats) == 13 * sizeof(double), "stats layout");
  PBDR_CUDA(cudaSetDevice(h->device));
  enqueue_stats(h, h->stats);
  PBDR_CUDA(cudaGetLastError());
  PBDR_CUDA(cudaMemcpyAsync(out, h->stats, sizeof(double) * 13 * h->nb, cudaMemcpyDeviceToHost, h->stream));
  PBDR_CUDA(cudaStreamSynchronize(h->stream));
  return PBDR_OK;
}

int pbdr_gpu_info(pbdr_handle* h, pbdr_info* o) {
  if (!h || !o) return set_error(PBDR_ERR_GENERIC, "null argument");
  o->num_particles = h->n;
  o->num_bodies = h->nb;
  o->num_ctas = h->ctas;
  o->hash_bits = h->hash_bits;
  o->sort_passes = h->passes;
  o->launches_per_frame = h->launches_per_frame;
  o->device_bytes = static_cast<int64_t>(h->device_bytes);
  o->device = h->device;
  o->sm_count = h->sm_count;
  o->cell_size = h->h;
  o->dt = h->dt;
  o->tile_kp = h->kp;
  o->scene_cluster = use_scene_clusters(h) ? h->scene_cluster : 0;
  return PBDR_OK;
}

// ---- Replay hooks ------------------------------------------------------------
int pbdr_gpu_debug_prologue(pbdr_handle* h) {
  if (!h) return set_error(PBDR_ERR_GENERIC, "null handle");
  PBDR_CUDA(cudaSetDevice(h->device));
  enqueue_substep(h, nullptr);
  h->debug_iter = 0;
  PBDR_CUDA(cudaGetLastError());
  return check_errors(h);
}

int pbdr_gpu_debug_iteration(pbdr_handle* h, int) {
  if (!h) return set_error(PBDR_ERR_GENERIC, "null handle");
  PBDR_CUDA(cudaSetDevice(h->device));
  enqueue_iteration(h, h->debug_iter % std::max(1, h->iters), nullptr);
  ++h->debug_iter;
  PBDR_CUDA(cudaGetLastError());
  return check_errors(h);
}

// Per-CTA clock64 stamps of one iteration launch: 8 per CTA (start, staged,
// phase A done, body math A done, phase B done, body math B done, end, smid).
int pbdr_gpu_debug_phase_timing(pbdr_handle* h, long long* out) {
  if (!h || !out) return set_error(PBDR_ERR_GENERIC, "null argument");
  if (h->slab) return set_error(PBDR_ERR_GENERIC, "phase timing is not available in slab mode");
  PBDR_CUDA(cudaSetDevice(h->device));
  if (!h->timing_buf) {
    void* p = nullptr;
    PBDR_CUDA(cudaMalloc(&p, sizeof(long long) * 16 * h->ctas));
    h->allocations.push_back(p);
    h->timing_buf = static_cast<long long*>(p);
  }
  PBDR_CUDA(cudaMemsetAsync(h->timing_buf, 0, sizeof(long long) * 16 * h->ctas, h->stream));
  h->timing = h->timing_buf;  // only this launch is instrumented
  enqueue_iteration(h, 0, nullptr);
  h->timing = nullptr;
  PBDR_CUDA(cudaMemcpyAsync(out, h->timing_buf, sizeof(long long) * 16 * h->ctas, cudaMemcpyDeviceToHost,
                            h->stream));
  PBDR_CUDA(cudaStreamSynchronize(h->stream));
  return check_errors(h);
}

int pbdr_gpu_debug_read_sorted(pbdr_handle* h, uint32_t* keys, uint32_t* vals) {
  if (!h) return set_error(PBDR_ERR_GENERIC, "null handle");
  PBDR_CUDA(cudaSetDevice(h->device));
  if (keys)
    PBDR_CUDA(cudaMemcpy(keys, h->keys[h->sorted_buf], sizeof(uint32_t) * h->n, cudaMemcpyDeviceToHost));
  if (vals)
    PBDR_CUDA(cudaMemcpy(vals, h->vals[h->sorted_buf], sizeof(uint32_t) * h->n, cudaMemcpyDeviceToHost));
  return PBDR_OK;
}

// Cell hash of every slot (from the last prologue's sorted pairs) and the
// integer cell coordinates recomputed by the host from the device positions.
int pbdr_gpu_debug_read_keys(pbdr_handle* h, uint32_t* cell_hash, int32_t* cell_xyz) {
  if (!h) return set_error(PBDR_ERR_GENERIC, "null handle");
  PBDR_CUDA(cudaSetDevice(h->device));
  if (cell_hash)
    PBDR_CUDA(cudaMemcpy(cell_hash, h->key_all, sizeof(uint32_t) * h->n, cudaMemcpyDeviceToHost));
  if (cell_xyz) {
    // Positions are still X~ between the prologue and the first iteration.
    std::vector<float4> xp(h->n);
    PBDR_CUDA(cudaMemcpy(xp.data(), h->pos[h->cur], sizeof(float4) * h->n, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < h->n; ++i) {
      cell_xyz[3 * i] = pbdr_cell_coord(xp[i].x, h->inv_h);
      cell_xyz[3 * i + 1] = pbdr_cell_coord(xp[i].y, h->inv_h);
      cell_xyz[3 * i + 2] = pbdr_cell_coord(xp[i].z, h->inv_h);
    }
  }
  return PBDR_OK;
}

int pbdr_gpu_debug_near_count(pbdr_handle* h, int64_t* count) {
  if (!h || !count) return set_error(PBDR_ERR_GENERIC, "null argument");
  PBDR_CUDA(cudaSetDevice(h->device));
  long long c = 0;
  PBDR_CUDA(cudaMemcpy(&c, h->near_count, sizeof c, cudaMemcpyDeviceToHost));
  *count = c;
  return PBDR_OK;
}

int pbdr_gpu_debug_read_candidates(pbdr_handle* h, int32_t* counts, int32_t* lists) {
  if (!h) return set_error(PBDR_ERR_GENERIC, "null handle");
  PBDR_CUDA(cudaSetDevice(h->device));
  std::vector<int32_t> c(h->n);
  PBDR_CUDA(cudaMemcpy(c.data(), h->ncand, sizeof(int32_t) * h->n, cudaMemcpyDeviceToHost));
  if (counts) std::memcpy(counts, c.data(), sizeof(int32_t) * h->n);
  if (lists) {
    std::vector<int32_t> sm(static_cast<size_t>(h->n) * PBDR_NBR_CAP);
    PBDR_CUDA(cudaMemcpy(sm.data(), h->cand_j, sizeof(int32_t) * sm.size(), cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < h->n; ++i)
      for (int k = 0; k < PBDR_NBR_CAP; ++k)
        lists[i * PBDR_NBR_CAP + k] = k < c[i] ? sm[static_cast<size_t>(k) * h->n + i] : -1;
  }
  return PBDR_OK;
}

int pbdr_gpu_debug_read_init(pbdr_handle* h, float* init4) {
  if (!h || !init4) return set_error(PBDR_ERR_GENERIC, "null argument");
  PBDR_CUDA(cudaSetDevice(h->device));
  PBDR_CUDA(cudaMemcpy(init4, h->init, sizeof(float4) * h->n, cudaMemcpyDeviceToHost));
  return PBDR_OK;
}

int pbdr_gpu_debug_read_anchor(pbdr_handle* h, float* anchor3) {
  if (!h || !anchor3) return set_error(PBDR_ERR_GENERIC, "null argument");
  PBDR_CUDA(cudaSetDevice(h->device));
  std::vector<float4> a(h->nb);
  PBDR_CUDA(cudaMemcpy(a.data(), h->anchor, sizeof(float4) * h->nb, cudaMemcpyDeviceToHost));
  for (int32_t b = 0; b < h->nb; ++b) {
    anchor3[3 * b] = a[b].x; anchor3[3 * b + 1] = a[b].y; anchor3[3 * b + 2] = a[b].z;
  }
  return PBDR_OK;
}

int pbdr_gpu_debug_read_rquat(pbdr_handle* h, float* q4) {
  if (!h || !q4) return set_error(PBDR_ERR_GENERIC, "null argument");
  PBDR_CUDA(cudaSetDevice(h->device));
  PBDR_CUDA(cudaMemcpy(q4, h->rquat, sizeof(float4) * h->nb, cudaMemcpyDeviceToHost));
  return PBDR_OK;
}

int pbdr_gpu_debug_write_rquat(pbdr_handle* h, const float* q4) {
  if (!h || !q4) return set_error(PBDR_ERR_GENERIC, "null argument");
  PBDR_CUDA(cudaSetDevice(h->device));
  PBDR_CUDA(cudaMemcpy(h->rquat, q4, sizeof(float4) * h->nb, cudaMemcpyHostToDevice));
  return PBDR_OK;
}

int pbdr_gpu_debug_write_anchor(pbdr_handle* h, const float* anchor3) {
  if (!h || !anchor3) return set_error(PBDR_ERR_GENERIC, "null argument");
  PBDR_CUDA(cudaSetDevice(h->device));
  std::vector<float4> a(h->nb);
  for (int32_t b = 0; b < h->nb; ++b) a[b] = make_float4(anchor3[3 * b], anchor3[3 * b + 1], anchor3[3 * b + 2], 0.0f);
  PBDR_CUDA(cudaMemcpy(h->anchor, a.data(), sizeof(float4) * h->nb, cudaMemcpyHostToDevice));
  return PBDR_OK;
}

// ---- Trajectory emission -----------------------------------------------------
int pbdr_gpu_trajectory_enable(pbdr_handle* h, int64_t capacity_frames) {
  if (!h) return set_error(PBDR_ERR_GENERIC, "null handle");
  PBDR_CUDA(cudaSetDevice(h->device));
  PBDR_CUDA(cudaStreamSynchronize(h->stream));
  if (h->traj) {
    cudaFree(h->traj);
    h->allocations.erase(std::find(h->allocations.begin(), h->allocations.end(), static_cast<void*>(h->traj)));
    h->traj = nullptr;
  }
  h->traj_cap = 0;
  h->traj_pending = 0;
  h->traj_t.clear();
  if (capacity_frames <= 0) return PBDR_OK;
  const int rc = dalloc(h, &h->traj, static_cast<size_t>(capacity_frames) * h->nb * 13);
  if (rc != PBDR_OK) return rc;
  h->traj_cap = capacity_frames;
  return PBDR_OK;
}

int pbdr_gpu_trajectory_drain(pbdr_handle* h, double* out, double* t, int64_t max_frames, int64_t* frames) {
  if (!h || !frames) return set_error(PBDR_ERR_GENERIC, "null argument");
  PBDR_CUDA(cudaSetDevice(h->device));
  PBDR_CUDA(cudaStreamSynchronize(h->stream));
  const int64_t k = std::min(h->traj_pending, max_frames);
  if (k < h->traj_pending)
    return set_error(PBDR_ERR_GENERIC, "trajectory drain: output holds fewer frames than pending");
  if (k > 0 && out)
    PBDR_CUDA(cudaMemcpy(out, h->traj, sizeof(double) * 13 * h->nb * k, cudaMemcpyDeviceToHost));
  if (t)
    for (int64_t f = 0; f < k; ++f) t[f] = h->traj_t[f];
  *frames = k;
  h->traj_pending = 0;
  h->traj_t.clear();
  return PBDR_OK;
}

// ---- Staged stepping and slab decomposition ------------------------------------
int pbdr_gpu_substep_begin(pbdr_handle* h) {
  if (!h) return set_error(PBDR_ERR_GENERIC, "null handle");
  PBDR_CUDA(cudaSetDevice(h->device));
  enqueue_substep(h, nullptr);
  h->stage_iter = 0;
  PBDR_CUDA(cudaGetLastError());
  return PBDR_OK;
}

int pbdr_gpu_substep_iteration(pbdr_handle* h) {
  if (!h) return set_error(PBDR_ERR_GENERIC, "null handle");
  PBDR_CUDA(cudaSetDevice(h->device));
  enqueue_iteration(h, h->stage_iter % std::max(1, h->iters), nullptr);
  if (++h->stage_iter == h->iters) h->substeps_done += 1;
  PBDR_CUDA(cudaGetLastError());
  return PBDR_OK;
}

int pbdr_gpu_sync(pbdr_handle* h) {
  if (!h) return set_error(PBDR_ERR_GENERIC, "null handle");
  pbdr_host::clear_error();
  PBDR_CUDA(cudaSetDevice(h->device));
  return check_errors(h);
}

int pbdr_gpu_stream(pbdr_handle* h, void** stream) {
  if (!h || !stream) return set_error(PBDR_ERR_GENERIC, "null argument");
  *stream = h->stream;
  return PBDR_OK;
}

int pbdr_gpu_set_roles(pbdr_handle* h, const int8_t* roles) {
  if (!h) return set_error(PBDR_ERR_GENERIC, "null handle");
  pbdr_host::clear_error();
  PBDR_CUDA(cudaSetDevice(h->device));
  PBDR_CUDA(cudaStreamSynchronize(h->stream));
  for (auto& g : h->graph)
    if (g) {
      cudaGraphExecDestroy(g);
      g = nullptr;
    }
  if (!roles) {  // back to the whole scene
    h->slab = false;
    h->pk_iter = h->pk_active = h->pk_full;
    h->p_lo = 0;
    h->p_hi = h->n;
    return PBDR_OK;
  }
  const int32_t nb = h->nb;
  if (!h->role) {
    int rc = PBDR_OK;
    rc |= dalloc(h, &h->role, nb);
    rc |= dalloc(h, &h->active_list, nb);
    rc |= dalloc(h, &h->slab_iter.cta, nb);
    rc |= dalloc(h, &h->slab_iter.warp, static_cast<size_t>(nb) * PBDR_CTA_WARPS);
    rc |= dalloc(h, &h->slab_iter.body, nb);
    rc |= dalloc(h, &h->slab_active.cta, nb);
    rc |= dalloc(h, &h->slab_active.warp, static_cast<size_t>(nb) * PBDR_CTA_WARPS);
    rc |= dalloc(h, &h->slab_active.body, nb);
    if (h->big_cluster > 0) {
      rc |= dalloc(h, &h->slab_iter.big, nb);
      rc |= dalloc(h, &h->slab_active.big, nb);
    }
    if (rc != PBDR_OK) return PBDR_ERR_CUDA;
  }
  std::vector<uint8_t> r(nb);
  std::vector<int> owned, active;
  int64_t lo = h->n, hi = 0;
  for (int32_t b = 0; b < nb; ++b) {
    if (roles[b] < 0 || roles[b] > 2) return set_config_error("roles", "role must be 0, 1 or 2");
    r[b] = static_cast<uint8_t>(roles[b]);
    if (r[b] == 0) continue;
    active.push_back(b);
    if (r[b] == 2) owned.push_back(b);
    lo = std::min(lo, h->h_bstart[b]);
    hi = std::max(hi, h->h_bstart[b] + h->h_bcount[b]);
  }
  std::vector<int4> cd, wd, bd(nb, make_int4(0, 0, 0, 0));
  std::vector<int> big;
  PBDR_CUDA(cudaMemcpy(h->role, r.data(), nb, cudaMemcpyHostToDevice));
  if (!active.empty())
    PBDR_CUDA(cudaMemcpy(h->active_list, active.data(), sizeof(int) * active.size(), cudaMemcpyHostToDevice));
  auto upload = [&](const std::vector<int>& list, pbdr_handle::Packing& dev) -> int {
    pack_bodies(list, h->h_bstart, h->h_bcount, h->h_bscene, h->kp, cd, wd, bd, big);
    dev.ctas = static_cast<int>(cd.size());
    dev.nbig = static_cast<int>(big.size());
    if (!big.empty())
      PBDR_CUDA(cudaMemcpy(dev.big, big.data(), sizeof(int) * big.size(), cudaMemcpyHostToDevice));
    if (!cd.empty()) {
      PBDR_CUDA(cudaMemcpy(dev.cta, cd.data(), sizeof(int4) * cd.size(), cudaMemcpyHostToDevice));
      PBDR_CUDA(cudaMemcpy(dev.warp, wd.data(), sizeof(int4) * wd.size(), cudaMemcpyHostToDevice));
    }
    if (!cd.empty() || !big.empty())
      PBDR_CUDA(cudaMemcpy(dev.body, bd.data(), sizeof(int4) * bd.size(), cudaMemcpyHostToDevice));
    return PBDR_OK;
  };
  int rc = upload(owned, h->slab_iter);
  h->h_iter_cdesc = cd;  // host copy of the owned tiles (native slab driver)
  if (rc == PBDR_OK) rc = upload(active, h->slab_active);
  if (rc != PBDR_OK) return rc;
  h->slab = true;
  h->pk_iter = h->slab_iter;
  h->pk_active = h->slab_active;
  h->n_active = static_cast<int>(active.size());
  h->p_lo = active.empty() ? 0 : lo;
  h->p_hi = active.empty() ? 0 : hi;
  return PBDR_OK;
}

static float4* exchange_field(pbdr_handle* h, int which, int64_t* limit) {
  switch (which) {
    case PBDR_FIELD_POSITION: *limit = h->n; return h->pos[h->cur];
    case PBDR_FIELD_VELOCITY: *limit = h->n; return h->vel;
    case PBDR_FIELD_ANCHOR: *limit = h->nb; return h->anchor;
    case PBDR_FIELD_ROTATION: *limit = h->nb; return h->rquat;
    default: return nullptr;
  }
}

int pbdr_gpu_gather(pbdr_handle* h, int which, const int32_t* index, int64_t count, void* dst) {
  if (!h || (count > 0 && (!index || !dst))) return set_error(PBDR_ERR_GENERIC, "null argument");
  int64_t limit = 0;
  const float4* src = exchange_field(h, which, &limit);
  if (!src) return set_config_error("field", "unknown exchange field");
  PBDR_CUDA(cudaSetDevice(h->device));
  pbdr_dev::launch_gather4(static_cast<float4*>(dst), src, index, count, h->stream);
  PBDR_CUDA(cudaGetLastError());
  return PBDR_OK;
}

int pbdr_gpu_scatter(pbdr_handle* h, int which, const int32_t* index, int64_t count, const void* src) {
  if (!h || (count > 0 && (!index || !src))) return set_error(PBDR_ERR_GENERIC, "null argument");
  int64_t limit = 0;
  float4* dst = exchange_field(h, which, &limit);
  if (!dst) return set_config_error("field", "unknown exchange field");
  PBDR_CUDA(cudaSetDevice(h->device));
  pbdr_dev::launch_scatter4(dst, static_cast<const float4*>(src), index, count, h->stream);
  PBDR_CUDA(cudaGetLastError());
  return PBDR_OK;
}

}  // extern "C"

// ---- Internal entry points for the native slab driver (pbdr_slab.cu) --------
namespace pbdr_engine {

int cuda_fail(cudaError_t e, const char* what) { return ::cuda_fail(e, what); }

int device_alloc(pbdr_handle* h, void** ptr, size_t bytes) {
  char* p = nullptr;
  const int rc = dalloc(h, &p, bytes);
  *ptr = p;
  return rc;
}

void enqueue_substep(pbdr_handle* h) { ::enqueue_substep(h, nullptr); }

void enqueue_iteration_tiles(pbdr_handle* h, int iter_index, const int* list, const int* count) {
  const int cur = h->cur;
  ::enqueue_iteration(h, iter_index, nullptr, 1, false, list, count);
  h->cur = cur;
}

void enqueue_body_stats(pbdr_handle* h, double* out) { enqueue_stats(h, out); }

int check_errors(pbdr_handle* h) { return ::check_errors(h); }

}  // namespace pbdr_engine
