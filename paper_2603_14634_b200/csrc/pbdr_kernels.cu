// sm_100a kernels of the PBD-R substep loop.
//
// Per substep:
//   k_integrate_key  x_init <- x; v~ = v + dt a; x~ = x + dt v~; cell key
//   [onesweep sort of (key, slot), pbdr_sort.cu]
//   k_cell_ranges    per-bucket [start, end) of the sorted array + body of
//                    every sorted entry
//   k_neighbours     per particle: contact candidates (other body, same scene,
//                    27-cell stencil, |x~_i - x~_j| < h), ascending slot order;
//                    the stencil is scanned as 9 x-rows, each one contiguous
//                    range of the sorted array (x-run cell keys)
//   k_iteration x N  fused: ground + particle-particle contact (Jacobi), shape
//                    matching (segmented com / Apq sums + fp64 polar), position
//                    and incremental velocity update, momentum constraint
//                    (Eq. 1 / Eq. 2) fused into the writeback
// The op order of every fp32 expression is pinned and
// mirrored by oracle/pbdr_oracle.cpp; the library is compiled with
// --fmad=false so the CUDA path and the oracle agree bit for bit.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <stdint.h>

#include "pbdr_kernels.cuh"
#include "pbdr_mat3.cuh"
#include "pbdr_pinned.h"

namespace pbdr_dev {

namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kWarps = PBDR_CTA_WARPS;
constexpr int kThreads = kWarps * 32;
constexpr uint32_t kEmpty = 0xFFFFFFFFu;

// Checked build (make checked -> lib/libpbdr_gpu_checked.so): device-side
// bounds and invariant checks on every index the kernels load or store
// through -- the substitute for compute-sanitizer, which this GPU pool does
// not run (profiles/r02_sanitizer_unavailable.md). A failed check traps
// (cudaErrorAssert / illegal instruction), so the calling test fails loudly.
#ifndef PBDR_CHECKED
#define PBDR_CHECKED 0
#endif
#if PBDR_CHECKED
// Checked build: a failed check writes (line, block, thread) into a record in
// mapped host memory -- readable after the context is gone -- and traps; the
// host appends the record to the CUDA error message (checked_failure()).
// No printf: its call frames would change the very code under test.
struct CheckRecord {
  int hit, line, block, thread;
};
__device__ CheckRecord* g_check_record = nullptr;
__device__ __noinline__ void check_fail(int line) {
  CheckRecord* r = g_check_record;
  if (r) {
    r->line = line;
    r->block = static_cast<int>(blockIdx.x);
    r->thread = static_cast<int>(threadIdx.x);
    r->hit = 1;
    __threadfence_system();
  }
  __trap();
}
#define PBDR_CHECK(cond)                 \
  do {                                   \
    if (!(cond)) check_fail(__LINE__);   \
  } while (0)
#else
#define PBDR_CHECK(cond) \
  do {                   \
  } while (0)
#endif

__device__ __forceinline__ void record_error(DevError* e, unsigned bits, int body,
                                             const long long* substep_counter,
                                             const double* axis = nullptr) {
  atomicOr(&e->bits, bits);
  const int prev = atomicMin(&e->body, body);
  atomicMin(reinterpret_cast<unsigned long long*>(&e->substep),
            static_cast<unsigned long long>(*substep_counter));
  if (axis && (prev > body)) {
    e->axis[0] = axis[0];
    e->axis[1] = axis[1];
    e->axis[2] = axis[2];
  }
}

__device__ __forceinline__ void cross3(const float a[3], const float b[3], float o[3]) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}

template <int F>
__device__ __forceinline__ void warp_butterfly(float (&acc)[F]) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1)
#pragma unroll
    for (int f = 0; f < F; ++f) acc[f] = acc[f] + __shfl_xor_sync(kFull, acc[f], off);
}

// Same reduction tree as warp_butterfly (xor offsets 16, 8, 4, 2, 1; every add
// combines the partial sums of lanes l and l^off), computed by recursive
// halving: at each offset a lane keeps half of the remaining fields and
// exchanges the other half, so F fields cost ~P-1 shuffles instead of 5F
// (P = F rounded up to a power of two). On return lane l holds the total of
// field l * P / 32 (every lane of a group of 32/P holds the same value);
// the totals are bit-identical to warp_butterfly's (IEEE add is commutative).
template <int F>
__device__ __forceinline__ float warp_reduce_scatter(const float (&acc)[F]) {
  constexpr int P = F <= 1 ? 1 : F <= 2 ? 2 : F <= 4 ? 4 : F <= 8 ? 8 : F <= 16 ? 16 : 32;
  static_assert(F <= 32, "at most 32 fields");
  const int lane = threadIdx.x & 31;
  float v[P];
#pragma unroll
  for (int f = 0; f < P; ++f) v[f] = f < F ? acc[f] : 0.0f;
  int c = P;
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    if (c > 1) {
      const bool up = (lane & off) != 0;
      const int h = c / 2;
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        if (k >= h) break;
        const float send = up ? v[k] : v[h + k];
        const float keep = up ? v[h + k] : v[k];
        v[k] = keep + __shfl_xor_sync(kFull, send, off);
      }
      c = h;
    } else {
      v[0] = v[0] + __shfl_xor_sync(kFull, v[0], off);
    }
  }
  return v[0];
}

// ---- TMA bulk staging (cp.async.bulk + mbarrier) ---------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ __attribute__((unused)) void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// L2 residency hints: descriptors and per-body tables are tiny and re-read by
// every launch, while particle state streams through (>> 126 MB L2). Keep the
// former (evict_last), stream the latter (evict_first on the bulk copies).
#ifndef PBDR_L2_HINTS
#define PBDR_L2_HINTS 1
#endif
template <typename T>
__device__ __forceinline__ T ld_keep_nc(const T* p) {
#if PBDR_L2_HINTS
  static_assert(sizeof(T) == 16 || sizeof(T) == 8, "vector loads only");
  T v;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  if constexpr (sizeof(T) == 16) {
    uint32_t* r = reinterpret_cast<uint32_t*>(&v);
    asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "l"(p), "l"(pol));
  } else {
    uint32_t* r = reinterpret_cast<uint32_t*>(&v);
    asm volatile("ld.global.nc.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;" : "=r"(r[0]), "=r"(r[1]) : "l"(p), "l"(pol));
  }
  return v;
#else
  return *p;
#endif
}

template <typename T>
__device__ __forceinline__ T ld_keep(const T* p) {  // coherent (data this kernel also writes)
#if PBDR_L2_HINTS
  static_assert(sizeof(T) == 16, "float4 only");
  T v;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  uint32_t* r = reinterpret_cast<uint32_t*>(&v);
  asm volatile("ld.global.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "l"(p), "l"(pol));
  return v;
#else
  return *p;
#endif
}

__device__ __forceinline__ void bulk_g2s_stream(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
#if PBDR_L2_HINTS
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
#else
  bulk_g2s(dst, src, bytes, bar);
#endif
}

// Bulk prefetch of a byte range into L2 (no shared memory, no registers): the
// next tile's staging ranges are pulled in while the current tile computes, so
// its bulk copies hit L2. Address rounded down / size up to 16 B.
__device__ __forceinline__ void bulk_prefetch_l2(const void* p, uint32_t bytes) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  const uintptr_t a0 = a & ~uintptr_t(15);
  const uint32_t sz = static_cast<uint32_t>((a - a0 + bytes + 15) & ~uintptr_t(15));
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"(sz) : "memory");
}

// Asynchronous global -> shared copies (no register staging) for the next
// tile's body table.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}

// ---------------------------------------------------------------------------
// integrate + cell key
// ---------------------------------------------------------------------------
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}
// PBDR_PREFETCH_L1: the iteration's staging-time prefetch of each particle's
// first candidate goes to L1 instead of L2.
#ifndef PBDR_PREFETCH_L1
#define PBDR_PREFETCH_L1 0
#endif

// Order-preserving float <-> uint encoding for atomicMin/atomicMax boxes.
__device__ __forceinline__ uint32_t f2ord(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u);
}

// integrate of one particle of body b:
// x_init <- x; v~ = v + dt a; x~ = x + dt v~, with a = gravity (unless
// exempt) + the body's active force program (F/M, alpha x (x - c)). Shared by
// k_integrate_key and the scene-cluster iteration kernel, which integrates the
// next substep in its final writeback.
__device__ __forceinline__ void integrate_one(const IntegrateArgs& A, int b, float4 x, float4 v, float4& xn,
                                              float4& vn) {
  BodyProgram pr{};
  if (A.has_programs) pr = A.programs[b];  // scenes without programs skip the 48-B record
  float a[3] = {0.0f, 0.0f, (pr.flags & 2) ? 0.0f : -A.gravity};
  const double t = static_cast<double>(*A.substep_counter) * A.dt_d;
  if ((pr.flags & 1) && t >= pr.t_start && t < pr.t_stop) {
    const float invM = A.body_mass[b].y;
    a[0] = a[0] + pr.fx * invM;
    a[1] = a[1] + pr.fy * invM;
    a[2] = a[2] + pr.fz * invM;
    if (pr.flags & 4) {
      const float4 c = A.wcom[b];
      const float4 al = A.walpha[b];
      const float r[3] = {x.x - c.x, x.y - c.y, x.z - c.z};
      const float alv[3] = {al.x, al.y, al.z};
      float ar[3];
      cross3(alv, r, ar);
      a[0] = a[0] + ar[0];
      a[1] = a[1] + ar[1];
      a[2] = a[2] + ar[2];
    }
  }
  vn.x = v.x + A.dt * a[0];
  vn.y = v.y + A.dt * a[1];
  vn.z = v.z + A.dt * a[2];
  vn.w = v.w;
  xn.x = x.x + A.dt * vn.x;
  xn.y = x.y + A.dt * vn.y;
  xn.z = x.z + A.dt * vn.z;
  xn.w = x.w;
}

__device__ __forceinline__ uint32_t integrate_key(const IntegrateArgs& A, int b, float4 xn) {
  const int32_t cx = pbdr_cell_coord(xn.x, A.inv_h);
  const int32_t cy = pbdr_cell_coord(xn.y, A.inv_h);
  const int32_t cz = pbdr_cell_coord(xn.z, A.inv_h);
  return pbdr_cell_key(cx, cy, cz, static_cast<uint32_t>(A.body_scene[b]), A.mask, A.layout);
}

__global__ void __launch_bounds__(256) k_integrate_key(IntegrateArgs A) {
  const int64_t p = A.p0 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  int b = p < A.n ? A.body_of[p] : -1;
  // State loads issued with the body id (not after it): the kernel is
  // latency-bound on these three streams.
  const float4 x = p < A.n ? A.pos[p] : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  const float4 v = p < A.n ? A.vel[p] : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  if (A.role && b >= 0 && A.role[b] == 0) b = -1;  // slab mode: not simulated here
  const bool valid = b >= 0;
  float4 xn = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  if (valid) {
    float4 vn;
    integrate_one(A, b, x, v, xn, vn);
    A.init[p] = make_float4(x.x, x.y, x.z, 0.0f);
    A.vel[p] = vn;
    A.pos[p] = xn;
    A.key_all[p] = integrate_key(A, b, xn);
  }
  // Body boxes of X~: warp-reduce when the warp holds at most two bodies, the
  // first lane's and the last lane's (the common case in body-major order:
  // a body of >= 32 particles), else one atomic per lane. min/max are exact
  // and order-free, so the boxes are deterministic.
  const int lane = threadIdx.x & 31;
  const int b0 = __shfl_sync(kFull, b, 0);
  const int b1 = __shfl_sync(kFull, b, 31);
  const bool two = __all_sync(kFull, b == b0 || b == b1) && b0 >= 0 && b1 >= 0;
  float lo[3] = {xn.x, xn.y, xn.z}, hi[3] = {xn.x, xn.y, xn.z};
  if (two) {
    // Group 0 = lanes of b0, group 1 = lanes of b1 (the same group when
    // b0 == b1); each lane folds only its own group's values.
    const bool g1 = b != b0;
    float lo0[3], hi0[3], lo1[3], hi1[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      lo0[c] = g1 ? INFINITY : lo[c];
      hi0[c] = g1 ? -INFINITY : hi[c];
      lo1[c] = g1 ? lo[c] : INFINITY;
      hi1[c] = g1 ? hi[c] : -INFINITY;
    }
    const uint32_t o_lo0[3] = {__reduce_min_sync(kFull, f2ord(lo0[0])), __reduce_min_sync(kFull, f2ord(lo0[1])),
                               __reduce_min_sync(kFull, f2ord(lo0[2]))};
    const uint32_t o_hi0[3] = {__reduce_max_sync(kFull, f2ord(hi0[0])), __reduce_max_sync(kFull, f2ord(hi0[1])),
                               __reduce_max_sync(kFull, f2ord(hi0[2]))};
    if (lane == 0)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        atomicMin(&A.box_min[3 * b0 + c], o_lo0[c]);
        atomicMax(&A.box_max[3 * b0 + c], o_hi0[c]);
      }
    if (b1 != b0) {
      const uint32_t o_lo1[3] = {__reduce_min_sync(kFull, f2ord(lo1[0])), __reduce_min_sync(kFull, f2ord(lo1[1])),
                                 __reduce_min_sync(kFull, f2ord(lo1[2]))};
      const uint32_t o_hi1[3] = {__reduce_max_sync(kFull, f2ord(hi1[0])), __reduce_max_sync(kFull, f2ord(hi1[1])),
                                 __reduce_max_sync(kFull, f2ord(hi1[2]))};
      if (lane == 31)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          atomicMin(&A.box_min[3 * b1 + c], o_lo1[c]);
          atomicMax(&A.box_max[3 * b1 + c], o_hi1[c]);
        }
    }
  } else if (valid) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      atomicMin(&A.box_min[3 * b + c], f2ord(lo[c]));
      atomicMax(&A.box_max[3 * b + c], f2ord(hi[c]));
    }
  }
}

// ---- body broadphase ----------------------------------------------------------
__device__ __forceinline__ void load_box(const uint32_t* bmin, const uint32_t* bmax, int b, float lo[3],
                                         float hi[3]) {
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    lo[c] = ord2f(bmin[3 * b + c]);
    hi[c] = ord2f(bmax[3 * b + c]);
  }
}

__global__ void __launch_bounds__(256) k_body_keys(BroadArgs A) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= A.nb) return;
  const int b = A.list ? A.list[t] : t;
  float lo[3], hi[3];
  load_box(A.box_min, A.box_max, b, lo, hi);
  // A box wider than the coarse cell (minus the inflation) would break the
  // 27-cell partner guarantee: then every body searches in full this substep.
  if (!(hi[0] - lo[0] <= A.max_extent && hi[1] - lo[1] <= A.max_extent && hi[2] - lo[2] <= A.max_extent))
    atomicOr(A.oversize, 1u);
  int32_t c[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) c[k] = pbdr_cell_coord(0.5f * (lo[k] + hi[k]), A.inv_cell);
  A.bkeys[t] = pbdr_cell_hash(c[0], c[1], c[2], static_cast<uint32_t>(A.body_scene[b]), A.mask);
  A.bvals[t] = static_cast<uint32_t>(b);
}

__global__ void __launch_bounds__(256) k_body_ranges(BroadArgs A) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= A.nb) return;
  const uint32_t k = A.sorted_bkeys[s];
  if (s == 0 || A.sorted_bkeys[s - 1] != k) A.bcells[k].x = static_cast<uint32_t>(s);
  if (s == A.nb - 1 || A.sorted_bkeys[s + 1] != k) A.bcells[k].y = static_cast<uint32_t>(s + 1);
}

// Partners of body b: other bodies of its scene whose box overlaps b's box
// inflated by h. The coarse cell is >= the largest box extent + h, so partner
// box centres lie in the 27 neighbouring coarse cells. One warp per body:
// lane t < 27 scans coarse cell t (lanes whose cells hash to the same bucket
// scan it once), hits are compacted with ballots. The partner list is only
// used as a set (near filter), so its order is immaterial; overflow (more than
// PBDR_PARTNER_CAP partners) marks the body for a full search.
__global__ void __launch_bounds__(256) k_body_partners(BroadArgs A) {
  const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= A.nb) return;  // warp-uniform
  const int b = A.list ? A.list[t] : t;
  if (*A.oversize) {
    if (lane == 0) A.npartners[b] = -1;
    return;
  }
  float lo[3], hi[3];
  load_box(A.box_min, A.box_max, b, lo, hi);
  const int sb = A.body_scene[b];
  int32_t c[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    c[k] = pbdr_cell_coord(0.5f * (lo[k] + hi[k]), A.inv_cell);
    lo[k] = lo[k] - (A.inflate + fabsf(lo[k]) * 1e-6f);
    hi[k] = hi[k] + (A.inflate + fabsf(hi[k]) * 1e-6f);
  }
  uint32_t key = 0xFFFFFFFFu;
  if (lane < 27)
    key = pbdr_cell_hash(c[0] + lane % 3 - 1, c[1] + (lane / 3) % 3 - 1, c[2] + lane / 9 - 1,
                         static_cast<uint32_t>(sb), A.mask);
  const unsigned same = __match_any_sync(kFull, key);
  const bool owner = lane < 27 && (__ffs(same) - 1) == lane;  // lowest lane of its bucket
  uint32_t s = 0, e = 0;
  if (owner) {
    const uint2 r = A.bcells[key];
    if (r.x != kEmpty) {
      s = r.x;
      e = r.y;
    }
  }
  int count = 0;
  while (__any_sync(kFull, s < e)) {
    bool hit = false;
    int o = -1;
    if (s < e) {
      o = static_cast<int>(A.sorted_bvals[s]);
      ++s;
      if (o != b && A.body_scene[o] == sb) {
        float olo[3], ohi[3];
        load_box(A.box_min, A.box_max, o, olo, ohi);
        hit = !(olo[0] > hi[0] || ohi[0] < lo[0] || olo[1] > hi[1] || ohi[1] < lo[1] || olo[2] > hi[2] ||
                ohi[2] < lo[2]);
      }
    }
    const unsigned m = __ballot_sync(kFull, hit);
    if (hit) {
      const int slot = count + __popc(m & ((1u << lane) - 1u));
      if (slot < PBDR_PARTNER_CAP) A.partners[static_cast<int64_t>(b) * PBDR_PARTNER_CAP + slot] = o;
    }
    count += __popc(m);
  }
  if (lane == 0) A.npartners[b] = count > PBDR_PARTNER_CAP ? -1 : count;
}

// Batched scenes of at most PBDR_PARTNER_CAP bodies, each scene a contiguous
// body range: partners by testing every body of the scene (lane l tests body
// first + l) with the same inflated-box overlap as k_body_partners. One launch
// replaces the coarse-grid keys, body sort, ranges and partner search; the
// partner set (all that the near filter uses) is the same.
__global__ void __launch_bounds__(256) k_scene_partners(BroadArgs A) {
  const int b = static_cast<int>((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (b >= A.nb) return;  // warp-uniform
  const int2 rng = A.scene_range[b];  // (first body, bodies) of b's scene
  float lo[3], hi[3];
  load_box(A.box_min, A.box_max, b, lo, hi);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    lo[k] = lo[k] - (A.inflate + fabsf(lo[k]) * 1e-6f);
    hi[k] = hi[k] + (A.inflate + fabsf(hi[k]) * 1e-6f);
  }
  const int o = rng.x + lane;
  bool hit = false;
  if (lane < rng.y && o != b) {
    float olo[3], ohi[3];
    load_box(A.box_min, A.box_max, o, olo, ohi);
    hit = !(olo[0] > hi[0] || ohi[0] < lo[0] || olo[1] > hi[1] || ohi[1] < lo[1] || olo[2] > hi[2] ||
            ohi[2] < lo[2]);
  }
  const unsigned m = __ballot_sync(kFull, hit);
  if (hit) A.partners[static_cast<int64_t>(b) * PBDR_PARTNER_CAP + __popc(m & ((1u << lane) - 1u))] = o;
  if (lane == 0) A.npartners[b] = __popc(m);
}

// Isolated tiles: every body of the tile has no partner this substep (so no
// particle of it has a candidate, and none is anyone's candidate: pairs are
// symmetric). They run all iterations of the substep in one launch with the
// state in shared memory; the other (contact) tiles iterate launch by
// launch. Lists are built with atomics: tiles are independent, so their
// order changes nothing.
__global__ void __launch_bounds__(256) k_classify_tiles(ClassifyArgs A) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= A.ntiles) return;
  const int4 cd = A.cta_desc[t];
  bool iso = true;
  for (int i = 0; i < cd.w && iso; ++i) iso = A.npartners[cd.z + i] == 0;
  const int c = atomicAdd(&A.counts[iso ? 0 : 1], 1);
  (iso ? A.iso_list : A.contact_list)[c] = t;
  if (A.iso_cd) {
    int4* cdo = iso ? A.iso_cd : A.contact_cd;
    int4* wdo = iso ? A.iso_wd : A.contact_wd;
    cdo[c] = cd;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) wdo[c * kWarps + w] = A.warp_desc[t * kWarps + w];
  }
}

// ---------------------------------------------------------------------------
// cell ranges: per-bucket (start, end) of the sorted array and the body of
// every sorted entry (slots ascend within a bucket, so bodies do too).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_cell_ranges(RangesArgs A) {
  const int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t m = *A.count;
  if (g == 0) {
    atomicAdd(reinterpret_cast<unsigned long long*>(A.substep_counter), 1ull);
    *A.prev_count = m;
  }
  for (int64_t s = g; s < m; s += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint32_t k = A.keys[s];
    const uint32_t v = A.vals[s];
    PBDR_CHECK(v < static_cast<uint64_t>(A.n) && (s == 0 || A.keys[s - 1] <= k));
    const int body = A.body_of[v];
    // X~ of the entry with its body in .w: the search reads one float4 per
    // entry (and a CTA stages runs of them, k_neighbours_staged).
    const float4 x = A.pos[v];
    A.sorted_pos[s] = make_float4(x.x, x.y, x.z, __int_as_float(body));
    // Entries of a bucket ascend by slot, hence by body: the first entry holds
    // the bucket's smallest body, the last its largest.
    if (s == 0 || A.keys[s - 1] != k) {
      A.cells[k].x = static_cast<uint32_t>(s);
      A.cells[k].z = static_cast<uint32_t>(body);
    }
    if (s == m - 1 || A.keys[s + 1] != k) {
      A.cells[k].y = static_cast<uint32_t>(s + 1);
      A.cells[k].w = static_cast<uint32_t>(body);
    }
  }
}


// ---------------------------------------------------------------------------
// Broadphase filter (exact): a candidate j of particle i lies in j's body box
// and within h of i, so i lies in the h-inflated box of a partner body. Only
// such "near" particles enter the hash grid and search it; the others have no
// candidates. Per body (one warp, partner boxes held in lanes): count the near
// particles; scan the body counts; write the near slots of each body at its
// offset. Bodies without partners cost no particle reads; the list is in slot
// order (bodies ascend, slots ascend within a body), so it is deterministic.
// ---------------------------------------------------------------------------
constexpr int kScanTile = 4096;

__device__ __forceinline__ void obb_axes(float4 q, float R[9]);

struct NearBoxes {
  float lo[3], hi[3];  // lane k < np: partner k's box inflated by h (+ relative guard)
  // PBDR_NEAR_FAST: partner k's oriented box, prepared once per body instead
  // of once per (particle, partner): frame R, centre, bounds with in_obb's
  // margins applied (the same float operations, so the same bits).
  float R[9], c[3], olo[3], ohi[3];
};
#ifndef PBDR_NEAR_FAST
#define PBDR_NEAR_FAST 1
#endif

__device__ __forceinline__ int near_body_setup(const NearArgs& A, int t, int lane, int& b, int& start, int& n,
                                               NearBoxes& bx) {
  b = A.list ? A.list[t] : t;
  const int4 bd = A.body_desc[b];
  start = bd.x;
  n = bd.y;
  int np = A.all_near ? -1 : A.npartners[b];
  if (A.role && A.role[b] == 0) np = 0;
  if (np > 0 && lane < np) {
    const int o = A.partners[static_cast<int64_t>(b) * PBDR_PARTNER_CAP + lane];
    float lo[3], hi[3];
    load_box(A.box_min, A.box_max, o, lo, hi);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const float m = A.inflate + fmaxf(fabsf(lo[c]), fabsf(hi[c])) * 1e-6f;
      bx.lo[c] = lo[c] - m;
      bx.hi[c] = hi[c] + m;
    }
#if PBDR_NEAR_FAST
    if (A.obb_q) {
      const float4 olo = A.obb_lo[o], ohi = A.obb_hi[o], oc = A.obb_c[o];
      obb_axes(A.obb_q[o], bx.R);
      bx.c[0] = oc.x; bx.c[1] = oc.y; bx.c[2] = oc.z;
      const float lv[3] = {olo.x, olo.y, olo.z}, hv[3] = {ohi.x, ohi.y, ohi.z};
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const float m = A.inflate * 1.0001f + 1e-5f * (fabsf(lv[k]) + fabsf(hv[k])) + 1e-6f;
        bx.olo[k] = lv[k] - m;
        bx.ohi[k] = hv[k] + m;
      }
    }
#endif
  }
  return np;
}

// Rotation of an oriented-box frame (columns = the frame axes) from a unit
// quaternion (w, x, y, z). The same function builds the bounds (k_body_obb)
// and tests against them, so both use the same bits.
__device__ __forceinline__ void obb_axes(float4 q, float R[9]) {
  const float w = q.x, x = q.y, y = q.z, z = q.w;
  R[0] = 1.0f - 2.0f * (y * y + z * z);
  R[1] = 2.0f * (x * y - w * z);
  R[2] = 2.0f * (x * z + w * y);
  R[3] = 2.0f * (x * y + w * z);
  R[4] = 1.0f - 2.0f * (x * x + z * z);
  R[5] = 2.0f * (y * z - w * x);
  R[6] = 2.0f * (x * z - w * y);
  R[7] = 2.0f * (y * z + w * x);
  R[8] = 1.0f - 2.0f * (x * x + y * y);
}

// Frame coordinates R^T (x - c).
__device__ __forceinline__ void obb_local(const float R[9], float4 c, float4 x, float r[3]) {
  const float d[3] = {x.x - c.x, x.y - c.y, x.z - c.z};
#pragma unroll
  for (int k = 0; k < 3; ++k) r[k] = (R[k] * d[0] + R[3 + k] * d[1]) + R[6 + k] * d[2];
}

// Oriented box of body b (one warp): frame from its warm-start rotation
// (normalised; identity before the first iteration), centre = anchor, and the
// exact bounds of its particles' X~ in that frame. Any frame bounds the body;
// a frame that follows its rotation bounds it tightly.
__device__ __forceinline__ void body_obb(const NearArgs& A, int t, int lane) {
  const int b = A.list ? A.list[t] : t;
  if (A.npartners[b] == 0 || (A.role && A.role[b] == 0)) return;
  float4 q = A.rquat[b];
  const float n2 = (q.x * q.x + q.y * q.y) + (q.z * q.z + q.w * q.w);
  if (!(n2 > 0.0f) || !isfinite(n2)) {
    q = make_float4(1.0f, 0.0f, 0.0f, 0.0f);
  } else {
    const float inv = rsqrtf(n2);
    q = make_float4(q.x * inv, q.y * inv, q.z * inv, q.w * inv);
  }
  const float4 c = A.anchor[b];
  float R[9];
  obb_axes(q, R);
  const int4 bd = A.body_desc[b];
  float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int qd = lane; qd < bd.y; qd += 32) {
    float r[3];
    obb_local(R, c, A.pos[bd.x + qd], r);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      lo[k] = fminf(lo[k], r[k]);
      hi[k] = fmaxf(hi[k], r[k]);
    }
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1)
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      lo[k] = fminf(lo[k], __shfl_xor_sync(kFull, lo[k], off));
      hi[k] = fmaxf(hi[k], __shfl_xor_sync(kFull, hi[k], off));
    }
  if (lane == 0) {
    A.obb_q[b] = q;
    A.obb_c[b] = c;
    A.obb_lo[b] = make_float4(lo[0], lo[1], lo[2], 0.0f);
    A.obb_hi[b] = make_float4(hi[0], hi[1], hi[2], 0.0f);
  }
}

__global__ void __launch_bounds__(256) k_body_obb(NearArgs A) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < A.nbl; t += nw)  // warp-uniform
    body_obb(A, t, lane);
}

// Inside partner o's oriented box inflated by h: a candidate j of o lies in
// o's box and within h of x (|R^T e|_inf <= |e|_2 for a rotation), with the
// inflation enlarged far beyond fp32 rounding of the frame coordinates.
__device__ __forceinline__ bool in_obb(const NearArgs& A, int o, float4 x) {
  const float4 lo = A.obb_lo[o], hi = A.obb_hi[o];
  float R[9];
  obb_axes(A.obb_q[o], R);
  float r[3];
  obb_local(R, A.obb_c[o], x, r);
  const float lv[3] = {lo.x, lo.y, lo.z}, hv[3] = {hi.x, hi.y, hi.z};
  bool in = true;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float m = A.inflate * 1.0001f + 1e-5f * (fabsf(lv[k]) + fabsf(hv[k])) + 1e-6f;
    in = in && r[k] >= lv[k] - m && r[k] <= hv[k] + m;
  }
  return in;
}

// Near test of particle slot p against the np partner boxes held by lanes
// (axis-aligned; then oriented when available).
__device__ __forceinline__ bool near_test(const NearArgs& A, bool valid, float4 xi, int np, const NearBoxes& bx,
                                          const int* partners) {
  bool in_any = false;
  for (int k = 0; k < np; ++k) {
    float lo[3], hi[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      lo[c] = __shfl_sync(kFull, bx.lo[c], k);
      hi[c] = __shfl_sync(kFull, bx.hi[c], k);
    }
    bool in = xi.x >= lo[0] && xi.x <= hi[0] && xi.y >= lo[1] && xi.y <= hi[1] && xi.z >= lo[2] && xi.z <= hi[2];
#if PBDR_NEAR_FAST
    // Oriented test with the partner's prepared frame, only when some lane
    // is inside the axis-aligned box; the warp stops once every lane is near.
    if (A.obb_q && __any_sync(kFull, in)) {
      float R[9], c[3], ol[3], oh[3];
#pragma unroll
      for (int e = 0; e < 9; ++e) R[e] = __shfl_sync(kFull, bx.R[e], k);
#pragma unroll
      for (int e = 0; e < 3; ++e) {
        c[e] = __shfl_sync(kFull, bx.c[e], k);
        ol[e] = __shfl_sync(kFull, bx.olo[e], k);
        oh[e] = __shfl_sync(kFull, bx.ohi[e], k);
      }
      const float d[3] = {xi.x - c[0], xi.y - c[1], xi.z - c[2]};
#pragma unroll
      for (int e = 0; e < 3; ++e) {
        const float r = (R[e] * d[0] + R[3 + e] * d[1]) + R[6 + e] * d[2];
        in = in && r >= ol[e] && r <= oh[e];
      }
    }
    in_any = in_any || in;
    if (__all_sync(kFull, in_any || !valid)) break;
#else
    if (in && A.obb_q) in = in_obb(A, partners[k], xi);
    in_any = in_any || in;
#endif
  }
  return valid && in_any;
}

// SPLIT warps per body (scenes of few bodies: config 3's 8192 bodies are
// 0.9 waves of warps at one warp per body, and a 1000-particle body with 15
// partners is a 19K-instruction serial loop): warp `sub` of a body takes
// every SPLIT-th chunk of 32 particles and adds its count to the body's
// (integer atomics on a zeroed array: the total does not depend on order).
template <int SPLIT>
__global__ void __launch_bounds__(256) k_near_count(NearArgs A) {
  const int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int t = wg / SPLIT, sub = wg % SPLIT;
  const int lane = threadIdx.x & 31;
  if (t >= A.nbl) return;  // warp-uniform
  int b, start, n;
  NearBoxes bx{};
  const int np = near_body_setup(A, t, lane, b, start, n, bx);
  uint32_t cnt = 0;
  if (np < 0) {
    cnt = sub == 0 ? static_cast<uint32_t>(n) : 0u;
  } else if (np > 0) {
    // The next chunk's positions are requested before this chunk is tested
    // (two loads in flight per warp: the loop is a chain of HBM round trips).
    auto load_x = [&](int base) {
      const int q = base + lane;
      return q < n ? A.pos[start + static_cast<int64_t>(q)] : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    };
    float4 xnext = load_x(32 * sub);
    for (int base = 32 * sub; base < n; base += 32 * SPLIT) {
      const int q = base + lane;
      const int64_t p = start + static_cast<int64_t>(q);
      const float4 xi = xnext;
      xnext = load_x(base + 32 * SPLIT);
      const bool near = near_test(A, q < n, xi, np, bx, A.partners + static_cast<int64_t>(b) * PBDR_PARTNER_CAP);
      if (q < n) A.near_flag[p] = near ? 1 : 0;  // k_near_write reuses the test
      cnt += __popc(__ballot_sync(kFull, near));
    }
  }
  if (lane == 0) {
    if (SPLIT == 1)
      A.body_near[t] = cnt;
    else if (cnt != 0u)
      atomicAdd(&A.body_near[t], cnt);
  }
}

__global__ void __launch_bounds__(256) k_near_write(NearArgs A) {
  const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= A.nbl) return;
  if (A.body_near[t] == 0u) return;  // warp-uniform
  const int b = A.list ? A.list[t] : t;
  const int4 bd = A.body_desc[b];
  const int start = bd.x, n = bd.y;
  const bool all = A.all_near || A.npartners[b] < 0;  // the count kernel took the same branch
  uint32_t off = A.body_off[t] + A.tile_off[t / kScanTile];
  for (int base = 0; base < n; base += 32) {
    const int q = base + lane;
    const int64_t p = start + static_cast<int64_t>(q);
    const bool near = q < n && (all || A.near_flag[p] != 0);
    const unsigned bal = __ballot_sync(kFull, near);
    if (near) {
      const uint32_t o = off + __popc(bal & ((1u << lane) - 1u));
      PBDR_CHECK(o < static_cast<uint32_t>(*A.count));
      A.near_list[o] = static_cast<int>(p);
      A.keys_c[o] = A.key_all[p];
      A.vals_c[o] = static_cast<uint32_t>(p);
    }
    off += __popc(bal);
  }
}

// Exclusive scan of the body near counts in two levels: k_near_scan_tiles
// scans tiles of 4096 counts (one CTA each, four consecutive counts per
// thread) and stores the tile totals; k_near_scan_top scans the tile totals
// (one CTA) and writes the near total; k_near_write adds the tile offset.
__device__ __forceinline__ uint32_t block_exclusive_scan_1024(uint32_t v, uint32_t* s_warp, uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, incl, off);
    if (lane >= off) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const uint32_t w = s_warp[lane];
    uint32_t wi = w;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, wi, off);
      if (lane >= off) wi += y;
    }
    s_warp[lane] = wi - w;
    if (lane == 31) *total = wi;
  }
  __syncthreads();
  return s_warp[warp] + (incl - v);
}

__global__ void __launch_bounds__(1024) k_near_scan_tiles(NearArgs A) {
  __shared__ uint32_t s_warp[32];
  __shared__ uint32_t s_total;
  const int i0 = blockIdx.x * kScanTile + 4 * threadIdx.x;
  uint32_t c[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) c[i] = (i0 + i < A.nbl) ? A.body_near[i0 + i] : 0u;
  const uint32_t sum = (c[0] + c[1]) + (c[2] + c[3]);
  uint32_t run = block_exclusive_scan_1024(sum, s_warp, &s_total);
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (i0 + i < A.nbl) {
      A.body_off[i0 + i] = run;
      run += c[i];
    }
  if (threadIdx.x == 0) A.tile_sum[blockIdx.x] = s_total;
}

__global__ void __launch_bounds__(1024) k_near_scan_top(NearArgs A) {
  __shared__ uint32_t s_warp[32];
  __shared__ uint32_t s_total;
  const int tiles = (A.nbl + kScanTile - 1) / kScanTile;  // <= 1024 (bodies < 4M)
  const uint32_t v = static_cast<int>(threadIdx.x) < tiles ? A.tile_sum[threadIdx.x] : 0u;
  const uint32_t ex = block_exclusive_scan_1024(v, s_warp, &s_total);
  if (static_cast<int>(threadIdx.x) < tiles) A.tile_off[threadIdx.x] = ex;
  if (threadIdx.x == 0) *A.count = static_cast<long long>(s_total);
}

// Candidate counts are only written for near particles (k_neighbours); the
// previous substep's near particles are reset to 0 first, so every particle
// outside the current near list reads 0 -- O(near) writes instead of O(N).
__global__ void __launch_bounds__(256) k_ncand_clear(int* ncand, const int* prev_near, const long long* prev_count) {
  const long long m = *prev_count;  // device-side count: grid-stride over a fixed grid
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < m;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x)
    ncand[prev_near[t]] = 0;
}

// Resets the buckets the previous substep wrote (instead of a full memset).
__global__ void __launch_bounds__(256) k_cell_clear(uint4* cells, const uint32_t* prev_keys,
                                                    const long long* prev_count) {
  const long long m = *prev_count;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < m;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x)
    cells[prev_keys[t]].x = kEmpty;  // keys are masked hashes: always inside the table
}

// ---------------------------------------------------------------------------
// contact candidates (pinned P4): {j : same scene, other body,
// |cell_j - cell_i|_inf <= 1, |x~_i - x~_j|^2 < h^2}, ascending j, <= CAP.
// ---------------------------------------------------------------------------
struct CandList {
  int j[PBDR_NBR_CAP];
  int count;
  bool overflow;
  // Sorted insert of a distinct j; keeps the CAP smallest.
  __device__ __forceinline__ void insert(int v) {
    int pos = count;
    while (pos > 0 && j[pos - 1] > v) --pos;
    if (pos > 0 && j[pos - 1] == v) return;  // seen through an aliased bucket
    if (count == PBDR_NBR_CAP) {
      overflow = true;
      if (pos == PBDR_NBR_CAP) return;
      --count;
    }
    for (int t = count; t > pos; --t) j[t] = j[t - 1];
    j[pos] = v;
    ++count;
  }
};

__device__ __forceinline__ void scan_range(const NeighbourArgs& A, uint32_t lo, uint32_t hi, int bi, int si,
                                           float4 xi, int32_t cx, int32_t cy, int32_t cz, CandList& L) {
  PBDR_CHECK(lo <= hi && hi <= static_cast<uint64_t>(*A.count));
  for (uint32_t s = lo; s < hi; ++s) {
    // Body, slot and position of the entry come from sorted-order copies
    // (k_cell_ranges), read side by side: no dependent gathers per entry.
    const float4 xj = A.sorted_pos[s];
    const int bj = __float_as_int(xj.w);
    if (bj == bi) continue;
    if (!A.single_scene && A.body_scene[bj] != si) continue;
    const int j = static_cast<int>(A.sorted_vals[s]);
    const int32_t jx = pbdr_cell_coord(xj.x, A.inv_h);
    const int32_t jy = pbdr_cell_coord(xj.y, A.inv_h);
    const int32_t jz = pbdr_cell_coord(xj.z, A.inv_h);
    if (jx < cx - 1 || jx > cx + 1 || jy < cy - 1 || jy > cy + 1 || jz < cz - 1 || jz > cz + 1) continue;
    const float ex = xi.x - xj.x, ey = xi.y - xj.y, ez = xi.z - xj.z;
    const float d2 = (ex * ex + ey * ey) + ez * ez;
    if (!(d2 < A.h2)) continue;
    L.insert(j);
  }
}

// Scans one bucket unless it is empty or holds only particle i's own body.
__device__ __forceinline__ void scan_bucket(const NeighbourArgs& A, uint32_t key, int bi, int si, float4 xi,
                                            int32_t cx, int32_t cy, int32_t cz, CandList& L) {
  const uint4 e = A.cells[key];
  if (e.x == kEmpty) return;
  if (e.z == static_cast<uint32_t>(bi) && e.w == static_cast<uint32_t>(bi)) return;
  scan_range(A, e.x, e.y, bi, si, xi, cx, cy, cz, L);
}

// PBDR_NBR_ROW_LOADS: a stencil row's three bucket heads are loaded together
// (landed C5 neighbour search 7.97 -> 7.30 ms per frame).
#ifndef PBDR_NBR_ROW_LOADS
#define PBDR_NBR_ROW_LOADS 1
#endif
__device__ __forceinline__ void scan_bucket_e(const NeighbourArgs& A, uint4 e, int bi, int si, float4 xi,
                                              int32_t cx, int32_t cy, int32_t cz, CandList& L) {
  if (e.x == kEmpty) return;
  if (e.z == static_cast<uint32_t>(bi) && e.w == static_cast<uint32_t>(bi)) return;
  scan_range(A, e.x, e.y, bi, si, xi, cx, cy, cz, L);
}

__device__ __forceinline__ void neighbours_one(const NeighbourArgs& A, int64_t t) {
  // Near particles in sorted (cell-key) order: neighbouring threads search
  // overlapping cells, so bucket entries are shared through L1/L2.
  const int64_t i = A.sorted_vals[t];
  PBDR_CHECK(i >= 0 && i < A.n);
  const float4 xi = A.sorted_pos[t];  // X~ of particle i, its body in .w
  const int bi = __float_as_int(xi.w);
  const int si = A.single_scene ? 0 : A.body_scene[bi];
  const int32_t cx = pbdr_cell_coord(xi.x, A.inv_h);
  const int32_t cy = pbdr_cell_coord(xi.y, A.inv_h);
  const int32_t cz = pbdr_cell_coord(xi.z, A.inv_h);
  const int xl = cx & ((1 << PBDR_XRUN_BITS) - 1);
  const bool linear = A.layout.linear != 0;
  // Consecutive keys for the row's three cells: inside an x-run (hashed
  // layout) or inside the box's x range (linear layout).
  const bool inner = linear ? static_cast<uint32_t>(cx - 1 - A.layout.ox) + 2u < (1u << A.layout.bx)
                            : (xl != 0 && xl != (1 << PBDR_XRUN_BITS) - 1);

  CandList L;
  L.count = 0;
  L.overflow = false;
  for (int r = 0; r < 9; ++r) {
    const int32_t yy = cy + (r % 3) - 1, zz = cz + (r / 3) - 1;
    // Row cells cx-1, cx, cx+1: consecutive keys inside an x-run.
    const uint32_t km = pbdr_cell_key(cx - 1, yy, zz, static_cast<uint32_t>(si), A.mask, A.layout);
    const uint32_t k0 = inner ? (km + 1) & A.mask : pbdr_cell_key(cx, yy, zz, static_cast<uint32_t>(si), A.mask, A.layout);
    const uint32_t kp = inner ? (km + 2) & A.mask : pbdr_cell_key(cx + 1, yy, zz, static_cast<uint32_t>(si), A.mask, A.layout);
#if PBDR_NBR_ROW_LOADS
    // The row's three bucket heads requested together (one line when the
    // keys are consecutive) before any of them is scanned.
    const uint4 em = A.cells[km], e0 = A.cells[k0], ep = A.cells[kp];
    scan_bucket_e(A, em, bi, si, xi, cx, cy, cz, L);
    scan_bucket_e(A, e0, bi, si, xi, cx, cy, cz, L);
    scan_bucket_e(A, ep, bi, si, xi, cx, cy, cz, L);
#else
    scan_bucket(A, km, bi, si, xi, cx, cy, cz, L);
    scan_bucket(A, k0, bi, si, xi, cx, cy, cz, L);
    scan_bucket(A, kp, bi, si, xi, cx, cy, cz, L);
#endif
  }
  if (L.overflow) record_error(A.err, PBDR_DEVERR_NBR_OVERFLOW, bi, A.substep_counter);
  A.ncand[i] = L.count;
  const float ri = A.rest[i].w;
  for (int k = 0; k < L.count; ++k) {
    const int j = L.j[k];
    A.cand_j[static_cast<int64_t>(k) * A.n + i] = j;
    A.cand_rr[static_cast<int64_t>(k) * A.n + i] = ri + A.rest[j].w;
  }
}

// Grid-stride over the device-side near count (the launch is sized for the
// worst case, so a fixed grid avoids launching N mostly-idle threads).
__global__ void __launch_bounds__(128) k_neighbours(NeighbourArgs A) {
  const long long m = *A.count;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < m;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x)
    neighbours_one(A, t);
}

// Staged search (single scenes with the linear key layout, P4). With linear
// keys a stencil row -- cells (cx-1..cx+1, y, z) -- is three consecutive keys,
// so its bucket entries are one contiguous run of the sorted arrays; and a
// CTA's chunk of kNbrChunk consecutive sorted near particles (one x-stretch of
// a few cell rows) needs, for each of the 9 (dy, dz) row offsets, one run of
// entries that is about as long as the chunk. The CTA reduces the 9 runs'
// bounds over its threads, merges overlapping runs, and stages them into
// shared memory with cp.async.bulk (one mbarrier); every thread then scans
// its rows from shared memory. Rows that are not three consecutive keys (the
// box's x edge, key wrap-around) or runs beyond the staging capacity are read
// from global memory bucket by bucket as in k_neighbours. The scanned entries
// are the same, and the candidate list keeps the CAP smallest distinct j
// whatever the order, so the result is bit-identical to k_neighbours.
#ifndef PBDR_NBR_STAGED
#define PBDR_NBR_STAGED 0
#endif
constexpr int kNbrChunk = 128;
constexpr int kNbrStage = 2048;  // staged entries per CTA (32 KB of float4)

__global__ void __launch_bounds__(kNbrChunk) k_neighbours_staged(NeighbourArgs A) {
  __shared__ __align__(16) float4 s_ent[kNbrStage];
  __shared__ __align__(8) uint64_t s_bar;
  __shared__ uint32_t s_lo[9], s_hi[9];
  __shared__ int s_base[9];  // shared index of entry s_lo[r], or -1 (row read from global)
  const long long m = *A.count;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) mbar_init(&s_bar, 1);
  __syncthreads();
  uint32_t parity = 0;
  for (int64_t c0 = static_cast<int64_t>(blockIdx.x) * kNbrChunk; c0 < m;
       c0 += static_cast<int64_t>(gridDim.x) * kNbrChunk, parity ^= 1u) {
    if (threadIdx.x < 9) {
      s_lo[threadIdx.x] = 0xFFFFFFFFu;
      s_hi[threadIdx.x] = 0u;
    }
    const int64_t t = c0 + threadIdx.x;
    const bool act = t < m;
    int64_t i = 0;
    float4 xi = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    int bi = -1;
    int32_t cx = 0, cy = 0, cz = 0;
    if (act) {
      i = A.sorted_vals[t];
      PBDR_CHECK(i >= 0 && i < A.n);
      xi = A.sorted_pos[t];
      bi = __float_as_int(xi.w);
      cx = pbdr_cell_coord(xi.x, A.inv_h);
      cy = pbdr_cell_coord(xi.y, A.inv_h);
      cz = pbdr_cell_coord(xi.z, A.inv_h);
    }
    const bool xin = static_cast<uint32_t>(cx - 1 - A.layout.ox) + 2u < (1u << A.layout.bx);
    // Per row: the contiguous run [lo, hi) of its three buckets (empty: lo =
    // hi = 0; not contiguous: lo = ~0, read bucket by bucket from global).
    uint32_t lo[9], hi[9];
    __syncthreads();  // s_lo / s_hi reset before the reductions below
#pragma unroll
    for (int r = 0; r < 9; ++r) {
      lo[r] = 0u;
      hi[r] = 0u;
      if (act) {
        const int32_t yy = cy + (r % 3) - 1, zz = cz + (r / 3) - 1;
        const uint32_t km = pbdr_cell_key(cx - 1, yy, zz, 0u, A.mask, A.layout);
        if (xin && km + 2u <= A.mask) {
          const uint4 e0 = A.cells[km], e1 = A.cells[km + 1], e2 = A.cells[km + 2];
          const bool n0 = e0.x != kEmpty, n1 = e1.x != kEmpty, n2 = e2.x != kEmpty;
          const uint32_t ub = static_cast<uint32_t>(bi);
          const bool own = (!n0 || (e0.z == ub && e0.w == ub)) && (!n1 || (e1.z == ub && e1.w == ub)) &&
                           (!n2 || (e2.z == ub && e2.w == ub));
          if ((n0 || n1 || n2) && !own) {
            lo[r] = n0 ? e0.x : (n1 ? e1.x : e2.x);
            hi[r] = n2 ? e2.y : (n1 ? e1.y : e0.y);
          }
        } else {
          lo[r] = 0xFFFFFFFFu;
        }
      }
      const bool has = lo[r] < hi[r];
      const uint32_t wl = __reduce_min_sync(kFull, has ? lo[r] : 0xFFFFFFFFu);
      const uint32_t wh = __reduce_max_sync(kFull, has ? hi[r] : 0u);
      if (lane == 0 && wl < wh) {
        atomicMin(&s_lo[r], wl);
        atomicMax(&s_hi[r], wh);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      // Merge the 9 runs (sorted by start) into disjoint segments, stage the
      // segments that fit, in ascending order.
      int ord[9], nr = 0;
      for (int r = 0; r < 9; ++r) {
        s_base[r] = -1;
        if (s_lo[r] < s_hi[r]) {
          int k = nr++;
          while (k > 0 && s_lo[ord[k - 1]] > s_lo[r]) {
            ord[k] = ord[k - 1];
            --k;
          }
          ord[k] = r;
        }
      }
      uint32_t bytes = 0;
      int used = 0;
      for (int a = 0; a < nr;) {
        uint32_t seg_lo = s_lo[ord[a]], seg_hi = s_hi[ord[a]];
        int b = a + 1;
        while (b < nr && s_lo[ord[b]] <= seg_hi) {
          seg_hi = max(seg_hi, s_hi[ord[b]]);
          ++b;
        }
        const int len = static_cast<int>(seg_hi - seg_lo);
        if (used + len <= kNbrStage) {
          for (int k = a; k < b; ++k) s_base[ord[k]] = used + static_cast<int>(s_lo[ord[k]] - seg_lo);
          bulk_g2s(&s_ent[used], A.sorted_pos + seg_lo, static_cast<uint32_t>(len) * 16u, &s_bar);
          used += len;
          bytes += static_cast<uint32_t>(len) * 16u;
        }
        a = b;
      }
      mbar_expect_tx(&s_bar, bytes);  // arrives once; the phase completes when the bytes have landed
    }
    __syncthreads();  // s_base published
    mbar_wait(&s_bar, parity);
    if (act) {
      CandList L;
      L.count = 0;
      L.overflow = false;
#pragma unroll 1
      for (int r = 0; r < 9; ++r) {
        if (lo[r] == 0xFFFFFFFFu) {  // row not contiguous: bucket by bucket from global
          const int32_t yy = cy + (r % 3) - 1, zz = cz + (r / 3) - 1;
          for (int dx = -1; dx <= 1; ++dx)
            scan_bucket(A, pbdr_cell_key(cx + dx, yy, zz, 0u, A.mask, A.layout), bi, 0, xi, cx, cy, cz, L);
          continue;
        }
        if (lo[r] >= hi[r]) continue;
        const int base = s_base[r];
        if (base < 0) {
          scan_range(A, lo[r], hi[r], bi, 0, xi, cx, cy, cz, L);
          continue;
        }
        const uint32_t r0 = s_lo[r];
        for (uint32_t s = lo[r]; s < hi[r]; ++s) {
          const float4 xj = s_ent[base + static_cast<int>(s - r0)];
          if (__float_as_int(xj.w) == bi) continue;
          const int32_t jx = pbdr_cell_coord(xj.x, A.inv_h);
          const int32_t jy = pbdr_cell_coord(xj.y, A.inv_h);
          const int32_t jz = pbdr_cell_coord(xj.z, A.inv_h);
          if (jx < cx - 1 || jx > cx + 1 || jy < cy - 1 || jy > cy + 1 || jz < cz - 1 || jz > cz + 1) continue;
          const float ex = xi.x - xj.x, ey = xi.y - xj.y, ez = xi.z - xj.z;
          const float d2 = (ex * ex + ey * ey) + ez * ez;
          if (!(d2 < A.h2)) continue;
          L.insert(static_cast<int>(A.sorted_vals[s]));
        }
      }
      if (L.overflow) record_error(A.err, PBDR_DEVERR_NBR_OVERFLOW, bi, A.substep_counter);
      A.ncand[i] = L.count;
      const float ri = A.rest[i].w;
      for (int k = 0; k < L.count; ++k) {
        const int j = L.j[k];
        A.cand_j[static_cast<int64_t>(k) * A.n + i] = j;
        A.cand_rr[static_cast<int64_t>(k) * A.n + i] = ri + A.rest[j].w;
      }
    }
    __syncthreads();  // staged entries read before the next chunk's copies overwrite them
  }
}

// ---------------------------------------------------------------------------
// One solver iteration, fused (pinned P1-P8). A CTA (8 warps) holds whole,
// consecutive bodies; its contiguous slot range of pos/vel/rest is staged in
// shared memory by three cp.async.bulk copies. A body of n particles owns
// W = ceil(n/(32 KP)) warps (KP = the scene's tile shape); lane l of body-warp
// wi owns q = k*32*W + wi*32 + l, k < KP. Warp 0 runs the per-body fp64 math
// for all bodies of the CTA, one lane per body. The same kernel runs one
// iteration per launch, all iterations of a substep on chip (MULTI: isolated
// tiles, one-wave cooperative grids, or one cluster per batched scene), and
// -- FUSE -- the substep's last iteration followed by the next integrate.
// ---------------------------------------------------------------------------
// PBDR_COST_PROBE (timing experiments only, results are wrong): bit 0 skips
// the polar, bit 1 the inertia solve -- what the per-body fp64 math costs.
#ifndef PBDR_GN_PROBE
#define PBDR_GN_PROBE 0
#endif
#ifndef PBDR_COST_PROBE
#define PBDR_COST_PROBE 0
#endif
// PBDR_CAND_ROLLED: keep the candidate loop rolled. The compiler otherwise
// unrolls it 4x for each of the KP particles of a lane: 10% more code, and
// the instruction-cache misses that costs (ncu: no_instruction stalls) are
// worth more than the extra loads in flight -- landed C5 iteration 245 -> 213
// ms per frame, C3 +4%, C4 +1%, bit-identical (tools/ab_landed.py, r02).
// PBDR_INTILE_SMEM: contact candidates inside the tile read X_j from the
// staged shared-memory copy.
#ifndef PBDR_INTILE_SMEM
#define PBDR_INTILE_SMEM 0
#endif
#ifndef PBDR_CAND_ROLLED
#define PBDR_CAND_ROLLED 1
#endif
// PBDR_PREFETCH_NEXT: after phase A, one lane pulls the next tile's staging
// ranges (pos, vel, rest) and its candidate counts into L2.
#ifndef PBDR_PREFETCH_NEXT
#define PBDR_PREFETCH_NEXT 0
#endif
// PBDR_DESC_SMEM: the next tile's descriptors are copied into shared memory
// by cp.async instead of being loaded into registers one tile ahead (ncu: 6%
// of the landed-C5 stall samples sat on those loads' first uses).
#ifndef PBDR_DESC_SMEM
#define PBDR_DESC_SMEM 1
#endif
// PBDR_ANCHOR_EARLY: body math A publishes the new anchor before the polar.
// PBDR_PREFETCH_COUNTS: after phase A the next tile's candidate counts and
// first-candidate rows are prefetched into L2.
#ifndef PBDR_PREFETCH_COUNTS
#define PBDR_PREFETCH_COUNTS 1
#endif
#ifndef PBDR_ANCHOR_EARLY
#define PBDR_ANCHOR_EARLY 1
#endif
// PBDR_PREFETCH_ALL_CANDS: the staging-time prefetch covers every candidate
// of a particle, not only the first.
#ifndef PBDR_PREFETCH_ALL_CANDS
#define PBDR_PREFETCH_ALL_CANDS 0
#endif
// Pinned fused multiply-adds (P8): only these explicit fmaf() are
// contracted (the library builds with --fmad=false); the oracle uses std::fmaf
// at the same places, and IEEE fma is correctly rounded on both sides.
__device__ __forceinline__ float dot3_fma(const float a[3], const float b[3]) {
  return fmaf(a[2], b[2], fmaf(a[1], b[1], a[0] * b[0]));
}
__device__ __forceinline__ void cross3_fma(const float a[3], const float b[3], float o[3]) {
  o[0] = fmaf(a[1], b[2], -(a[2] * b[1]));
  o[1] = fmaf(a[2], b[0], -(a[0] * b[2]));
  o[2] = fmaf(a[0], b[1], -(a[1] * b[0]));
}

// One particle-particle contact of particle i (slot p, X_i = x, inverse mass
// w) against candidate j: Jacobi delta accumulated into dPP.
__device__ __forceinline__ void pp_contact(const float x[3], float w, int64_t p, float4 xj, int j, float rr,
                                           float relax, float dPP[3]) {
  const float e[3] = {x[0] - xj.x, x[1] - xj.y, x[2] - xj.z};
  const float d2 = dot3_fma(e, e);
  if (d2 < rr * rr) {
    const float dist = sqrtf(d2);
    float nrm[3];
    if (dist > PBDR_COINCIDENT_EPS) {
      const float inv = 1.0f / dist;
      nrm[0] = e[0] * inv; nrm[1] = e[1] * inv; nrm[2] = e[2] * inv;
    } else {
      nrm[0] = p < j ? 1.0f : -1.0f; nrm[1] = 0.0f; nrm[2] = 0.0f;
    }
    const float C = dist - rr;
    const float kk = (relax * (w / (w + xj.w))) * C;
    dPP[0] = fmaf(-kk, nrm[0], dPP[0]);
    dPP[1] = fmaf(-kk, nrm[1], dPP[1]);
    dPP[2] = fmaf(-kk, nrm[2], dPP[2]);
  }
}

// Barrier between the iterations of a multi-iteration launch with pairs: the
// whole grid (cooperative launch, one-wave scenes) or the CTA cluster that
// holds one batched scene (multi_pairs == 2; candidates never leave a scene,
// pinned P4). Both release this CTA's X_{i+1} stores (L2) and acquire the
// others' before the next iteration's gathers.
__device__ __forceinline__ void multi_barrier(const IterArgs& A) {
  if (A.multi_pairs == 2)
    cooperative_groups::this_cluster().sync();
  else
    cooperative_groups::this_grid().sync();
}

// Phase A of one particle (slot p; X_i = x4, V = v4, rest = r4, nc candidates):
// ground/wall contacts with friction, Jacobi particle contacts, and the
// particle's terms of the 21 bsm body sums (com, dX, Apq, P_bsm, L_bsm).
template <bool MULTI>
__device__ __forceinline__ void phase_a_particle(const IterArgs& A, int it, int64_t p, float4 x4, float4 v4,
                                                 float4 r4, int nc, const float a[3], float (&dXk)[3],
                                                 float (&acc)[21], const float4* s_tile, int tile_first,
                                                 int tile_count, const float* dpp_pre = nullptr) {
  const float x[3] = {x4.x, x4.y, x4.z};
  const float m = v4.w;

  float dPG[3] = {0.0f, 0.0f, 0.0f};
  // Kept rolled: unrolled plane tests cost the KP = 4 kernels registers (and
  // spills) for every particle (C3 +5%, C5 +4% rolled).
#pragma unroll 1
  for (int pl = 0; pl < A.planes.count; ++pl) {
    const float* Pp = A.planes.p[pl];
    const float* Pn = A.planes.n[pl];
    const float xp[3] = {x[0] - Pp[0], x[1] - Pp[1], x[2] - Pp[2]};
    const float d = dot3_fma(xp, Pn) - r4.w;
    if (d < 0.0f) {
      const float push = -(A.relax * d);
      dPG[0] = fmaf(push, Pn[0], dPG[0]);
      dPG[1] = fmaf(push, Pn[1], dPG[1]);
      dPG[2] = fmaf(push, Pn[2], dPG[2]);
      const float mu = A.planes.mu[pl];
      if (mu > 0.0f) {
        const float4 xi = A.init[p];
        const float t[3] = {x[0] - xi.x, x[1] - xi.y, x[2] - xi.z};
        const float tn = dot3_fma(t, Pn);
        const float tt[3] = {fmaf(-tn, Pn[0], t[0]), fmaf(-tn, Pn[1], t[1]), fmaf(-tn, Pn[2], t[2])};
        const float len2 = dot3_fma(tt, tt);
        if (len2 > 0.0f) {
          const float len = sqrtf(len2);
          const float lim = mu * (-d);
          if (len <= lim) {
            dPG[0] = dPG[0] - tt[0];
            dPG[1] = dPG[1] - tt[1];
            dPG[2] = dPG[2] - tt[2];
          } else {
            const float fr = lim / len;
            dPG[0] = fmaf(-tt[0], fr, dPG[0]);
            dPG[1] = fmaf(-tt[1], fr, dPG[1]);
            dPG[2] = fmaf(-tt[2], fr, dPG[2]);
          }
        }
      }
    }
  }
  float dPP[3] = {0.0f, 0.0f, 0.0f};
  if (dpp_pre) {  // contacts already summed (PBDR_CAND_COLUMNS), same order
    dPP[0] = dpp_pre[0];
    dPP[1] = dpp_pre[1];
    dPP[2] = dpp_pre[2];
    nc = 0;
  }
#if PBDR_CAND_ROLLED
#pragma unroll 1
#endif
  for (int c = 0; c < nc; ++c) {
    const int j = A.cand_j[static_cast<int64_t>(c) * A.n + p];
    PBDR_CHECK(c < PBDR_NBR_CAP && j >= 0 && j < A.n && j != p);
#ifdef PBDR_RR_UNIFORM  // A/B probe only: every contact radius sum is this constant
    const float rr = PBDR_RR_UNIFORM;
#else
    const float rr = A.cand_rr[static_cast<int64_t>(c) * A.n + p];
#endif
    // Multi-iteration launch with pairs: neighbours' X_i come from the
    // buffer the previous iteration wrote (after a grid barrier; L2 only).
#if PBDR_INTILE_SMEM
    // Candidates in this tile's own slot range are read from the staged X_i
    // in shared memory (identical values: the same snapshot) instead of L2.
    const uint32_t jt = static_cast<uint32_t>(j - tile_first);
    const float4 xj = jt < static_cast<uint32_t>(tile_count)
                          ? s_tile[jt]
                          : ((MULTI && A.multi_pairs) ? __ldcg(&A.pos_b[it & 1][j]) : A.pos_in[j]);
#else
    (void)s_tile; (void)tile_first; (void)tile_count;
    const float4 xj = (MULTI && A.multi_pairs) ? __ldcg(&A.pos_b[it & 1][j]) : A.pos_in[j];
#endif
    pp_contact(x, x4.w, p, xj, j, rr, A.relax, dPP);
  }
  const float v[3] = {v4.x, v4.y, v4.z};
  const float q0[3] = {r4.x, r4.y, r4.z};
  // Body sums: product fields accumulate with one fma per particle (the
  // first stage of the pinned reduction tree), cross products are summed.
  float pp[3], pb[3], mp[3], vb[3], mvb[3], kb[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    dXk[c] = dPG[c] + dPP[c];
    pp[c] = x[c] - a[c];
    pb[c] = pp[c] + dXk[c];
    vb[c] = fmaf(dXk[c], A.inv_dt, v[c]);
    mp[c] = m * pp[c];
    mvb[c] = m * vb[c];
  }
  cross3_fma(pb, mvb, kb);
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    acc[c] = fmaf(m, pp[c], acc[c]);
    acc[3 + c] = fmaf(m, dXk[c], acc[3 + c]);
    acc[15 + c] = fmaf(m, vb[c], acc[15 + c]);
    acc[18 + c] = acc[18 + c] + kb[c];
  }
#pragma unroll
  for (int rI = 0; rI < 3; ++rI)
#pragma unroll
    for (int cI = 0; cI < 3; ++cI) acc[6 + 3 * rI + cI] = fmaf(mp[rI], q0[cI], acc[6 + 3 * rI + cI]);
}

// Final state of one particle in a launch that ends the substep: X and V
// out, or -- with fuse -- the next substep's integrate on them (the integrate
// kernel's arithmetic): X~ and V~ out, X_init and the cell key, the body box
// folded into lo/hi (ordered uints) for warp_box_commit.
__device__ __forceinline__ void store_final(const IterArgs& A, int64_t p, int b, float4 xo, float4 vo, bool fuse,
                                            uint32_t (&lo)[3], uint32_t (&hi)[3]) {
  if (!fuse) {
    A.pos_out[p] = xo;
    A.vel[p] = vo;
    return;
  }
  float4 xn, vn;
  integrate_one(A.ia, b, xo, vo, xn, vn);
  A.ia.init[p] = make_float4(xo.x, xo.y, xo.z, 0.0f);
  A.pos_out[p] = xn;
  A.vel[p] = vn;
  A.ia.key_all[p] = integrate_key(A.ia, b, xn);
  const uint32_t o[3] = {f2ord(xn.x), f2ord(xn.y), f2ord(xn.z)};
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    lo[c] = min(lo[c], o[c]);
    hi[c] = max(hi[c], o[c]);
  }
}

// The warp's particles (one body) fold into the body box. All lanes.
__device__ __forceinline__ void warp_box_commit(const IterArgs& A, int b, const uint32_t (&lo)[3],
                                                const uint32_t (&hi)[3], int lane) {
  uint32_t l[3], h[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    l[c] = __reduce_min_sync(kFull, lo[c]);
    h[c] = __reduce_max_sync(kFull, hi[c]);
  }
  if (lane == 0)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      atomicMin(&A.ia.box_min[3 * b + c], l[c]);
      atomicMax(&A.ia.box_max[3 * b + c], h[c]);
    }
}

// Cross-warp body sums (stage 3 of the P7 tree): S[f] = ((w0 + w1) + w2) ...
// over the body's warps nw, in warp order. PBDR_PART_VEC reads each warp's
// partials as float4 (rows padded to 24 floats): 6 shared loads instead of
// 21 -- warp 0 runs this while the other CTAs of the SM keep the L1/shared
// pipeline busy with contact gathers, where every load instruction queues.
#ifndef PBDR_PART_VEC
#define PBDR_PART_VEC 1
#endif
#ifndef PBDR_PART_UNROLL
#define PBDR_PART_UNROLL 1
#endif
constexpr int kPartStride = PBDR_PART_VEC ? 24 : 21;
constexpr int kPartUnroll = PBDR_PART_UNROLL;
template <int F>
__device__ __forceinline__ void part_sum(const float* part, int fw, int nw, float (&S)[F]) {
#if PBDR_PART_VEC
  constexpr int V = (F + 3) / 4;
  const float4* r = reinterpret_cast<const float4*>(part + fw * kPartStride);
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const float4 t = r[v];
    const float tv[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (4 * v + e < F) S[4 * v + e] = tv[e];
  }
  // Kept rolled (with the plane loop: smaller code, C3 +5%, C5 +3%).
#pragma unroll kPartUnroll
  for (int u = 1; u < nw; ++u) {
    r = reinterpret_cast<const float4*>(part + (fw + u) * kPartStride);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const float4 t = r[v];
      const float tv[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (4 * v + e < F) S[4 * v + e] = S[4 * v + e] + tv[e];
    }
  }
#else
#pragma unroll
  for (int f = 0; f < F; ++f) S[f] = part[fw * kPartStride + f];
#pragma unroll 1
  for (int u = 1; u < nw; ++u)
#pragma unroll
    for (int f = 0; f < F; ++f) S[f] = S[f] + part[(fw + u) * kPartStride + f];
#endif
}

constexpr int kResF = 32;
constexpr int kTimingSlots = 16;  // debug phase clocks per CTA (pbdr_gpu_debug_phase_timing)
enum ResSlot {
  kResC = 0,      // c (3), anchor-relative com of X_i
  kResLb = 3,     // L_bsm (3)
  kResPb = 6,     // P_bsm (3)
  kResR = 9,      // R (9)
  kResSmOk = 18,  // shape-matching valid flag
  kResCa = 19,    // c_asm (3)
  kResDv = 22,    // dv (3)
  kResW = 25,     // omega (3)
  kResA = 28,     // anchor a (3)
};

// Per-body math A from the 21 bsm sums S of body bb (anchor an, 1/M):
// com c, P_bsm, L_bsm about the predicted com, warm-started polar of Apq;
// results into R (kRes* slots), new anchor and rotation to global memory.
template <bool kStore = true>  // false: the caller stores rquat / anchor (after a cluster barrier)
__device__ __forceinline__ void body_math_a(const IterArgs& A, int bb, const float (&S)[21], float4 an,
                                            float invM, float4 rq4, float* R, float4& rq_new,
                                            float4& an_new, long long* stamp = nullptr,
                                            float4* an_slot = nullptr) {
  bool finite = true;
#pragma unroll
  for (int f = 0; f < 21; ++f) finite = finite && isfinite(S[f]);
  if (!finite) record_error(A.err, PBDR_DEVERR_NONFINITE, bb, A.substep_counter);
  float c[3], cb[3], Pb[3], tmp[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    c[k] = S[k] * invM;
    cb[k] = c[k] + S[3 + k] * invM;
    Pb[k] = S[15 + k];
  }
  cross3(cb, Pb, tmp);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    R[kResC + k] = c[k];
    R[kResPb + k] = Pb[k];
    R[kResLb + k] = S[18 + k] - tmp[k];
  }
  // The new anchor does not depend on the polar: with an_slot (the tile's
  // table entry) it is published now, so that neither it nor an / c stays
  // live (spilled: ncu showed their reloads missing the small L1) across it.
  an_new = make_float4(an.x + c[0], an.y + c[1], an.z + c[2], 0.0f);
  if (kStore && an_slot) {
    A.anchor[bb] = an_new;
    *an_slot = an_new;
  }
  double qd[4];
  const float rq[4] = {rq4.x, rq4.y, rq4.z, rq4.w};
  if (stamp) stamp[0] = clock64();  // debug phase clocks: polar start
#if PBDR_COST_PROBE & 1  // cost probe only (wrong results): no polar, identity rotation
  const bool ok = true;
  qd[0] = 1.0; qd[1] = qd[2] = qd[3] = 0.0;
#pragma unroll
  for (int k = 0; k < 9; ++k) R[kResR + k] = (k % 4 == 0) ? 1.0f : 0.0f;
#else
#if PBDR_GN_PROBE  // debug: Gauss-Newton steps of this body (15 = cold polar) into the phase stamps
  int steps = 0;
  const bool ok = polar_warm_f(&S[6], rq, &R[kResR], qd, &steps);
  if (A.timing) atomicAdd(reinterpret_cast<unsigned long long*>(A.timing + kTimingSlots * static_cast<int64_t>(blockIdx.x) + 7),
                          1ull << (16 + 4 * (steps <= 4 ? steps : 5)));
#else
  const bool ok = polar_warm_f(&S[6], rq, &R[kResR], qd);
#endif
#endif
  if (stamp) stamp[1] = clock64();  // polar end
  R[kResSmOk] = ok ? 1.0f : 0.0f;
  rq_new = ok ? make_float4(static_cast<float>(qd[0]), static_cast<float>(qd[1]), static_cast<float>(qd[2]),
                            static_cast<float>(qd[3]))
              : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  if (kStore) A.rquat[bb] = rq_new;
  if (!ok) record_error(A.err, PBDR_DEVERR_DEGENERATE, bb, A.substep_counter);
  if (kStore && !an_slot) A.anchor[bb] = an_new;
}

// Phase B of one particle: shape-matching delta (R q0 + c - p, when the polar
// is valid), X_a = X_i + dX and V_a (incremental or legacy velocity update).
__device__ __forceinline__ void phase_b_particle(const IterArgs& A, int64_t p, float4 x4, float4 v4, float4 r4,
                                                 const float a[3], bool sm_ok, const float (&Rf)[9],
                                                 const float (&c)[3], float (&dXk)[3], float (&xa)[3],
                                                 float (&va)[3], float (&pa)[3]) {
  const float x[3] = {x4.x, x4.y, x4.z};
  const float v[3] = {v4.x, v4.y, v4.z};
  const float q0[3] = {r4.x, r4.y, r4.z};
  float xi[3] = {0.0f, 0.0f, 0.0f};
  if (!A.incremental) {
    const float4 i4 = A.init[p];
    xi[0] = i4.x; xi[1] = i4.y; xi[2] = i4.z;
  }
#pragma unroll
  for (int cI = 0; cI < 3; ++cI) {
    const float pk = x[cI] - a[cI];
    float dsm = 0.0f;
    if (sm_ok) {
      const float Rrow[3] = {Rf[3 * cI], Rf[3 * cI + 1], Rf[3 * cI + 2]};
      const float g = dot3_fma(Rrow, q0);
      dsm = g - (pk - c[cI]);
    }
    dXk[cI] = dXk[cI] + dsm;
    xa[cI] = x[cI] + dXk[cI];
    va[cI] = A.incremental ? fmaf(dXk[cI], A.inv_dt, v[cI]) : (xa[cI] - xi[cI]) * A.inv_dt;
    pa[cI] = pk + dXk[cI];
  }
}

// The particle's terms of the 15 asm sums: dX, P_asm, L_asm and the inertia
// (anchor-relative; parallel axis applied in body_math_b).
__device__ __forceinline__ void accum_b(float mk, const float (&dXk)[3], const float (&va)[3],
                                        const float (&pa)[3], float (&accB)[15]) {
  const float mva[3] = {mk * va[0], mk * va[1], mk * va[2]};
  float ka[3];
  cross3_fma(pa, mva, ka);
  const float s2 = dot3_fma(pa, pa);
#pragma unroll
  for (int cI = 0; cI < 3; ++cI) {
    accB[cI] = fmaf(mk, dXk[cI], accB[cI]);
    accB[3 + cI] = fmaf(mk, va[cI], accB[3 + cI]);
    accB[6 + cI] = accB[6 + cI] + ka[cI];
    accB[9 + cI] = fmaf(mk, fmaf(-pa[cI], pa[cI], s2), accB[9 + cI]);
  }
  accB[12] = fmaf(-mk, pa[0] * pa[1], accB[12]);
  accB[13] = fmaf(-mk, pa[0] * pa[2], accB[13]);
  accB[14] = fmaf(-mk, pa[1] * pa[2], accB[14]);
}

// Per-body math B from the 15 asm sums S of body bb: com c_asm, P_asm,
// L_asm; the SM-induced momentum change (accumulated over the substep for
// kPerSubstep); linear fix dv = dP/M and angular fix omega = pinv(I) dL.
// Reads kResC/kResPb/kResLb and writes kResCa/kResDv/kResW of R.
__device__ __forceinline__ void body_math_b(const IterArgs& A, int bb, const float (&S)[15], float2 mass,
                                            float* R, int iter_index, int last_iter) {
  bool finite = true;
#pragma unroll
  for (int f = 0; f < 15; ++f) finite = finite && isfinite(S[f]);
  if (!finite) record_error(A.err, PBDR_DEVERR_NONFINITE, bb, A.substep_counter);
  const float M = mass.x, invM = mass.y;
  float ca[3], Pa[3], La[3], tmp[3], dv[3] = {0.0f, 0.0f, 0.0f}, om[3] = {0.0f, 0.0f, 0.0f};
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    ca[k] = R[kResC + k] + S[k] * invM;
    Pa[k] = S[3 + k];
  }
  cross3(ca, Pa, tmp);
#pragma unroll
  for (int k = 0; k < 3; ++k) La[k] = S[6 + k] - tmp[k];
  // SM-induced momentum change of this iteration (P_bsm - P_asm, L_asm - L_bsm).
  float dP[3], dL[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    dP[k] = R[kResPb + k] - Pa[k];
    dL[k] = La[k] - R[kResLb + k];
  }
  bool correct = true;
  if (A.per_substep) {
    // kPerSubstep: accumulate over the substep's iterations, correct once.
    float4 aP = make_float4(0.0f, 0.0f, 0.0f, 0.0f), aL = aP;
    if (iter_index > 0) {
      aP = A.mom_acc[2 * bb];
      aL = A.mom_acc[2 * bb + 1];
    }
    aP.x = aP.x + dP[0]; aP.y = aP.y + dP[1]; aP.z = aP.z + dP[2];
    aL.x = aL.x + dL[0]; aL.y = aL.y + dL[1]; aL.z = aL.z + dL[2];
    A.mom_acc[2 * bb] = aP;
    A.mom_acc[2 * bb + 1] = aL;
    dP[0] = aP.x; dP[1] = aP.y; dP[2] = aP.z;
    dL[0] = aL.x; dL[1] = aL.y; dL[2] = aL.z;
    correct = last_iter != 0;
  }
  if (A.linfix && correct)
#pragma unroll
    for (int k = 0; k < 3; ++k) dv[k] = dP[k] * invM;
  if (A.angfix && correct) {
    float If[6];
    If[0] = S[9] - M * (ca[1] * ca[1] + ca[2] * ca[2]);
    If[1] = S[10] - M * (ca[0] * ca[0] + ca[2] * ca[2]);
    If[2] = S[11] - M * (ca[0] * ca[0] + ca[1] * ca[1]);
    If[3] = S[12] + M * (ca[0] * ca[1]);
    If[4] = S[13] + M * (ca[0] * ca[2]);
    If[5] = S[14] + M * (ca[1] * ca[2]);
    double nax[3];
#if PBDR_COST_PROBE & 2  // cost probe only (wrong results): no inertia solve
    const unsigned e = 0u;
    (void)If;
#else
    const unsigned e = inertia_solve_f(If, dL, om, nax);
#endif
    if (e) record_error(A.err, e, bb, A.substep_counter, nax);
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    R[kResCa + k] = ca[k];
    R[kResDv + k] = dv[k];
    R[kResW + k] = om[k];
  }
}

// Phase C of one particle: momentum corrections (Eq. 1 then Eq. 2) on top of
// X_a, V_a: v = V_a + dv - omega x r, x = X_a + dt dv - dt omega x r.
__device__ __forceinline__ void phase_c_particle(const IterArgs& A, int64_t p, float4 x4, float4 v4,
                                                 const float a[3], const float (&dXk)[3], const float (&ca)[3],
                                                 const float (&dv)[3], const float (&om)[3], float (&xo)[3],
                                                 float (&vo)[3]) {
  float xi[3] = {0.0f, 0.0f, 0.0f};
  if (!A.incremental) {
    const float4 i4 = A.init[p];
    xi[0] = i4.x; xi[1] = i4.y; xi[2] = i4.z;
  }
  const float x[3] = {x4.x, x4.y, x4.z};
  const float v[3] = {v4.x, v4.y, v4.z};
  float xa[3], va[3], r[3], wr[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    xa[c] = x[c] + dXk[c];
    va[c] = A.incremental ? fmaf(dXk[c], A.inv_dt, v[c]) : (xa[c] - xi[c]) * A.inv_dt;
    r[c] = ((x[c] - a[c]) + dXk[c]) - ca[c];
  }
  cross3_fma(om, r, wr);
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    vo[c] = (va[c] + dv[c]) - wr[c];
    xo[c] = fmaf(-wr[c], A.dt, fmaf(dv[c], A.dt, xa[c]));
  }
}

// KP = 8 particles per lane, 8-warp CTAs: 96 KB of staged state per CTA, so
// two CTAs per SM with up to 128 registers (no spills). Measured on C4:
// 0.382 ms per iteration vs 0.436 for KP = 4 at three CTAs per SM (80
// registers, spills) -- more particles in flight per SM, fewer warps per body.
// PBDR_CAND_COLUMNS (KP <= 4 tiles; needs the rolled layout's s_dx): the
// particle-particle contacts of a lane's KP particles run side by side,
// candidate rank by rank, in a pass of their own before phase A, with all of
// a rank's loads issued before any arithmetic (2; 3 also overlaps the next
// rank's slot loads) -- KP gather chains in flight per lane instead of one,
// only in the warps that have a candidate at all. Per particle the deltas are
// still summed in ascending candidate order, so results are bit-identical.
// Landed C5 iteration -8.7%, C3 -2.5% together with PBDR_DESC_SMEM and
// PBDR_ANCHOR_EARLY (tools/ab_landed.py, round 2). 1 = the first version
// (loads inside per-particle branches: no overlap, slower than off).
// 4 = the same pass worked off by the whole CTA from a shared list of the
// tile's particles that have candidates (kCoop in k_iteration), one particle
// per thread with two ranks' loads in flight: the contact work no
// longer sits on the few warps that own those particles while the others
// wait at the barrier -- landed C3 iteration -7.4%, C5 -0.9%.
#ifndef PBDR_CAND_COLUMNS
#define PBDR_CAND_COLUMNS 4
#endif
// Ranks in flight per listed particle in the CTA-wide pass. Two, not four:
// the four-rank version's extra registers came out of the kernel's 80 as
// spills (local loads x4), which cost the landing frames of C5 4% and its
// landed frames everything the pass had gained (tools/scratch A/B, r02).
#ifndef PBDR_COOP_BATCH
#define PBDR_COOP_BATCH 2
#endif
// Rolled particle loops with the deltas in shared memory (KP <= 4 tiles only:
// at KP >= 7 the extra 32 KB would cost a CTA per SM).
#ifndef PBDR_ROLL_PARTICLES
#define PBDR_ROLL_PARTICLES 1
#endif
template <int KP>
constexpr bool iter_rolled() { return PBDR_ROLL_PARTICLES != 0 && KP <= 4; }
#ifndef PBDR_SMALL_KP_WARPS
#define PBDR_SMALL_KP_WARPS 24  // resident warps per SM requested for KP <= 4 (sets the register cap)
#endif
template <int KP>
constexpr int iter_min_blocks() { return (KP >= 7 ? 16 : PBDR_SMALL_KP_WARPS) / kWarps; }  // 16 or 24 warps per SM

// FUSE (single-iteration launches only): the launch ends the substep and
// integrates the next one in its writeback (a separate instantiation, so the
// other iterations keep their register allocation).
template <int KP, bool MULTI, bool FUSE = false>
__global__ void __launch_bounds__(kThreads, iter_min_blocks<KP>()) k_iteration(IterArgs A) {
  constexpr int kSlots = kThreads * KP;  // particle slots staged per CTA
  constexpr bool kRoll = PBDR_ROLL_PARTICLES != 0 && KP <= 4;  // iter_rolled<KP>()
  // Single-iteration launches only: the multi-iteration launches are the
  // isolated tiles (no candidates at all) and small latency-bound scenes, and
  // the extra pass cost their instantiation spills (C3 / C5 free flight -6%).
  constexpr bool kColumns = kRoll && PBDR_CAND_COLUMNS != 0 && !MULTI;
  // kCoop (PBDR_CAND_COLUMNS == 4): the tile's particles that have candidates
  // are listed in shared memory during the prelude and the whole CTA works the
  // list off, one particle per thread, spread over the warps -- instead of the
  // few warps that own those particles doing it while the others wait at the
  // next barrier. Each particle's candidates are still summed in rank order.
  constexpr bool kCoop = kColumns && PBDR_CAND_COLUMNS == 4;
  constexpr int kCoopBatch = PBDR_COOP_BATCH;  // candidate ranks in flight per listed particle
  __shared__ unsigned short s_clist[kCoop ? kThreads * KP : 1];
  __shared__ int s_ccount;
  extern __shared__ float4 s_stage[];  // pos | vel | rest [| dX], kSlots each
  __shared__ __align__(16) float s_part[kWarps][kPartStride];
  __shared__ float s_res[kWarps][kResF];
  __shared__ __align__(8) uint64_t s_bar;

  float4* s_pos = s_stage;
  float4* s_vel = s_stage + kSlots;
  float4* s_rest = s_stage + 2 * kSlots;
  float4* s_dx = s_stage + 3 * kSlots;  // kRoll only

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // Per-body table of a tile (anchor, masses, body descriptor, warm-start
  // rotation), double-buffered: the next tile's table is copied in with
  // cp.async while the current tile computes.
  __shared__ float4 s_tanc[2][kWarps];
  __shared__ float2 s_tmass[2][kWarps];
  __shared__ int4 s_tdesc[2][kWarps];
  __shared__ float4 s_trq[2][kWarps];
  __shared__ int s_next;
  // Tile and warp descriptors of the current / next tile, double-buffered like
  // the body table and filled by cp.async: no register waits on them
  // (kDescSmem: the single-iteration launches, whose persistent CTAs walk
  // many tiles; the multi-iteration launches keep them in registers).
  constexpr bool kDescSmem = PBDR_DESC_SMEM != 0 && !MULTI;
  static_assert(!(PBDR_DESC_SMEM != 0 && PBDR_PREFETCH_NEXT != 0), "the next-tile prefetch reads cd_n from registers");
  __shared__ int4 s_cd[2];
  __shared__ int4 s_wd[2][kWarps];
  const bool fixes = A.linfix || A.angfix;
  const long long t_entry = A.timing ? clock64() : 0;  // phase clocks (debug launches only)
  // One CTA per tile (grid == ntiles): static; otherwise tiles are claimed
  // dynamically, in increasing order. With a device-side tile list (isolated /
  // contact tiles of this substep) claim c is tile tile_list[c] of tile_count.
  const int ntiles = A.tile_count ? *A.tile_count : A.ntiles;
  const bool dynamic = A.tile_count != nullptr || static_cast<int>(gridDim.x) < ntiles;
  auto tid = [&](int c) { return A.tile_list ? A.tile_list[c] : c; };
  if (threadIdx.x == 0) {
    mbar_init(&s_bar, 1);
    s_next = dynamic ? atomicAdd(A.tile_ctr, 1) : static_cast<int>(blockIdx.x);
    s_ccount = 0;
  }
  __syncthreads();
  int tile = s_next;
  int tb = 0;  // table buffer of the current tile
  int4 cd_n = make_int4(0, 0, 0, 0), wd_n = make_int4(-1, 0, 0, 1 << 16);
  if (tile < ntiles) {
    const int t0 = tid(tile);
    cd_n = ld_keep_nc(&A.cta_desc[t0]);
    wd_n = ld_keep_nc(&A.warp_desc[t0 * kWarps + warp]);
    if (warp == 0 && lane < cd_n.w) {  // first tile's table: synchronous
      const int bb = cd_n.z + lane;
      s_tdesc[0][lane] = ld_keep_nc(&A.body_desc[bb]);
      s_tanc[0][lane] = ld_keep(&A.anchor[bb]);
      s_tmass[0][lane] = ld_keep_nc(&A.body_mass[bb]);
      s_trq[0][lane] = ld_keep(&A.rquat[bb]);
    }
    if constexpr (kDescSmem) {
      if (lane == 0) s_wd[0][warp] = wd_n;
      if (threadIdx.x == 0) s_cd[0] = cd_n;
    }
  }
  if constexpr (kDescSmem) __syncthreads();
  for (uint32_t it_parity = 0; tile < ntiles; it_parity ^= 1u) {
  const int4 cd = kDescSmem ? s_cd[tb] : cd_n;  // first slot, slot count, first body, bodies
  const int4 wd = kDescSmem ? s_wd[tb][warp] : wd_n;
  const int first = cd.x;

  if (threadIdx.x == 0) {
    const uint32_t bytes = static_cast<uint32_t>(cd.y) * 16u;
    PBDR_CHECK(cd.y > 0 && cd.y <= kSlots && cd.x >= 0 && cd.x + cd.y <= A.n && cd.w >= 1 && cd.w <= kWarps);
    mbar_expect_tx(&s_bar, 3u * bytes);
    bulk_g2s_stream(s_pos, A.pos_in + first, bytes, &s_bar);
    bulk_g2s_stream(s_vel, A.vel + first, bytes, &s_bar);
    bulk_g2s_stream(s_rest, A.rest + first, bytes, &s_bar);
    s_next = dynamic ? atomicAdd(A.tile_ctr, 1) : ntiles;  // the tile after this one
  }
  cp_async_wait_all();  // this tile's table (prefetched during the previous tile)

  const int b = wd.x;
  const int wi = wd.y;
  const bool live = b >= 0;
  const int lb = live ? b - cd.z : 0;  // body index within the CTA
  const int start = wd.z, n = wd.w & 0xFFFF, W = wd.w >> 16;
  PBDR_CHECK(!live || (start >= first && start - first + n <= cd.y && W >= 1 && wi < W && n <= 32 * KP * W &&
                       lb >= 0 && lb < cd.w));
  // Candidate counts of the lane's particles (prefetched: off the phase-A
  // chain); kRoll packs them 8 bits each (<= PBDR_NBR_CAP) so that the rolled
  // particle loops index them without local memory.
  int ncs_a[kRoll ? 1 : KP];
  uint32_t ncs_pk = 0;
#pragma unroll
  for (int k = 0; k < KP; ++k) {
    const int q = k * 32 * W + wi * 32 + lane;
    const int c = (live && q < n) ? A.ncand[start + q] : 0;
    if constexpr (kRoll)
      ncs_pk |= static_cast<uint32_t>(c) << (8 * k);
    else
      ncs_a[k] = c;
  }
  auto ncs = [&](int k) -> int {
    if constexpr (kRoll)
      return static_cast<int>((ncs_pk >> (8 * k)) & 0xFFu);
    else
      return ncs_a[k];
  };
  if constexpr (kCoop) {
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      if (ncs(k) > 0) {
        const int idx = (start - first) + k * 32 * W + wi * 32 + lane;
        PBDR_CHECK(idx >= 0 && idx < kSlots && ncs(k) <= 32);
        s_clist[atomicAdd(&s_ccount, 1)] = static_cast<unsigned short>(((ncs(k) - 1) << 10) | idx);
      }
    }
  }
  // First candidate of each particle: its slot now, and its position and
  // contact radius pulled into L2, while the tile's staging copies are in
  // flight -- in contact-rich states phase A otherwise waits on two dependent
  // HBM round trips per particle (-5% iteration time in a settled C5 pile).
  if (!MULTI || !A.multi_pairs) {
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      if (ncs(k) > 0) {
        const int64_t p = start + k * 32 * W + wi * 32 + lane;
        const int j = __ldg(&A.cand_j[p]);
        PBDR_CHECK(j >= 0 && j < A.n);
#if PBDR_PREFETCH_L1
        prefetch_l1(&A.pos_in[j]);
        prefetch_l1(&A.cand_rr[p]);
#else
        prefetch_l2(&A.pos_in[j]);
        prefetch_l2(&A.cand_rr[p]);
#endif
#if PBDR_PREFETCH_ALL_CANDS == 1
        // ... and every further candidate (settled piles: p90 phase A was
        // one dependent L2/HBM round trip per candidate, in series).
#pragma unroll 1
        for (int c = 1; c < ncs(k); ++c) {
          const int jc = __ldg(&A.cand_j[static_cast<int64_t>(c) * A.n + p]);
          prefetch_l2(&A.pos_in[jc]);
          prefetch_l2(&A.cand_rr[static_cast<int64_t>(c) * A.n + p]);
        }
#endif
      }
    }
#if PBDR_PREFETCH_ALL_CANDS >= 2
    // Candidates 1 .. kPfDepth of every particle of the lane: all their slot
    // loads issued back to back (independent, up to KP * kPfDepth in flight),
    // then all the position prefetches -- the per-candidate chain
    // (slot load -> position gather) of phase A then finds both in L1 / L2.
    constexpr int kPfDepth = PBDR_PREFETCH_ALL_CANDS;
    int jc[KP][kPfDepth];
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      const int64_t p = start + k * 32 * W + wi * 32 + lane;
#pragma unroll
      for (int c = 1; c <= kPfDepth; ++c)
        jc[k][c - 1] = c < ncs(k) ? __ldg(&A.cand_j[static_cast<int64_t>(c) * A.n + p]) : -1;
    }
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      const int64_t p = start + k * 32 * W + wi * 32 + lane;
#pragma unroll
      for (int c = 1; c <= kPfDepth; ++c)
        if (jc[k][c - 1] >= 0) {
          prefetch_l2(&A.pos_in[jc[k][c - 1]]);
          prefetch_l2(&A.cand_rr[static_cast<int64_t>(c) * A.n + p]);
        }
    }
#endif
  }
  const int off = start - first;

  long long* tm = A.timing ? A.timing + kTimingSlots * static_cast<int64_t>(tile) : nullptr;
  if (tm && threadIdx.x == 0) tm[0] = t_entry;  // CTA entry: stage = descriptors + table + bulk copies
  __syncthreads();  // barrier initialised, per-body table filled, next tile claimed
  const int tile_next = s_next;
  if constexpr (kDescSmem) {
    if (tile_next < ntiles && warp == kWarps - 1 && lane <= kWarps) {
      // Next tile's descriptors into the other buffer (asynchronous; complete
      // before the tile-end barrier through cp.async.wait_all there).
      const int t1 = tid(tile_next);
      if (lane < kWarps)
        cp_async16(&s_wd[tb ^ 1][lane], &A.warp_desc[t1 * kWarps + lane]);
      else
        cp_async16(&s_cd[tb ^ 1], &A.cta_desc[t1]);
      cp_async_commit();
    }
  } else if (tile_next < ntiles) {  // next tile's descriptors, consumed at its start
    const int t1 = tid(tile_next);
    cd_n = ld_keep_nc(&A.cta_desc[t1]);
    wd_n = ld_keep_nc(&A.warp_desc[t1 * kWarps + warp]);
  }
#if PBDR_PREFETCH_NEXT == 2
  // Next tile's staging ranges pulled into L2 as soon as its descriptor is
  // known: two tiles' worth of HBM reads in flight per CTA.
  if (warp == kWarps - 1 && lane == 0 && tile_next < ntiles) {
    const uint32_t bytes = static_cast<uint32_t>(cd_n.y) * 16u;
    bulk_prefetch_l2(A.pos_in + cd_n.x, bytes);
    bulk_prefetch_l2(A.vel + cd_n.x, bytes);
    bulk_prefetch_l2(A.rest + cd_n.x, bytes);
    bulk_prefetch_l2(A.ncand + cd_n.x, static_cast<uint32_t>(cd_n.y) * 4u);
  }
#endif
  mbar_wait(&s_bar, it_parity);
  if (tm && threadIdx.x == 0) tm[1] = clock64();

  // Scenes without candidate pairs (one body per scene) run all iterations of
  // the substep in one launch: a body's iteration reads only its own
  // particles, so the state stays in shared memory between iterations.
  const int n_iters = MULTI ? A.n_iters : 1;
  for (int it = 0; it < n_iters; ++it) {
  const int iter_index = A.iter_index + it;
  const int last_iter = MULTI ? (A.last_iter && it == n_iters - 1) : A.last_iter;
  // Previous iteration's state and table in smem (the grid / cluster barrier
  // that ended it already synchronised this CTA).
  if (it > 0 && !A.multi_pairs) __syncthreads();
  float a[3];
  {
    const float4 an = s_tanc[tb][lb];
    a[0] = an.x; a[1] = an.y; a[2] = an.z;
  }

  // Per-particle deltas dX: registers (unrolled particle loops), or -- kRoll
  // -- shared memory next to the staged state, so the three particle loops
  // stay rolled (a quarter of the code: the tile loop then fits the SM's
  // instruction cache better) and no delta is live across the body math.
  float dX[kRoll ? 1 : KP][3];
  if constexpr (!kRoll) {
#pragma unroll
    for (int k = 0; k < KP; ++k) dX[k][0] = dX[k][1] = dX[k][2] = 0.0f;
  }
  auto dx_load = [&](int k, int q, float (&d)[3]) {
    if constexpr (kRoll) {
      const float4 t = s_dx[off + q];
      d[0] = t.x; d[1] = t.y; d[2] = t.z;
    } else {
      d[0] = dX[k][0]; d[1] = dX[k][1]; d[2] = dX[k][2];
    }
  };
  auto dx_store = [&](int k, int q, const float (&d)[3]) {
    if constexpr (kRoll) {
      s_dx[off + q] = make_float4(d[0], d[1], d[2], 0.0f);
    } else {
      dX[k][0] = d[0]; dX[k][1] = d[1]; dX[k][2] = d[2];
    }
  };

  // ---- Phase A: contacts, bsm sums -----------------------------------------
  float acc[21];
#pragma unroll
  for (int f = 0; f < 21; ++f) acc[f] = 0.0f;
  bool warp_has_cands = false;  // kColumns
  if constexpr (kColumns) {
    // Phase A1: the particle-particle contacts of the lane's KP particles side
    // by side, candidate rank by rank -- up to KP independent gathers in flight
    // where the per-particle loop has one -- summed per particle in ascending
    // candidate order as before, and parked in s_dx for phase A2.
    // ncs_pk != 0 <=> some particle of the lane has a candidate. Warps without
    // any (most warps: contacts sit on a few faces) skip the pass and its
    // round trip through s_dx.
    warp_has_cands = __any_sync(kFull, ncs_pk != 0u);
    if constexpr (kCoop) {
      const int count = s_ccount;  // complete since the first barrier of the tile
      // Entry e goes to warp e % 8, lane e / 8: the list spreads over the warps.
      for (int e = lane * kWarps + warp; e < count; e += kThreads) {
        const int ent = s_clist[e];
        const int idx = ent & 1023, nc = (ent >> 10) + 1;
        const int64_t p = first + idx;
        const float4 x4 = s_pos[idx];
        const float x[3] = {x4.x, x4.y, x4.z};
        float d[3] = {0.0f, 0.0f, 0.0f};
#pragma unroll 1
        for (int c0 = 0; c0 < nc; c0 += kCoopBatch) {
          int jq[kCoopBatch];
          float rq[kCoopBatch];
          float4 xq[kCoopBatch];
#pragma unroll
          for (int u = 0; u < kCoopBatch; ++u) {
            jq[u] = -1;
            rq[u] = 0.0f;
            if (c0 + u < nc) {  // predicated loads, no branch
              const int64_t at = static_cast<int64_t>(c0 + u) * A.n + p;
              jq[u] = __ldg(&A.cand_j[at]);
              rq[u] = __ldg(&A.cand_rr[at]);
            }
          }
#pragma unroll
          for (int u = 0; u < kCoopBatch; ++u) {
            xq[u] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
            if (jq[u] >= 0) xq[u] = A.pos_in[jq[u]];
          }
#pragma unroll
          for (int u = 0; u < kCoopBatch; ++u) {
            if (jq[u] >= 0) {
              PBDR_CHECK(jq[u] < A.n && jq[u] != p);
              pp_contact(x, x4.w, p, xq[u], jq[u], rq[u], A.relax, d);
            }
          }
        }
        s_dx[idx] = make_float4(d[0], d[1], d[2], 0.0f);
      }
      __syncthreads();  // every listed particle's contact delta is in s_dx
    }
    if (!kCoop && warp_has_cands) {
    float dpp[KP][3];
#pragma unroll
    for (int k = 0; k < KP; ++k) dpp[k][0] = dpp[k][1] = dpp[k][2] = 0.0f;
    int maxc = 0;
#pragma unroll
    for (int k = 0; k < KP; ++k) maxc = max(maxc, ncs(k));
#if PBDR_CAND_COLUMNS >= 2
    // All of a rank's loads first (slots and radii, then the positions they
    // point at: KP independent chains in flight), arithmetic afterwards.
    // With PBDR_CAND_COLUMNS == 3 the next rank's slots and radii are loaded
    // while this rank's positions are in flight (one dependent round trip
    // per rank instead of two).
    int jj[KP];
    float rrk[KP];
    auto load_rank = [&](int c, int (&jo)[KP], float (&ro)[KP]) {
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        jo[k] = -1;
        ro[k] = 0.0f;
        if (c < ncs(k)) {  // predicated loads, no branch
          const int64_t at = static_cast<int64_t>(c) * A.n + (start + k * 32 * W + wi * 32 + lane);
          jo[k] = __ldg(&A.cand_j[at]);
          ro[k] = __ldg(&A.cand_rr[at]);
        }
      }
    };
    if (PBDR_CAND_COLUMNS == 3) load_rank(0, jj, rrk);
#pragma unroll 1
    for (int c = 0; c < maxc; ++c) {
      float4 xjk[KP];
      if (PBDR_CAND_COLUMNS == 2) load_rank(c, jj, rrk);
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        xjk[k] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        if (jj[k] >= 0) xjk[k] = (MULTI && A.multi_pairs) ? __ldcg(&A.pos_b[it & 1][jj[k]]) : A.pos_in[jj[k]];
      }
      int jn[KP];
      float rn[KP];
      if (PBDR_CAND_COLUMNS == 3) load_rank(c + 1, jn, rn);
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        if (jj[k] >= 0) {
          const int q = k * 32 * W + wi * 32 + lane;
          const int64_t p = start + q;
          PBDR_CHECK(jj[k] < A.n && jj[k] != p);
          const float4 x4 = s_pos[off + q];
          const float x[3] = {x4.x, x4.y, x4.z};
          pp_contact(x, x4.w, p, xjk[k], jj[k], rrk[k], A.relax, dpp[k]);
        }
      }
      if (PBDR_CAND_COLUMNS == 3) {
#pragma unroll
        for (int k = 0; k < KP; ++k) {
          jj[k] = jn[k];
          rrk[k] = rn[k];
        }
      }
    }
#else
#pragma unroll 1
    for (int c = 0; c < maxc; ++c) {
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        if (c < ncs(k)) {
          const int q = k * 32 * W + wi * 32 + lane;
          const int64_t p = start + q;
          const int j = A.cand_j[static_cast<int64_t>(c) * A.n + p];
          PBDR_CHECK(j >= 0 && j < A.n && j != p);
          const float rr = A.cand_rr[static_cast<int64_t>(c) * A.n + p];
          const float4 xj = (MULTI && A.multi_pairs) ? __ldcg(&A.pos_b[it & 1][j]) : A.pos_in[j];
          const float4 x4 = s_pos[off + q];
          const float x[3] = {x4.x, x4.y, x4.z};
          pp_contact(x, x4.w, p, xj, j, rr, A.relax, dpp[k]);
        }
      }
    }
#endif
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      const int q = k * 32 * W + wi * 32 + lane;
      if (live && q < n) s_dx[off + q] = make_float4(dpp[k][0], dpp[k][1], dpp[k][2], 0.0f);
    }
    }  // warp_has_cands
  }
  auto phase_a_k = [&](int k) {
    const int q = k * 32 * W + wi * 32 + lane;
    if (!(live && q < n)) return;
    const int64_t p = start + q;
    float d[3] = {0.0f, 0.0f, 0.0f};
    if constexpr (kColumns) {
      float pre[3] = {0.0f, 0.0f, 0.0f};
      if (kCoop ? ncs(k) > 0 : warp_has_cands) {
        const float4 t = s_dx[off + q];
        pre[0] = t.x; pre[1] = t.y; pre[2] = t.z;
      }
      phase_a_particle<MULTI>(A, it, p, s_pos[off + q], s_vel[off + q], s_rest[off + q], 0, a, d, acc, s_pos,
                              first, cd.y, pre);
    } else {
      phase_a_particle<MULTI>(A, it, p, s_pos[off + q], s_vel[off + q], s_rest[off + q], ncs(k), a, d, acc,
                              s_pos, first, cd.y);
    }
    dx_store(k, q, d);
  };
  if constexpr (kRoll) {
#pragma unroll 1
    for (int k = 0; k < KP; ++k) phase_a_k(k);
  } else {
#pragma unroll
    for (int k = 0; k < KP; ++k) phase_a_k(k);
  }
  if (live) {
    // 21 fields as 16 + 5 (each its own power-of-two reduce-scatter: fewer
    // shuffles than padding to 32; every field's tree is the same butterfly).
    float a16[16], a5[5];
#pragma unroll
    for (int f = 0; f < 16; ++f) a16[f] = acc[f];
#pragma unroll
    for (int f = 0; f < 5; ++f) a5[f] = acc[16 + f];
    const float t16 = warp_reduce_scatter<16>(a16);  // lanes 2f, 2f+1: field f
    const float t5 = warp_reduce_scatter<5>(a5);     // lanes 4f..4f+3: field 16 + f
    if ((lane & 1) == 0) s_part[warp][lane >> 1] = t16;
    if ((lane & 3) == 0 && (lane >> 2) < 5) s_part[warp][16 + (lane >> 2)] = t5;
  }
#if PBDR_PREFETCH_NEXT == 1
  if (it == 0 && warp == kWarps - 1 && lane == 0 && tile_next < ntiles) {
    const uint32_t bytes = static_cast<uint32_t>(cd_n.y) * 16u;
    bulk_prefetch_l2(A.pos_in + cd_n.x, bytes);
    bulk_prefetch_l2(A.vel + cd_n.x, bytes);
    bulk_prefetch_l2(A.rest + cd_n.x, bytes);
    bulk_prefetch_l2(A.ncand + cd_n.x, static_cast<uint32_t>(cd_n.y) * 4u);
  }
#endif
#if PBDR_PREFETCH_COUNTS
  if constexpr (kDescSmem) {
    // The next tile's candidate counts and first-candidate slots and radii
    // (contiguous ranges: row 0 of the candidate arrays) pulled into L2 now,
    // a phase and the body math ahead of their use at its start -- the two
    // dependent loads there were 9% of the landed-C5 stall samples. The
    // descriptor copies issued at this tile's start have long landed.
    if (warp == kWarps - 1 && tile_next < ntiles) {
      cp_async_wait_all();
      __syncwarp();
      if (lane == 0) {
        const int4 cdx = s_cd[tb ^ 1];
        const uint32_t bytes = static_cast<uint32_t>(cdx.y) * 4u;
        bulk_prefetch_l2(A.ncand + cdx.x, bytes);
        bulk_prefetch_l2(A.cand_j + cdx.x, bytes);
        bulk_prefetch_l2(A.cand_rr + cdx.x, bytes);
        if (PBDR_PREFETCH_COUNTS & 2) {  // second candidate row
          bulk_prefetch_l2(A.cand_j + A.n + cdx.x, bytes);
          bulk_prefetch_l2(A.cand_rr + A.n + cdx.x, bytes);
        }
        if (PBDR_PREFETCH_COUNTS & 4) {  // the staging ranges themselves
          bulk_prefetch_l2(A.pos_in + cdx.x, 4u * bytes);
          bulk_prefetch_l2(A.vel + cdx.x, 4u * bytes);
          bulk_prefetch_l2(A.rest + cdx.x, 4u * bytes);
        }
      }
    }
  }
#endif
  __syncthreads();
  if (tm && threadIdx.x == 0) tm[2] = clock64();

  // ---- per-body math A (warp 0, lane = body of the CTA) ---------------------
  // kDescSmem: the body count is re-read from shared memory, so the predicate
  // is rebuilt after the barrier instead of being kept (spilled) across the
  // particle phase.
  if ((warp == 0 && lane < (kDescSmem ? s_cd[tb].w : cd.w))) {
    const int bb = cd.z + lane;
    const float4 an = make_float4(s_tanc[tb][lane].x, s_tanc[tb][lane].y,
                                  s_tanc[tb][lane].z, s_tmass[tb][lane].x);
    const float invM = s_tmass[tb][lane].y;
    const int2 bw = make_int2(s_tdesc[tb][lane].w, s_tdesc[tb][lane].z);
    const int fw = bw.x;
    float S[21];
    part_sum(&s_part[0][0], fw, bw.y, S);
    float4 rq_new, an_new;
    if (tm && lane == 0) tm[8] = clock64();  // body sums read
#if PBDR_ANCHOR_EARLY
    body_math_a(A, bb, S, an, invM, s_trq[tb][lane], &s_res[lane][0], rq_new, an_new,
                (tm && lane == 0) ? tm + 12 : nullptr, &s_tanc[tb][lane]);
    if (tm && lane == 0) tm[9] = clock64();
    s_trq[tb][lane] = rq_new;   // next iteration of a multi-iteration launch
#else
    body_math_a(A, bb, S, an, invM, s_trq[tb][lane], &s_res[lane][0], rq_new, an_new,
                (tm && lane == 0) ? tm + 12 : nullptr);
    if (tm && lane == 0) tm[9] = clock64();
    s_trq[tb][lane] = rq_new;   // next iteration of a multi-iteration launch
    s_tanc[tb][lane] = an_new;
#endif
  }
  __syncthreads();
  if (tm && threadIdx.x == 0) tm[3] = clock64();

  // ---- Phase B: shape matching, position + velocity update ----------------
  // kDescSmem: the body's index in the tile is rebuilt from the shared
  // descriptors (two LDS) rather than reloaded from a spill slot after the
  // barrier (ncu: an LDL that misses the small L1).
  int lb_b = live ? lb : 0;
  if constexpr (kDescSmem) lb_b = live ? s_wd[tb][warp].x - s_cd[tb].z : 0;
  const float* res = &s_res[lb_b][0];
  float accB[15];
#pragma unroll
  for (int f = 0; f < 15; ++f) accB[f] = 0.0f;
  // Launch that ends the substep and integrates the next one (not MULTI:
  // the multi-iteration tail below does its own).
  const bool fuse_out = FUSE && !MULTI && last_iter;
  uint32_t flo[3] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu}, fhi[3] = {0u, 0u, 0u};
  if (live) {
    const bool sm_ok = res[kResSmOk] != 0.0f;
    float Rf[9], c[3];
#pragma unroll
    for (int f = 0; f < 9; ++f) Rf[f] = res[kResR + f];
#pragma unroll
    for (int k = 0; k < 3; ++k) c[k] = res[kResC + k];
    auto phase_b_k = [&](int k) {
      const int q = k * 32 * W + wi * 32 + lane;
      if (!(q < n)) return;
      const float4 x4 = s_pos[off + q];
      const float4 v4 = s_vel[off + q];
      float xa[3], va[3], pa[3], d[3];
      dx_load(k, q, d);
      phase_b_particle(A, start + q, x4, v4, s_rest[off + q], a, sm_ok, Rf, c, d, xa, va, pa);
      dx_store(k, q, d);
      if (fixes) {
        accum_b(v4.w, d, va, pa, accB);
      } else {
        const int64_t p = start + q;
        if (MULTI) {
          s_pos[off + q] = make_float4(xa[0], xa[1], xa[2], x4.w);
          s_vel[off + q] = make_float4(va[0], va[1], va[2], v4.w);
          // Only particles with candidates are gathered by others (the
          // candidate relation is symmetric, P4), so only they are published.
          if (A.multi_pairs && it + 1 < n_iters && ncs(k) > 0) __stcg(&A.pos_b[(it + 1) & 1][p], s_pos[off + q]);
        } else {
          store_final(A, p, b, make_float4(xa[0], xa[1], xa[2], x4.w), make_float4(va[0], va[1], va[2], v4.w),
                      fuse_out, flo, fhi);
        }
      }
    };
    if constexpr (kRoll) {
#pragma unroll 1
      for (int k = 0; k < KP; ++k) phase_b_k(k);
    } else {
#pragma unroll
      for (int k = 0; k < KP; ++k) phase_b_k(k);
    }
    if (fuse_out && !fixes) warp_box_commit(A, b, flo, fhi, lane);
  }
  if (fixes) {

  if (live) {
    const float tot = warp_reduce_scatter<15>(accB);  // lanes 2f, 2f+1: field f
    if ((lane & 1) == 0 && (lane >> 1) < 15) s_part[warp][lane >> 1] = tot;
  }
  __syncthreads();
  if (tm && threadIdx.x == 0) tm[4] = clock64();

  // ---- per-body math B: momentum corrections -------------------------------
  // kDescSmem: the body count is re-read from shared memory, so the predicate
  // is rebuilt after the barrier instead of being kept (spilled) across the
  // particle phase.
  if ((warp == 0 && lane < (kDescSmem ? s_cd[tb].w : cd.w))) {
    const int bb = cd.z + lane;
    const float2 mass = s_tmass[tb][lane];
    const int2 bw = make_int2(s_tdesc[tb][lane].w, s_tdesc[tb][lane].z);
    const int fw = bw.x;
    float S[15];
    part_sum(&s_part[0][0], fw, bw.y, S);
    if (tm && lane == 0) tm[10] = clock64();
    body_math_b(A, bb, S, mass, &s_res[lane][0], iter_index, last_iter);
    if (tm && lane == 0) tm[11] = clock64();
  }
  __syncthreads();
  if (tm && threadIdx.x == 0) tm[5] = clock64();

  // ---- Phase C: momentum corrections (Eq. 1 then Eq. 2), writeback --------
  if (live) {
  float ca[3], dv[3], om[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    ca[k] = res[kResCa + k];
    dv[k] = res[kResDv + k];
    om[k] = res[kResW + k];
  }
  auto phase_c_k = [&](int k) {
    const int q = k * 32 * W + wi * 32 + lane;
    if (!(q < n)) return;
    const float4 x4 = s_pos[off + q];
    const float4 v4 = s_vel[off + q];
    const int64_t p = start + q;
    float xo[3], vo[3], d[3];
    dx_load(k, q, d);
    phase_c_particle(A, p, x4, v4, a, d, ca, dv, om, xo, vo);
    if (MULTI) {
      s_pos[off + q] = make_float4(xo[0], xo[1], xo[2], x4.w);
      s_vel[off + q] = make_float4(vo[0], vo[1], vo[2], v4.w);
      if (A.multi_pairs && it + 1 < n_iters && ncs(k) > 0) __stcg(&A.pos_b[(it + 1) & 1][p], s_pos[off + q]);
    } else {
      store_final(A, p, b, make_float4(xo[0], xo[1], xo[2], x4.w), make_float4(vo[0], vo[1], vo[2], v4.w),
                  fuse_out, flo, fhi);
    }
  };
  if constexpr (kRoll) {
#pragma unroll 1
    for (int k = 0; k < KP; ++k) phase_c_k(k);
  } else {
#pragma unroll
    for (int k = 0; k < KP; ++k) phase_c_k(k);
  }
  if (fuse_out) warp_box_commit(A, b, flo, fhi, lane);
  }  // live
  }  // fixes
  if (MULTI && A.multi_pairs && it + 1 < n_iters) multi_barrier(A);
  }  // iterations of this launch
  if (MULTI) {
    // With pairs and an even count the last iteration gathered neighbours
    // from pos_b[1] == pos_out: every CTA of the barrier group must be past
    // that phase A before the final state overwrites it.
    if (A.multi_pairs && !(n_iters & 1)) multi_barrier(A);
    __syncthreads();
    if (live && A.fuse_integrate) {
      // Next substep's integrate on the final state (the same arithmetic as
      // k_integrate_key): X~ and V~ go out instead of X and V, X_init = X,
      // the cell keys, and the body box from one warp reduction per warp.
      uint32_t lo[3] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu}, hi[3] = {0u, 0u, 0u};
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        const int q = k * 32 * W + wi * 32 + lane;
        if (q < n) {
          const int64_t p = start + q;
          const float4 x4 = s_pos[off + q];
          float4 xn, vn;
          integrate_one(A.ia, b, x4, s_vel[off + q], xn, vn);
          A.ia.init[p] = make_float4(x4.x, x4.y, x4.z, 0.0f);
          A.pos_out[p] = xn;
          A.vel[p] = vn;
          A.ia.key_all[p] = integrate_key(A.ia, b, xn);
          const uint32_t o[3] = {f2ord(xn.x), f2ord(xn.y), f2ord(xn.z)};
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            lo[c] = min(lo[c], o[c]);
            hi[c] = max(hi[c], o[c]);
          }
        }
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        lo[c] = __reduce_min_sync(kFull, lo[c]);
        hi[c] = __reduce_max_sync(kFull, hi[c]);
      }
      if (lane == 0)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          atomicMin(&A.ia.box_min[3 * b + c], lo[c]);
          atomicMax(&A.ia.box_max[3 * b + c], hi[c]);
        }
    } else if (live) {
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        const int q = k * 32 * W + wi * 32 + lane;
        if (q < n) {
          A.pos_out[start + q] = s_pos[off + q];
          A.vel[start + q] = s_vel[off + q];
        }
      }
    }
  }
  if (tm && threadIdx.x == 0) {
    tm[6] = clock64();
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
#if PBDR_GN_PROBE
    atomicAdd(reinterpret_cast<unsigned long long*>(&tm[7]), static_cast<unsigned long long>(smid));
#else
    tm[7] = smid;
#endif
  }
  constexpr int kTableWarp = kDescSmem ? kWarps - 1 : 0;  // the warp that copied the descriptors also copies the table
  if constexpr (kDescSmem) {
    if (tile_next < ntiles && warp == kTableWarp) {
      cp_async_wait_all();  // its own descriptor copies, issued at this tile's start
      __syncwarp();
      cd_n = s_cd[tb ^ 1];
    }
  }
  if (tile_next < ntiles && warp == kTableWarp && lane < cd_n.w) {
    const int bb = cd_n.z + lane;
    cp_async16(&s_tdesc[tb ^ 1][lane], &A.body_desc[bb]);
    cp_async16(&s_tanc[tb ^ 1][lane], &A.anchor[bb]);
    cp_async8(&s_tmass[tb ^ 1][lane], &A.body_mass[bb]);
    cp_async16(&s_trq[tb ^ 1][lane], &A.rquat[bb]);
  }
  cp_async_commit();
  if (kCoop && threadIdx.x == 0) s_ccount = 0;  // every thread read it long ago (phase A)
  __syncthreads();  // the next tile's bulk copies overwrite the staging buffers
  tile = tile_next;
  tb ^= 1;
  }  // tiles
  if (dynamic && threadIdx.x == 0) {
    // The last CTA out resets the claim counter for the next launch.
    __threadfence();
    if (atomicAdd(A.tile_ctr + 1, 1) == static_cast<int>(gridDim.x) - 1) {
      A.tile_ctr[0] = 0;
      A.tile_ctr[1] = 0;
    }
  }
}

// ---------------------------------------------------------------------------
// Bodies larger than one CTA (W = pbdr_body_warps(n, 8) > 8 warps): one
// thread-block cluster per body. CTA r of the cluster (w = blockDim/32 warps,
// w = ceil(W / cluster) <= 8 so that the warps spread evenly) stages and
// computes the body's warps r*w .. r*w+w-1 with the same slot -> (warp, lane, k) map, the
// same per-particle code and the same reduction tree as k_iteration: lane
// sums over k, xor butterfly, then the per-warp partials -- written into the
// leader CTA's shared memory over DSMEM -- summed serially in warp order by
// the leader, which runs the per-body math; the other CTAs read the results
// back over DSMEM. Cluster barriers order the phases (release/acquire, so the
// remote stores are visible after them). KP = 8: a scene with such a body
// always reduces with the KP = 8 tree (pbdr_choose_kp).
// ---------------------------------------------------------------------------
constexpr int kBigMaxWarps = PBDR_MAX_CLUSTER_CTAS * kWarps;  // 128 warps = 32768 particles

// Cluster barrier without release/acquire semantics: for the barriers that
// only order execution (every CTA started; no CTA exits while another still
// reads its shared memory -- those reads have completed, their values were
// stored to local shared memory before a __syncthreads). The default
// cluster.sync() releases, which waits for this CTA's outstanding global
// stores (the phase-C writeback) -- measured as membar stalls.
__device__ __forceinline__ void cluster_sync_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}

__global__ void __launch_bounds__(kThreads, 2) k_iteration_big(IterArgs A) {
  constexpr int KP = PBDR_KP_MAX;
  const int nt = blockDim.x;           // 32 * warps per CTA (launch_iteration_big)
  const int kSlots = nt * KP;
  extern __shared__ float4 s_stage[];  // pos | vel | rest of this CTA's warps, [k][warp][lane]
  __shared__ float s_part[kBigMaxWarps][21];  // leader: per-warp partials of the body
  __shared__ float s_res[kResF];              // leader: per-body results; others: their copy
  __shared__ float s_sum[21];                 // leader: body sums
  __shared__ float4 s_rq;                     // leader: warm-start rotation across iterations
  __shared__ __align__(8) uint64_t s_bar;
  float4* s_pos = s_stage;
  float4* s_vel = s_stage + kSlots;
  float4* s_rest = s_stage + 2 * kSlots;

  cooperative_groups::cluster_group cluster = cooperative_groups::this_cluster();
  const int r = static_cast<int>(cluster.block_rank());
  const int ncl = static_cast<int>(cluster.num_blocks());
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int b = A.big_list[blockIdx.x / ncl];
  const int4 bd = A.body_desc[b];
  const int start = bd.x, n = bd.y, W = bd.z;
  const int wi = r * (nt >> 5) + warp;
  const bool live = wi < W;
  const int K = pbdr_body_slots(n, W);
  const bool fixes = A.linfix || A.angfix;
  const int n_iters = A.multi_pairs ? 1 : A.n_iters;  // several only without pairs (state stays in smem)
  float* lead_part = cluster.map_shared_rank(&s_part[0][0], 0);
  const float* lead_res = cluster.map_shared_rank(&s_res[0], 0);

  if (threadIdx.x == 0) {
    mbar_init(&s_bar, 1);
    // Row k of the body holds slots k*32*W .. (k+1)*32*W; this CTA's part of
    // it is the nt slots from k*32*W + r*nt (clipped to the row and to n).
    uint32_t total = 0;
    for (int k = 0; k < K; ++k) {
      const int q0 = k * 32 * W + r * nt;
      const int q1 = min(min(q0 + nt, (k + 1) * 32 * W), n);
      if (q1 > q0) total += 3u * 16u * static_cast<uint32_t>(q1 - q0);
    }
    mbar_expect_tx(&s_bar, total);
    for (int k = 0; k < K; ++k) {
      const int q0 = k * 32 * W + r * nt;
      const int q1 = min(min(q0 + nt, (k + 1) * 32 * W), n);
      if (q1 <= q0) continue;
      const uint32_t bytes = 16u * static_cast<uint32_t>(q1 - q0);
      bulk_g2s_stream(s_pos + k * nt, A.pos_in + start + q0, bytes, &s_bar);
      bulk_g2s_stream(s_vel + k * nt, A.vel + start + q0, bytes, &s_bar);
      bulk_g2s_stream(s_rest + k * nt, A.rest + start + q0, bytes, &s_bar);
    }
    if (r == 0) s_rq = A.rquat[b];
  }
  if (threadIdx.x < 3) s_res[kResA + threadIdx.x] = (&A.anchor[b].x)[threadIdx.x];
  int ncs[KP];
#pragma unroll
  for (int k = 0; k < KP; ++k) {
    const int q = k * 32 * W + wi * 32 + lane;
    ncs[k] = (live && q < n) ? A.ncand[start + q] : 0;
  }
  __syncthreads();         // s_res anchor, barrier init (CTA-local ordering)
  cluster_sync_relaxed();  // every CTA of the cluster running (DSMEM targets exist)
  mbar_wait(&s_bar, 0);

  for (int it = 0; it < n_iters; ++it) {
    const int iter_index = A.iter_index + it;
    const int last_iter = A.last_iter && it == n_iters - 1;
    const float a[3] = {s_res[kResA], s_res[kResA + 1], s_res[kResA + 2]};
    float dX[KP][3];

    // ---- Phase A ----------------------------------------------------------
    float acc[21];
#pragma unroll
    for (int f = 0; f < 21; ++f) acc[f] = 0.0f;
#pragma unroll
    for (int k = 0; k < KP; ++k) dX[k][0] = dX[k][1] = dX[k][2] = 0.0f;
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      const int q = k * 32 * W + wi * 32 + lane;
      if (!(live && q < n)) continue;
      const int li = k * nt + threadIdx.x;
      phase_a_particle<false>(A, it, start + q, s_pos[li], s_vel[li], s_rest[li], ncs[k], a, dX[k], acc, nullptr, 0,
                              0);
    }
    if (live) {
      float a16[16], a5[5];  // 16 + 5 fields, as in k_iteration
#pragma unroll
      for (int f = 0; f < 16; ++f) a16[f] = acc[f];
#pragma unroll
      for (int f = 0; f < 5; ++f) a5[f] = acc[16 + f];
      const float t16 = warp_reduce_scatter<16>(a16);
      const float t5 = warp_reduce_scatter<5>(a5);
      if ((lane & 1) == 0) lead_part[wi * 21 + (lane >> 1)] = t16;
      if ((lane & 3) == 0 && (lane >> 2) < 5) lead_part[wi * 21 + 16 + (lane >> 2)] = t5;
    }
    cluster.sync();
    if (r == 0) {
      // Stage 3 of the tree: per field, serially over the warps (one thread
      // per field), then the body math on one thread.
      if (threadIdx.x < 21) {
        float t = s_part[0][threadIdx.x];
        for (int u = 1; u < W; ++u) t = t + s_part[u][threadIdx.x];
        s_sum[threadIdx.x] = t;
      }
      __syncthreads();
    }
    if (r == 0 && threadIdx.x == 0) {
      float S[21];
#pragma unroll
      for (int f = 0; f < 21; ++f) S[f] = s_sum[f];
      const float4 an = make_float4(a[0], a[1], a[2], 0.0f);
      float4 rq_new, an_new;
      body_math_a<false>(A, b, S, an, A.body_mass[b].y, s_rq, s_res, rq_new, an_new);
      s_rq = rq_new;
      s_res[kResA] = an_new.x;
      s_res[kResA + 1] = an_new.y;
      s_res[kResA + 2] = an_new.z;
    }
    cluster.sync();
    if (r != 0 && threadIdx.x < kResF) s_res[threadIdx.x] = lead_res[threadIdx.x];
    if (r == 0 && threadIdx.x == 0) {  // after the barrier: its release need not wait for them
      A.rquat[b] = s_rq;
      A.anchor[b] = make_float4(s_res[kResA], s_res[kResA + 1], s_res[kResA + 2], 0.0f);
    }
    __syncthreads();

    // ---- Phase B ----------------------------------------------------------
    float accB[15];
#pragma unroll
    for (int f = 0; f < 15; ++f) accB[f] = 0.0f;
    if (live) {
      const bool sm_ok = s_res[kResSmOk] != 0.0f;
      float Rf[9], c[3];
#pragma unroll
      for (int f = 0; f < 9; ++f) Rf[f] = s_res[kResR + f];
#pragma unroll
      for (int k = 0; k < 3; ++k) c[k] = s_res[kResC + k];
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        const int q = k * 32 * W + wi * 32 + lane;
        if (!(q < n)) continue;
        const int li = k * nt + threadIdx.x;
        const float4 x4 = s_pos[li];
        const float4 v4 = s_vel[li];
        float xa[3], va[3], pa[3];
        phase_b_particle(A, start + q, x4, v4, s_rest[li], a, sm_ok, Rf, c, dX[k], xa, va, pa);
        if (fixes) {
          accum_b(v4.w, dX[k], va, pa, accB);
        } else if (n_iters > 1) {
          s_pos[li] = make_float4(xa[0], xa[1], xa[2], x4.w);
          s_vel[li] = make_float4(va[0], va[1], va[2], v4.w);
        } else {
          A.pos_out[start + q] = make_float4(xa[0], xa[1], xa[2], x4.w);
          A.vel[start + q] = make_float4(va[0], va[1], va[2], v4.w);
        }
      }
    }
    if (fixes) {
      if (live) {
        const float tot = warp_reduce_scatter<15>(accB);  // lanes 2f, 2f+1: field f
        if ((lane & 1) == 0 && (lane >> 1) < 15) lead_part[wi * 21 + (lane >> 1)] = tot;
      }
      cluster.sync();
      if (r == 0) {
        if (threadIdx.x < 15) {
          float t = s_part[0][threadIdx.x];
          for (int u = 1; u < W; ++u) t = t + s_part[u][threadIdx.x];
          s_sum[threadIdx.x] = t;
        }
        __syncthreads();
      }
      if (r == 0 && threadIdx.x == 0) {
        float S[15];
#pragma unroll
        for (int f = 0; f < 15; ++f) S[f] = s_sum[f];
        body_math_b(A, b, S, A.body_mass[b], s_res, iter_index, last_iter);
      }
      cluster.sync();
      if (r != 0 && threadIdx.x < kResF) s_res[threadIdx.x] = lead_res[threadIdx.x];
      __syncthreads();

      // ---- Phase C --------------------------------------------------------
      if (live) {
        float ca[3], dv[3], om[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          ca[k] = s_res[kResCa + k];
          dv[k] = s_res[kResDv + k];
          om[k] = s_res[kResW + k];
        }
#pragma unroll
        for (int k = 0; k < KP; ++k) {
          const int q = k * 32 * W + wi * 32 + lane;
          if (!(q < n)) continue;
          const int li = k * nt + threadIdx.x;
          const float4 x4 = s_pos[li];
          const float4 v4 = s_vel[li];
          float xo[3], vo[3];
          phase_c_particle(A, start + q, x4, v4, a, dX[k], ca, dv, om, xo, vo);
          if (n_iters > 1) {
            s_pos[li] = make_float4(xo[0], xo[1], xo[2], x4.w);
            s_vel[li] = make_float4(vo[0], vo[1], vo[2], v4.w);
          } else {
            A.pos_out[start + q] = make_float4(xo[0], xo[1], xo[2], x4.w);
            A.vel[start + q] = make_float4(vo[0], vo[1], vo[2], v4.w);
          }
        }
      }
    }
    __syncthreads();  // s_res (anchor) and the staged state of the next iteration
  }
  if (n_iters > 1 && live)
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      const int q = k * 32 * W + wi * 32 + lane;
      if (q < n) {
        const int li = k * nt + threadIdx.x;
        A.pos_out[start + q] = s_pos[li];
        A.vel[start + q] = s_vel[li];
      }
    }
  cluster_sync_relaxed();  // the leader's shared memory outlives every remote read
}

// ---------------------------------------------------------------------------
// Per-body trajectory sample: com, orientation (extract_pose), P, L.
// ---------------------------------------------------------------------------
// Terms of particle p in the 18 trajectory sums (anchor-relative m x, Apq, P,
// L about the anchor).
__device__ __forceinline__ void stats_accum(const StatsArgs& A, int64_t p, const float a[3], float (&acc)[18]) {
  const float4 x4 = A.pos[p];
  const float4 v4 = A.vel[p];
  const float4 r4 = A.rest[p];
  const float mk = v4.w;
  const float pp[3] = {x4.x - a[0], x4.y - a[1], x4.z - a[2]};
  const float mp[3] = {mk * pp[0], mk * pp[1], mk * pp[2]};
  const float mv[3] = {mk * v4.x, mk * v4.y, mk * v4.z};
  const float q0[3] = {r4.x, r4.y, r4.z};
  float kk[3];
  cross3(pp, mv, kk);
  acc[0] = acc[0] + mp[0];
  acc[1] = acc[1] + mp[1];
  acc[2] = acc[2] + mp[2];
#pragma unroll
  for (int rI = 0; rI < 3; ++rI)
#pragma unroll
    for (int cI = 0; cI < 3; ++cI) acc[3 + 3 * rI + cI] = acc[3 + 3 * rI + cI] + mp[rI] * q0[cI];
  acc[12] = acc[12] + mv[0];
  acc[13] = acc[13] + mv[1];
  acc[14] = acc[14] + mv[2];
  acc[15] = acc[15] + kk[0];
  acc[16] = acc[16] + kk[1];
  acc[17] = acc[17] + kk[2];
}

// Trajectory sample of body bb from its 18 sums: com, orientation, P, L.
__device__ __forceinline__ void stats_body_out(const StatsArgs& A, int bb, const float (&S)[18]) {
  const float4 an = A.anchor[bb];
  const float a[3] = {an.x, an.y, an.z};
  const float invM = A.body_mass[bb].y;
  float c[3], P[3], tmp[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    c[k] = S[k] * invM;
    P[k] = S[12 + k];
  }
  cross3(c, P, tmp);
  float Rf[9];
  double qd[4];
  if (!polar_rotation_f(&S[3], Rf, qd)) {
    qd[0] = 1.0; qd[1] = 0.0; qd[2] = 0.0; qd[3] = 0.0;
  }
  double* o = A.out + 13 * static_cast<int64_t>(bb);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    o[k] = static_cast<double>(a[k]) + static_cast<double>(c[k]);
    o[7 + k] = static_cast<double>(P[k]);
    o[10 + k] = static_cast<double>(S[15 + k] - tmp[k]);
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) o[3 + k] = qd[k];
}

template <int KP>
__global__ void __launch_bounds__(kThreads) k_body_stats(StatsArgs A) {
  __shared__ float s_part[kWarps][18];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int4 cd = A.cta_desc[blockIdx.x];
  const int4 wd = A.warp_desc[blockIdx.x * kWarps + warp];
  const int b = wd.x;
  const int wi = wd.y;
  const bool live = b >= 0;
  float acc[18];
#pragma unroll
  for (int f = 0; f < 18; ++f) acc[f] = 0.0f;
  if (live) {
    const int4 bd = make_int4(wd.z, wd.w & 0xFFFF, wd.w >> 16, 0);
    const float4 an = A.anchor[b];
    const float a[3] = {an.x, an.y, an.z};
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      const int q = k * 32 * bd.z + wi * 32 + lane;
      if (q >= bd.y) continue;
      stats_accum(A, bd.x + q, a, acc);
    }
    warp_butterfly<18>(acc);
    if (lane == 0)
#pragma unroll
      for (int f = 0; f < 18; ++f) s_part[warp][f] = acc[f];
  }
  __syncthreads();
  if (!(warp == 0 && lane < cd.w)) return;
  const int bb = cd.z + lane;
  const int4 bd = A.body_desc[bb];
  float S[18];
#pragma unroll
  for (int f = 0; f < 18; ++f) S[f] = s_part[bd.w][f];
  for (int u = 1; u < bd.z; ++u)
#pragma unroll
    for (int f = 0; f < 18; ++f) S[f] = S[f] + s_part[bd.w + u][f];
  stats_body_out(A, bb, S);
}


// Trajectory sample of a body larger than one CTA: one CTA per body, each warp
// loops over the body's warps wi = warp, warp + 8, ... (same tree).
__global__ void __launch_bounds__(kThreads) k_body_stats_big(StatsArgs A) {
  __shared__ float s_part[kBigMaxWarps][18];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int b = A.big_list[blockIdx.x];
  const int4 bd = A.body_desc[b];
  const float4 an = A.anchor[b];
  const float a[3] = {an.x, an.y, an.z};
  for (int wi = warp; wi < bd.z; wi += kWarps) {
    float acc[18];
#pragma unroll
    for (int f = 0; f < 18; ++f) acc[f] = 0.0f;
#pragma unroll
    for (int k = 0; k < PBDR_KP_MAX; ++k) {
      const int q = k * 32 * bd.z + wi * 32 + lane;
      if (q < bd.y) stats_accum(A, bd.x + q, a, acc);
    }
    warp_butterfly<18>(acc);
    if (lane == 0)
#pragma unroll
      for (int f = 0; f < 18; ++f) s_part[wi][f] = acc[f];
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  float S[18];
#pragma unroll
  for (int f = 0; f < 18; ++f) S[f] = s_part[0][f];
  for (int u = 1; u < bd.z; ++u)
#pragma unroll
    for (int f = 0; f < 18; ++f) S[f] = S[f] + s_part[u][f];
  stats_body_out(A, b, S);
}

// ---------------------------------------------------------------------------
// Torque programs: per-body com, inertia and alpha = pinv(I) tau of X at the
// substep start (distribute_wrench, body.cpp:126-150). Same reduction tree as
// every body sum (pbdr_pinned.h); the oracle mirrors it (integrate()).
// ---------------------------------------------------------------------------
// Terms of particle p in the 9 wrench sums (anchor-relative m x and inertia).
__device__ __forceinline__ void wrench_accum(const WrenchArgs& A, int64_t p, const float a[3], float (&acc)[9]) {
  const float4 x4 = A.pos[p];
  const float mk = A.vel[p].w;
  const float pp[3] = {x4.x - a[0], x4.y - a[1], x4.z - a[2]};
  const float s2 = (pp[0] * pp[0] + pp[1] * pp[1]) + pp[2] * pp[2];
  acc[0] = acc[0] + mk * pp[0];
  acc[1] = acc[1] + mk * pp[1];
  acc[2] = acc[2] + mk * pp[2];
  acc[3] = acc[3] + mk * (s2 - pp[0] * pp[0]);
  acc[4] = acc[4] + mk * (s2 - pp[1] * pp[1]);
  acc[5] = acc[5] + mk * (s2 - pp[2] * pp[2]);
  acc[6] = acc[6] + -(mk * (pp[0] * pp[1]));
  acc[7] = acc[7] + -(mk * (pp[0] * pp[2]));
  acc[8] = acc[8] + -(mk * (pp[1] * pp[2]));
}

// com, inertia and alpha = pinv(I) tau of body bb from its 9 sums.
__device__ __forceinline__ void wrench_body_out(const WrenchArgs& A, int bb, const float (&S)[9],
                                                const BodyProgram& pr) {
  const float2 mass = A.body_mass[bb];
  const float M = mass.x, invM = mass.y;
  const float4 an = A.anchor[bb];
  float c[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) c[k] = S[k] * invM;
  float If[6];
  If[0] = S[3] - M * (c[1] * c[1] + c[2] * c[2]);
  If[1] = S[4] - M * (c[0] * c[0] + c[2] * c[2]);
  If[2] = S[5] - M * (c[0] * c[0] + c[1] * c[1]);
  If[3] = S[6] + M * (c[0] * c[1]);
  If[4] = S[7] + M * (c[0] * c[2]);
  If[5] = S[8] + M * (c[1] * c[2]);
  const float tau[3] = {pr.tx, pr.ty, pr.tz};
  float al[3];
  double nax[3];
  const unsigned e = inertia_solve_f(If, tau, al, nax);
  if (e) record_error(A.err, e, bb, A.substep_counter, nax);
  A.wcom[bb] = make_float4(an.x + c[0], an.y + c[1], an.z + c[2], 0.0f);
  A.walpha[bb] = make_float4(al[0], al[1], al[2], 0.0f);
}

template <int KP>
__global__ void __launch_bounds__(kThreads) k_body_wrench(WrenchArgs A) {
  __shared__ float s_part[kWarps][9];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int4 cd = A.cta_desc[blockIdx.x];
  const int4 wd = A.warp_desc[blockIdx.x * kWarps + warp];
  const int b = wd.x;
  const int wi = wd.y;
  const bool live = b >= 0 && (A.programs[b].flags & 4);
  float acc[9];
#pragma unroll
  for (int f = 0; f < 9; ++f) acc[f] = 0.0f;
  if (live) {
    const int start = wd.z, n = wd.w & 0xFFFF, W = wd.w >> 16;
    const float4 an = A.anchor[b];
    const float a[3] = {an.x, an.y, an.z};
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      const int q = k * 32 * W + wi * 32 + lane;
      if (q >= n) continue;
      wrench_accum(A, start + q, a, acc);
    }
    warp_butterfly<9>(acc);
    if (lane == 0)
#pragma unroll
      for (int f = 0; f < 9; ++f) s_part[warp][f] = acc[f];
  }
  __syncthreads();
  if (!(warp == 0 && lane < cd.w)) return;
  const int bb = cd.z + lane;
  const BodyProgram pr = A.programs[bb];
  if (!(pr.flags & 4)) return;
  const int4 bd = A.body_desc[bb];
  float S[9];
#pragma unroll
  for (int f = 0; f < 9; ++f) S[f] = s_part[bd.w][f];
  for (int u = 1; u < bd.z; ++u)
#pragma unroll
    for (int f = 0; f < 9; ++f) S[f] = S[f] + s_part[bd.w + u][f];
  wrench_body_out(A, bb, S, pr);
}


// Torque prepass of a body larger than one CTA (one CTA per body, looping warps).
__global__ void __launch_bounds__(kThreads) k_body_wrench_big(WrenchArgs A) {
  __shared__ float s_part[kBigMaxWarps][9];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int b = A.big_list[blockIdx.x];
  const BodyProgram pr = A.programs[b];
  if (!(pr.flags & 4)) return;  // CTA-uniform
  const int4 bd = A.body_desc[b];
  const float4 an = A.anchor[b];
  const float a[3] = {an.x, an.y, an.z};
  for (int wi = warp; wi < bd.z; wi += kWarps) {
    float acc[9];
#pragma unroll
    for (int f = 0; f < 9; ++f) acc[f] = 0.0f;
#pragma unroll
    for (int k = 0; k < PBDR_KP_MAX; ++k) {
      const int q = k * 32 * bd.z + wi * 32 + lane;
      if (q < bd.y) wrench_accum(A, bd.x + q, a, acc);
    }
    warp_butterfly<9>(acc);
    if (lane == 0)
#pragma unroll
      for (int f = 0; f < 9; ++f) s_part[wi][f] = acc[f];
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  float S[9];
#pragma unroll
  for (int f = 0; f < 9; ++f) S[f] = s_part[0][f];
  for (int u = 1; u < bd.z; ++u)
#pragma unroll
    for (int f = 0; f < 9; ++f) S[f] = S[f] + s_part[u][f];
  wrench_body_out(A, b, S, pr);
}

}  // namespace

size_t iteration_smem_bytes(int kp) {
  return sizeof(float4) * ((PBDR_ROLL_PARTICLES != 0 && kp <= 4) ? 4 : 3) * kThreads * kp;
}

void launch_integrate(const IntegrateArgs& a, cudaStream_t s) {
  const unsigned blocks = static_cast<unsigned>((a.n - a.p0 + 255) / 256);
  if (blocks == 0) return;
  k_integrate_key<<<blocks, 256, 0, s>>>(a);
}

void launch_body_keys(const BroadArgs& a, cudaStream_t s) {
  if (a.nb == 0) return;
  k_body_keys<<<(a.nb + 255) / 256, 256, 0, s>>>(a);
}

void launch_body_ranges(const BroadArgs& a, cudaStream_t s) {
  if (a.nb == 0) return;
  k_body_ranges<<<(a.nb + 255) / 256, 256, 0, s>>>(a);
}

void launch_classify_tiles(const ClassifyArgs& a, cudaStream_t s) {
  if (a.ntiles <= 0) return;
  k_classify_tiles<<<(a.ntiles + 255) / 256, 256, 0, s>>>(a);
}

void launch_scene_partners(const BroadArgs& a, cudaStream_t s) {
  if (a.nb <= 0) return;
  k_scene_partners<<<static_cast<unsigned>((static_cast<int64_t>(a.nb) * 32 + 255) / 256), 256, 0, s>>>(a);
}

void launch_body_partners(const BroadArgs& a, cudaStream_t s) {
  if (a.nb == 0) return;
  k_body_partners<<<static_cast<unsigned>((static_cast<int64_t>(a.nb) * 32 + 255) / 256), 256, 0, s>>>(a);
}

void launch_near(const NearArgs& a, cudaStream_t s) {
  if (a.nbl > 0) {
    const unsigned wblocks = static_cast<unsigned>((static_cast<int64_t>(a.nbl) * 32 + 255) / 256);
    if (a.obb_q && !a.all_near)
      k_body_obb<<<std::min<unsigned>(wblocks, 148u * 16u), 256, 0, s>>>(a);
    // One warp per body fills the GPU from ~64K bodies on; below that, eight.
    if (a.nbl >= (1 << 16)) {
      k_near_count<1><<<wblocks, 256, 0, s>>>(a);
    } else {
      constexpr int kSplit = 8;
      cudaMemsetAsync(a.body_near, 0, sizeof(uint32_t) * static_cast<size_t>(a.nbl), s);
      k_near_count<kSplit><<<static_cast<unsigned>((static_cast<int64_t>(a.nbl) * kSplit * 32 + 255) / 256), 256, 0, s>>>(a);
    }
    k_near_scan_tiles<<<(a.nbl + kScanTile - 1) / kScanTile, 1024, 0, s>>>(a);
    k_near_scan_top<<<1, 1024, 0, s>>>(a);
    k_near_write<<<wblocks, 256, 0, s>>>(a);
  } else {
    cudaMemsetAsync(a.count, 0, sizeof(long long), s);
  }
}

// Slab halo exchange: float4 records by index (particle slots or body ids).
__global__ void __launch_bounds__(256) k_gather4(float4* __restrict__ dst, const float4* __restrict__ src,
                                                 const int* __restrict__ idx, int64_t count) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < count) {
    PBDR_CHECK(idx[t] >= 0);
    dst[t] = src[idx[t]];
  }
}

__global__ void __launch_bounds__(256) k_scatter4(float4* __restrict__ dst, const float4* __restrict__ src,
                                                  const int* __restrict__ idx, int64_t count) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < count) {
    PBDR_CHECK(idx[t] >= 0);
    dst[idx[t]] = src[t];
  }
}

void launch_gather4(float4* dst, const float4* src, const int* idx, int64_t count, cudaStream_t s) {
  if (count > 0) k_gather4<<<static_cast<unsigned>((count + 255) / 256), 256, 0, s>>>(dst, src, idx, count);
}

void launch_scatter4(float4* dst, const float4* src, const int* idx, int64_t count, cudaStream_t s) {
  if (count > 0) k_scatter4<<<static_cast<unsigned>((count + 255) / 256), 256, 0, s>>>(dst, src, idx, count);
}

static unsigned stride_grid(int64_t n_max) {
  const int64_t want = (n_max + 255) / 256;
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(want, 148 * 16)));
}

// pbdr_gpu_write_particles / read_particles on the device: the caller's fp64
// Scene::particles arrays (position[3i..], velocity[3i..], body.hpp:11-17) are
// staged in HBM and converted (round to nearest) and permuted into the
// body-major float4 slots, or the reverse. Slot s holds caller particle
// slot_particle[s]; .w (inverse mass / mass) is kept.
__global__ void __launch_bounds__(256) k_particles_in(float4* __restrict__ pos, float4* __restrict__ vel,
                                                      const double* __restrict__ x, const double* __restrict__ v,
                                                      const int* __restrict__ slot_particle, int64_t n) {
  for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < n;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = slot_particle[s];
    PBDR_CHECK(i >= 0 && i < n);
    if (x) {
      float4 p = pos[s];
      p.x = static_cast<float>(x[3 * i]);
      p.y = static_cast<float>(x[3 * i + 1]);
      p.z = static_cast<float>(x[3 * i + 2]);
      pos[s] = p;
    }
    if (v) {
      float4 q = vel[s];
      q.x = static_cast<float>(v[3 * i]);
      q.y = static_cast<float>(v[3 * i + 1]);
      q.z = static_cast<float>(v[3 * i + 2]);
      vel[s] = q;
    }
  }
}

__global__ void __launch_bounds__(256) k_particles_out(const float4* __restrict__ pos,
                                                       const float4* __restrict__ vel, double* __restrict__ x,
                                                       double* __restrict__ v,
                                                       const int* __restrict__ slot_particle, int64_t n) {
  for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < n;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = slot_particle[s];
    if (x) {
      const float4 p = pos[s];
      x[3 * i] = p.x;
      x[3 * i + 1] = p.y;
      x[3 * i + 2] = p.z;
    }
    if (v) {
      const float4 q = vel[s];
      v[3 * i] = q.x;
      v[3 * i + 1] = q.y;
      v[3 * i + 2] = q.z;
    }
  }
}

// After new positions: each body's anchor (origin of its fp32 body sums) is
// its first slot's position, as at create.
__global__ void __launch_bounds__(256) k_anchor_reset(float4* __restrict__ anchor, const int4* __restrict__ body_desc,
                                                      const float4* __restrict__ pos, int nb) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < nb) {
    const float4 p = pos[body_desc[b].x];
    anchor[b] = make_float4(p.x, p.y, p.z, 0.0f);
  }
}

void launch_particles_in(float4* pos, float4* vel, const double* x, const double* v, const int* slot_particle,
                         int64_t n, cudaStream_t s) {
  if (n > 0) k_particles_in<<<stride_grid(n), 256, 0, s>>>(pos, vel, x, v, slot_particle, n);
}

void launch_particles_out(const float4* pos, const float4* vel, double* x, double* v, const int* slot_particle,
                          int64_t n, cudaStream_t s) {
  if (n > 0) k_particles_out<<<stride_grid(n), 256, 0, s>>>(pos, vel, x, v, slot_particle, n);
}

void launch_anchor_reset(float4* anchor, const int4* body_desc, const float4* pos, int nb, cudaStream_t s) {
  if (nb > 0) k_anchor_reset<<<(nb + 255) / 256, 256, 0, s>>>(anchor, body_desc, pos, nb);
}

__global__ void k_tick(long long* substep_counter) {
  atomicAdd(reinterpret_cast<unsigned long long*>(substep_counter), 1ull);
}

void launch_tick(long long* substep_counter, cudaStream_t s) { k_tick<<<1, 1, 0, s>>>(substep_counter); }

void launch_ncand_clear(int* ncand, const int* prev_near, const long long* prev_count, int64_t n_max,
                        cudaStream_t s) {
  k_ncand_clear<<<stride_grid(n_max), 256, 0, s>>>(ncand, prev_near, prev_count);
}

void launch_cell_clear(uint4* cells, const uint32_t* prev_keys, const long long* prev_count, int64_t n_max,
                       cudaStream_t s) {
  k_cell_clear<<<stride_grid(n_max), 256, 0, s>>>(cells, prev_keys, prev_count);
}

void launch_ranges(const RangesArgs& a, cudaStream_t s) {
  k_cell_ranges<<<stride_grid(a.n), 256, 0, s>>>(a);
}

void launch_neighbours(const NeighbourArgs& a, cudaStream_t s) {
  static const bool staged = [] {
    const char* e = std::getenv("PBDR_NBR_STAGED");
    return PBDR_NBR_STAGED != 0 && !(e && e[0] == '0');
  }();
  if (staged && a.layout.linear && a.single_scene) {
    // Persistent: 6 CTAs of 128 threads (33 KB shared) per SM.
    const unsigned blocks = static_cast<unsigned>(
        std::max<int64_t>(1, std::min<int64_t>((a.n + kNbrChunk - 1) / kNbrChunk, 148 * 6)));
    k_neighbours_staged<<<blocks, kNbrChunk, 0, s>>>(a);
    return;
  }
  const unsigned blocks = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((a.n + 127) / 128, 148 * 64)));
  k_neighbours<<<blocks, 128, 0, s>>>(a);
}

static int g_iter_grid_cap[9] = {0};  // resident iteration CTAs on the device, per KP (persistent grid)
static int g_iter_coop_cap[9] = {0};  // resident multi-iteration CTAs (cooperative launch), per KP

template <int KP>
static cudaError_t prepare_one() {
  cudaError_t e = cudaFuncSetAttribute(k_iteration<KP, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(iteration_smem_bytes(KP)));
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k_iteration<KP, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(iteration_smem_bytes(KP)));
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k_iteration<KP, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(iteration_smem_bytes(KP)));
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_iteration<KP, false>, kThreads, iteration_smem_bytes(KP));
  g_iter_grid_cap[KP] = sms * per_sm;
  // Debug/test cap on the persistent grid (PBDR_ITER_GRID_CAP=k): small scenes
  // then take the multi-tile path (dynamic claims, next-tile table prefetch)
  // that otherwise only BASELINE-size scenes reach. Re-read at every create.
  if (const char* cap = std::getenv("PBDR_ITER_GRID_CAP")) {
    const int c = std::atoi(cap);
    if (c > 0) g_iter_grid_cap[KP] = std::min(g_iter_grid_cap[KP], c);
  }
  int per_sm_multi = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_multi, k_iteration<KP, true>, kThreads, iteration_smem_bytes(KP));
  g_iter_coop_cap[KP] = sms * per_sm_multi;
#ifdef PBDR_ITER_CARVEOUT
  return cudaFuncSetAttribute(k_iteration<KP, false>, cudaFuncAttributePreferredSharedMemoryCarveout, PBDR_ITER_CARVEOUT);
#else
  return cudaSuccess;
#endif
}

#if PBDR_CHECKED
static CheckRecord* g_check_host = nullptr;
#endif
// Checked build: the failed device check behind a CUDA error, if any
// ("pbdr_kernels.cu:LINE block B thread T"); empty otherwise.
std::string checked_failure() {
#if PBDR_CHECKED
  if (g_check_host && g_check_host->hit) {
    char buf[160];
    std::snprintf(buf, sizeof(buf), " [PBDR_CHECK failed at pbdr_kernels.cu:%d block %d thread %d]",
                  g_check_host->line, g_check_host->block, g_check_host->thread);
    return buf;
  }
#endif
  return std::string();
}

cudaError_t prepare_iteration_kernel() {
#if PBDR_CHECKED
  if (!g_check_host) {
    cudaError_t ce = cudaHostAlloc(reinterpret_cast<void**>(&g_check_host), sizeof(CheckRecord), cudaHostAllocMapped);
    if (ce != cudaSuccess) return ce;
    *g_check_host = CheckRecord{0, 0, 0, 0};
    CheckRecord* dev = nullptr;
    ce = cudaHostGetDevicePointer(reinterpret_cast<void**>(&dev), g_check_host, 0);
    if (ce == cudaSuccess) ce = cudaMemcpyToSymbol(g_check_record, &dev, sizeof(dev));
    if (ce != cudaSuccess) return ce;
  }
#endif
  cudaError_t e = prepare_one<2>();
  if (e == cudaSuccess) e = prepare_one<4>();
  if (e == cudaSuccess) e = prepare_one<7>();
  if (e == cudaSuccess) e = prepare_one<8>();
  return e;
}

// Persistent grid: one wave of resident CTAs claims tiles dynamically and
// prefetches each next tile's descriptors and body table.
#ifndef PBDR_ITER_PERSISTENT
#define PBDR_ITER_PERSISTENT 1
#endif

template <int KP>
static void launch_iteration_kp(const IterArgs& a, int ctas, cudaStream_t s) {
  IterArgs b = a;
  b.ntiles = ctas;
  int grid = ctas;
  if (PBDR_ITER_PERSISTENT && g_iter_grid_cap[KP] > 0 && !a.timing) grid = std::min(ctas, g_iter_grid_cap[KP]);
  if (a.tile_count && g_iter_grid_cap[KP] > 0) grid = std::min(ctas, g_iter_grid_cap[KP]);  // count on the device
  if (a.n_iters > 1 && a.multi_pairs == 2) {
    // Batched scenes: one cluster of a.cluster CTAs per scene (its tiles),
    // one tile per CTA, iterating together with cluster barriers.
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(ctas));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = iteration_smem_bytes(KP);
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = static_cast<unsigned>(a.cluster);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
#ifndef PBDR_CLUSTER_POLICY
#define PBDR_CLUSTER_POLICY cudaClusterSchedulingPolicySpread
#endif
    attr[1].id = cudaLaunchAttributeClusterSchedulingPolicyPreference;
    attr[1].val.clusterSchedulingPolicyPreference = PBDR_CLUSTER_POLICY;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    cudaLaunchKernelEx(&cfg, k_iteration<KP, true>, b);
  } else if (a.n_iters > 1 && a.multi_pairs) {
    // One wave of tiles iterating together: grid barriers need a cooperative
    // launch (every CTA resident; the engine checks iteration_coop_capacity).
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(ctas));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = iteration_smem_bytes(KP);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_iteration<KP, true>, b);
  } else if (a.n_iters > 1) {
    k_iteration<KP, true><<<grid, kThreads, iteration_smem_bytes(KP), s>>>(b);
  } else
    if (a.fuse_integrate)
      k_iteration<KP, false, true><<<grid, kThreads, iteration_smem_bytes(KP), s>>>(b);
    else
      k_iteration<KP, false><<<grid, kThreads, iteration_smem_bytes(KP), s>>>(b);
}

int iteration_coop_capacity(int kp) { return g_iter_coop_cap[kp == 2 ? 2 : (kp == 4 ? 4 : (kp == 7 ? 7 : 8))]; }

template <int KP>
static int scene_clusters_kp(int cluster) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(cluster));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = iteration_smem_bytes(KP);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(cluster);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, k_iteration<KP, true>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int iteration_scene_clusters(int kp, int cluster) {
  switch (kp) {
    case 2: return scene_clusters_kp<2>(cluster);
    case 4: return scene_clusters_kp<4>(cluster);
    case 7: return scene_clusters_kp<7>(cluster);
    default: return scene_clusters_kp<8>(cluster);
  }
}

void launch_iteration(const IterArgs& a, int ctas, int kp, cudaStream_t s) {
  switch (kp) {
    case 2: launch_iteration_kp<2>(a, ctas, s); break;
    case 4: launch_iteration_kp<4>(a, ctas, s); break;
    case 7: launch_iteration_kp<7>(a, ctas, s); break;
    default: launch_iteration_kp<8>(a, ctas, s); break;
  }
}

void launch_wrench(const WrenchArgs& a, int ctas, int kp, cudaStream_t s) {
  switch (kp) {
    case 2: k_body_wrench<2><<<ctas, kThreads, 0, s>>>(a); break;
    case 4: k_body_wrench<4><<<ctas, kThreads, 0, s>>>(a); break;
    case 7: k_body_wrench<7><<<ctas, kThreads, 0, s>>>(a); break;
    default: k_body_wrench<8><<<ctas, kThreads, 0, s>>>(a); break;
  }
}

void launch_stats(const StatsArgs& a, int ctas, int kp, cudaStream_t s) {
  switch (kp) {
    case 2: k_body_stats<2><<<ctas, kThreads, 0, s>>>(a); break;
    case 4: k_body_stats<4><<<ctas, kThreads, 0, s>>>(a); break;
    case 7: k_body_stats<7><<<ctas, kThreads, 0, s>>>(a); break;
    default: k_body_stats<8><<<ctas, kThreads, 0, s>>>(a); break;
  }
}

// ---- bodies larger than one CTA ---------------------------------------------
int big_cluster_size(int max_warps) { return (max_warps + kWarps - 1) / kWarps; }

static bool g_big_prepared = false;
static cudaError_t prepare_big() {
  if (g_big_prepared) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(k_iteration_big, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(iteration_smem_bytes(PBDR_KP_MAX)));
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_iteration_big, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  g_big_prepared = e == cudaSuccess;
  return e;
}

static cudaLaunchConfig_t big_config(unsigned grid, int cluster, int warps, cudaStream_t s,
                                     cudaLaunchAttribute* attr) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(32 * warps);
  cfg.dynamicSmemBytes = sizeof(float4) * 3 * 32 * warps * PBDR_KP_MAX;
  cfg.stream = s;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(cluster);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cfg;
}

int big_cta_warps(int max_warps, int cluster) { return (max_warps + cluster - 1) / cluster; }

cudaError_t big_cluster_check(int cluster, int warps) {
  if (cluster < 1 || cluster > PBDR_MAX_CLUSTER_CTAS || warps < 1 || warps > kWarps) return cudaErrorInvalidValue;
  cudaError_t e = prepare_big();
  if (e != cudaSuccess) return e;
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = big_config(static_cast<unsigned>(cluster), cluster, warps, nullptr, attr);
  int active = 0;
  e = cudaOccupancyMaxActiveClusters(&active, k_iteration_big, &cfg);
  if (e != cudaSuccess) return e;
  return active > 0 ? cudaSuccess : cudaErrorInvalidClusterSize;
}

void launch_iteration_big(const IterArgs& a, int nbig, int cluster, int warps, cudaStream_t s) {
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = big_config(static_cast<unsigned>(nbig * cluster), cluster, warps, s, attr);
  cudaLaunchKernelEx(&cfg, k_iteration_big, a);
}

void launch_stats_big(const StatsArgs& a, int nbig, cudaStream_t s) {
  k_body_stats_big<<<nbig, kThreads, 0, s>>>(a);
}

void launch_wrench_big(const WrenchArgs& a, int nbig, cudaStream_t s) {
  k_body_wrench_big<<<nbig, kThreads, 0, s>>>(a);
}

}  // namespace pbdr_dev
