/* Pinned constants shared by the CUDA path and the CPU oracle.
 *
 * The reference's solver (proj/src/solver.cpp, listed at proj/CMakeLists.txt:20)
 * is absent, so several choices its code would have fixed are pinned here once
 * and documented in DESIGN.md section "Pinned semantics". Only data-format
 * facts live in this header (the cell hash, the per-body reduction topology and
 * numeric thresholds); the physics formulas are written independently in the
 * CUDA kernels and in oracle/pbdr_oracle.cpp, so the bit-exact parity tests
 * compare two implementations rather than one shared one.
 *
 * Plain C99 so that both nvcc and g++ (oracle) include it.
 */
#ifndef PBDR_PINNED_H
#define PBDR_PINNED_H

#include <math.h>
#include <stdint.h>

#if defined(__CUDACC__)
#define PBDR_HD __host__ __device__ __forceinline__
#else
#define PBDR_HD static inline
#endif

/* ---- Per-body reduction topology ---------------------------------------
 * A body with n particles is reduced by W = ceil(n / (32*KP)) warps (KP: the
 * scene's tile shape, pbdr_choose_kp). Lane l of
 * warp wi owns the particles q = k*32*W + wi*32 + l for k = 0..K-1 with
 * K = ceil(n / (32*W)) (q < n). Every body sum is, in this order:
 *   1. per lane, serially over k ascending, starting from +0.0f;
 *   2. per warp, xor-butterfly with offsets 16, 8, 4, 2, 1 (a + b per level);
 *   3. per body, serially over warps wi ascending, starting from warp 0's value.
 * This plays the role of the reference's fixed-chunk deterministic reduction
 * (proj/include/pbdr/parallel.hpp:15-18, 40-63): results are independent of
 * scheduling, and the oracle reproduces the tree exactly.
 */
#define PBDR_KP_MAX 8             /* particles per lane per body, largest tile */
#ifndef PBDR_CTA_WARPS
#define PBDR_CTA_WARPS 8          /* warps per iteration CTA                */
#endif
#define PBDR_MAX_BODY_PARTICLES (PBDR_KP_MAX * 32 * PBDR_CTA_WARPS) /* 2048: one CTA */
/* Larger bodies take a thread-block cluster of up to 16 CTAs (same slot ->
 * warp map and reduction tree, W up to 128 warps). */
#define PBDR_MAX_CLUSTER_CTAS 16
#define PBDR_MAX_BODY_PARTICLES_BIG (PBDR_MAX_BODY_PARTICLES * PBDR_MAX_CLUSTER_CTAS) /* 32768 */

PBDR_HD int pbdr_body_warps(int n, int kp) { return (n + 32 * kp - 1) / (32 * kp); }
PBDR_HD int pbdr_body_slots(int n, int w) { return (n + 32 * w - 1) / (32 * w); }

/* Tile shape KP (particles per lane), one per scene, chosen from the scene's
 * size (measured on B200): small scenes are latency-bound
 * and want the most parallel layout (KP = 2); scenes whose mean body fits one
 * warp at KP = 8 (<= 256 particles) run best with KP = 8 (two CTAs per SM);
 * larger or mixed bodies with KP = 4 (three CTAs per SM). KP is raised until
 * the largest body fits one CTA, or to PBDR_KP_MAX when it does not (such a
 * body runs on a CTA cluster). `forced` (scene_desc.tile_kp) overrides. The
 * oracle applies the same rule, so both sides reduce with the same tree. */
PBDR_HD int pbdr_choose_kp(long long n_particles, int n_bodies, int max_body, int forced) {
  int kp;
  if (forced == 2 || forced == 4 || forced == 8)
    kp = forced;
  else if (n_particles < 131072)
    kp = 2;
  else if (n_particles <= 256LL * n_bodies)
    kp = 8;
  else
    kp = 4;
  while (kp < PBDR_KP_MAX && max_body > kp * 32 * PBDR_CTA_WARPS) kp *= 2;
  return kp;
}

/* ---- Uniform hash grid ----------------------------------------------------
 * Cell edge h = 2 * max radius. Cell coordinate per axis is
 * floorf(x * inv_h) in fp32 (inv_h = 1.0f / h_f), clamped to +-2^24 before the
 * int conversion so that runaway particles cannot overflow. The clamp is
 * monotone and non-expansive, so two particles closer than h still land in
 * adjacent cells.
 *
 * Bucket key: cells are grouped into x-runs of 16; the run (scene, cz, cy,
 * cx >> 4) is scrambled with a murmur3-finalised mix of the Teschner primes and
 * the low 4 bits keep cx & 15. So the three x-adjacent cells of a stencil row
 * are consecutive keys -- one contiguous range of the sorted array -- unless
 * the row crosses a run boundary. Scene ids keep batched scenes apart.
 */
#define PBDR_CELL_CLAMP 16777216.0f
#define PBDR_XRUN_BITS 4

PBDR_HD uint32_t pbdr_cell_hash(int32_t cx, int32_t cy, int32_t cz, uint32_t scene,
                                uint32_t mask) {
  uint32_t h = ((uint32_t)(cx >> PBDR_XRUN_BITS) * 73856093u) ^ ((uint32_t)cy * 19349663u) ^
               ((uint32_t)cz * 83492791u) ^ (scene * 2654435761u);
  h ^= h >> 16;
  h *= 0x85ebca6bu;
  h ^= h >> 13;
  h *= 0xc2b2ae35u;
  h ^= h >> 16;
  return ((h << PBDR_XRUN_BITS) | ((uint32_t)cx & ((1u << PBDR_XRUN_BITS) - 1u))) & mask;
}

/* Hash table size T = 2^bits, the smallest power of two >= max(n, 1024). */
PBDR_HD int pbdr_hash_bits(int64_t n) {
  int b = 10;
  while (b < 31 && ((int64_t)1 << b) < n) ++b;
  return b;
}

/* Spatially ordered bucket keys for single scenes. With hashed x-runs (above)
 * the 9 stencil rows of a cell sit at random places of the sorted arrays, so
 * the neighbour search streams them from DRAM once per row that reads them.
 * A scene whose cells fit a 2^29-bucket box instead gets the LINEAR key
 * ((cz - oz) << (bx + by)) + ((cy - oy) << bx) + (cx - ox) (mod the table): x-
 * neighbours are consecutive keys, y- and z-neighbours a fixed stride away, so
 * the sweep over sorted particles touches each row's entries while they are
 * in L2. The box is the scene's cell range at creation, padded by an eighth
 * of its extent + 32 cells per side in x and y and + 40 in z; cells that
 * later leave it alias into other rows of the table -- bucket collisions, which
 * the search already tolerates (it re-checks cell coordinates). The layout is
 * chosen from the fp32 positions the device and the oracle both start from,
 * and changes no candidate (P4: the set is geometric). */
typedef struct pbdr_key_layout {
  int32_t linear;      /* 0: hashed x-runs */
  int32_t bits;        /* table bits */
  int32_t bx, by;      /* bits of the x and y ranges (linear) */
  int32_t ox, oy, oz;  /* cell origin of the box (linear) */
} pbdr_key_layout;

PBDR_HD int pbdr_ceil_log2(int64_t v) {
  int b = 0;
  while (((int64_t)1 << b) < v) ++b;
  return b;
}

PBDR_HD pbdr_key_layout pbdr_choose_key_layout(int single_scene, const int32_t cmin[3], const int32_t cmax[3],
                                               int64_t n_particles) {
  pbdr_key_layout L;
  L.linear = 0;
  L.bits = pbdr_hash_bits(n_particles);
  L.bx = L.by = 0;
  L.ox = L.oy = L.oz = 0;
  if (!single_scene) return L;
  const int64_t ex = (int64_t)cmax[0] - cmin[0] + 1, ey = (int64_t)cmax[1] - cmin[1] + 1;
  const int64_t ez = (int64_t)cmax[2] - cmin[2] + 1;
  const int64_t px = ex / 8 + 32, py = ey / 8 + 32;
  const int bx = pbdr_ceil_log2(ex + 2 * px), by = pbdr_ceil_log2(ey + 2 * py);
  const int bz = pbdr_ceil_log2(ez + ez / 8 + 40 + 16);
  if (bx + by > 24 || bx + by + bz > 29) return L;
  L.linear = 1;
  L.bx = bx;
  L.by = by;
  L.ox = (int32_t)(cmin[0] - px);
  L.oy = (int32_t)(cmin[1] - py);
  L.oz = cmin[2] - 16;
  if (bx + by + bz > L.bits) L.bits = bx + by + bz;
  return L;
}

PBDR_HD uint32_t pbdr_cell_key(int32_t cx, int32_t cy, int32_t cz, uint32_t scene, uint32_t mask,
                               pbdr_key_layout L) {
  if (!L.linear) return pbdr_cell_hash(cx, cy, cz, scene, mask);
  return (((uint32_t)(cz - L.oz) << (L.bx + L.by)) + ((uint32_t)(cy - L.oy) << L.bx) + (uint32_t)(cx - L.ox)) &
         mask;
}

PBDR_HD int32_t pbdr_cell_coord(float x, float inv_h) {
  float c = floorf(x * inv_h);
  c = fminf(fmaxf(c, -PBDR_CELL_CLAMP), PBDR_CELL_CLAMP);
  return (int32_t)c;
}

/* Maximum contact candidates per particle per substep. More raises
 * PBDR_ERR_SIMULATION (never silently dropped). */
#define PBDR_NBR_CAP 32

/* Body-broadphase partners kept per body; more disables the skip for that
 * body (its particles always run the full stencil search). */
#define PBDR_PARTNER_CAP 32

/* Maximum planes (ground + walls) per scene. */
#define PBDR_MAX_PLANES 8

/* ---- Numeric thresholds (double, per body) --------------------------------
 * Polar decomposition (math.cpp:170-210 semantics, scaled Newton, tol 1e-9,
 * <= 64 iterations). The reference's absolute det(A) <= 1e-12 test
 * (math.cpp:172) rejects small-but-valid bodies, so the
 * degeneracy test is scale-relative: det(A) <= 1e-12 * (||A||_F / sqrt 3)^3,
 * evaluated without roots as det <= 0 or det^2 <= 1e-24 * (||A||_F^2 / 3)^3.
 */
#define PBDR_POLAR_TOL 1e-9
#define PBDR_POLAR_TOL2 1e-18     /* convergence: |dX|_F^2 <= tol^2 |X|_F^2  */
#define PBDR_POLAR_SCALE_REL2 1e-4 /* keep the 1-inf scaling while |dX|/|X| > 1e-2 */
#define PBDR_POLAR_TOLQ 1e-12     /* unscaled step with |dX|^2 <= 1e-12 |X|^2 leaves ~1e-12 */
#define PBDR_POLAR_MAX_IT 64
#define PBDR_POLAR_REL_DET 1e-12
#define PBDR_ONE_THIRD (1.0 / 3.0)
/* Warm-started rotation extraction: Gauss-Newton steps from the previous
 * iteration's rotation (see polar_warm in oracle_math.hpp / pbdr_mat3.cuh). */
#define PBDR_POLAR_WARM_STEPS 4
#define PBDR_POLAR_WARM_MAX2 0.25
/* A Gauss-Newton step of squared size <= 1e-10 (|w| <= 1e-5 rad) is the last:
 * the step is quadratically convergent, so the rotation it returns is within
 * O(|w|^2) ~ 1e-10 rad of the polar factor -- below the reference polar's own
 * 1e-9 tolerance and three orders below fp32 particle resolution. Most
 * iterations after the first of a substep need one step. */
#define PBDR_POLAR_WARM_TOLQ 1e-10
/* Arithmetic of the warm Gauss-Newton steps: 1 = fp32 (the warm start is an
 * fp32 quaternion and the returned rotation is rounded to fp32 anyway; the
 * step's fp32 noise, ~1e-7 rad, sits far below the 1e-5 stop threshold),
 * 0 = fp64. Both sides (pbdr_mat3.cuh, oracle_math.hpp) follow the switch, so
 * parity stays bit-exact either way; the degeneracy test and the cold polar
 * stay fp64. */
#ifndef PBDR_POLAR_WARM_F32
#define PBDR_POLAR_WARM_F32 0
#endif
/* fp32 warm-up stage of the polar (then fp64 polish to PBDR_POLAR_TOL). */
#define PBDR_POLAR_F32_TOL2 1e-12f
#define PBDR_POLAR_F32_TOLQ 1e-7f
#define PBDR_POLAR_F32_MAX_IT 32

/* Inertia inverse for the angular-momentum fix: pseudo-inverse semantics of
 * math.cpp:90-108 (rank cut at eigenvalue < 1e-10 * trace). When
 * det(I) >= 1e-6 * trace(I)^3 the matrix is provably full rank under that cut
 * and the adjugate inverse is used; otherwise the cyclic-Jacobi eigen path runs.
 * dL along a null axis below 1e-12 is projected out; above it the body raises
 * RankDeficientError. */
#define PBDR_PINV_REL_TOL 1e-10
#define PBDR_PINV_FAST_DET 1e-6
#define PBDR_NULL_AXIS_TOL 1e-12

/* Coincident-centre fallback axis for particle-particle contact:
 * distance below this uses +x for the lower particle index, -x for the higher. */
#define PBDR_COINCIDENT_EPS 1e-9f

/* Device error word bits (mapped to pbdr::errors classes by the host). */
#define PBDR_DEVERR_DEGENERATE 1u     /* polar: det at/below tolerance      */
#define PBDR_DEVERR_RANK_DEFICIENT 2u /* dL along a singular inertia axis   */
#define PBDR_DEVERR_NBR_OVERFLOW 4u   /* > PBDR_NBR_CAP contact candidates  */
#define PBDR_DEVERR_NONFINITE 8u      /* NaN/Inf in a body sum              */

#endif /* PBDR_PINNED_H */
