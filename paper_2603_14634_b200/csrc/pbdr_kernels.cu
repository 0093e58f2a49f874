// sm_100a kernels of the PBD-R substep loop.
//
// Per substep:
//   integrate_key  x_init <- x; v~ = v + dt a; x~ = x + dt v~ ; cell hash key
//   [onesweep sort of (key, slot), pbdr_sort.cu]
//   cell_ranges    per-bucket [start, end) in sorted order + sorted copy of x~
//   neighbours     per particle: contact candidates (other body, same scene,
//                  27-cell stencil, |x~_i - x~_j| < h), ascending slot order
//   iteration x N  fused: ground + particle-particle contact (Jacobi), shape
//                  matching (segmented com / Apq sums + fp64 polar), position
//                  and incremental velocity update, momentum constraint
//                  (Eq. 1 / Eq. 2) fused into the writeback
// The op order of every fp32 expression is pinned and mirrored by
// oracle/pbdr_oracle.cpp; the library is compiled with --fmad=false so the
// CUDA path and the oracle agree bit for bit.
#include <cuda_runtime.h>
#include <stdint.h>

#include "pbdr_kernels.cuh"
#include "pbdr_mat3.cuh"
#include "pbdr_pinned.h"

namespace pbdr_dev {

namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kIterThreads = PBDR_CTA_WARPS * 32;

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

// ---------------------------------------------------------------------------
// integrate + cell key
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_integrate_key(IntegrateArgs A) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= A.n) return;
  const int b = A.body_of[p];
  const double t = static_cast<double>(*A.substep_counter) * A.dt_d;
  const BodyProgram pr = A.programs[b];
  float a[3] = {0.0f, 0.0f, (pr.flags & 2) ? 0.0f : -A.gravity};
  if ((pr.flags & 1) && t >= pr.t_start && t < pr.t_stop) {
    const float invM = A.body_mass[b].y;
    a[0] = a[0] + pr.fx * invM;
    a[1] = a[1] + pr.fy * invM;
    a[2] = a[2] + pr.fz * invM;
  }
  const float4 x = A.pos[p];
  const float4 v = A.vel[p];
  A.init[p] = make_float4(x.x, x.y, x.z, 0.0f);
  float4 vn, xn;
  vn.x = v.x + A.dt * a[0];
  vn.y = v.y + A.dt * a[1];
  vn.z = v.z + A.dt * a[2];
  vn.w = v.w;
  xn.x = x.x + A.dt * vn.x;
  xn.y = x.y + A.dt * vn.y;
  xn.z = x.z + A.dt * vn.z;
  xn.w = x.w;
  A.vel[p] = vn;
  A.pos[p] = xn;
  const int32_t cx = pbdr_cell_coord(xn.x, A.inv_h);
  const int32_t cy = pbdr_cell_coord(xn.y, A.inv_h);
  const int32_t cz = pbdr_cell_coord(xn.z, A.inv_h);
  A.keys[p] = pbdr_cell_hash(cx, cy, cz, static_cast<uint32_t>(A.body_scene[b]), A.mask);
  A.vals[p] = static_cast<uint32_t>(p);
}

// ---------------------------------------------------------------------------
// cell ranges: per-bucket [start, end) in sorted order, and the body of every
// sorted entry (slots are ascending within a bucket, so bodies are too).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_cell_ranges(RangesArgs A) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s == 0) atomicAdd(reinterpret_cast<unsigned long long*>(A.substep_counter), 1ull);
  if (s >= A.n) return;
  const uint32_t k = A.keys[s];
  if (s == 0 || A.keys[s - 1] != k) A.cell_start[k] = static_cast<uint32_t>(s);
  if (s == A.n - 1 || A.keys[s + 1] != k) A.cell_end[k] = static_cast<uint32_t>(s + 1);
  A.sorted_body[s] = A.body_of[A.vals[s]];
}

// ---------------------------------------------------------------------------
// contact candidates (pinned P4): {j : same scene, other body,
// |cell_j - cell_i|_inf <= 1, |x~_i - x~_j|^2 < h^2}, ascending j, <= CAP.
// A bucket whose first and last entries belong to particle i's own body holds
// only own-body particles and is skipped without a scan (most buckets).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) k_neighbours(NeighbourArgs A) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= A.n) return;
  const float4 xi = A.pos[i];
  const float ri = A.rest[i].w;
  const int bi = A.body_of[i];
  const int si = A.body_scene[bi];
  const int32_t cx = pbdr_cell_coord(xi.x, A.inv_h);
  const int32_t cy = pbdr_cell_coord(xi.y, A.inv_h);
  const int32_t cz = pbdr_cell_coord(xi.z, A.inv_h);

  int cand[PBDR_NBR_CAP];
  float cr[PBDR_NBR_CAP];
  int count = 0;
  bool overflow = false;
  uint32_t visited[27];
#pragma unroll
  for (int t = 0; t < 27; ++t) {
    const int dz = t / 9 - 1, dy = (t / 3) % 3 - 1, dx = t % 3 - 1;
    const uint32_t hb = pbdr_cell_hash(cx + dx, cy + dy, cz + dz, static_cast<uint32_t>(si), A.mask);
    bool dup = false;
#pragma unroll
    for (int u = 0; u < t; ++u) dup = dup || (visited[u] == hb);
    visited[t] = hb;
    if (dup) continue;
    const uint32_t s0 = A.cell_start[hb];
    if (s0 == 0xFFFFFFFFu) continue;
    const uint32_t s1 = A.cell_end[hb];
    if (A.sorted_body[s0] == bi && A.sorted_body[s1 - 1] == bi) continue;
    for (uint32_t s = s0; s < s1; ++s) {
      const int bj = A.sorted_body[s];
      if (bj == bi) continue;
      if (A.body_scene[bj] != si) continue;
      const int j = static_cast<int>(A.sorted_vals[s]);
      const float4 xj = A.pos[j];
      const int32_t jx = pbdr_cell_coord(xj.x, A.inv_h);
      const int32_t jy = pbdr_cell_coord(xj.y, A.inv_h);
      const int32_t jz = pbdr_cell_coord(xj.z, A.inv_h);
      if (jx < cx - 1 || jx > cx + 1 || jy < cy - 1 || jy > cy + 1 || jz < cz - 1 || jz > cz + 1)
        continue;
      const float ex = xi.x - xj.x, ey = xi.y - xj.y, ez = xi.z - xj.z;
      const float d2 = (ex * ex + ey * ey) + ez * ez;
      if (!(d2 < A.h2)) continue;
      // Keep the CAP smallest j in ascending order.
      if (count == PBDR_NBR_CAP) {
        overflow = true;
        if (j > cand[PBDR_NBR_CAP - 1]) continue;
        --count;
      }
      int pos = count;
      while (pos > 0 && cand[pos - 1] > j) {
        cand[pos] = cand[pos - 1];
        cr[pos] = cr[pos - 1];
        --pos;
      }
      cand[pos] = j;
      cr[pos] = ri + A.rest[j].w;
      ++count;
    }
  }
  if (overflow) record_error(A.err, PBDR_DEVERR_NBR_OVERFLOW, bi, A.substep_counter);
  A.ncand[i] = count;
  for (int k = 0; k < count; ++k) {
    A.cand_j[static_cast<int64_t>(k) * A.n + i] = cand[k];
    A.cand_rr[static_cast<int64_t>(k) * A.n + i] = cr[k];
  }
}

// ---------------------------------------------------------------------------
// One solver iteration, fused (pinned P1-P8). CTA = 16 warps; each body owns
// W = ceil(n/64) consecutive warps; lane l of body-warp wi owns particles
// q = k*32*W + wi*32 + l, k < 2.
// ---------------------------------------------------------------------------
constexpr int kResF = 32;
enum ResSlot {
  kResC = 0,     // c (3)
  kResLb = 3,    // L_bsm (3)
  kResPb = 6,    // P_bsm (3)
  kResR = 9,     // R (9)
  kResSmOk = 18, // shape-matching valid flag
  kResCa = 19,   // c_asm (3)
  kResDv = 22,   // dv (3)
  kResW = 25,    // omega (3)
};

__global__ void __launch_bounds__(kIterThreads, 2) k_iteration(IterArgs A) {
  __shared__ float s_part[PBDR_CTA_WARPS][21];
  __shared__ float s_res[PBDR_CTA_WARPS][kResF];

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int2 wd = A.warp_desc[blockIdx.x * PBDR_CTA_WARPS + warp];
  const int b = wd.x;
  const int wi = wd.y;
  const bool live = b >= 0;
  int4 bd = make_int4(0, 0, 1, 0);
  float a[3] = {0.0f, 0.0f, 0.0f};
  float2 mass = make_float2(0.0f, 0.0f);
  if (live) {
    bd = A.body_desc[b];
    const float4 an = A.anchor[b];
    a[0] = an.x; a[1] = an.y; a[2] = an.z;
    mass = A.body_mass[b];
  }
  const int start = bd.x, n = bd.y, W = bd.z, fw = bd.w;
  const bool fixes = A.linfix || A.angfix;

  float x[PBDR_KP][3], w[PBDR_KP], v[PBDR_KP][3], m[PBDR_KP], q0[PBDR_KP][3], dc[PBDR_KP][3];
  bool act[PBDR_KP];
  int64_t pidx[PBDR_KP];

  // ---- Phase A: contacts, bsm sums -----------------------------------------
  float acc[21];
#pragma unroll
  for (int f = 0; f < 21; ++f) acc[f] = 0.0f;
#pragma unroll
  for (int k = 0; k < PBDR_KP; ++k) {
    const int q = k * 32 * W + wi * 32 + lane;
    act[k] = live && q < n;
    pidx[k] = start + q;
    if (!act[k]) continue;
    const int64_t p = pidx[k];
    const float4 x4 = A.pos_in[p];
    const float4 v4 = A.vel[p];
    const float4 r4 = A.rest[p];
    x[k][0] = x4.x; x[k][1] = x4.y; x[k][2] = x4.z; w[k] = x4.w;
    v[k][0] = v4.x; v[k][1] = v4.y; v[k][2] = v4.z; m[k] = v4.w;
    q0[k][0] = r4.x; q0[k][1] = r4.y; q0[k][2] = r4.z;
    const float r = r4.w;

    float dPG[3] = {0.0f, 0.0f, 0.0f};
    for (int pl = 0; pl < A.planes.count; ++pl) {
      const float* Pp = A.planes.p[pl];
      const float* Pn = A.planes.n[pl];
      const float d = (((x[k][0] - Pp[0]) * Pn[0] + (x[k][1] - Pp[1]) * Pn[1]) +
                       (x[k][2] - Pp[2]) * Pn[2]) - r;
      if (d < 0.0f) {
        const float push = -(A.relax * d);
        dPG[0] = dPG[0] + push * Pn[0];
        dPG[1] = dPG[1] + push * Pn[1];
        dPG[2] = dPG[2] + push * Pn[2];
        const float mu = A.planes.mu[pl];
        if (mu > 0.0f) {
          const float4 xi = A.init[p];
          const float t[3] = {x[k][0] - xi.x, x[k][1] - xi.y, x[k][2] - xi.z};
          const float tn = (t[0] * Pn[0] + t[1] * Pn[1]) + t[2] * Pn[2];
          const float tt[3] = {t[0] - tn * Pn[0], t[1] - tn * Pn[1], t[2] - tn * Pn[2]};
          const float len2 = (tt[0] * tt[0] + tt[1] * tt[1]) + tt[2] * tt[2];
          if (len2 > 0.0f) {
            const float len = sqrtf(len2);
            const float lim = mu * (-d);
            if (len <= lim) {
              dPG[0] = dPG[0] - tt[0];
              dPG[1] = dPG[1] - tt[1];
              dPG[2] = dPG[2] - tt[2];
            } else {
              const float fr = lim / len;
              dPG[0] = dPG[0] - tt[0] * fr;
              dPG[1] = dPG[1] - tt[1] * fr;
              dPG[2] = dPG[2] - tt[2] * fr;
            }
          }
        }
      }
    }
    float dPP[3] = {0.0f, 0.0f, 0.0f};
    const int nc = A.ncand[p];
    for (int c = 0; c < nc; ++c) {
      const int j = A.cand_j[static_cast<int64_t>(c) * A.n + p];
      const float rr = A.cand_rr[static_cast<int64_t>(c) * A.n + p];
      const float4 xj = A.pos_in[j];
      const float e[3] = {x[k][0] - xj.x, x[k][1] - xj.y, x[k][2] - xj.z};
      const float d2 = (e[0] * e[0] + e[1] * e[1]) + e[2] * e[2];
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
        const float kk = (A.relax * (w[k] / (w[k] + xj.w))) * C;
        dPP[0] = dPP[0] - kk * nrm[0];
        dPP[1] = dPP[1] - kk * nrm[1];
        dPP[2] = dPP[2] - kk * nrm[2];
      }
    }
    float pp[3], pb[3], mp[3], mvb[3], kb[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      dc[k][c] = dPG[c] + dPP[c];
      pp[c] = x[k][c] - a[c];
      pb[c] = pp[c] + dc[k][c];
      const float vb = v[k][c] + dc[k][c] * A.inv_dt;
      mp[c] = m[k] * pp[c];
      mvb[c] = m[k] * vb;
    }
    cross3(pb, mvb, kb);
    acc[0] = acc[0] + mp[0];
    acc[1] = acc[1] + mp[1];
    acc[2] = acc[2] + mp[2];
    acc[3] = acc[3] + m[k] * dc[k][0];
    acc[4] = acc[4] + m[k] * dc[k][1];
    acc[5] = acc[5] + m[k] * dc[k][2];
#pragma unroll
    for (int rI = 0; rI < 3; ++rI)
#pragma unroll
      for (int cI = 0; cI < 3; ++cI) acc[6 + 3 * rI + cI] = acc[6 + 3 * rI + cI] + mp[rI] * q0[k][cI];
    acc[15] = acc[15] + mvb[0];
    acc[16] = acc[16] + mvb[1];
    acc[17] = acc[17] + mvb[2];
    acc[18] = acc[18] + kb[0];
    acc[19] = acc[19] + kb[1];
    acc[20] = acc[20] + kb[2];
  }
  if (live) {
    warp_butterfly<21>(acc);
    if (lane == 0)
#pragma unroll
      for (int f = 0; f < 21; ++f) s_part[warp][f] = acc[f];
  }
  __syncthreads();

  if (live && wi == 0 && lane == 0) {
    float S[21];
#pragma unroll
    for (int f = 0; f < 21; ++f) S[f] = s_part[warp][f];
    for (int u = 1; u < W; ++u)
#pragma unroll
      for (int f = 0; f < 21; ++f) S[f] = S[f] + s_part[warp + u][f];
    bool finite = true;
#pragma unroll
    for (int f = 0; f < 21; ++f) finite = finite && isfinite(S[f]);
    if (!finite) record_error(A.err, PBDR_DEVERR_NONFINITE, b, A.substep_counter);
    float c[3], cb[3], Pb[3], tmp[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      c[k] = S[k] * mass.y;
      cb[k] = c[k] + S[3 + k] * mass.y;
      Pb[k] = S[15 + k];
    }
    cross3(cb, Pb, tmp);
    float* R = &s_res[warp][0];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      R[kResC + k] = c[k];
      R[kResPb + k] = Pb[k];
      R[kResLb + k] = S[18 + k] - tmp[k];
    }
    double qd[4];
    const bool ok = polar_rotation_f(&S[6], &R[kResR], qd);
    R[kResSmOk] = ok ? 1.0f : 0.0f;
    if (!ok) record_error(A.err, PBDR_DEVERR_DEGENERATE, b, A.substep_counter);
    A.anchor[b] = make_float4(a[0] + c[0], a[1] + c[1], a[2] + c[2], 0.0f);
  }
  __syncthreads();

  // ---- Phase B: shape matching, position + velocity update ----------------
  float xa[PBDR_KP][3], va[PBDR_KP][3], pa[PBDR_KP][3];
  float accB[15];
#pragma unroll
  for (int f = 0; f < 15; ++f) accB[f] = 0.0f;
  const float* res = &s_res[fw][0];
  if (live) {
    const bool sm_ok = res[kResSmOk] != 0.0f;
    float Rf[9], c[3];
#pragma unroll
    for (int f = 0; f < 9; ++f) Rf[f] = res[kResR + f];
#pragma unroll
    for (int k = 0; k < 3; ++k) c[k] = res[kResC + k];
#pragma unroll
    for (int k = 0; k < PBDR_KP; ++k) {
      if (!act[k]) continue;
      float dX[3];
      float4 xi = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
      if (!A.incremental) xi = A.init[pidx[k]];
      const float xiv[3] = {xi.x, xi.y, xi.z};
#pragma unroll
      for (int cI = 0; cI < 3; ++cI) {
        const float pk = x[k][cI] - a[cI];
        float dsm = 0.0f;
        if (sm_ok) {
          const float g = (Rf[3 * cI] * q0[k][0] + Rf[3 * cI + 1] * q0[k][1]) + Rf[3 * cI + 2] * q0[k][2];
          dsm = g - (pk - c[cI]);
        }
        dX[cI] = dc[k][cI] + dsm;
        xa[k][cI] = x[k][cI] + dX[cI];
        va[k][cI] = A.incremental ? v[k][cI] + dX[cI] * A.inv_dt : (xa[k][cI] - xiv[cI]) * A.inv_dt;
        pa[k][cI] = pk + dX[cI];
      }
      if (fixes) {
        const float mk = m[k];
        const float mva[3] = {mk * va[k][0], mk * va[k][1], mk * va[k][2]};
        float ka[3];
        cross3(pa[k], mva, ka);
        const float s2 = (pa[k][0] * pa[k][0] + pa[k][1] * pa[k][1]) + pa[k][2] * pa[k][2];
        accB[0] = accB[0] + mk * dX[0];
        accB[1] = accB[1] + mk * dX[1];
        accB[2] = accB[2] + mk * dX[2];
        accB[3] = accB[3] + mva[0];
        accB[4] = accB[4] + mva[1];
        accB[5] = accB[5] + mva[2];
        accB[6] = accB[6] + ka[0];
        accB[7] = accB[7] + ka[1];
        accB[8] = accB[8] + ka[2];
        accB[9] = accB[9] + mk * (s2 - pa[k][0] * pa[k][0]);
        accB[10] = accB[10] + mk * (s2 - pa[k][1] * pa[k][1]);
        accB[11] = accB[11] + mk * (s2 - pa[k][2] * pa[k][2]);
        accB[12] = accB[12] + -(mk * (pa[k][0] * pa[k][1]));
        accB[13] = accB[13] + -(mk * (pa[k][0] * pa[k][2]));
        accB[14] = accB[14] + -(mk * (pa[k][1] * pa[k][2]));
      }
    }
  }

  if (!fixes) {
#pragma unroll
    for (int k = 0; k < PBDR_KP; ++k) {
      if (!act[k]) continue;
      const int64_t p = pidx[k];
      A.pos_out[p] = make_float4(xa[k][0], xa[k][1], xa[k][2], w[k]);
      A.vel[p] = make_float4(va[k][0], va[k][1], va[k][2], m[k]);
    }
    return;
  }

  if (live) {
    warp_butterfly<15>(accB);
    if (lane == 0)
#pragma unroll
      for (int f = 0; f < 15; ++f) s_part[warp][f] = accB[f];
  }
  __syncthreads();

  if (live && wi == 0 && lane == 0) {
    float S[15];
#pragma unroll
    for (int f = 0; f < 15; ++f) S[f] = s_part[warp][f];
    for (int u = 1; u < W; ++u)
#pragma unroll
      for (int f = 0; f < 15; ++f) S[f] = S[f] + s_part[warp + u][f];
    bool finite = true;
#pragma unroll
    for (int f = 0; f < 15; ++f) finite = finite && isfinite(S[f]);
    if (!finite) record_error(A.err, PBDR_DEVERR_NONFINITE, b, A.substep_counter);
    float* R = &s_res[warp][0];
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
    if (A.linfix)
#pragma unroll
      for (int k = 0; k < 3; ++k) dv[k] = (R[kResPb + k] - Pa[k]) * invM;
    if (A.angfix) {
      float If[6];
      If[0] = S[9] - M * (ca[1] * ca[1] + ca[2] * ca[2]);
      If[1] = S[10] - M * (ca[0] * ca[0] + ca[2] * ca[2]);
      If[2] = S[11] - M * (ca[0] * ca[0] + ca[1] * ca[1]);
      If[3] = S[12] + M * (ca[0] * ca[1]);
      If[4] = S[13] + M * (ca[0] * ca[2]);
      If[5] = S[14] + M * (ca[1] * ca[2]);
      const float dL[3] = {La[0] - R[kResLb], La[1] - R[kResLb + 1], La[2] - R[kResLb + 2]};
      double nax[3];
      const unsigned e = inertia_solve_f(If, dL, om, nax);
      if (e) record_error(A.err, e, b, A.substep_counter, nax);
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      R[kResCa + k] = ca[k];
      R[kResDv + k] = dv[k];
      R[kResW + k] = om[k];
    }
  }
  __syncthreads();

  // ---- Phase C: momentum corrections (Eq. 1 then Eq. 2), writeback --------
  if (!live) return;
  float ca[3], dv[3], om[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    ca[k] = res[kResCa + k];
    dv[k] = res[kResDv + k];
    om[k] = res[kResW + k];
  }
#pragma unroll
  for (int k = 0; k < PBDR_KP; ++k) {
    if (!act[k]) continue;
    float r[3], wr[3], xo[3], vo[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) r[c] = pa[k][c] - ca[c];
    cross3(om, r, wr);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      float vv = va[k][c] + dv[c];
      vv = vv - wr[c];
      float xx = xa[k][c] + dv[c] * A.dt;
      xx = xx - wr[c] * A.dt;
      vo[c] = vv;
      xo[c] = xx;
    }
    const int64_t p = pidx[k];
    A.pos_out[p] = make_float4(xo[0], xo[1], xo[2], w[k]);
    A.vel[p] = make_float4(vo[0], vo[1], vo[2], m[k]);
  }
}

// ---------------------------------------------------------------------------
// Per-body trajectory sample: com, orientation (extract_pose), P, L.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kIterThreads) k_body_stats(StatsArgs A) {
  __shared__ float s_part[PBDR_CTA_WARPS][18];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int2 wd = A.warp_desc[blockIdx.x * PBDR_CTA_WARPS + warp];
  const int b = wd.x;
  const int wi = wd.y;
  const bool live = b >= 0;
  int4 bd = make_int4(0, 0, 1, 0);
  float a[3] = {0.0f, 0.0f, 0.0f};
  if (live) {
    bd = A.body_desc[b];
    const float4 an = A.anchor[b];
    a[0] = an.x; a[1] = an.y; a[2] = an.z;
  }
  const int start = bd.x, n = bd.y, W = bd.z;
  float acc[18];
#pragma unroll
  for (int f = 0; f < 18; ++f) acc[f] = 0.0f;
  if (live) {
#pragma unroll
    for (int k = 0; k < PBDR_KP; ++k) {
      const int q = k * 32 * W + wi * 32 + lane;
      if (q >= n) continue;
      const int64_t p = start + q;
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
    warp_butterfly<18>(acc);
    if (lane == 0)
#pragma unroll
      for (int f = 0; f < 18; ++f) s_part[warp][f] = acc[f];
  }
  __syncthreads();
  if (!(live && wi == 0 && lane == 0)) return;
  float S[18];
#pragma unroll
  for (int f = 0; f < 18; ++f) S[f] = s_part[warp][f];
  for (int u = 1; u < W; ++u)
#pragma unroll
    for (int f = 0; f < 18; ++f) S[f] = S[f] + s_part[warp + u][f];
  const float invM = A.body_mass[b].y;
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
  double* o = A.out + 13 * static_cast<int64_t>(b);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    o[k] = static_cast<double>(a[k]) + static_cast<double>(c[k]);
    o[7 + k] = static_cast<double>(P[k]);
    o[10 + k] = static_cast<double>(S[15 + k] - tmp[k]);
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) o[3 + k] = qd[k];
}

}  // namespace

void launch_integrate(const IntegrateArgs& a, cudaStream_t s) {
  const unsigned blocks = static_cast<unsigned>((a.n + 255) / 256);
  k_integrate_key<<<blocks, 256, 0, s>>>(a);
}

void launch_ranges(const RangesArgs& a, cudaStream_t s) {
  const unsigned blocks = static_cast<unsigned>((a.n + 255) / 256);
  k_cell_ranges<<<blocks, 256, 0, s>>>(a);
}

void launch_neighbours(const NeighbourArgs& a, cudaStream_t s) {
  const unsigned blocks = static_cast<unsigned>((a.n + 127) / 128);
  k_neighbours<<<blocks, 128, 0, s>>>(a);
}

void launch_iteration(const IterArgs& a, int ctas, cudaStream_t s) {
  k_iteration<<<ctas, kIterThreads, 0, s>>>(a);
}

void launch_stats(const StatsArgs& a, int ctas, cudaStream_t s) {
  k_body_stats<<<ctas, kIterThreads, 0, s>>>(a);
}

}  // namespace pbdr_dev
