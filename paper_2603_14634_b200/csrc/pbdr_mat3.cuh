// Per-body fp64 3x3 numerics on the device: scaled-Newton polar rotation and
// the inertia solve for the angular-momentum fix.
//
// Semantics: math.cpp:8-24 (adjugate inverse), :26-71 (cyclic Jacobi),
// :90-108 (SPD pseudo-inverse), :117-146 (quaternion from matrix), :170-210
// (scaled Newton polar, tol 1e-9, <= 64 iterations); op order pinned in
// DESIGN.md so the result matches the CPU oracle bit for bit (the library is
// built with --fmad=false; IEEE div/sqrt on both sides).
//
// One thread per body runs these; the matrices live in registers / local
// memory of that thread only.
#pragma once

#include <stdint.h>

#include "pbdr_pinned.h"

namespace pbdr_dev {

struct D3 {
  double a[3][3];
};

__device__ __forceinline__ double d3_det(const D3& m) {
  return m.a[0][0] * (m.a[1][1] * m.a[2][2] - m.a[1][2] * m.a[2][1]) -
         m.a[0][1] * (m.a[1][0] * m.a[2][2] - m.a[1][2] * m.a[2][0]) +
         m.a[0][2] * (m.a[1][0] * m.a[2][1] - m.a[1][1] * m.a[2][0]);
}

__device__ __forceinline__ double d3_frob(const D3& m) {
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) s = s + m.a[i][j] * m.a[i][j];
  return sqrt(s);
}

__device__ __forceinline__ D3 d3_adj_inverse(const D3& m, double d) {
  const double id = 1.0 / d;
  D3 r;
  r.a[0][0] = (m.a[1][1] * m.a[2][2] - m.a[1][2] * m.a[2][1]) * id;
  r.a[0][1] = (m.a[0][2] * m.a[2][1] - m.a[0][1] * m.a[2][2]) * id;
  r.a[0][2] = (m.a[0][1] * m.a[1][2] - m.a[0][2] * m.a[1][1]) * id;
  r.a[1][0] = (m.a[1][2] * m.a[2][0] - m.a[1][0] * m.a[2][2]) * id;
  r.a[1][1] = (m.a[0][0] * m.a[2][2] - m.a[0][2] * m.a[2][0]) * id;
  r.a[1][2] = (m.a[0][2] * m.a[1][0] - m.a[0][0] * m.a[1][2]) * id;
  r.a[2][0] = (m.a[1][0] * m.a[2][1] - m.a[1][1] * m.a[2][0]) * id;
  r.a[2][1] = (m.a[0][1] * m.a[2][0] - m.a[0][0] * m.a[2][1]) * id;
  r.a[2][2] = (m.a[0][0] * m.a[1][1] - m.a[0][1] * m.a[1][0]) * id;
  return r;
}

__device__ __forceinline__ double d3_norm1_inf(const D3& m) {
  double c = 0.0, r = 0.0;
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const double s = (fabs(m.a[0][j]) + fabs(m.a[1][j])) + fabs(m.a[2][j]);
    c = s > c ? s : c;
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double s = (fabs(m.a[i][0]) + fabs(m.a[i][1])) + fabs(m.a[i][2]);
    r = s > r ? s : r;
  }
  return c * r;
}

__device__ __forceinline__ void d3_quat_from(const D3& x, double q[4]) {
  const double tr = (x.a[0][0] + x.a[1][1]) + x.a[2][2];
  double w, qx, qy, qz;
  if (tr > 0.0) {
    const double s = sqrt(tr + 1.0) * 2.0;
    w = 0.25 * s;
    qx = (x.a[2][1] - x.a[1][2]) / s;
    qy = (x.a[0][2] - x.a[2][0]) / s;
    qz = (x.a[1][0] - x.a[0][1]) / s;
  } else if (x.a[0][0] > x.a[1][1] && x.a[0][0] > x.a[2][2]) {
    const double s = sqrt(((1.0 + x.a[0][0]) - x.a[1][1]) - x.a[2][2]) * 2.0;
    w = (x.a[2][1] - x.a[1][2]) / s;
    qx = 0.25 * s;
    qy = (x.a[0][1] + x.a[1][0]) / s;
    qz = (x.a[0][2] + x.a[2][0]) / s;
  } else if (x.a[1][1] > x.a[2][2]) {
    const double s = sqrt(((1.0 + x.a[1][1]) - x.a[0][0]) - x.a[2][2]) * 2.0;
    w = (x.a[0][2] - x.a[2][0]) / s;
    qx = (x.a[0][1] + x.a[1][0]) / s;
    qy = 0.25 * s;
    qz = (x.a[1][2] + x.a[2][1]) / s;
  } else {
    const double s = sqrt(((1.0 + x.a[2][2]) - x.a[0][0]) - x.a[1][1]) * 2.0;
    w = (x.a[1][0] - x.a[0][1]) / s;
    qx = (x.a[0][2] + x.a[2][0]) / s;
    qy = (x.a[1][2] + x.a[2][1]) / s;
    qz = 0.25 * s;
  }
  const double n = sqrt(((w * w + qx * qx) + qy * qy) + qz * qz);
  if (n > 0.0) {
    w = w / n; qx = qx / n; qy = qy / n; qz = qz / n;
  } else {
    w = 1.0; qx = 0.0; qy = 0.0; qz = 0.0;
  }
  q[0] = w; q[1] = qx; q[2] = qy; q[3] = qz;
}

__device__ __forceinline__ void d3_quat_to(const double q[4], float R[9]) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  const double xx = x * x, yy = y * y, zz = z * z;
  const double xy = x * y, xz = x * z, yz = y * z;
  const double wx = w * x, wy = w * y, wz = w * z;
  R[0] = static_cast<float>(1.0 - 2.0 * (yy + zz));
  R[1] = static_cast<float>(2.0 * (xy - wz));
  R[2] = static_cast<float>(2.0 * (xz + wy));
  R[3] = static_cast<float>(2.0 * (xy + wz));
  R[4] = static_cast<float>(1.0 - 2.0 * (xx + zz));
  R[5] = static_cast<float>(2.0 * (yz - wx));
  R[6] = static_cast<float>(2.0 * (xz - wy));
  R[7] = static_cast<float>(2.0 * (yz + wx));
  R[8] = static_cast<float>(1.0 - 2.0 * (xx + yy));
}

// Rotation of the polar decomposition of A (row-major fp32 sums). Returns
// false when A is degenerate (non-finite or det <= rel. tolerance).
__device__ __noinline__ bool polar_rotation_f(const float Af[9], float R[9], double q[4]) {
  D3 A;
  bool finite = true;
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    A.a[i / 3][i % 3] = static_cast<double>(Af[i]);
    finite = finite && isfinite(Af[i]);
  }
  if (!finite) return false;
  const double s = d3_frob(A) / sqrt(3.0);
  if (d3_det(A) <= PBDR_POLAR_REL_DET * ((s * s) * s)) return false;
  D3 X = A;
  for (int it = 0; it < PBDR_POLAR_MAX_IT; ++it) {
    const double d = d3_det(X);
    if (d == 0.0 || !isfinite(d)) return false;
    const D3 inv = d3_adj_inverse(X, d);
    D3 xit;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) xit.a[i][j] = inv.a[j][i];
    const double xn = d3_norm1_inf(X);
    const double in = d3_norm1_inf(xit);
    const double g = (xn > 0.0 && in > 0.0) ? sqrt(sqrt(in / xn)) : 1.0;
    const double ig = 1.0 / g;
    D3 nx, dx;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        nx.a[i][j] = 0.5 * (g * X.a[i][j] + xit.a[i][j] * ig);
        dx.a[i][j] = nx.a[i][j] - X.a[i][j];
      }
    const double delta = d3_frob(dx);
    X = nx;
    const double fx = d3_frob(X);
    if (delta <= PBDR_POLAR_TOL * (fx > 1e-300 ? fx : 1e-300)) break;
  }
  d3_quat_from(X, q);
  d3_quat_to(q, R);
  return true;
}

__device__ void d3_sym_eigen(const D3& m, double ev[3], D3& V) {
  double A[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) A[i][j] = 0.5 * (m.a[i][j] + m.a[j][i]);
  double U[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  for (int sweep = 0; sweep < 32; ++sweep) {
    const double off = (fabs(A[0][1]) + fabs(A[0][2])) + fabs(A[1][2]);
    const double scale = (fabs(A[0][0]) + fabs(A[1][1])) + fabs(A[2][2]);
    if (off <= 1e-15 * (scale > 1e-300 ? scale : 1e-300)) break;
    for (int p = 0; p < 2; ++p)
      for (int qq = p + 1; qq < 3; ++qq) {
        if (A[p][qq] == 0.0) continue;
        const double theta = (A[qq][qq] - A[p][p]) / (2.0 * A[p][qq]);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0);
        const double s = t * c;
        const double app = A[p][p], aqq = A[qq][qq], apq = A[p][qq];
        A[p][p] = ((c * c) * app - ((2.0 * s) * c) * apq) + (s * s) * aqq;
        A[qq][qq] = ((s * s) * app + ((2.0 * s) * c) * apq) + (c * c) * aqq;
        A[p][qq] = 0.0;
        A[qq][p] = 0.0;
        for (int k = 0; k < 3; ++k) {
          if (k == p || k == qq) continue;
          const double akp = A[k][p], akq = A[k][qq];
          A[k][p] = c * akp - s * akq;
          A[p][k] = A[k][p];
          A[k][qq] = s * akp + c * akq;
          A[qq][k] = A[k][qq];
        }
        for (int k = 0; k < 3; ++k) {
          const double vkp = U[k][p], vkq = U[k][qq];
          U[k][p] = c * vkp - s * vkq;
          U[k][qq] = s * vkp + c * vkq;
        }
      }
  }
  int order[3] = {0, 1, 2};
  const double d[3] = {A[0][0], A[1][1], A[2][2]};
  for (int i = 1; i < 3; ++i) {
    const int o = order[i];
    int j = i - 1;
    while (j >= 0 && d[order[j]] > d[o]) {
      order[j + 1] = order[j];
      --j;
    }
    order[j + 1] = o;
  }
  for (int i = 0; i < 3; ++i) {
    ev[i] = d[order[i]];
    for (int k = 0; k < 3; ++k) V.a[k][i] = U[k][order[i]];
  }
}

// omega = pinv(I) dL (fp32 inputs, fp64 solve). Returns 0 or
// PBDR_DEVERR_RANK_DEFICIENT (omega = 0, null axis filled).
__device__ __noinline__ unsigned inertia_solve_f(const float If[6] /* xx yy zz xy xz yz */,
                                                  const float dLf[3], float w[3],
                                                  double null_axis[3]) {
  D3 I;
  I.a[0][0] = If[0]; I.a[1][1] = If[1]; I.a[2][2] = If[2];
  I.a[0][1] = If[3]; I.a[1][0] = If[3];
  I.a[0][2] = If[4]; I.a[2][0] = If[4];
  I.a[1][2] = If[5]; I.a[2][1] = If[5];
  const double dL[3] = {static_cast<double>(dLf[0]), static_cast<double>(dLf[1]),
                        static_cast<double>(dLf[2])};
  const double tr = (I.a[0][0] + I.a[1][1]) + I.a[2][2];
  const double d = d3_det(I);
  w[0] = w[1] = w[2] = 0.0f;
  if (tr > 0.0 && d >= PBDR_PINV_FAST_DET * ((tr * tr) * tr)) {
    const D3 inv = d3_adj_inverse(I, d);
#pragma unroll
    for (int r = 0; r < 3; ++r)
      w[r] = static_cast<float>((inv.a[r][0] * dL[0] + inv.a[r][1] * dL[1]) + inv.a[r][2] * dL[2]);
    return 0u;
  }
  double ev[3];
  D3 V;
  d3_sym_eigen(I, ev, V);
  const double atr = fabs(tr);
  const double cut = PBDR_PINV_REL_TOL * (atr > 1e-300 ? atr : 1e-300);
  D3 P;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) P.a[i][j] = 0.0;
  int rank = 0;
  double nax[3] = {0.0, 0.0, 0.0};
  for (int k = 0; k < 3; ++k) {
    const double u[3] = {V.a[0][k], V.a[1][k], V.a[2][k]};
    if (ev[k] >= cut) {
      const double il = 1.0 / ev[k];
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) P.a[i][j] = P.a[i][j] + (u[i] * u[j]) * il;
      ++rank;
    } else {
      nax[0] = u[0]; nax[1] = u[1]; nax[2] = u[2];
    }
  }
  if (rank < 3) {
    const double along = fabs((dL[0] * nax[0] + dL[1] * nax[1]) + dL[2] * nax[2]);
    if (along > PBDR_NULL_AXIS_TOL) {
      null_axis[0] = nax[0]; null_axis[1] = nax[1]; null_axis[2] = nax[2];
      return PBDR_DEVERR_RANK_DEFICIENT;
    }
  }
  for (int r = 0; r < 3; ++r)
    w[r] = static_cast<float>((P.a[r][0] * dL[0] + P.a[r][1] * dL[1]) + P.a[r][2] * dL[2]);
  return 0u;
}

}  // namespace pbdr_dev
