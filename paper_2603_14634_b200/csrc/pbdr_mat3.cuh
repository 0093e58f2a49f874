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
    const double is = 1.0 / s;
    w = 0.25 * s;
    qx = (x.a[2][1] - x.a[1][2]) * is;
    qy = (x.a[0][2] - x.a[2][0]) * is;
    qz = (x.a[1][0] - x.a[0][1]) * is;
  } else if (x.a[0][0] > x.a[1][1] && x.a[0][0] > x.a[2][2]) {
    const double s = sqrt(((1.0 + x.a[0][0]) - x.a[1][1]) - x.a[2][2]) * 2.0;
    const double is = 1.0 / s;
    w = (x.a[2][1] - x.a[1][2]) * is;
    qx = 0.25 * s;
    qy = (x.a[0][1] + x.a[1][0]) * is;
    qz = (x.a[0][2] + x.a[2][0]) * is;
  } else if (x.a[1][1] > x.a[2][2]) {
    const double s = sqrt(((1.0 + x.a[1][1]) - x.a[0][0]) - x.a[2][2]) * 2.0;
    const double is = 1.0 / s;
    w = (x.a[0][2] - x.a[2][0]) * is;
    qx = (x.a[0][1] + x.a[1][0]) * is;
    qy = 0.25 * s;
    qz = (x.a[1][2] + x.a[2][1]) * is;
  } else {
    const double s = sqrt(((1.0 + x.a[2][2]) - x.a[0][0]) - x.a[1][1]) * 2.0;
    const double is = 1.0 / s;
    w = (x.a[1][0] - x.a[0][1]) * is;
    qx = (x.a[0][2] + x.a[2][0]) * is;
    qy = (x.a[1][2] + x.a[2][1]) * is;
    qz = 0.25 * s;
  }
  const double n = sqrt(((w * w + qx * qx) + qy * qy) + qz * qz);
  if (n > 0.0) {
    const double in = 1.0 / n;
    w = w * in; qx = qx * in; qy = qy * in; qz = qz * in;
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

// R = r * |q|^2 R(q) (homogeneous form; r = 1/|q|^2 gives the rotation of a
// non-unit q), rounded to float.
__device__ __forceinline__ void d3_quat_to_h(const double q[4], double r, float R[9]) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  const double w2 = w * w, xx = x * x, yy = y * y, zz = z * z;
  const double xy = x * y, xz = x * z, yz = y * z;
  const double wx = w * x, wy = w * y, wz = w * z;
  R[0] = static_cast<float>(((w2 + xx) - (yy + zz)) * r);
  R[1] = static_cast<float>((2.0 * (xy - wz)) * r);
  R[2] = static_cast<float>((2.0 * (xz + wy)) * r);
  R[3] = static_cast<float>((2.0 * (xy + wz)) * r);
  R[4] = static_cast<float>(((w2 + yy) - (xx + zz)) * r);
  R[5] = static_cast<float>((2.0 * (yz - wx)) * r);
  R[6] = static_cast<float>((2.0 * (xz - wy)) * r);
  R[7] = static_cast<float>((2.0 * (yz + wx)) * r);
  R[8] = static_cast<float>(((w2 + zz) - (xx + yy)) * r);
}

__device__ __forceinline__ double d3_frob2(const D3& m) {
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) s = s + m.a[i][j] * m.a[i][j];
  return s;
}

// Pinned Newton polar loop (float or double), mirrored line by line from
// oracle/oracle_math.hpp newton_polar(). Returns iterations used, -1 if singular.
template <typename T>
__device__ __forceinline__ int newton_polar(T X[3][3], T tol2, T tolq, T scale_rel2, int max_it, bool scaled) {
  for (int it = 0; it < max_it; ++it) {
    const T d = X[0][0] * (X[1][1] * X[2][2] - X[1][2] * X[2][1]) -
                X[0][1] * (X[1][0] * X[2][2] - X[1][2] * X[2][0]) +
                X[0][2] * (X[1][0] * X[2][1] - X[1][1] * X[2][0]);
    if (d == T(0) || !isfinite(d)) return -1;
    const T id = T(1) / d;
    T inv[3][3];
    inv[0][0] = (X[1][1] * X[2][2] - X[1][2] * X[2][1]) * id;
    inv[0][1] = (X[0][2] * X[2][1] - X[0][1] * X[2][2]) * id;
    inv[0][2] = (X[0][1] * X[1][2] - X[0][2] * X[1][1]) * id;
    inv[1][0] = (X[1][2] * X[2][0] - X[1][0] * X[2][2]) * id;
    inv[1][1] = (X[0][0] * X[2][2] - X[0][2] * X[2][0]) * id;
    inv[1][2] = (X[0][2] * X[1][0] - X[0][0] * X[1][2]) * id;
    inv[2][0] = (X[1][0] * X[2][1] - X[1][1] * X[2][0]) * id;
    inv[2][1] = (X[0][1] * X[2][0] - X[0][0] * X[2][1]) * id;
    inv[2][2] = (X[0][0] * X[1][1] - X[0][1] * X[1][0]) * id;
    T g = T(1), ig = T(1);
    if (scaled) {
      float c = 0.0f, r = 0.0f, ci = 0.0f, ri = 0.0f;
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const float s1 = static_cast<float>((fabs(X[0][j]) + fabs(X[1][j])) + fabs(X[2][j]));
        const float s2 = static_cast<float>((fabs(inv[0][j]) + fabs(inv[1][j])) + fabs(inv[2][j]));
        c = s1 > c ? s1 : c;
        ci = s2 > ci ? s2 : ci;
      }
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const float s1 = static_cast<float>((fabs(X[i][0]) + fabs(X[i][1])) + fabs(X[i][2]));
        const float s2 = static_cast<float>((fabs(inv[i][0]) + fabs(inv[i][1])) + fabs(inv[i][2]));
        r = s1 > r ? s1 : r;
        ri = s2 > ri ? s2 : ri;
      }
      const float xn = c * r, in = ci * ri;
      if (xn > 0.0f && in > 0.0f && isfinite(in / xn)) {
        const float gf = sqrtf(sqrtf(in / xn));
        g = static_cast<T>(gf);
        ig = static_cast<T>(1.0f / gf);
      }
    }
    T dd[9], ff[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const T nx = T(0.5) * (g * X[i][j] + inv[j][i] * ig);
        const T dx = nx - X[i][j];
        dd[3 * i + j] = dx * dx;
        ff[3 * i + j] = nx * nx;
        X[i][j] = nx;
      }
    const T delta2 = (((dd[0] + dd[1]) + (dd[2] + dd[3])) + ((dd[4] + dd[5]) + (dd[6] + dd[7]))) + dd[8];
    const T fx2 = (((ff[0] + ff[1]) + (ff[2] + ff[3])) + ((ff[4] + ff[5]) + (ff[6] + ff[7]))) + ff[8];
    const T fx = fx2 > T(1e-30) ? fx2 : T(1e-30);
    if (delta2 <= tol2 * fx || (!scaled && delta2 <= tolq * fx)) return it + 1;
    scaled = delta2 > scale_rel2 * fx;
  }
  return max_it;
}

// Rotation of the polar decomposition of A (row-major fp32 sums): fp32 scaled
// Newton on A / (||A||_F / sqrt3), then unscaled fp64 Newton to 1e-9, then the
// quaternion round trip (math.cpp:207-209). Returns false when A is degenerate.
__device__ __noinline__ bool polar_rotation_f(const float Af[9], float R[9], double q[4]) {
  D3 A;
  bool finite = true;
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    A.a[i / 3][i % 3] = static_cast<double>(Af[i]);
    finite = finite && isfinite(Af[i]);
  }
  if (!finite) return false;
  const double d0 = d3_det(A);
  const double c3 = d3_frob2(A) * PBDR_ONE_THIRD;
  if (!(d0 > 0.0) || d0 * d0 <= (PBDR_POLAR_REL_DET * PBDR_POLAR_REL_DET) * ((c3 * c3) * c3)) return false;
  const double is = 1.0 / sqrt(c3);
  float Xf[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) Xf[i][j] = static_cast<float>(A.a[i][j] * is);
  double X[3][3];
  const int f_it = newton_polar<float>(Xf, PBDR_POLAR_F32_TOL2, PBDR_POLAR_F32_TOLQ,
                                       static_cast<float>(PBDR_POLAR_SCALE_REL2), PBDR_POLAR_F32_MAX_IT, true);
  D3 Xm;
  if (f_it > 0) {
    // fp64 polish: one unscaled Newton step re-orthonormalises the fp32
    // iterate (R0), then one first-order rotation correction solves the
    // symmetry condition of B = R0^T A: axial(B - B^T) = (tr(S) I - S) w,
    // S = sym(B), and R = R0 (I + [w]x) (error O(|w|^2) ~ 1e-14).
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) X[i][j] = static_cast<double>(Xf[i][j]);
    if (newton_polar<double>(X, 0.0, 0.0, 0.0, 1, false) < 0) return false;
    double B[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j)
        B[i][j] = (X[0][i] * A.a[0][j] + X[1][i] * A.a[1][j]) + X[2][i] * A.a[2][j];
    const double sv[3] = {B[2][1] - B[1][2], B[0][2] - B[2][0], B[1][0] - B[0][1]};
    double M[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) M[i][j] = -(0.5 * (B[i][j] + B[j][i]));
    const double tr = (-M[0][0] + -M[1][1]) + -M[2][2];
    M[0][0] = tr + M[0][0];
    M[1][1] = tr + M[1][1];
    M[2][2] = tr + M[2][2];
    const double dm = M[0][0] * (M[1][1] * M[2][2] - M[1][2] * M[2][1]) -
                      M[0][1] * (M[1][0] * M[2][2] - M[1][2] * M[2][0]) +
                      M[0][2] * (M[1][0] * M[2][1] - M[1][1] * M[2][0]);
    double w[3] = {0.0, 0.0, 0.0};
    if (dm != 0.0 && isfinite(dm)) {
      const double idm = 1.0 / dm;
      const double c00 = (M[1][1] * M[2][2] - M[1][2] * M[2][1]) * idm;
      const double c01 = (M[0][2] * M[2][1] - M[0][1] * M[2][2]) * idm;
      const double c02 = (M[0][1] * M[1][2] - M[0][2] * M[1][1]) * idm;
      const double c11 = (M[0][0] * M[2][2] - M[0][2] * M[2][0]) * idm;
      const double c12 = (M[0][2] * M[1][0] - M[0][0] * M[1][2]) * idm;
      const double c22 = (M[0][0] * M[1][1] - M[0][1] * M[1][0]) * idm;
      w[0] = (c00 * sv[0] + c01 * sv[1]) + c02 * sv[2];
      w[1] = (c01 * sv[0] + c11 * sv[1]) + c12 * sv[2];
      w[2] = (c02 * sv[0] + c12 * sv[1]) + c22 * sv[2];
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      Xm.a[i][0] = X[i][0] + (X[i][1] * w[2] - X[i][2] * w[1]);
      Xm.a[i][1] = X[i][1] + (X[i][2] * w[0] - X[i][0] * w[2]);
      Xm.a[i][2] = X[i][2] + (X[i][0] * w[1] - X[i][1] * w[0]);
    }
  } else {
    // fp32 stage broke down: full scaled fp64 Newton from A.
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) X[i][j] = A.a[i][j];
    if (newton_polar<double>(X, PBDR_POLAR_TOL2, PBDR_POLAR_TOLQ, PBDR_POLAR_SCALE_REL2, PBDR_POLAR_MAX_IT, true) < 0)
      return false;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) Xm.a[i][j] = X[i][j];
  }
  d3_quat_from(Xm, q);
  d3_quat_to(q, R);
  return true;
}

// Warm-started rotation extraction (pinned): starting from the body's rotation
// of the previous solver iteration (quaternion rq, all-zero = none), apply
// Gauss-Newton corrections of the polar factor's symmetry condition -- with
// B = R^T A and S = sym(B): axial(B - B^T) = (tr(S) I - S) w, then
// q <- q (x) (1, w/2), unnormalised (R built homogeneously as |q|^2 R(q)), until
// |w|^2 <= 1e-10; the last q is normalised (the step leaves an O(|w|^2) error). Converges quadratically from any nearby R whatever the
// conditioning of S. A missing warm start, |w|^2 > 0.25 (not local), a
// singular solve, or 4 steps without convergence fall back to the cold
// two-stage Newton polar. The result is the same polar factor to 1e-12.
// PBDR_GN_ROLLED: keep the Gauss-Newton step loop rolled (code size).
#ifndef PBDR_GN_ROLLED
#define PBDR_GN_ROLLED 0
#endif
#ifndef PBDR_WARM_INLINE
#define PBDR_WARM_INLINE 1
#endif
#if PBDR_WARM_INLINE
__device__ __forceinline__  // inlined: no call frame / spills around it (measured -5% per iteration)
#else
__device__ __noinline__
#endif
bool polar_warm_f(const float Af[9], const float rq[4], float R[9], double q[4], int* steps_used = nullptr) {
  D3 A;
  bool finite = true;
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    A.a[i / 3][i % 3] = static_cast<double>(Af[i]);
    finite = finite && isfinite(Af[i]);
  }
  // Degeneracy is decided here but only acted on at the exits, so the checks
  // overlap the first Gauss-Newton step instead of preceding it.
  const double d0 = d3_det(A);
  const double c3 = d3_frob2(A) * PBDR_ONE_THIRD;
  const bool bad =
      !finite || !(d0 > 0.0) || d0 * d0 <= (PBDR_POLAR_REL_DET * PBDR_POLAR_REL_DET) * ((c3 * c3) * c3);
#if PBDR_POLAR_WARM_F32
  if (rq[0] != 0.0f || rq[1] != 0.0f || rq[2] != 0.0f || rq[3] != 0.0f) {
    // The same homogeneous Gauss-Newton iteration in fp32 (mirrors oracle
    // polar_warm_f32): A is the fp32 body sum itself.
    float qc[4] = {rq[0], rq[1], rq[2], rq[3]};
#if PBDR_GN_ROLLED
#pragma unroll 1
#endif
    for (int step = 0; step < PBDR_POLAR_WARM_STEPS; ++step) {
      const float w = qc[0], x = qc[1], y = qc[2], z = qc[3];
      const float w2 = w * w, xx = x * x, yy = y * y, zz = z * z;
      const float xy = x * y, xz = x * z, yz = y * z;
      const float wx = w * x, wy = w * y, wz = w * z;
      float R0[3][3];
      R0[0][0] = (w2 + xx) - (yy + zz);
      R0[0][1] = 2.0f * (xy - wz);
      R0[0][2] = 2.0f * (xz + wy);
      R0[1][0] = 2.0f * (xy + wz);
      R0[1][1] = (w2 + yy) - (xx + zz);
      R0[1][2] = 2.0f * (yz - wx);
      R0[2][0] = 2.0f * (xz - wy);
      R0[2][1] = 2.0f * (yz + wx);
      R0[2][2] = (w2 + zz) - (xx + yy);
      float B[3][3];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) B[i][j] = (R0[0][i] * Af[j] + R0[1][i] * Af[3 + j]) + R0[2][i] * Af[6 + j];
      const float sv[3] = {B[2][1] - B[1][2], B[0][2] - B[2][0], B[1][0] - B[0][1]};
      float M[3][3];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) M[i][j] = -(0.5f * (B[i][j] + B[j][i]));
      const float tr = (-M[0][0] + -M[1][1]) + -M[2][2];
      M[0][0] = tr + M[0][0];
      M[1][1] = tr + M[1][1];
      M[2][2] = tr + M[2][2];
      const float dm = M[0][0] * (M[1][1] * M[2][2] - M[1][2] * M[2][1]) -
                       M[0][1] * (M[1][0] * M[2][2] - M[1][2] * M[2][0]) +
                       M[0][2] * (M[1][0] * M[2][1] - M[1][1] * M[2][0]);
      if (!(dm > 0.0f) || !isfinite(dm)) break;
      const float idm = 1.0f / dm;
      const float c00 = (M[1][1] * M[2][2] - M[1][2] * M[2][1]) * idm;
      const float c01 = (M[0][2] * M[2][1] - M[0][1] * M[2][2]) * idm;
      const float c02 = (M[0][1] * M[1][2] - M[0][2] * M[1][1]) * idm;
      const float c11 = (M[0][0] * M[2][2] - M[0][2] * M[2][0]) * idm;
      const float c12 = (M[0][2] * M[1][0] - M[0][0] * M[1][2]) * idm;
      const float c22 = (M[0][0] * M[1][1] - M[0][1] * M[1][0]) * idm;
      const float h[3] = {0.5f * ((c00 * sv[0] + c01 * sv[1]) + c02 * sv[2]),
                          0.5f * ((c01 * sv[0] + c11 * sv[1]) + c12 * sv[2]),
                          0.5f * ((c02 * sv[0] + c12 * sv[1]) + c22 * sv[2])};
      const float ww = 4.0f * ((h[0] * h[0] + h[1] * h[1]) + h[2] * h[2]);
      if (!(ww <= static_cast<float>(PBDR_POLAR_WARM_MAX2))) break;
      float qn[4];
      qn[0] = qc[0] - ((qc[1] * h[0] + qc[2] * h[1]) + qc[3] * h[2]);
      qn[1] = (qc[0] * h[0] + qc[1]) + (qc[2] * h[2] - qc[3] * h[1]);
      qn[2] = (qc[0] * h[1] + qc[2]) + (qc[3] * h[0] - qc[1] * h[2]);
      qn[3] = (qc[0] * h[2] + qc[3]) + (qc[1] * h[1] - qc[2] * h[0]);
      if (ww <= static_cast<float>(PBDR_POLAR_WARM_TOLQ)) {
        if (steps_used) *steps_used = step + 1;
        if (bad) return false;
        const float n2 = ((qn[0] * qn[0] + qn[1] * qn[1]) + qn[2] * qn[2]) + qn[3] * qn[3];
        const float r = 1.0f / n2;
        const float s = 1.5f - 0.5f * n2;
        const float a = qn[0], b = qn[1], c = qn[2], d = qn[3];
        const float a2 = a * a, bb = b * b, cc = c * c, dd = d * d;
        const float bc = b * c, bd = b * d, cd = c * d, ab = a * b, ac = a * c, ad = a * d;
        R[0] = ((a2 + bb) - (cc + dd)) * r;
        R[1] = (2.0f * (bc - ad)) * r;
        R[2] = (2.0f * (bd + ac)) * r;
        R[3] = (2.0f * (bc + ad)) * r;
        R[4] = ((a2 + cc) - (bb + dd)) * r;
        R[5] = (2.0f * (cd - ab)) * r;
        R[6] = (2.0f * (bd - ac)) * r;
        R[7] = (2.0f * (cd + ab)) * r;
        R[8] = ((a2 + dd) - (bb + cc)) * r;
#pragma unroll
        for (int k = 0; k < 4; ++k) q[k] = static_cast<double>(qn[k] * s);
        return true;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) qc[k] = qn[k];
    }
  }
#else
  if (rq[0] != 0.0f || rq[1] != 0.0f || rq[2] != 0.0f || rq[3] != 0.0f) {
    // Homogeneous iterate (mirrors oracle polar_warm): qc is not renormalised
    // between steps; R0 = |qc|^2 R(qc) and the step h is scale invariant.
    double qc[4] = {rq[0], rq[1], rq[2], rq[3]};
#if PBDR_GN_ROLLED
#pragma unroll 1
#endif
    for (int step = 0; step < PBDR_POLAR_WARM_STEPS; ++step) {
      const double w = qc[0], x = qc[1], y = qc[2], z = qc[3];
      const double w2 = w * w, xx = x * x, yy = y * y, zz = z * z;
      const double xy = x * y, xz = x * z, yz = y * z;
      const double wx = w * x, wy = w * y, wz = w * z;
      double R0[3][3];
      R0[0][0] = (w2 + xx) - (yy + zz);
      R0[0][1] = 2.0 * (xy - wz);
      R0[0][2] = 2.0 * (xz + wy);
      R0[1][0] = 2.0 * (xy + wz);
      R0[1][1] = (w2 + yy) - (xx + zz);
      R0[1][2] = 2.0 * (yz - wx);
      R0[2][0] = 2.0 * (xz - wy);
      R0[2][1] = 2.0 * (yz + wx);
      R0[2][2] = (w2 + zz) - (xx + yy);
      double B[3][3];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
          B[i][j] = (R0[0][i] * A.a[0][j] + R0[1][i] * A.a[1][j]) + R0[2][i] * A.a[2][j];
      const double sv[3] = {B[2][1] - B[1][2], B[0][2] - B[2][0], B[1][0] - B[0][1]};
      double M[3][3];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) M[i][j] = -(0.5 * (B[i][j] + B[j][i]));
      const double tr = (-M[0][0] + -M[1][1]) + -M[2][2];
      M[0][0] = tr + M[0][0];
      M[1][1] = tr + M[1][1];
      M[2][2] = tr + M[2][2];
      const double dm = M[0][0] * (M[1][1] * M[2][2] - M[1][2] * M[2][1]) -
                        M[0][1] * (M[1][0] * M[2][2] - M[1][2] * M[2][0]) +
                        M[0][2] * (M[1][0] * M[2][1] - M[1][1] * M[2][0]);
      if (!(dm > 0.0) || !isfinite(dm)) break;
      const double idm = 1.0 / dm;
      const double c00 = (M[1][1] * M[2][2] - M[1][2] * M[2][1]) * idm;
      const double c01 = (M[0][2] * M[2][1] - M[0][1] * M[2][2]) * idm;
      const double c02 = (M[0][1] * M[1][2] - M[0][2] * M[1][1]) * idm;
      const double c11 = (M[0][0] * M[2][2] - M[0][2] * M[2][0]) * idm;
      const double c12 = (M[0][2] * M[1][0] - M[0][0] * M[1][2]) * idm;
      const double c22 = (M[0][0] * M[1][1] - M[0][1] * M[1][0]) * idm;
      const double h[3] = {0.5 * ((c00 * sv[0] + c01 * sv[1]) + c02 * sv[2]),
                           0.5 * ((c01 * sv[0] + c11 * sv[1]) + c12 * sv[2]),
                           0.5 * ((c02 * sv[0] + c12 * sv[1]) + c22 * sv[2])};
      const double ww = 4.0 * ((h[0] * h[0] + h[1] * h[1]) + h[2] * h[2]);
      if (!(ww <= PBDR_POLAR_WARM_MAX2)) break;
      double qn[4];
      qn[0] = qc[0] - ((qc[1] * h[0] + qc[2] * h[1]) + qc[3] * h[2]);
      qn[1] = (qc[0] * h[0] + qc[1]) + (qc[2] * h[2] - qc[3] * h[1]);
      qn[2] = (qc[0] * h[1] + qc[2]) + (qc[3] * h[0] - qc[1] * h[2]);
      qn[3] = (qc[0] * h[2] + qc[3]) + (qc[1] * h[1] - qc[2] * h[0]);
      if (ww <= PBDR_POLAR_WARM_TOLQ) {
        if (steps_used) *steps_used = step + 1;
        if (bad) return false;
        // R = |qn|^-2 (homogeneous rotation of qn); the stored quaternion gets
        // one Newton step of 1/sqrt from |qn|^2 ~ 1 (error O((|qn|^2 - 1)^2)).
        const double n2 = ((qn[0] * qn[0] + qn[1] * qn[1]) + qn[2] * qn[2]) + qn[3] * qn[3];
        const double r = 1.0 / n2;
        const double s = 1.5 - 0.5 * n2;
        d3_quat_to_h(qn, r, R);
#pragma unroll
        for (int k = 0; k < 4; ++k) q[k] = qn[k] * s;
        return true;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) qc[k] = qn[k];
    }
  }
#endif
  if (steps_used) *steps_used = 15;  // cold fallback
  if (bad) return false;
  // Cold path through copies: no array of the caller's hot path has its
  // address taken (address-taken arrays live in local memory on every path,
  // and in contact-rich states those local loads miss L1).
  float Ac[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) Ac[i] = Af[i];
  double qc[4];
  const bool ok = polar_rotation_f(Ac, R, qc);
#pragma unroll
  for (int k = 0; k < 4; ++k) q[k] = qc[k];
  return ok;
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
__device__ __noinline__ unsigned inertia_solve_slow(const D3& I, const double dL[3], float w[3],
                                                     double null_axis[3]);

__device__ __forceinline__ unsigned inertia_solve_f(const float If[6] /* xx yy zz xy xz yz */,
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
  // Through copies, as polar_warm_f's cold path (keeps the callers' arrays
  // out of local memory).
  D3 Ic = I;
  double dLc[3] = {dL[0], dL[1], dL[2]}, nc[3] = {0.0, 0.0, 0.0};
  float wc[3];
  const unsigned e = inertia_solve_slow(Ic, dLc, wc, nc);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    w[k] = wc[k];
    null_axis[k] = nc[k];
  }
  return e;
}

// Cyclic-Jacobi pseudo-inverse path (rank-deficient or ill-conditioned I).
__device__ __noinline__ unsigned inertia_solve_slow(const D3& I, const double dL[3], float w[3],
                                                     double null_axis[3]) {
  const double tr = (I.a[0][0] + I.a[1][1]) + I.a[2][2];
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
