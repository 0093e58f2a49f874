// TEST INFRASTRUCTURE ONLY — part of the CPU oracle (see pbdr_oracle.cpp).
//
// Double-precision 3x3 numerics restated from the reference's math module,
// with the op order pinned so that the CUDA
// path's per-body math is bit-identical:
//   * adjugate inverse            — math.cpp:8-24
//   * cyclic Jacobi eigen         — math.cpp:26-71
//   * SPD pseudo-inverse          — math.cpp:90-108
//   * quaternion from/to matrix   — math.cpp:117-146, math.hpp:217-227
//   * scaled-Newton polar         — math.cpp:170-210
// Deviations from the reference (all documented in DESIGN.md):
//   * g = (in/xn)^(1/4) is evaluated as sqrt(sqrt(.)) (correctly rounded on
//     both CPU and GPU) instead of std::pow; X^-T/g as X^-T * (1/g); the
//     scaling is applied only while the relative change exceeds 1e-2 (then
//     plain Newton, which converges quadratically near the polar factor);
//     root-free degeneracy and convergence tests;
//   * the polar degeneracy test is scale-relative (pbdr_pinned.h);
//   * the inertia inverse takes the adjugate branch when provably full rank.
// These functions are checked against the reference's own compiled math
// (oracle/_ref) by tests/test_oracle_golden.py.
#pragma once

#include <cmath>

#include "pbdr_pinned.h"

namespace orc {

struct M3 {
  double a[3][3];
};

inline double det3(const M3& m) {
  return m.a[0][0] * (m.a[1][1] * m.a[2][2] - m.a[1][2] * m.a[2][1]) -
         m.a[0][1] * (m.a[1][0] * m.a[2][2] - m.a[1][2] * m.a[2][0]) +
         m.a[0][2] * (m.a[1][0] * m.a[2][1] - m.a[1][1] * m.a[2][0]);
}

inline double frob(const M3& m) {
  double s = 0.0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) s = s + m.a[i][j] * m.a[i][j];
  return std::sqrt(s);
}

inline bool finite3(const M3& m) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      if (!std::isfinite(m.a[i][j])) return false;
  return true;
}

// Adjugate / det. Caller guarantees det != 0.
inline M3 adj_inverse(const M3& m, double d) {
  const double id = 1.0 / d;
  const double(*a)[3] = m.a;
  M3 r;
  r.a[0][0] = (a[1][1] * a[2][2] - a[1][2] * a[2][1]) * id;
  r.a[0][1] = (a[0][2] * a[2][1] - a[0][1] * a[2][2]) * id;
  r.a[0][2] = (a[0][1] * a[1][2] - a[0][2] * a[1][1]) * id;
  r.a[1][0] = (a[1][2] * a[2][0] - a[1][0] * a[2][2]) * id;
  r.a[1][1] = (a[0][0] * a[2][2] - a[0][2] * a[2][0]) * id;
  r.a[1][2] = (a[0][2] * a[1][0] - a[0][0] * a[1][2]) * id;
  r.a[2][0] = (a[1][0] * a[2][1] - a[1][1] * a[2][0]) * id;
  r.a[2][1] = (a[0][1] * a[2][0] - a[0][0] * a[2][1]) * id;
  r.a[2][2] = (a[0][0] * a[1][1] - a[0][1] * a[1][0]) * id;
  return r;
}

// max column abs-sum times max row abs-sum.
inline double norm1_inf(const M3& m) {
  double c = 0.0, r = 0.0;
  for (int j = 0; j < 3; ++j) {
    const double s = (std::fabs(m.a[0][j]) + std::fabs(m.a[1][j])) + std::fabs(m.a[2][j]);
    c = s > c ? s : c;
  }
  for (int i = 0; i < 3; ++i) {
    const double s = (std::fabs(m.a[i][0]) + std::fabs(m.a[i][1])) + std::fabs(m.a[i][2]);
    r = s > r ? s : r;
  }
  return c * r;
}

// Unit quaternion (w, x, y, z) from a near-rotation matrix, largest-pivot
// branch (one reciprocal of the pivot), then normalised by one reciprocal.
inline void quat_from(const M3& x, double q[4]) {
  const double(*m)[3] = x.a;
  const double tr = (m[0][0] + m[1][1]) + m[2][2];
  double w, qx, qy, qz;
  if (tr > 0.0) {
    const double s = std::sqrt(tr + 1.0) * 2.0;
    const double is = 1.0 / s;
    w = 0.25 * s;
    qx = (m[2][1] - m[1][2]) * is;
    qy = (m[0][2] - m[2][0]) * is;
    qz = (m[1][0] - m[0][1]) * is;
  } else if (m[0][0] > m[1][1] && m[0][0] > m[2][2]) {
    const double s = std::sqrt(((1.0 + m[0][0]) - m[1][1]) - m[2][2]) * 2.0;
    const double is = 1.0 / s;
    w = (m[2][1] - m[1][2]) * is;
    qx = 0.25 * s;
    qy = (m[0][1] + m[1][0]) * is;
    qz = (m[0][2] + m[2][0]) * is;
  } else if (m[1][1] > m[2][2]) {
    const double s = std::sqrt(((1.0 + m[1][1]) - m[0][0]) - m[2][2]) * 2.0;
    const double is = 1.0 / s;
    w = (m[0][2] - m[2][0]) * is;
    qx = (m[0][1] + m[1][0]) * is;
    qy = 0.25 * s;
    qz = (m[1][2] + m[2][1]) * is;
  } else {
    const double s = std::sqrt(((1.0 + m[2][2]) - m[0][0]) - m[1][1]) * 2.0;
    const double is = 1.0 / s;
    w = (m[1][0] - m[0][1]) * is;
    qx = (m[0][2] + m[2][0]) * is;
    qy = (m[1][2] + m[2][1]) * is;
    qz = 0.25 * s;
  }
  const double n = std::sqrt(((w * w + qx * qx) + qy * qy) + qz * qz);
  if (n > 0.0) {
    const double in = 1.0 / n;
    w = w * in; qx = qx * in; qy = qy * in; qz = qz * in;
  } else {
    w = 1.0; qx = qy = qz = 0.0;
  }
  q[0] = w; q[1] = qx; q[2] = qy; q[3] = qz;
}

inline M3 quat_to(const double q[4]) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  const double xx = x * x, yy = y * y, zz = z * z;
  const double xy = x * y, xz = x * z, yz = y * z;
  const double wx = w * x, wy = w * y, wz = w * z;
  M3 r;
  r.a[0][0] = 1.0 - 2.0 * (yy + zz);
  r.a[0][1] = 2.0 * (xy - wz);
  r.a[0][2] = 2.0 * (xz + wy);
  r.a[1][0] = 2.0 * (xy + wz);
  r.a[1][1] = 1.0 - 2.0 * (xx + zz);
  r.a[1][2] = 2.0 * (yz - wx);
  r.a[2][0] = 2.0 * (xz - wy);
  r.a[2][1] = 2.0 * (yz + wx);
  r.a[2][2] = 1.0 - 2.0 * (xx + yy);
  return r;
}

// |q|^2 R(q) for a non-unit quaternion (homogeneous form).
inline M3 quat_to_h(const double q[4]) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  const double w2 = w * w, xx = x * x, yy = y * y, zz = z * z;
  const double xy = x * y, xz = x * z, yz = y * z;
  const double wx = w * x, wy = w * y, wz = w * z;
  M3 r;
  r.a[0][0] = (w2 + xx) - (yy + zz);
  r.a[0][1] = 2.0 * (xy - wz);
  r.a[0][2] = 2.0 * (xz + wy);
  r.a[1][0] = 2.0 * (xy + wz);
  r.a[1][1] = (w2 + yy) - (xx + zz);
  r.a[1][2] = 2.0 * (yz - wx);
  r.a[2][0] = 2.0 * (xz - wy);
  r.a[2][1] = 2.0 * (yz + wx);
  r.a[2][2] = (w2 + zz) - (xx + yy);
  return r;
}

inline double frob2(const M3& m) {
  double s = 0.0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) s = s + m.a[i][j] * m.a[i][j];
  return s;
}

// One pinned Newton polar loop on a 3x3 of float or double (the same code
// runs in fp32 and fp64): X <- (g X + X^-T / g) / 2, with the 1-inf scaling g
// (formed in fp32) while the relative change exceeds 1e-2. Stops when the
// change is below tol, or -- after an unscaled step, whose remaining error is
// O(change^2) -- below sqrt(tol). Returns the iterations used, or -1 when the
// iterate became singular.
template <typename T>
int newton_polar(T X[3][3], T tol2, T tolq, T scale_rel2, int max_it, bool scaled) {
  for (int it = 0; it < max_it; ++it) {
    const T d = X[0][0] * (X[1][1] * X[2][2] - X[1][2] * X[2][1]) -
                X[0][1] * (X[1][0] * X[2][2] - X[1][2] * X[2][0]) +
                X[0][2] * (X[1][0] * X[2][1] - X[1][1] * X[2][0]);
    if (d == T(0) || !std::isfinite(d)) return -1;
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
      for (int j = 0; j < 3; ++j) {
        const float s1 = static_cast<float>((std::fabs(X[0][j]) + std::fabs(X[1][j])) + std::fabs(X[2][j]));
        const float s2 = static_cast<float>((std::fabs(inv[0][j]) + std::fabs(inv[1][j])) + std::fabs(inv[2][j]));
        c = s1 > c ? s1 : c;
        ci = s2 > ci ? s2 : ci;
      }
      for (int i = 0; i < 3; ++i) {
        const float s1 = static_cast<float>((std::fabs(X[i][0]) + std::fabs(X[i][1])) + std::fabs(X[i][2]));
        const float s2 = static_cast<float>((std::fabs(inv[i][0]) + std::fabs(inv[i][1])) + std::fabs(inv[i][2]));
        r = s1 > r ? s1 : r;
        ri = s2 > ri ? s2 : ri;
      }
      const float xn = c * r, in = ci * ri;
      if (xn > 0.0f && in > 0.0f && std::isfinite(in / xn)) {
        const float gf = std::sqrt(std::sqrt(in / xn));
        g = static_cast<T>(gf);
        ig = static_cast<T>(1.0f / gf);
      }
    }
    T dd[9], ff[9];
    for (int i = 0; i < 3; ++i)
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

// Returns false when degenerate. On success fills R (rotation matrix from the
// normalised quaternion) and q. Two stages (pinned): a scaled Newton loop in
// fp32 on A normalised by ||A||_F/sqrt3, then unscaled fp64 Newton steps to
// the 1e-9 tolerance (one step, since the fp32 stage leaves ~1e-7); if the fp32
// stage breaks down, the fp64 loop runs from A with scaling.
inline bool polar_rotation(const M3& A, M3& R, double q[4]) {
  if (!finite3(A)) return false;
  const double d0 = det3(A);
  const double c3 = frob2(A) * PBDR_ONE_THIRD;
  if (!(d0 > 0.0) || d0 * d0 <= (PBDR_POLAR_REL_DET * PBDR_POLAR_REL_DET) * ((c3 * c3) * c3)) return false;
  const double is = 1.0 / std::sqrt(c3);
  float Xf[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) Xf[i][j] = static_cast<float>(A.a[i][j] * is);
  double X[3][3];
  const int f_it = newton_polar<float>(Xf, PBDR_POLAR_F32_TOL2, PBDR_POLAR_F32_TOLQ,
                                       static_cast<float>(PBDR_POLAR_SCALE_REL2), PBDR_POLAR_F32_MAX_IT, true);
  M3 Xm;
  if (f_it > 0) {
    // fp64 polish: one unscaled Newton step re-orthonormalises the fp32
    // iterate (R0), then one first-order rotation correction solves the
    // symmetry condition of B = R0^T A: axial(B - B^T) = (tr(S) I - S) w,
    // S = sym(B), and R = R0 (I + [w]x) (error O(|w|^2) ~ 1e-14).
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) X[i][j] = static_cast<double>(Xf[i][j]);
    if (newton_polar<double>(X, 0.0, 0.0, 0.0, 1, false) < 0) return false;
    double B[3][3];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j)
        B[i][j] = (X[0][i] * A.a[0][j] + X[1][i] * A.a[1][j]) + X[2][i] * A.a[2][j];
    const double sv[3] = {B[2][1] - B[1][2], B[0][2] - B[2][0], B[1][0] - B[0][1]};
    double M[3][3];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) M[i][j] = -(0.5 * (B[i][j] + B[j][i]));
    const double tr = (-M[0][0] + -M[1][1]) + -M[2][2];
    M[0][0] = tr + M[0][0];
    M[1][1] = tr + M[1][1];
    M[2][2] = tr + M[2][2];
    const double dm = M[0][0] * (M[1][1] * M[2][2] - M[1][2] * M[2][1]) -
                      M[0][1] * (M[1][0] * M[2][2] - M[1][2] * M[2][0]) +
                      M[0][2] * (M[1][0] * M[2][1] - M[1][1] * M[2][0]);
    double w[3] = {0.0, 0.0, 0.0};
    if (dm != 0.0 && std::isfinite(dm)) {
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
    for (int i = 0; i < 3; ++i) {
      Xm.a[i][0] = X[i][0] + (X[i][1] * w[2] - X[i][2] * w[1]);
      Xm.a[i][1] = X[i][1] + (X[i][2] * w[0] - X[i][0] * w[2]);
      Xm.a[i][2] = X[i][2] + (X[i][0] * w[1] - X[i][1] * w[0]);
    }
  } else {
    // fp32 stage broke down: full scaled fp64 Newton from A.
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) X[i][j] = A.a[i][j];
    if (newton_polar<double>(X, PBDR_POLAR_TOL2, PBDR_POLAR_TOLQ, PBDR_POLAR_SCALE_REL2, PBDR_POLAR_MAX_IT, true) < 0)
      return false;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) Xm.a[i][j] = X[i][j];
  }
  quat_from(Xm, q);
  R = quat_to(q);
  return true;
}

// Warm-started rotation extraction (pinned): starting from the body's rotation
// of the previous solver iteration (quaternion rq, all-zero = none), apply
// Gauss-Newton corrections of the polar factor's symmetry condition -- with
// B = R^T A and S = sym(B): axial(B - B^T) = (tr(S) I - S) w, then
// q <- normalise(q (x) (1, w/2)) -- until |w|^2 <= 1e-12 (the step then leaves
// an O(|w|^2) error). Converges quadratically from any nearby R whatever the
// conditioning of S. A missing warm start, |w|^2 > 0.25 (not local), a
// singular solve, or 4 steps without convergence fall back to the cold
// two-stage Newton polar. The result is the same polar factor to 1e-12.
// PBDR_POLAR_WARM_F32 (pbdr_pinned.h): the same iteration in fp32 on the
// fp32 body sum A (exactly representable: A holds float values).
inline bool polar_warm_f32(const M3& A, const float rq[4], M3& R, double q[4], bool bad) {
  float Af[9];
  for (int i = 0; i < 9; ++i) Af[i] = static_cast<float>(A.a[i / 3][i % 3]);
  float qc[4] = {rq[0], rq[1], rq[2], rq[3]};
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
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) B[i][j] = (R0[0][i] * Af[j] + R0[1][i] * Af[3 + j]) + R0[2][i] * Af[6 + j];
    const float sv[3] = {B[2][1] - B[1][2], B[0][2] - B[2][0], B[1][0] - B[0][1]};
    float M[3][3];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) M[i][j] = -(0.5f * (B[i][j] + B[j][i]));
    const float tr = (-M[0][0] + -M[1][1]) + -M[2][2];
    M[0][0] = tr + M[0][0];
    M[1][1] = tr + M[1][1];
    M[2][2] = tr + M[2][2];
    const float dm = M[0][0] * (M[1][1] * M[2][2] - M[1][2] * M[2][1]) -
                     M[0][1] * (M[1][0] * M[2][2] - M[1][2] * M[2][0]) +
                     M[0][2] * (M[1][0] * M[2][1] - M[1][1] * M[2][0]);
    if (!(dm > 0.0f) || !std::isfinite(dm)) break;
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
      if (bad) return false;
      const float n2 = ((qn[0] * qn[0] + qn[1] * qn[1]) + qn[2] * qn[2]) + qn[3] * qn[3];
      const float r = 1.0f / n2;
      const float s = 1.5f - 0.5f * n2;
      const float a = qn[0], b = qn[1], c = qn[2], d = qn[3];
      const float a2 = a * a, bb = b * b, cc = c * c, dd = d * d;
      const float bc = b * c, bd = b * d, cd = c * d, ab = a * b, ac = a * c, ad = a * d;
      const float Rf[9] = {((a2 + bb) - (cc + dd)) * r, (2.0f * (bc - ad)) * r, (2.0f * (bd + ac)) * r,
                           (2.0f * (bc + ad)) * r, ((a2 + cc) - (bb + dd)) * r, (2.0f * (cd - ab)) * r,
                           (2.0f * (bd - ac)) * r, (2.0f * (cd + ab)) * r, ((a2 + dd) - (bb + cc)) * r};
      for (int i = 0; i < 9; ++i) R.a[i / 3][i % 3] = static_cast<double>(Rf[i]);
      for (int k = 0; k < 4; ++k) q[k] = static_cast<double>(qn[k] * s);
      return true;
    }
    for (int k = 0; k < 4; ++k) qc[k] = qn[k];
  }
  if (bad) return false;
  return polar_rotation(A, R, q);
}

inline bool polar_warm(const M3& A, const float rq[4], M3& R, double q[4]) {
  const double d0 = det3(A);
  const double c3 = frob2(A) * PBDR_ONE_THIRD;
  const bool bad =
      !finite3(A) || !(d0 > 0.0) || d0 * d0 <= (PBDR_POLAR_REL_DET * PBDR_POLAR_REL_DET) * ((c3 * c3) * c3);
#if PBDR_POLAR_WARM_F32
  if (rq[0] != 0.0f || rq[1] != 0.0f || rq[2] != 0.0f || rq[3] != 0.0f) return polar_warm_f32(A, rq, R, q, bad);
#endif
  if (rq[0] != 0.0f || rq[1] != 0.0f || rq[2] != 0.0f || rq[3] != 0.0f) {
    // Homogeneous iterate: qc is not renormalised between steps; R0 below is
    // |qc|^2 R(qc), and the step h is invariant under that uniform scale.
    double qc[4] = {rq[0], rq[1], rq[2], rq[3]};
    for (int step = 0; step < PBDR_POLAR_WARM_STEPS; ++step) {
      const M3 R0 = quat_to_h(qc);
      double B[3][3];
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
          B[i][j] = (R0.a[0][i] * A.a[0][j] + R0.a[1][i] * A.a[1][j]) + R0.a[2][i] * A.a[2][j];
      const double sv[3] = {B[2][1] - B[1][2], B[0][2] - B[2][0], B[1][0] - B[0][1]};
      double M[3][3];
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) M[i][j] = -(0.5 * (B[i][j] + B[j][i]));
      const double tr = (-M[0][0] + -M[1][1]) + -M[2][2];
      M[0][0] = tr + M[0][0];
      M[1][1] = tr + M[1][1];
      M[2][2] = tr + M[2][2];
      const double dm = M[0][0] * (M[1][1] * M[2][2] - M[1][2] * M[2][1]) -
                        M[0][1] * (M[1][0] * M[2][2] - M[1][2] * M[2][0]) +
                        M[0][2] * (M[1][0] * M[2][1] - M[1][1] * M[2][0]);
      if (!(dm > 0.0) || !std::isfinite(dm)) break;
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
        if (bad) return false;
        const double n2 = ((qn[0] * qn[0] + qn[1] * qn[1]) + qn[2] * qn[2]) + qn[3] * qn[3];
        const double r = 1.0 / n2;
        const double s = 1.5 - 0.5 * n2;
        R = quat_to_h(qn);
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) R.a[i][j] = R.a[i][j] * r;
        for (int k = 0; k < 4; ++k) q[k] = qn[k] * s;
        return true;
      }
      for (int k = 0; k < 4; ++k) qc[k] = qn[k];
    }
  }
  if (bad) return false;
  return polar_rotation(A, R, q);
}

// Cyclic Jacobi on the symmetrised matrix; ascending eigenvalues, eigenvector
// columns in V.
inline void sym_eigen(const M3& m, double ev[3], M3& V) {
  double A[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) A[i][j] = 0.5 * (m.a[i][j] + m.a[j][i]);
  double U[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  for (int sweep = 0; sweep < 32; ++sweep) {
    const double off = (std::fabs(A[0][1]) + std::fabs(A[0][2])) + std::fabs(A[1][2]);
    const double scale = (std::fabs(A[0][0]) + std::fabs(A[1][1])) + std::fabs(A[2][2]);
    if (off <= 1e-15 * (scale > 1e-300 ? scale : 1e-300)) break;
    for (int p = 0; p < 2; ++p)
      for (int qq = p + 1; qq < 3; ++qq) {
        if (A[p][qq] == 0.0) continue;
        const double theta = (A[qq][qq] - A[p][p]) / (2.0 * A[p][qq]);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) /
                         (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0);
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
  // Stable insertion sort, ascending.
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

// omega = pinv(I) * dL with the reference's rank cut. Returns 0, or
// PBDR_DEVERR_RANK_DEFICIENT (omega = 0, null axis filled).
inline unsigned inertia_solve(const M3& I, const double dL[3], double w[3], double null_axis[3]) {
  const double tr = (I.a[0][0] + I.a[1][1]) + I.a[2][2];
  const double d = det3(I);
  w[0] = w[1] = w[2] = 0.0;
  if (tr > 0.0 && d >= PBDR_PINV_FAST_DET * ((tr * tr) * tr)) {
    const M3 inv = adj_inverse(I, d);
    for (int r = 0; r < 3; ++r)
      w[r] = (inv.a[r][0] * dL[0] + inv.a[r][1] * dL[1]) + inv.a[r][2] * dL[2];
    return 0u;
  }
  double ev[3];
  M3 V;
  sym_eigen(I, ev, V);
  const double atr = std::fabs(tr);
  const double cut = PBDR_PINV_REL_TOL * (atr > 1e-300 ? atr : 1e-300);
  M3 P = {{{0, 0, 0}, {0, 0, 0}, {0, 0, 0}}};
  int rank = 0;
  double nax[3] = {0, 0, 0};
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
    const double along = std::fabs((dL[0] * nax[0] + dL[1] * nax[1]) + dL[2] * nax[2]);
    if (along > PBDR_NULL_AXIS_TOL) {
      null_axis[0] = nax[0]; null_axis[1] = nax[1]; null_axis[2] = nax[2];
      return PBDR_DEVERR_RANK_DEFICIENT;
    }
  }
  for (int r = 0; r < 3; ++r) w[r] = (P.a[r][0] * dL[0] + P.a[r][1] * dL[1]) + P.a[r][2] * dL[2];
  return 0u;
}

}  // namespace orc
