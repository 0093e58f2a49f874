// ============================================================================
// TEST INFRASTRUCTURE ONLY -- the independent fp64 oracle of the PBD-R step.
//
// A second CPU restatement of the substep loop, written to share nothing with
// the CUDA path but the semantic decisions (P1-P6): no fp32, no
// anchored sums, no warp-tree reduction order, no warm-started polar, no
// header of the product. It follows the reference's own numerics:
//   * every per-body quantity is a plain fp64 sum in particle order, as
//     compute_com / compute_inertia / compute_momentum (body.cpp:50-83);
//   * shape matching's rotation is the reference's scaled-Newton
//     polar_decompose (math.cpp:170-210: 1-inf norm scaling, tolerance 1e-9,
//     at most 64 iterations), from a cold start every iteration;
//   * the inertia solve is pseudo_invert_spd (math.cpp:90-108, cyclic Jacobi
//     math.cpp:26-71) with the null-axis rule of SPEC.md:321;
//   * enforce_momentum re-measures L after the linear fix literally
//      instead of using L_asm;
//   * integrate, contacts, friction and the velocity update follow
//     PAPER.md:136-172 / SPEC.md:272-316 in fp64.
// Pinned choices kept (they are semantics, not numerics): Jacobi across
// constraints (P1), the bsm capture point (P2), the candidate rule on the
// predicted positions with cell h = 2 r_max (P4, here in fp64), friction on
// x - x_init (P5), and the scale-relative polar degeneracy test (the
// reference's absolute 1e-12 rejects config 3's small bodies).
//
// The GPU (fp32 state) is compared with this oracle at the north_star
// tolerances (tests/test_gpu_fp64_oracle.py), so an error the GPU and the
// bit-exact fp32 oracle (pbdr_oracle.cpp) shared would show up here.
// ============================================================================
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <tuple>
#include <vector>

#include "pbdr_gpu.h"

namespace {

// Error bits of this oracle's record (o64_error); the status codes returned
// are the C-ABI's (errors.hpp classes).
enum : unsigned { kNonFinite = 1u, kDegenerate = 2u, kOverflow = 4u, kRankDeficient = 8u };

struct V3 {
  double x = 0, y = 0, z = 0;
};
inline V3 operator+(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 operator-(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 operator*(V3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
inline double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline V3 cross(V3 a, V3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }

struct M {
  double a[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
};
inline V3 mul(const M& m, V3 v) {
  return {m.a[0][0] * v.x + m.a[0][1] * v.y + m.a[0][2] * v.z, m.a[1][0] * v.x + m.a[1][1] * v.y + m.a[1][2] * v.z,
          m.a[2][0] * v.x + m.a[2][1] * v.y + m.a[2][2] * v.z};
}
inline double det(const M& m) {
  return m.a[0][0] * (m.a[1][1] * m.a[2][2] - m.a[1][2] * m.a[2][1]) -
         m.a[0][1] * (m.a[1][0] * m.a[2][2] - m.a[1][2] * m.a[2][0]) +
         m.a[0][2] * (m.a[1][0] * m.a[2][1] - m.a[1][1] * m.a[2][0]);
}
inline double frob(const M& m) {
  double s = 0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) s += m.a[i][j] * m.a[i][j];
  return std::sqrt(s);
}

bool invert(const M& m, M& out) {
  const double d = det(m);
  if (!(std::fabs(d) > 1e-300)) return false;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      // cofactor C_ji / det (adjugate = transposed cofactors)
      const int r0 = (j + 1) % 3, r1 = (j + 2) % 3, c0 = (i + 1) % 3, c1 = (i + 2) % 3;
      out.a[i][j] = (m.a[r0][c0] * m.a[r1][c1] - m.a[r0][c1] * m.a[r1][c0]) / d;
    }
  return true;
}

double norm_1(const M& m) {  // max column sum
  double b = 0;
  for (int j = 0; j < 3; ++j) b = std::max(b, std::fabs(m.a[0][j]) + std::fabs(m.a[1][j]) + std::fabs(m.a[2][j]));
  return b;
}
double norm_inf(const M& m) {  // max row sum
  double b = 0;
  for (int i = 0; i < 3; ++i) b = std::max(b, std::fabs(m.a[i][0]) + std::fabs(m.a[i][1]) + std::fabs(m.a[i][2]));
  return b;
}

// Orthogonal polar factor by scaled Newton (math.cpp:170-210 semantics);
// false when degenerate (scale-relative determinant test) or singular.
bool polar_R(const M& A, M& R) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      if (!std::isfinite(A.a[i][j])) return false;
  const double s = frob(A) / std::sqrt(3.0);
  if (!(det(A) > 1e-12 * s * s * s)) return false;
  M X = A;
  for (int it = 0; it < 64; ++it) {
    M Xi;
    if (!invert(X, Xi)) return false;
    M XiT;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) XiT.a[i][j] = Xi.a[j][i];
    const double xn = norm_1(X) * norm_inf(X), in = norm_1(XiT) * norm_inf(XiT);
    const double g = (xn > 0 && in > 0) ? std::pow(in / xn, 0.25) : 1.0;
    M N;
    double d2 = 0;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        N.a[i][j] = 0.5 * (g * X.a[i][j] + XiT.a[i][j] / g);
        d2 += (N.a[i][j] - X.a[i][j]) * (N.a[i][j] - X.a[i][j]);
      }
    X = N;
    if (std::sqrt(d2) <= 1e-9 * std::max(frob(X), 1e-300)) break;
  }
  R = X;
  return true;
}

void jacobi_eigen(const M& m, double ev[3], M& V) {
  M A;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) A.a[i][j] = 0.5 * (m.a[i][j] + m.a[j][i]);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) V.a[i][j] = i == j ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 32; ++sweep) {
    const double off = std::fabs(A.a[0][1]) + std::fabs(A.a[0][2]) + std::fabs(A.a[1][2]);
    const double dg = std::fabs(A.a[0][0]) + std::fabs(A.a[1][1]) + std::fabs(A.a[2][2]);
    if (off <= 1e-15 * std::max(dg, 1e-300)) break;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        if (A.a[p][q] == 0.0) continue;
        const double th = (A.a[q][q] - A.a[p][p]) / (2.0 * A.a[p][q]);
        const double t = (th >= 0 ? 1.0 : -1.0) / (std::fabs(th) + std::sqrt(th * th + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        // A <- J^T A J with J = rotation in the (p, q) plane.
        for (int k = 0; k < 3; ++k) {
          const double akp = A.a[k][p], akq = A.a[k][q];
          A.a[k][p] = c * akp - s * akq;
          A.a[k][q] = s * akp + c * akq;
        }
        for (int k = 0; k < 3; ++k) {
          const double apk = A.a[p][k], aqk = A.a[q][k];
          A.a[p][k] = c * apk - s * aqk;
          A.a[q][k] = s * apk + c * aqk;
        }
        for (int k = 0; k < 3; ++k) {
          const double vkp = V.a[k][p], vkq = V.a[k][q];
          V.a[k][p] = c * vkp - s * vkq;
          V.a[k][q] = s * vkp + c * vkq;
        }
      }
  }
  int o[3] = {0, 1, 2};
  std::sort(o, o + 3, [&](int i, int j) { return A.a[i][i] < A.a[j][j]; });
  M W;
  for (int k = 0; k < 3; ++k) {
    ev[k] = A.a[o[k]][o[k]];
    for (int r = 0; r < 3; ++r) W.a[r][k] = V.a[r][o[k]];
  }
  V = W;
}

// omega = pinv(I) dL; a dL component above 1e-12 along a dropped (null) axis
// is RankDeficientError, below it is projected out.
bool pinv_solve(const M& I, V3 dL, V3& w, V3& null_axis) {
  double ev[3];
  M V;
  jacobi_eigen(I, ev, V);
  const double tr = std::fabs(I.a[0][0] + I.a[1][1] + I.a[2][2]);
  w = {0, 0, 0};
  bool ok = true;
  for (int k = 0; k < 3; ++k) {
    const V3 u{V.a[0][k], V.a[1][k], V.a[2][k]};
    const double proj = dot(u, dL);
    if (ev[k] >= 1e-10 * std::max(tr, 1e-300)) {
      w = w + u * (proj / ev[k]);
    } else if (std::fabs(proj) > 1e-12) {
      ok = false;
      null_axis = u;
    }
  }
  return ok;
}

struct Plane {
  V3 p, n;
  double mu;
};

struct O64 {
  int64_t n = 0;
  int32_t nb = 0;
  std::vector<V3> x, v, xinit;
  std::vector<double> w, m, r;
  std::vector<int32_t> body, scene;  // per particle
  std::vector<int64_t> boff;         // CSR
  std::vector<int32_t> bidx;
  std::vector<V3> q0;                // per CSR entry
  std::vector<double> M;             // per body
  std::vector<pbdr_force_program> prog;
  bool has_prog = false;
  std::vector<Plane> planes;
  double dt = 0, g = 0, relax = 1, h = 0;
  int iters = 10;
  bool incremental = true, linfix = true, angfix = true, per_substep = false;
  int64_t substep = 0;
  std::vector<std::vector<int64_t>> cand;
  unsigned err = 0;
  int32_t err_body = -1;
  V3 err_axis;
  int threads = 1;
};

void flag(O64& s, unsigned bits, int32_t b, const V3* axis = nullptr) {
#pragma omp critical(o64_err)
  {
    s.err |= bits;
    if (s.err_body < 0 || b < s.err_body) {
      s.err_body = b;
      if (axis) s.err_axis = *axis;
    }
  }
}

V3 body_com(const O64& s, int32_t b, const std::vector<V3>& X) {
  V3 c;
  double Mb = 0;
  for (int64_t k = s.boff[b]; k < s.boff[b + 1]; ++k) {
    const int64_t i = s.bidx[k];
    c = c + X[i] * s.m[i];
    Mb += s.m[i];
  }
  return c * (1.0 / Mb);
}

M body_inertia(const O64& s, int32_t b, const std::vector<V3>& X, V3 c) {
  M I;
  for (int64_t k = s.boff[b]; k < s.boff[b + 1]; ++k) {
    const int64_t i = s.bidx[k];
    const V3 r = X[i] - c;
    const double rr[3] = {r.x, r.y, r.z}, r2 = dot(r, r);
    for (int a = 0; a < 3; ++a)
      for (int bb = 0; bb < 3; ++bb) I.a[a][bb] += s.m[i] * ((a == bb ? r2 : 0.0) - rr[a] * rr[bb]);
  }
  return I;
}

void integrate(O64& s) {
  const double t = static_cast<double>(s.substep) * s.dt;
  std::vector<V3> alpha(static_cast<size_t>(s.nb)), com(static_cast<size_t>(s.nb));
  std::vector<char> on(static_cast<size_t>(s.nb), 0), torque(static_cast<size_t>(s.nb), 0);
  for (int32_t b = 0; b < s.nb; ++b) {
    if (!s.has_prog) break;
    const pbdr_force_program& p = s.prog[b];
    on[b] = t >= p.t_start && t < p.t_stop;
    const V3 tau{p.torque[0], p.torque[1], p.torque[2]};
    if (on[b] && dot(tau, tau) > 0) {  // distribute_wrench (body.cpp:126-150)
      torque[b] = 1;
      com[b] = body_com(s, b, s.x);
      V3 ax;
      if (!pinv_solve(body_inertia(s, b, s.x, com[b]), tau, alpha[b], ax))
        flag(s, kRankDeficient, b, &ax);
    }
  }
  for (int64_t i = 0; i < s.n; ++i) {
    const int32_t b = s.body[i];
    V3 a{0, 0, (s.has_prog && s.prog[b].gravity_exempt) ? 0.0 : -s.g};
    if (s.has_prog && on[b]) {
      a = a + V3{s.prog[b].force[0], s.prog[b].force[1], s.prog[b].force[2]} * (1.0 / s.M[b]);
      if (torque[b]) a = a + cross(alpha[b], s.x[i] - com[b]);
    }
    s.xinit[i] = s.x[i];
    s.v[i] = s.v[i] + a * s.dt;
    s.x[i] = s.x[i] + s.v[i] * s.dt;
  }
}

void candidates(O64& s) {
  using Key = std::tuple<int32_t, int64_t, int64_t, int64_t>;
  auto cell = [&](double c) { return static_cast<int64_t>(std::floor(c / s.h)); };
  std::vector<std::pair<Key, int64_t>> keys(static_cast<size_t>(s.n));
  for (int64_t i = 0; i < s.n; ++i)
    keys[i] = {Key{s.scene[i], cell(s.x[i].x), cell(s.x[i].y), cell(s.x[i].z)}, i};
  std::sort(keys.begin(), keys.end());
  s.cand.assign(static_cast<size_t>(s.n), {});
#pragma omp parallel for num_threads(s.threads) schedule(dynamic, 1024)
  for (int64_t i = 0; i < s.n; ++i) {
    const int64_t cx = cell(s.x[i].x), cy = cell(s.x[i].y), cz = cell(s.x[i].z);
    std::vector<int64_t>& out = s.cand[i];
    for (int dx = -1; dx <= 1; ++dx)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dz = -1; dz <= 1; ++dz) {
          const Key k{s.scene[i], cx + dx, cy + dy, cz + dz};
          auto it = std::lower_bound(keys.begin(), keys.end(), std::make_pair(k, int64_t(-1)));
          for (; it != keys.end() && it->first == k; ++it) {
            const int64_t j = it->second;
            if (s.body[j] == s.body[i]) continue;
            const V3 e = s.x[i] - s.x[j];
            if (dot(e, e) < s.h * s.h) out.push_back(j);
          }
        }
    std::sort(out.begin(), out.end());
    if (out.size() > 32) flag(s, kOverflow, s.body[i]);
  }
}

void iteration(O64& s, int it, std::vector<V3>& accP, std::vector<V3>& accL) {
  const std::vector<V3> X = s.x;  // X_i snapshot (P1)
  const std::vector<V3> Vi = s.v;
  const double idt = 1.0 / s.dt;
#pragma omp parallel for num_threads(s.threads) schedule(dynamic, 4)
  for (int32_t b = 0; b < s.nb; ++b) {
    const int64_t k0 = s.boff[b], k1 = s.boff[b + 1];
    const int64_t nk = k1 - k0;
    const double Mb = s.M[b];
    std::vector<V3> dC(static_cast<size_t>(nk));
    for (int64_t k = k0; k < k1; ++k) {
      const int64_t i = s.bidx[k];
      V3 d;
      for (const Plane& P : s.planes) {  // ground / walls with friction (P5)
        const double dist = dot(X[i] - P.p, P.n) - s.r[i];
        if (!(dist < 0)) continue;
        d = d + P.n * (-s.relax * dist);
        if (!(P.mu > 0)) continue;
        const V3 t = X[i] - s.xinit[i];
        const V3 tt = t - P.n * dot(t, P.n);
        const double len = std::sqrt(dot(tt, tt));
        if (!(len > 0)) continue;
        const double lim = P.mu * (-dist);
        d = d - (len <= lim ? tt : tt * (lim / len));
      }
      for (const int64_t j : s.cand[i]) {  // particle-particle
        const V3 e = X[i] - X[j];
        const double rr = s.r[i] + s.r[j];
        const double d2 = dot(e, e);
        if (!(d2 < rr * rr)) continue;
        const double dist = std::sqrt(d2);
        const V3 nrm = dist > 1e-9 ? e * (1.0 / dist) : V3{i < j ? 1.0 : -1.0, 0, 0};
        d = d - nrm * (s.relax * (s.w[i] / (s.w[i] + s.w[j])) * (dist - rr));
      }
      dC[k - k0] = d;
    }
    // Shape matching on X_i (com c, Apq = sum m (x - c) q0^T) and the bsm momenta.
    V3 c, cb;
    for (int64_t k = k0; k < k1; ++k) {
      const int64_t i = s.bidx[k];
      c = c + X[i] * s.m[i];
      cb = cb + (X[i] + dC[k - k0]) * s.m[i];
    }
    c = c * (1.0 / Mb);
    cb = cb * (1.0 / Mb);
    M A;
    V3 Pb, Lb;
    for (int64_t k = k0; k < k1; ++k) {
      const int64_t i = s.bidx[k];
      const V3 p = X[i] - c, q = s.q0[k];
      const double pv[3] = {p.x, p.y, p.z}, qv[3] = {q.x, q.y, q.z};
      for (int a = 0; a < 3; ++a)
        for (int bb = 0; bb < 3; ++bb) A.a[a][bb] += s.m[i] * pv[a] * qv[bb];
      const V3 vb = Vi[i] + dC[k - k0] * idt;
      Pb = Pb + vb * s.m[i];
      Lb = Lb + cross(X[i] + dC[k - k0] - cb, vb * s.m[i]);
    }
    M R;
    const bool sm = polar_R(A, R);
    if (!sm) flag(s, kDegenerate, b);
    std::vector<V3> xa(static_cast<size_t>(nk)), va(static_cast<size_t>(nk));
    for (int64_t k = k0; k < k1; ++k) {
      const int64_t i = s.bidx[k];
      const V3 dsm = sm ? (mul(R, s.q0[k]) + c) - X[i] : V3{};
      const V3 dX = dC[k - k0] + dsm;
      xa[k - k0] = X[i] + dX;
      va[k - k0] = s.incremental ? Vi[i] + dX * idt : (xa[k - k0] - s.xinit[i]) * idt;
    }
    // enforce_momentum: linear, then L re-measured, angular.
    V3 ca, Pa;
    for (int64_t k = k0; k < k1; ++k) {
      const int64_t i = s.bidx[k];
      ca = ca + xa[k - k0] * s.m[i];
      Pa = Pa + va[k - k0] * s.m[i];
    }
    ca = ca * (1.0 / Mb);
    V3 dP = Pb - Pa;
    bool correct = true;
    if (s.per_substep) {
      if (it == 0) accP[b] = accL[b] = V3{};
      accP[b] = accP[b] + dP;
      dP = accP[b];
      correct = it == s.iters - 1;
    }
    if (s.linfix && correct) {
      const V3 dv = dP * (1.0 / Mb);
      for (int64_t k = 0; k < nk; ++k) {
        va[k] = va[k] + dv;
        xa[k] = xa[k] + dv * s.dt;
      }
    }
    V3 c2, La;
    for (int64_t k = k0; k < k1; ++k) c2 = c2 + xa[k - k0] * s.m[s.bidx[k]];
    c2 = c2 * (1.0 / Mb);
    for (int64_t k = k0; k < k1; ++k) {
      const int64_t i = s.bidx[k];
      La = La + cross(xa[k - k0] - c2, va[k - k0] * s.m[i]);
    }
    V3 dL = La - Lb;
    if (s.per_substep) {
      accL[b] = accL[b] + dL;
      dL = accL[b];
    }
    if (s.angfix && correct) {
      M I;
      for (int64_t k = k0; k < k1; ++k) {
        const V3 r = xa[k - k0] - c2;
        const double rr[3] = {r.x, r.y, r.z}, r2 = dot(r, r), mk = s.m[s.bidx[k]];
        for (int a = 0; a < 3; ++a)
          for (int bb = 0; bb < 3; ++bb) I.a[a][bb] += mk * ((a == bb ? r2 : 0.0) - rr[a] * rr[bb]);
      }
      V3 om, ax;
      if (!pinv_solve(I, dL, om, ax)) flag(s, kRankDeficient, b, &ax);
      for (int64_t k = 0; k < nk; ++k) {
        const V3 wr = cross(om, xa[k] - c2);
        va[k] = va[k] - wr;
        xa[k] = xa[k] - wr * s.dt;
      }
    }
    for (int64_t k = k0; k < k1; ++k) {
      const int64_t i = s.bidx[k];
      s.x[i] = xa[k - k0];
      s.v[i] = va[k - k0];
    }
  }
}

}  // namespace

extern "C" {

int o64_create(const pbdr_scene_desc* d, const pbdr_solver_cfg* c, int threads, void** out) {
  *out = nullptr;
  if (!d || !c || d->num_particles <= 0 || d->num_bodies <= 0) return PBDR_ERR_CONFIG;
  O64* s = new O64();
  s->threads = threads > 0 ? threads : 1;
  s->n = d->num_particles;
  s->nb = d->num_bodies;
  const int64_t n = s->n;
  s->x.resize(n);
  s->v.resize(n);
  s->xinit.resize(n);
  s->w.resize(n);
  s->m.resize(n);
  s->r.resize(n);
  s->body.resize(n);
  s->scene.resize(n);
  double rmax = 0;
  for (int64_t i = 0; i < n; ++i) {
    s->x[i] = {d->position[3 * i], d->position[3 * i + 1], d->position[3 * i + 2]};
    s->v[i] = {d->velocity[3 * i], d->velocity[3 * i + 1], d->velocity[3 * i + 2]};
    s->w[i] = d->inv_mass[i];
    s->m[i] = 1.0 / d->inv_mass[i];
    s->r[i] = d->radius[i];
    rmax = std::max(rmax, s->r[i]);
  }
  s->boff.assign(d->body_offsets, d->body_offsets + s->nb + 1);
  s->bidx.assign(d->body_indices, d->body_indices + s->boff.back());
  s->q0.resize(s->bidx.size());
  for (size_t k = 0; k < s->bidx.size(); ++k)
    s->q0[k] = {d->rest_offsets[3 * k], d->rest_offsets[3 * k + 1], d->rest_offsets[3 * k + 2]};
  s->M.resize(s->nb);
  for (int32_t b = 0; b < s->nb; ++b) {
    double Mb = 0;
    for (int64_t k = s->boff[b]; k < s->boff[b + 1]; ++k) {
      s->body[s->bidx[k]] = b;
      s->scene[s->bidx[k]] = d->body_scene ? d->body_scene[b] : 0;
      Mb += s->m[s->bidx[k]];
    }
    s->M[b] = Mb;  // plain sum of the member masses (body.cpp:16-48 make_body)
  }
  if (d->programs) {
    s->has_prog = true;
    s->prog.assign(d->programs, d->programs + s->nb);
  }
  auto plane = [](const pbdr_plane& p) {
    return Plane{{p.point[0], p.point[1], p.point[2]}, {p.normal[0], p.normal[1], p.normal[2]}, p.friction};
  };
  if (d->has_ground) s->planes.push_back(plane(d->ground));
  for (int k = 0; k < d->num_walls; ++k) s->planes.push_back(plane(d->walls[k]));
  s->dt = 1.0 / (c->frame_rate * c->substeps);
  s->g = c->gravity;
  s->relax = d->contact_relaxation;
  s->h = 2.0 * rmax;
  s->iters = c->solver_iterations;
  s->incremental = c->velocity_update == PBDR_VELOCITY_INCREMENTAL;
  s->linfix = c->linear_momentum_fix != 0;
  s->angfix = c->angular_momentum_fix != 0;
  s->per_substep = c->momentum_frequency == PBDR_MOMENTUM_PER_SUBSTEP;
  *out = s;
  return PBDR_OK;
}

void o64_destroy(void* h) { delete static_cast<O64*>(h); }

// Advances `substeps` substeps; returns a pbdr_status (errors as the device).
int o64_step(void* h, int64_t substeps) {
  O64& s = *static_cast<O64*>(h);
  std::vector<V3> accP(static_cast<size_t>(s.nb)), accL(static_cast<size_t>(s.nb));
  for (int64_t k = 0; k < substeps; ++k) {
    integrate(s);
    candidates(s);
    for (int it = 0; it < s.iters; ++it) iteration(s, it, accP, accL);
    ++s.substep;
    if (s.err & (kNonFinite | kOverflow)) return PBDR_ERR_SIMULATION;
    if (s.err & kRankDeficient) return PBDR_ERR_RANK_DEFICIENT;
    if (s.err & kDegenerate) return PBDR_ERR_DEGENERATE;
  }
  return PBDR_OK;
}

// Caller-order fp64 state (3 doubles per particle); either may be null.
void o64_read(void* h, double* pos, double* vel) {
  const O64& s = *static_cast<O64*>(h);
  for (int64_t i = 0; i < s.n; ++i) {
    if (pos) { pos[3 * i] = s.x[i].x; pos[3 * i + 1] = s.x[i].y; pos[3 * i + 2] = s.x[i].z; }
    if (vel) { vel[3 * i] = s.v[i].x; vel[3 * i + 1] = s.v[i].y; vel[3 * i + 2] = s.v[i].z; }
  }
}

void o64_write(void* h, const double* pos, const double* vel) {
  O64& s = *static_cast<O64*>(h);
  for (int64_t i = 0; i < s.n; ++i) {
    if (pos) s.x[i] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
    if (vel) s.v[i] = {vel[3 * i], vel[3 * i + 1], vel[3 * i + 2]};
  }
}

// Per body: com[3], quat[4] (extract_pose: polar of sum m (x - com) q0^T),
// P[3], L[3] about the com (compute_momentum) -- the pbdr_body_stats layout.
void o64_body_stats(void* h, double* out) {
  const O64& s = *static_cast<O64*>(h);
  for (int32_t b = 0; b < s.nb; ++b) {
    const V3 c = body_com(s, b, s.x);
    M A;
    V3 P, L;
    for (int64_t k = s.boff[b]; k < s.boff[b + 1]; ++k) {
      const int64_t i = s.bidx[k];
      const V3 p = s.x[i] - c, q = s.q0[k];
      const double pv[3] = {p.x, p.y, p.z}, qv[3] = {q.x, q.y, q.z};
      for (int a = 0; a < 3; ++a)
        for (int bb = 0; bb < 3; ++bb) A.a[a][bb] += s.m[i] * pv[a] * qv[bb];
      P = P + s.v[i] * s.m[i];
      L = L + cross(p, s.v[i] * s.m[i]);
    }
    M R;
    double q[4] = {1, 0, 0, 0};
    if (polar_R(A, R)) {  // quaternion of R (largest-pivot branch)
      const double tr = R.a[0][0] + R.a[1][1] + R.a[2][2];
      if (tr > 0) {
        const double t = 2 * std::sqrt(1 + tr);
        q[0] = 0.25 * t; q[1] = (R.a[2][1] - R.a[1][2]) / t;
        q[2] = (R.a[0][2] - R.a[2][0]) / t; q[3] = (R.a[1][0] - R.a[0][1]) / t;
      } else if (R.a[0][0] > R.a[1][1] && R.a[0][0] > R.a[2][2]) {
        const double t = 2 * std::sqrt(1 + R.a[0][0] - R.a[1][1] - R.a[2][2]);
        q[0] = (R.a[2][1] - R.a[1][2]) / t; q[1] = 0.25 * t;
        q[2] = (R.a[0][1] + R.a[1][0]) / t; q[3] = (R.a[0][2] + R.a[2][0]) / t;
      } else if (R.a[1][1] > R.a[2][2]) {
        const double t = 2 * std::sqrt(1 + R.a[1][1] - R.a[0][0] - R.a[2][2]);
        q[0] = (R.a[0][2] - R.a[2][0]) / t; q[1] = (R.a[0][1] + R.a[1][0]) / t;
        q[2] = 0.25 * t; q[3] = (R.a[1][2] + R.a[2][1]) / t;
      } else {
        const double t = 2 * std::sqrt(1 + R.a[2][2] - R.a[0][0] - R.a[1][1]);
        q[0] = (R.a[1][0] - R.a[0][1]) / t; q[1] = (R.a[0][2] + R.a[2][0]) / t;
        q[2] = (R.a[1][2] + R.a[2][1]) / t; q[3] = 0.25 * t;
      }
      const double nq = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
      for (double& e : q) e /= nq;
    }
    double* o = out + 13 * static_cast<int64_t>(b);
    o[0] = c.x; o[1] = c.y; o[2] = c.z;
    for (int k = 0; k < 4; ++k) o[3 + k] = q[k];
    o[7] = P.x; o[8] = P.y; o[9] = P.z;
    o[10] = L.x; o[11] = L.y; o[12] = L.z;
  }
}

int o64_error(void* h, uint32_t* bits, int32_t* body, double* axis) {
  const O64& s = *static_cast<O64*>(h);
  if (bits) *bits = s.err;
  if (body) *body = s.err_body;
  if (axis) { axis[0] = s.err_axis.x; axis[1] = s.err_axis.y; axis[2] = s.err_axis.z; }
  return s.err ? 1 : 0;
}

}  // extern "C"
