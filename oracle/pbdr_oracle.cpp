// ============================================================================
// TEST INFRASTRUCTURE ONLY — the CPU oracle for the PBD-R substep loop.
//
// This file is the parity checker and the CPU baseline ("kind": "port"). Only
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference legs may load it; the product library never links it, and the
// product path fails loudly when its CUDA library is missing.
//
// What it restates. The reference's solver (proj/src/solver.cpp, listed at
// proj/CMakeLists.txt:20) is absent, so this is a restatement of:
//   * PAPER.md:136-155 Algorithm 1 (integrate; per iteration ground contact,
//     particle-particle contact, shape matching, position update, velocity
//     update, momentum enforcement),
//   * PAPER.md:157-172 incremental velocity update,
//   * PAPER.md:177-219 momentum-conservation constraint (Eq. 1, Eq. 2),
//   * SPEC.md:253-365 solver module (worked examples, design decisions
//     SPEC.md:343-351, open questions :362-364),
// with the reference's shipped helpers' semantics: compute_com / inertia /
// momentum (body.cpp:50-83), extract_pose (body.cpp:103-124), polar and SPD
// pseudo-inverse (math.cpp:90-108, 170-210), the fixed-order deterministic
// reduction idea (parallel.hpp:40-63) and scene.hpp:17-82 types.
//
// Pinned semantics (DESIGN.md "Pinned semantics" states each one and why):
//   P1 Jacobi across constraints: PG, PP and SM all read the X_i snapshot.
//   P2 bsm state = (X_i + dC, V_i + dC/dt) with dC = dPG + dPP; asm state =
//      (X_{i+1}, V_{i+1}) after the position and velocity update.
//   P3 incremental update V_{i+1} = V_i + dX/dt (legacy: (X_{i+1}-X_init)/dt).
//   P4 hash grid built once per substep on the predicted positions; the
//      candidate set is {j: same scene, other body, |cell_j - cell_i|_inf <= 1,
//      |x~_i - x~_j|^2 < h^2}, h = 2 r_max; the contact predicate
//      d^2 < (r_i + r_j)^2 is evaluated on X_i every iteration.
//   P5 ground/wall friction on the tangential part of (x - x_init), clamped to
//      mu*|d|, measured before the normal push.
//   P6 enforce_momentum: linear first, then angular with L "re-measured" after
//      the linear fix (algebraically equal to L_asm).
//   P7 all body sums are fp32 in anchored coordinates (p = x - a_b, a_b the
//      body's com from the previous iteration) and reduced in the fixed tree of
//      pbdr_pinned.h; per-body 3x3 math is fp64 (oracle_math.hpp).
//   P8 fp32 state, round-to-nearest casts from the caller's fp64 at upload; no
//      FMA contraction anywhere (built with -ffp-contract=off, GPU with
//      --fmad=false), so the CUDA path reproduces this file bit for bit.
//
// Parity pins: the 3x3 math, com/inertia/momentum and pose are checked
// against the reference's own compiled code (oracle/_ref, golden fixtures in
// tests/golden/); the solver-level SPEC.md worked examples
// are known-answer tests in tests/test_oracle_kat.py. The step() loop itself
// has no reference implementation or trajectory fixture to pin against.
// ============================================================================
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <tuple>
#include <vector>

#if defined(_OPENMP)
#include <omp.h>
#endif

#include "oracle_math.hpp"
#include "pbdr_gpu.h"
#include "pbdr_pinned.h"

namespace {

struct Plane4 {
  float p[3], n[3], mu;
};

struct State {
  int64_t n = 0;
  int32_t nb = 0;
  std::vector<int64_t> slot_to_particle;  // body-major slot -> caller index
  std::vector<float> pos, vel, rest, init;  // 4 floats per slot
  std::vector<int32_t> body_of;
  std::vector<int64_t> bstart;
  std::vector<float> bM, binvM, anchor, bforce;
  std::vector<float> rquat;  // per body: last rotation (w, x, y, z), 0 = none
  std::vector<float> mom_acc;  // per body kPerSubstep accumulators (P, L)
  bool per_substep = false;
  bool any_torque = false;
  int iter_in_substep = 0;
  std::vector<int32_t> bscene, bexempt, bprog;
  std::vector<float> btorque;       // 3 per body
  std::vector<int32_t> btorque_on;  // nonzero torque program
  std::vector<float> wcom, walpha;  // 3 per body: com and alpha at the substep start
  std::vector<double> tstart, tstop;
  std::vector<Plane4> planes;
  float dt = 0, inv_dt = 0, g = 0, relax = 1, h = 0, inv_h = 0, h2 = 0;
  double dt_d = 0;
  int iters = 10, substeps = 10;
  bool incremental = true, linfix = true, angfix = true;
  int64_t substep_index = 0;
  uint32_t mask = 0;
  pbdr_key_layout layout{};
  std::vector<int32_t> ncand, cand;
  std::vector<float> cand_rr;
  uint32_t err_bits = 0;
  int32_t err_body = -1;
  double err_axis[3] = {0, 0, 0};
  int threads = 1;
  int kp = 2;  // tile shape of the reduction trees (pbdr_choose_kp)
  std::vector<int8_t> role;  // slab mode: 0 inactive, 1 ghost, 2 owned (empty = all owned)
};

inline int role_of(const State& s, int32_t b) { return s.role.empty() ? 2 : s.role[b]; }

inline void flag(State& s, uint32_t bits, int32_t body, const double* axis = nullptr) {
#pragma omp critical(oracle_err)
  {
    s.err_bits |= bits;
    if (s.err_body < 0 || body < s.err_body) {
      s.err_body = body;
      if (axis) std::memcpy(s.err_axis, axis, sizeof s.err_axis);
    }
  }
}

// ---- Fixed-topology body sum (pbdr_pinned.h) --------------------------------
template <int F>
void tree_sum(int kp, int n, const float* vals, float out[F]) {
  const int W = pbdr_body_warps(n, kp);
  const int K = pbdr_body_slots(n, W);
  float lane[32][F], nxt[32][F];
  for (int wi = 0; wi < W; ++wi) {
    for (int l = 0; l < 32; ++l) {
      for (int f = 0; f < F; ++f) lane[l][f] = 0.0f;
      for (int k = 0; k < K; ++k) {
        const int q = k * 32 * W + wi * 32 + l;
        if (q < n)
          for (int f = 0; f < F; ++f) lane[l][f] = lane[l][f] + vals[static_cast<size_t>(q) * F + f];
      }
    }
    for (int off = 16; off >= 1; off >>= 1) {
      for (int l = 0; l < 32; ++l)
        for (int f = 0; f < F; ++f) nxt[l][f] = lane[l][f] + lane[l ^ off][f];
      std::memcpy(lane, nxt, sizeof lane);
    }
    if (wi == 0) {
      for (int f = 0; f < F; ++f) out[f] = lane[0][f];
    } else {
      for (int f = 0; f < F; ++f) out[f] = out[f] + lane[0][f];
    }
  }
}

// Same tree with fused first stage: per lane acc = fma(a_q, b_q, acc) over k
// ascending (b = 1 for summed fields: fma(a, 1, acc) == a + acc exactly).
template <int F>
void tree_sum_fma(int kp, int n, const float* va, const float* vb, float out[F]) {
  const int W = pbdr_body_warps(n, kp);
  const int K = pbdr_body_slots(n, W);
  float lane[32][F], nxt[32][F];
  for (int wi = 0; wi < W; ++wi) {
    for (int l = 0; l < 32; ++l) {
      for (int f = 0; f < F; ++f) lane[l][f] = 0.0f;
      for (int k = 0; k < K; ++k) {
        const int q = k * 32 * W + wi * 32 + l;
        if (q < n)
          for (int f = 0; f < F; ++f) {
            const size_t i = static_cast<size_t>(q) * F + f;
            lane[l][f] = std::fmaf(va[i], vb[i], lane[l][f]);
          }
      }
    }
    for (int off = 16; off >= 1; off >>= 1) {
      for (int l = 0; l < 32; ++l)
        for (int f = 0; f < F; ++f) nxt[l][f] = lane[l][f] + lane[l ^ off][f];
      std::memcpy(lane, nxt, sizeof lane);
    }
    if (wi == 0) {
      for (int f = 0; f < F; ++f) out[f] = lane[0][f];
    } else {
      for (int f = 0; f < F; ++f) out[f] = out[f] + lane[0][f];
    }
  }
}

// Pinned explicit fused multiply-adds (mirrors the kernels' fmaf()).
inline float dot3_fma(const float a[3], const float b[3]) {
  return std::fmaf(a[2], b[2], std::fmaf(a[1], b[1], a[0] * b[0]));
}
inline void cross3_fma(const float a[3], const float b[3], float o[3]) {
  o[0] = std::fmaf(a[1], b[2], -(a[2] * b[1]));
  o[1] = std::fmaf(a[2], b[0], -(a[0] * b[2]));
  o[2] = std::fmaf(a[0], b[1], -(a[1] * b[0]));
}

inline void cross3(const float a[3], const float b[3], float o[3]) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}

// ---- integrate ---------------------------
// distribute_wrench (body.cpp:126-150): alpha = pinv(I) tau with the com and
// inertia of X at the substep start, anchored fp32 sums in the pinned tree.
void wrench_prepass(State& s) {
#pragma omp parallel for num_threads(s.threads) schedule(dynamic, 8)
  for (int32_t b = 0; b < s.nb; ++b) {
    if (!s.btorque_on[b] || role_of(s, b) == 0) continue;
    const int64_t start = s.bstart[b];
    const int n = static_cast<int>(s.bstart[b + 1] - start);
    const float a[3] = {s.anchor[3 * b], s.anchor[3 * b + 1], s.anchor[3 * b + 2]};
    std::vector<float> vals(9 * static_cast<size_t>(n));
    for (int q = 0; q < n; ++q) {
      const int64_t p = start + q;
      const float mk = s.vel[4 * p + 3];
      const float pp[3] = {s.pos[4 * p] - a[0], s.pos[4 * p + 1] - a[1], s.pos[4 * p + 2] - a[2]};
      const float s2 = (pp[0] * pp[0] + pp[1] * pp[1]) + pp[2] * pp[2];
      float* o = &vals[9 * static_cast<size_t>(q)];
      o[0] = mk * pp[0]; o[1] = mk * pp[1]; o[2] = mk * pp[2];
      o[3] = mk * (s2 - pp[0] * pp[0]);
      o[4] = mk * (s2 - pp[1] * pp[1]);
      o[5] = mk * (s2 - pp[2] * pp[2]);
      o[6] = -(mk * (pp[0] * pp[1]));
      o[7] = -(mk * (pp[0] * pp[2]));
      o[8] = -(mk * (pp[1] * pp[2]));
    }
    float S[9] = {};
    tree_sum<9>(s.kp, n, vals.data(), S);
    const float M = s.bM[b], invM = s.binvM[b];
    float c[3];
    for (int k = 0; k < 3; ++k) c[k] = S[k] * invM;
    const float Ixx = S[3] - M * (c[1] * c[1] + c[2] * c[2]);
    const float Iyy = S[4] - M * (c[0] * c[0] + c[2] * c[2]);
    const float Izz = S[5] - M * (c[0] * c[0] + c[1] * c[1]);
    const float Ixy = S[6] + M * (c[0] * c[1]);
    const float Ixz = S[7] + M * (c[0] * c[2]);
    const float Iyz = S[8] + M * (c[1] * c[2]);
    orc::M3 I = {{{Ixx, Ixy, Ixz}, {Ixy, Iyy, Iyz}, {Ixz, Iyz, Izz}}};
    const double tau[3] = {s.btorque[3 * b], s.btorque[3 * b + 1], s.btorque[3 * b + 2]};
    double al[3], nax[3];
    const unsigned e = orc::inertia_solve(I, tau, al, nax);
    if (e) flag(s, e, b, nax);
    for (int k = 0; k < 3; ++k) {
      s.wcom[3 * b + k] = a[k] + c[k];
      s.walpha[3 * b + k] = static_cast<float>(al[k]);
    }
  }
}

void integrate(State& s) {
  s.iter_in_substep = 0;
  if (s.any_torque) wrench_prepass(s);
  const double t = static_cast<double>(s.substep_index) * s.dt_d;
#pragma omp parallel for num_threads(s.threads) schedule(static)
  for (int64_t p = 0; p < s.n; ++p) {
    const int32_t b = s.body_of[p];
    if (role_of(s, b) == 0) continue;  // slab mode: not simulated on this rank
    float a[3] = {0.0f, 0.0f, s.bexempt[b] ? 0.0f : -s.g};
    float* x = &s.pos[4 * p];
    if (s.bprog[b] && t >= s.tstart[b] && t < s.tstop[b]) {
      for (int k = 0; k < 3; ++k) a[k] = a[k] + s.bforce[3 * b + k] * s.binvM[b];
      if (s.btorque_on[b]) {
        const float r[3] = {x[0] - s.wcom[3 * b], x[1] - s.wcom[3 * b + 1], x[2] - s.wcom[3 * b + 2]};
        float ar[3];
        cross3(&s.walpha[3 * b], r, ar);
        for (int k = 0; k < 3; ++k) a[k] = a[k] + ar[k];
      }
    }
    float* v = &s.vel[4 * p];
    float* xi = &s.init[4 * p];
    for (int k = 0; k < 3; ++k) {
      xi[k] = x[k];
      v[k] = v[k] + s.dt * a[k];
      x[k] = x[k] + s.dt * v[k];
    }
    xi[3] = 0.0f;
  }
}

// ---- hash-grid candidates (pinned P4) -------------------
void build_candidates(State& s) {
  struct Key {
    int32_t scene, cz, cy, cx;
    bool operator<(const Key& o) const {
      return std::tie(scene, cz, cy, cx) < std::tie(o.scene, o.cz, o.cy, o.cx);
    }
    bool operator==(const Key& o) const {
      return scene == o.scene && cz == o.cz && cy == o.cy && cx == o.cx;
    }
  };
  std::vector<Key> key(static_cast<size_t>(s.n));
  for (int64_t p = 0; p < s.n; ++p) {
    const float* x = &s.pos[4 * p];
    key[p] = {s.bscene[s.body_of[p]], pbdr_cell_coord(x[2], s.inv_h), pbdr_cell_coord(x[1], s.inv_h),
              pbdr_cell_coord(x[0], s.inv_h)};
  }
  // Slab mode: only owned + ghost particles enter the grid.
  std::vector<int64_t> order;
  order.reserve(static_cast<size_t>(s.n));
  for (int64_t p = 0; p < s.n; ++p)
    if (role_of(s, s.body_of[p]) != 0) order.push_back(p);
  std::stable_sort(order.begin(), order.end(),
                   [&](int64_t a, int64_t b) { return key[a] < key[b]; });
  std::vector<Key> sorted(order.size());
  for (size_t k = 0; k < order.size(); ++k) sorted[k] = key[order[k]];

  s.ncand.assign(static_cast<size_t>(s.n), 0);
  s.cand.assign(static_cast<size_t>(s.n) * PBDR_NBR_CAP, -1);
  s.cand_rr.assign(static_cast<size_t>(s.n) * PBDR_NBR_CAP, 0.0f);
#pragma omp parallel for num_threads(s.threads) schedule(dynamic, 1024)
  for (int64_t i = 0; i < s.n; ++i) {
    if (role_of(s, s.body_of[i]) == 0) continue;
    const Key ki = key[i];
    const float* xi = &s.pos[4 * i];
    std::vector<int64_t> found;
    for (int dz = -1; dz <= 1; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          const Key kn{ki.scene, ki.cz + dz, ki.cy + dy, ki.cx + dx};
          auto range = std::equal_range(sorted.begin(), sorted.end(), kn);
          for (auto it = range.first; it != range.second; ++it) {
            const int64_t j = order[static_cast<size_t>(it - sorted.begin())];
            if (s.body_of[j] == s.body_of[i]) continue;
            const float* xj = &s.pos[4 * j];
            const float ex = xi[0] - xj[0], ey = xi[1] - xj[1], ez = xi[2] - xj[2];
            const float d2 = (ex * ex + ey * ey) + ez * ez;
            if (d2 < s.h2) found.push_back(j);
          }
        }
    std::sort(found.begin(), found.end());
    if (static_cast<int>(found.size()) > PBDR_NBR_CAP) {
      flag(s, PBDR_DEVERR_NBR_OVERFLOW, s.body_of[i]);
      found.resize(PBDR_NBR_CAP);
    }
    s.ncand[i] = static_cast<int32_t>(found.size());
    for (size_t k = 0; k < found.size(); ++k) {
      const int64_t j = found[k];
      s.cand[static_cast<size_t>(i) * PBDR_NBR_CAP + k] = static_cast<int32_t>(j);
      s.cand_rr[static_cast<size_t>(i) * PBDR_NBR_CAP + k] = s.rest[4 * i + 3] + s.rest[4 * j + 3];
    }
  }
}

// ---- constraint components -------------

// Ground / wall contact for one particle against all planes (SPEC.md:281-289,
// pinned P5). `xinit` is only read when the particle penetrates a plane with
// friction. Accumulates into dPG (starting from +0).
void ground_delta(const std::vector<Plane4>& planes, float relax, const float x[3],
                  const float* xinit, float r, float dPG[3]) {
  for (const Plane4& P : planes) {
    const float xp[3] = {x[0] - P.p[0], x[1] - P.p[1], x[2] - P.p[2]};
    const float d = dot3_fma(xp, P.n) - r;
    if (!(d < 0.0f)) continue;
    const float push = -(relax * d);
    for (int k = 0; k < 3; ++k) dPG[k] = std::fmaf(push, P.n[k], dPG[k]);
    if (!(P.mu > 0.0f)) continue;
    const float t[3] = {x[0] - xinit[0], x[1] - xinit[1], x[2] - xinit[2]};
    const float tn = dot3_fma(t, P.n);
    const float tt[3] = {std::fmaf(-tn, P.n[0], t[0]), std::fmaf(-tn, P.n[1], t[1]), std::fmaf(-tn, P.n[2], t[2])};
    const float len2 = dot3_fma(tt, tt);
    if (!(len2 > 0.0f)) continue;
    const float len = std::sqrt(len2);
    const float lim = P.mu * (-d);
    if (len <= lim) {
      for (int k = 0; k < 3; ++k) dPG[k] = dPG[k] - tt[k];
    } else {
      const float f = lim / len;
      for (int k = 0; k < 3; ++k) dPG[k] = std::fmaf(-tt[k], f, dPG[k]);
    }
  }
}

// One particle-particle pair seen from particle i: mass-
// weighted push along n = (x_i - x_j)/|x_i - x_j|; accumulates into dPP.
void pp_delta(const float x[3], float w, int64_t i, const float xj[3], float wj, int64_t j,
              float rr, float relax, float dPP[3]) {
  const float e[3] = {x[0] - xj[0], x[1] - xj[1], x[2] - xj[2]};
  const float d2 = dot3_fma(e, e);
  if (!(d2 < rr * rr)) return;
  const float dist = std::sqrt(d2);
  float nrm[3];
  if (dist > PBDR_COINCIDENT_EPS) {
    const float inv = 1.0f / dist;
    for (int k = 0; k < 3; ++k) nrm[k] = e[k] * inv;
  } else {
    nrm[0] = i < j ? 1.0f : -1.0f;
    nrm[1] = 0.0f;
    nrm[2] = 0.0f;
  }
  const float C = dist - rr;
  const float kk = (relax * (w / (w + wj))) * C;
  for (int k = 0; k < 3; ++k) dPP[k] = std::fmaf(-kk, nrm[k], dPP[k]);
}

struct BodyIn {
  int n;
  const float* x;     // 3n, X_i
  const float* v;     // 3n, V_i
  const float* m;     // n
  const float* q0;    // 3n rest offsets
  const float* dc;    // 3n contact deltas dPG + dPP
  const float* init;  // 3n X_init (legacy update only)
  float a[3];         // anchor
  float* rq;          // warm-start quaternion (in/out), 4 floats
  float M, invM, dt, inv_dt;
  bool incremental, linfix, angfix;
  float* acc = nullptr;  // kPerSubstep accumulators (6 floats) or null
  bool reset = false;    // first iteration of the substep
  bool last = true;      // last iteration of the substep
  int kp = 2;            // tile shape of the reduction tree (pbdr_choose_kp)
};

struct BodyOut {
  float* x;  // 3n, X_{i+1}
  float* v;  // 3n, V_{i+1}
  float c[3];  // anchor-relative com of X_i
  unsigned err = 0;
  double axis[3] = {0, 0, 0};
};

// Momentum enforcement (Eq. 1 then Eq. 2).
// Inputs are the asm state (xa, va), its anchored positions pa, the per-particle
// update dX (so c_asm = c + sum m dX / M) and the bsm momenta.
// kPerSubstep (acc != null): the SM-induced changes (P_bsm - P_asm,
// L_asm - L_bsm) are accumulated over the substep's iterations (acc reset at
// iteration 0) and corrected once, in the last iteration (correct == true).
void momentum_fix(int n, const float* m, const float* xa, const float* va, const float* pa,
                  const float* dX, const float c[3], const float Pb[3], const float Lb[3], float M,
                  float invM, float dt, bool linfix, bool angfix, float* xo, float* vo,
                  unsigned& err, double axis[3], float* acc = nullptr, bool reset = false,
                  bool last = true, int kp = 2) {
  // (a, b) per field: the tree's first stage is acc = fma(a, b, acc).
  std::vector<float> fa(15 * static_cast<size_t>(n)), fb(15 * static_cast<size_t>(n), 1.0f);
  for (int q = 0; q < n; ++q) {
    const float mk = m[q];
    const float* P = &pa[3 * q];
    const float mva[3] = {mk * va[3 * q], mk * va[3 * q + 1], mk * va[3 * q + 2]};
    float ka[3];
    cross3_fma(P, mva, ka);
    const float s2 = dot3_fma(P, P);
    float* a = &fa[15 * static_cast<size_t>(q)];
    float* b = &fb[15 * static_cast<size_t>(q)];
    for (int k = 0; k < 3; ++k) {
      a[k] = mk; b[k] = dX[3 * q + k];
      a[3 + k] = mk; b[3 + k] = va[3 * q + k];
      a[6 + k] = ka[k];
      a[9 + k] = mk; b[9 + k] = std::fmaf(-P[k], P[k], s2);
    }
    a[12] = -mk; b[12] = P[0] * P[1];
    a[13] = -mk; b[13] = P[0] * P[2];
    a[14] = -mk; b[14] = P[1] * P[2];
  }
  float SB[15];
  tree_sum_fma<15>(kp, n, fa.data(), fb.data(), SB);
  bool fin = true;
  for (float f : SB) fin = fin && std::isfinite(f);
  if (!fin) err |= PBDR_DEVERR_NONFINITE;
  float ca[3], Pa[3], La[3], tmp[3], dv[3] = {0, 0, 0}, om[3] = {0, 0, 0};
  for (int k = 0; k < 3; ++k) {
    ca[k] = c[k] + SB[k] * invM;
    Pa[k] = SB[3 + k];
  }
  cross3(ca, Pa, tmp);
  for (int k = 0; k < 3; ++k) La[k] = SB[6 + k] - tmp[k];
  float dP[3], dLf[3];
  for (int k = 0; k < 3; ++k) {
    dP[k] = Pb[k] - Pa[k];
    dLf[k] = La[k] - Lb[k];
  }
  bool correct = true;
  if (acc) {
    for (int k = 0; k < 3; ++k) {
      const float p0 = reset ? 0.0f : acc[k];
      const float l0 = reset ? 0.0f : acc[3 + k];
      acc[k] = p0 + dP[k];
      acc[3 + k] = l0 + dLf[k];
      dP[k] = acc[k];
      dLf[k] = acc[3 + k];
    }
    correct = last;
  }
  if (linfix && correct)
    for (int k = 0; k < 3; ++k) dv[k] = dP[k] * invM;
  if (angfix && correct) {
    const float Ixx = SB[9] - M * (ca[1] * ca[1] + ca[2] * ca[2]);
    const float Iyy = SB[10] - M * (ca[0] * ca[0] + ca[2] * ca[2]);
    const float Izz = SB[11] - M * (ca[0] * ca[0] + ca[1] * ca[1]);
    const float Ixy = SB[12] + M * (ca[0] * ca[1]);
    const float Ixz = SB[13] + M * (ca[0] * ca[2]);
    const float Iyz = SB[14] + M * (ca[1] * ca[2]);
    orc::M3 I = {{{Ixx, Ixy, Ixz}, {Ixy, Iyy, Iyz}, {Ixz, Iyz, Izz}}};
    const double dL[3] = {static_cast<double>(dLf[0]), static_cast<double>(dLf[1]),
                          static_cast<double>(dLf[2])};
    double wd[3];
    const unsigned e = orc::inertia_solve(I, dL, wd, axis);
    err |= e;
    for (int k = 0; k < 3; ++k) om[k] = static_cast<float>(wd[k]);
  }
  for (int q = 0; q < n; ++q) {
    float r[3], wr[3];
    for (int k = 0; k < 3; ++k) r[k] = pa[3 * q + k] - ca[k];
    cross3_fma(om, r, wr);
    for (int k = 0; k < 3; ++k) {
      vo[3 * q + k] = (va[3 * q + k] + dv[k]) - wr[k];
      xo[3 * q + k] = std::fmaf(-wr[k], dt, std::fmaf(dv[k], dt, xa[3 * q + k]));
    }
  }
}

// Shape matching + position/velocity update + momentum fix for one body, given
// its contact deltas (pinned P1-P3, P6, P7).
void body_iteration(const BodyIn& in, BodyOut& out) {
  const int n = in.n;
  std::vector<float> fa(21 * static_cast<size_t>(n)), fb(21 * static_cast<size_t>(n), 1.0f);
  for (int q = 0; q < n; ++q) {
    const float* x = &in.x[3 * q];
    const float* v = &in.v[3 * q];
    const float m = in.m[q];
    const float* dc = &in.dc[3 * q];
    const float* q0 = &in.q0[3 * q];
    float pp[3], pb[3], mp[3], vb[3], mvb[3], kb[3];
    for (int k = 0; k < 3; ++k) {
      pp[k] = x[k] - in.a[k];
      pb[k] = pp[k] + dc[k];
      vb[k] = std::fmaf(dc[k], in.inv_dt, v[k]);
      mp[k] = m * pp[k];
      mvb[k] = m * vb[k];
    }
    cross3_fma(pb, mvb, kb);
    float* a = &fa[21 * static_cast<size_t>(q)];
    float* b = &fb[21 * static_cast<size_t>(q)];
    for (int k = 0; k < 3; ++k) {
      a[k] = m; b[k] = pp[k];
      a[3 + k] = m; b[3 + k] = dc[k];
      a[15 + k] = m; b[15 + k] = vb[k];
      a[18 + k] = kb[k];
    }
    for (int rI = 0; rI < 3; ++rI)
      for (int cI = 0; cI < 3; ++cI) {
        a[6 + 3 * rI + cI] = mp[rI];
        b[6 + 3 * rI + cI] = q0[cI];
      }
  }
  float SA[21];
  tree_sum_fma<21>(in.kp, n, fa.data(), fb.data(), SA);
  bool finite = true;
  for (float f : SA) finite = finite && std::isfinite(f);
  if (!finite) out.err |= PBDR_DEVERR_NONFINITE;

  float c[3], cb[3], Pb[3], Lb[3], tmp[3];
  for (int k = 0; k < 3; ++k) {
    c[k] = SA[k] * in.invM;
    cb[k] = c[k] + SA[3 + k] * in.invM;
    Pb[k] = SA[15 + k];
    out.c[k] = c[k];
  }
  cross3(cb, Pb, tmp);
  for (int k = 0; k < 3; ++k) Lb[k] = SA[18 + k] - tmp[k];

  orc::M3 A;
  for (int rI = 0; rI < 3; ++rI)
    for (int cI = 0; cI < 3; ++cI) A.a[rI][cI] = static_cast<double>(SA[6 + 3 * rI + cI]);
  orc::M3 R;
  double qd[4];
  const bool sm_ok = orc::polar_warm(A, in.rq, R, qd);
  if (!sm_ok) out.err |= PBDR_DEVERR_DEGENERATE;
  for (int k = 0; k < 4; ++k) in.rq[k] = sm_ok ? static_cast<float>(qd[k]) : 0.0f;
  float Rf[3][3];
  for (int rI = 0; rI < 3; ++rI)
    for (int cI = 0; cI < 3; ++cI) Rf[rI][cI] = static_cast<float>(R.a[rI][cI]);

  std::vector<float> xa(3 * n), va(3 * n), pa(3 * n), dXv(3 * n);
  for (int q = 0; q < n; ++q) {
    const float* x = &in.x[3 * q];
    const float* v = &in.v[3 * q];
    const float* q0 = &in.q0[3 * q];
    const float* dc = &in.dc[3 * q];
    for (int k = 0; k < 3; ++k) {
      const float pk = x[k] - in.a[k];
      float dsm = 0.0f;
      if (sm_ok) {
        const float gk = dot3_fma(Rf[k], q0);
        dsm = gk - (pk - c[k]);
      }
      const float dX = dc[k] + dsm;
      dXv[3 * q + k] = dX;
      xa[3 * q + k] = x[k] + dX;
      if (in.incremental)
        va[3 * q + k] = std::fmaf(dX, in.inv_dt, v[k]);
      else
        va[3 * q + k] = (xa[3 * q + k] - in.init[3 * q + k]) * in.inv_dt;
      pa[3 * q + k] = pk + dX;
    }
  }
  if (in.linfix || in.angfix) {
    momentum_fix(n, in.m, xa.data(), va.data(), pa.data(), dXv.data(), c, Pb, Lb, in.M, in.invM,
                 in.dt, in.linfix, in.angfix, out.x, out.v, out.err, out.axis, in.acc, in.reset, in.last,
                 in.kp);
  } else {
    std::memcpy(out.x, xa.data(), sizeof(float) * 3 * n);
    std::memcpy(out.v, va.data(), sizeof(float) * 3 * n);
  }
}

// ---- one solver iteration ----------------------------------
void iteration(State& s) {
  const std::vector<float> X = s.pos;  // X_i snapshot (P1)
#pragma omp parallel for num_threads(s.threads) schedule(dynamic, 8)
  for (int32_t b = 0; b < s.nb; ++b) {
    if (role_of(s, b) != 2) continue;  // slab mode: only owned bodies are solved
    const int64_t start = s.bstart[b];
    const int n = static_cast<int>(s.bstart[b + 1] - start);
    std::vector<float> x(3 * n), v(3 * n), m(n), q0(3 * n), dc(3 * n), init(3 * n), xo(3 * n), vo(3 * n);
    for (int q = 0; q < n; ++q) {
      const int64_t p = start + q;
      const float* xp = &X[4 * p];
      for (int k = 0; k < 3; ++k) {
        x[3 * q + k] = xp[k];
        v[3 * q + k] = s.vel[4 * p + k];
        q0[3 * q + k] = s.rest[4 * p + k];
        init[3 * q + k] = s.init[4 * p + k];
      }
      m[q] = s.vel[4 * p + 3];
      float dPG[3] = {0.0f, 0.0f, 0.0f};
      ground_delta(s.planes, s.relax, xp, &s.init[4 * p], s.rest[4 * p + 3], dPG);
      float dPP[3] = {0.0f, 0.0f, 0.0f};
      const int nc = s.ncand[p];
      for (int c = 0; c < nc; ++c) {
        const int64_t j = s.cand[static_cast<size_t>(p) * PBDR_NBR_CAP + c];
        const float rr = s.cand_rr[static_cast<size_t>(p) * PBDR_NBR_CAP + c];
        pp_delta(xp, xp[3], p, &X[4 * j], X[4 * j + 3], j, rr, s.relax, dPP);
      }
      for (int k = 0; k < 3; ++k) dc[3 * q + k] = dPG[k] + dPP[k];
    }
    BodyIn in{n, x.data(), v.data(), m.data(), q0.data(), dc.data(), init.data(),
              {s.anchor[3 * b], s.anchor[3 * b + 1], s.anchor[3 * b + 2]}, &s.rquat[4 * b],
              s.bM[b], s.binvM[b], s.dt, s.inv_dt, s.incremental, s.linfix, s.angfix};
    in.kp = s.kp;
    if (s.per_substep) {
      in.acc = &s.mom_acc[6 * b];
      in.reset = s.iter_in_substep == 0;
      in.last = s.iter_in_substep == s.iters - 1;
    }
    BodyOut out{xo.data(), vo.data(), {0, 0, 0}};
    body_iteration(in, out);
    if (out.err) flag(s, out.err, b, out.axis);
    for (int q = 0; q < n; ++q) {
      const int64_t p = start + q;
      for (int k = 0; k < 3; ++k) {
        s.pos[4 * p + k] = xo[3 * q + k];
        s.vel[4 * p + k] = vo[3 * q + k];
      }
    }
    for (int k = 0; k < 3; ++k) s.anchor[3 * b + k] = in.a[k] + out.c[k];
  }
  ++s.iter_in_substep;
}

// ---- per-body trajectory sample (body.cpp:72-83, 103-124) --------------------
void body_stats(State& s, pbdr_body_stats* out) {
#pragma omp parallel for num_threads(s.threads) schedule(dynamic, 8)
  for (int32_t b = 0; b < s.nb; ++b) {
    if (role_of(s, b) != 2) continue;
    const int64_t start = s.bstart[b];
    const int n = static_cast<int>(s.bstart[b + 1] - start);
    const float a[3] = {s.anchor[3 * b], s.anchor[3 * b + 1], s.anchor[3 * b + 2]};
    std::vector<float> vals(18 * static_cast<size_t>(n));
    for (int q = 0; q < n; ++q) {
      const int64_t p = start + q;
      const float* x = &s.pos[4 * p];
      const float* v = &s.vel[4 * p];
      const float m = v[3];
      const float* q0 = &s.rest[4 * p];
      float mp[3], mv[3], pp[3], kk[3];
      for (int k = 0; k < 3; ++k) {
        pp[k] = x[k] - a[k];
        mp[k] = m * pp[k];
        mv[k] = m * v[k];
      }
      cross3(pp, mv, kk);
      float* o = &vals[18 * static_cast<size_t>(q)];
      o[0] = mp[0]; o[1] = mp[1]; o[2] = mp[2];
      for (int rI = 0; rI < 3; ++rI)
        for (int cI = 0; cI < 3; ++cI) o[3 + 3 * rI + cI] = mp[rI] * q0[cI];
      o[12] = mv[0]; o[13] = mv[1]; o[14] = mv[2];
      o[15] = kk[0]; o[16] = kk[1]; o[17] = kk[2];
    }
    float S[18];
    tree_sum<18>(s.kp, n, vals.data(), S);
    float c[3], P[3], tmp[3];
    for (int k = 0; k < 3; ++k) {
      c[k] = S[k] * s.binvM[b];
      P[k] = S[12 + k];
    }
    cross3(c, P, tmp);
    orc::M3 A;
    for (int rI = 0; rI < 3; ++rI)
      for (int cI = 0; cI < 3; ++cI) A.a[rI][cI] = static_cast<double>(S[3 + 3 * rI + cI]);
    orc::M3 R;
    double qd[4];
    if (!orc::polar_rotation(A, R, qd)) {
      qd[0] = 1.0; qd[1] = qd[2] = qd[3] = 0.0;
    }
    pbdr_body_stats& o = out[b];
    for (int k = 0; k < 3; ++k) {
      o.com[k] = static_cast<double>(a[k]) + static_cast<double>(c[k]);
      o.linear[k] = static_cast<double>(P[k]);
      o.angular[k] = static_cast<double>(S[15 + k] - tmp[k]);
    }
    for (int k = 0; k < 4; ++k) o.quat[k] = qd[k];
  }
}

int finish_substep_errors(State& s) {
  if (!s.err_bits) return PBDR_OK;
  if (s.err_bits & (PBDR_DEVERR_NONFINITE | PBDR_DEVERR_NBR_OVERFLOW)) return PBDR_ERR_SIMULATION;
  if (s.err_bits & PBDR_DEVERR_RANK_DEFICIENT) return PBDR_ERR_RANK_DEFICIENT;
  return PBDR_ERR_DEGENERATE;
}

}  // namespace

extern "C" {

int oracle_create(const pbdr_scene_desc* d, const pbdr_solver_cfg* cfg, int threads, void** out) {
  *out = nullptr;
  if (!d || !cfg || d->num_particles <= 0 || d->num_bodies <= 0) return PBDR_ERR_CONFIG;
  State* s = new State();
  s->threads = threads > 0 ? threads : 1;
  s->n = d->num_particles;
  s->nb = d->num_bodies;
  const int64_t n = s->n;
  s->slot_to_particle.resize(static_cast<size_t>(n));
  s->pos.resize(4 * n);
  s->vel.resize(4 * n);
  s->rest.resize(4 * n);
  s->init.assign(4 * n, 0.0f);
  s->body_of.resize(n);
  s->bstart.resize(s->nb + 1);
  s->bM.resize(s->nb);
  s->binvM.resize(s->nb);
  s->anchor.resize(3 * s->nb);
  s->rquat.assign(4 * s->nb, 0.0f);
  s->mom_acc.assign(6 * s->nb, 0.0f);
  s->bforce.assign(3 * s->nb, 0.0f);
  s->btorque.assign(3 * s->nb, 0.0f);
  s->btorque_on.assign(s->nb, 0);
  s->wcom.assign(3 * s->nb, 0.0f);
  s->walpha.assign(3 * s->nb, 0.0f);
  s->bscene.resize(s->nb);
  s->bexempt.assign(s->nb, 0);
  s->bprog.assign(s->nb, 0);
  s->tstart.assign(s->nb, 0.0);
  s->tstop.assign(s->nb, 0.0);
  double rmax = 0.0;
  int64_t slot = 0;
  for (int32_t b = 0; b < s->nb; ++b) {
    s->bstart[b] = slot;
    for (int64_t k = d->body_offsets[b]; k < d->body_offsets[b + 1]; ++k, ++slot) {
      const int64_t i = d->body_indices[k];
      s->slot_to_particle[slot] = i;
      for (int c = 0; c < 3; ++c) {
        s->pos[4 * slot + c] = static_cast<float>(d->position[3 * i + c]);
        s->vel[4 * slot + c] = static_cast<float>(d->velocity[3 * i + c]);
        s->rest[4 * slot + c] = static_cast<float>(d->rest_offsets[3 * k + c]);
      }
      s->pos[4 * slot + 3] = static_cast<float>(d->inv_mass[i]);
      s->vel[4 * slot + 3] = static_cast<float>(1.0 / d->inv_mass[i]);
      s->rest[4 * slot + 3] = static_cast<float>(d->radius[i]);
      s->body_of[slot] = b;
      rmax = std::max(rmax, d->radius[i]);
    }
    s->bM[b] = static_cast<float>(d->total_mass[b]);
    s->binvM[b] = static_cast<float>(1.0 / d->total_mass[b]);
    const int64_t first = s->bstart[b];
    for (int c = 0; c < 3; ++c) s->anchor[3 * b + c] = s->pos[4 * first + c];
    s->bscene[b] = d->body_scene ? d->body_scene[b] : 0;
    if (d->programs) {
      const pbdr_force_program& pr = d->programs[b];
      s->bexempt[b] = pr.gravity_exempt ? 1 : 0;
      s->bprog[b] = 1;
      s->tstart[b] = pr.t_start;
      s->tstop[b] = pr.t_stop;
      for (int c = 0; c < 3; ++c) {
        s->bforce[3 * b + c] = static_cast<float>(pr.force[c]);
        s->btorque[3 * b + c] = static_cast<float>(pr.torque[c]);
      }
      s->btorque_on[b] = (pr.torque[0] != 0.0 || pr.torque[1] != 0.0 || pr.torque[2] != 0.0) ? 1 : 0;
      s->any_torque = s->any_torque || s->btorque_on[b];
    }
  }
  s->bstart[s->nb] = slot;
  if (slot != n) {
    delete s;
    return PBDR_ERR_CONFIG;
  }
  {
    int max_body = 0;
    for (int32_t b = 0; b < s->nb; ++b)
      max_body = std::max(max_body, static_cast<int>(s->bstart[b + 1] - s->bstart[b]));
    s->kp = pbdr_choose_kp(n, s->nb, max_body, d->tile_kp);
  }
  if (d->has_ground) {
    Plane4 P;
    for (int c = 0; c < 3; ++c) {
      P.p[c] = static_cast<float>(d->ground.point[c]);
      P.n[c] = static_cast<float>(d->ground.normal[c]);
    }
    P.mu = static_cast<float>(d->ground.friction);
    s->planes.push_back(P);
  }
  for (int w = 0; w < d->num_walls; ++w) {
    Plane4 P;
    for (int c = 0; c < 3; ++c) {
      P.p[c] = static_cast<float>(d->walls[w].point[c]);
      P.n[c] = static_cast<float>(d->walls[w].normal[c]);
    }
    P.mu = static_cast<float>(d->walls[w].friction);
    s->planes.push_back(P);
  }
  s->substeps = cfg->substeps;
  s->iters = cfg->solver_iterations;
  s->dt_d = 1.0 / (cfg->frame_rate * cfg->substeps);
  s->dt = static_cast<float>(s->dt_d);
  s->inv_dt = static_cast<float>(cfg->frame_rate * cfg->substeps);
  s->g = static_cast<float>(cfg->gravity);
  s->relax = static_cast<float>(d->contact_relaxation);
  s->incremental = cfg->velocity_update == PBDR_VELOCITY_INCREMENTAL;
  s->linfix = cfg->linear_momentum_fix != 0;
  s->angfix = cfg->angular_momentum_fix != 0;
  s->per_substep = cfg->momentum_frequency == PBDR_MOMENTUM_PER_SUBSTEP;
  s->h = static_cast<float>(2.0 * rmax);
  s->inv_h = 1.0f / s->h;
  s->h2 = s->h * s->h;
  {
    // Bucket key layout: the library's rule on the same fp32 positions.
    bool single = true;
    for (int32_t b = 0; b < s->nb && single; ++b) single = s->bscene[b] == 0;
    int32_t cmin[3] = {INT32_MAX, INT32_MAX, INT32_MAX}, cmax[3] = {INT32_MIN, INT32_MIN, INT32_MIN};
    for (int64_t p = 0; p < n; ++p)
      for (int a = 0; a < 3; ++a) {
        const int32_t c = pbdr_cell_coord(s->pos[4 * p + a], s->inv_h);
        cmin[a] = std::min(cmin[a], c);
        cmax[a] = std::max(cmax[a], c);
      }
    s->layout = pbdr_choose_key_layout(single ? 1 : 0, cmin, cmax, n);
    if (const char* e = std::getenv("PBDR_LINEAR_KEYS"))
      if (std::atoi(e) == 0) s->layout = pbdr_choose_key_layout(0, cmin, cmax, n);
  }
  s->mask = static_cast<uint32_t>((uint64_t(1) << s->layout.bits) - 1u);
  *out = s;
  return PBDR_OK;
}

void oracle_destroy(void* st) { delete static_cast<State*>(st); }

void oracle_integrate(void* st) { integrate(*static_cast<State*>(st)); }
void oracle_candidates(void* st) { build_candidates(*static_cast<State*>(st)); }
void oracle_iteration(void* st) { iteration(*static_cast<State*>(st)); }
void oracle_end_substep(void* st) { ++static_cast<State*>(st)->substep_index; }

int oracle_step(void* st, int64_t substeps) {
  State& s = *static_cast<State*>(st);
  for (int64_t k = 0; k < substeps; ++k) {
    integrate(s);
    build_candidates(s);
    for (int it = 0; it < s.iters; ++it) iteration(s);
    ++s.substep_index;
    const int e = finish_substep_errors(s);
    if (e != PBDR_OK) return e;
  }
  return PBDR_OK;
}

int oracle_error(void* st, uint32_t* bits, int32_t* body, double* axis) {
  State& s = *static_cast<State*>(st);
  if (bits) *bits = s.err_bits;
  if (body) *body = s.err_body;
  if (axis) std::memcpy(axis, s.err_axis, sizeof s.err_axis);
  return finish_substep_errors(s);
}

// Slab decomposition (mirrors pbdr_gpu_set_roles / _gather / _scatter).
void oracle_set_roles(void* st, const int8_t* roles) {
  State& s = *static_cast<State*>(st);
  if (!roles) {
    s.role.clear();
    return;
  }
  s.role.assign(roles, roles + s.nb);
}

void oracle_gather(void* st, int field, const int32_t* index, int64_t count, float* dst) {
  State& s = *static_cast<State*>(st);
  for (int64_t t = 0; t < count; ++t) {
    const int64_t i = index[t];
    float* o = &dst[4 * t];
    switch (field) {
      case PBDR_FIELD_POSITION: std::memcpy(o, &s.pos[4 * i], 16); break;
      case PBDR_FIELD_VELOCITY: std::memcpy(o, &s.vel[4 * i], 16); break;
      case PBDR_FIELD_ANCHOR: std::memcpy(o, &s.anchor[3 * i], 12); o[3] = 0.0f; break;
      case PBDR_FIELD_ROTATION: std::memcpy(o, &s.rquat[4 * i], 16); break;
      default: break;
    }
  }
}

void oracle_scatter(void* st, int field, const int32_t* index, int64_t count, const float* src) {
  State& s = *static_cast<State*>(st);
  for (int64_t t = 0; t < count; ++t) {
    const int64_t i = index[t];
    const float* o = &src[4 * t];
    switch (field) {
      case PBDR_FIELD_POSITION: std::memcpy(&s.pos[4 * i], o, 16); break;
      case PBDR_FIELD_VELOCITY: std::memcpy(&s.vel[4 * i], o, 16); break;
      case PBDR_FIELD_ANCHOR: std::memcpy(&s.anchor[3 * i], o, 12); break;
      case PBDR_FIELD_ROTATION: std::memcpy(&s.rquat[4 * i], o, 16); break;
      default: break;
    }
  }
}

void oracle_read_f32(void* st, float* pos4, float* vel4) {
  State& s = *static_cast<State*>(st);
  if (pos4) std::memcpy(pos4, s.pos.data(), s.pos.size() * sizeof(float));
  if (vel4) std::memcpy(vel4, s.vel.data(), s.vel.size() * sizeof(float));
}

void oracle_write_f32(void* st, const float* pos4, const float* vel4) {
  State& s = *static_cast<State*>(st);
  if (pos4) std::memcpy(s.pos.data(), pos4, s.pos.size() * sizeof(float));
  if (vel4) std::memcpy(s.vel.data(), vel4, s.vel.size() * sizeof(float));
}

void oracle_read_init(void* st, float* init4) {
  State& s = *static_cast<State*>(st);
  std::memcpy(init4, s.init.data(), s.init.size() * sizeof(float));
}

void oracle_write_init(void* st, const float* init4) {
  State& s = *static_cast<State*>(st);
  std::memcpy(s.init.data(), init4, s.init.size() * sizeof(float));
}

void oracle_read_anchor(void* st, float* a) {
  State& s = *static_cast<State*>(st);
  std::memcpy(a, s.anchor.data(), s.anchor.size() * sizeof(float));
}

void oracle_write_anchor(void* st, const float* a) {
  State& s = *static_cast<State*>(st);
  std::memcpy(s.anchor.data(), a, s.anchor.size() * sizeof(float));
}

void oracle_read_rquat(void* st, float* q) {
  State& s = *static_cast<State*>(st);
  std::memcpy(q, s.rquat.data(), s.rquat.size() * sizeof(float));
}

void oracle_write_rquat(void* st, const float* q) {
  State& s = *static_cast<State*>(st);
  std::memcpy(s.rquat.data(), q, s.rquat.size() * sizeof(float));
}

void oracle_read_particles(void* st, double* pos, double* vel) {
  State& s = *static_cast<State*>(st);
  for (int64_t slot = 0; slot < s.n; ++slot) {
    const int64_t i = s.slot_to_particle[slot];
    for (int c = 0; c < 3; ++c) {
      if (pos) pos[3 * i + c] = static_cast<double>(s.pos[4 * slot + c]);
      if (vel) vel[3 * i + c] = static_cast<double>(s.vel[4 * slot + c]);
    }
  }
}

// Cell coordinates and hash of the current positions (replay checks).
void oracle_read_keys(void* st, uint32_t* hash, int32_t* cell) {
  State& s = *static_cast<State*>(st);
  for (int64_t p = 0; p < s.n; ++p) {
    const float* x = &s.pos[4 * p];
    const int32_t cx = pbdr_cell_coord(x[0], s.inv_h);
    const int32_t cy = pbdr_cell_coord(x[1], s.inv_h);
    const int32_t cz = pbdr_cell_coord(x[2], s.inv_h);
    if (cell) {
      cell[3 * p] = cx; cell[3 * p + 1] = cy; cell[3 * p + 2] = cz;
    }
    if (hash) hash[p] = pbdr_cell_key(cx, cy, cz, static_cast<uint32_t>(s.bscene[s.body_of[p]]), s.mask, s.layout);
  }
}

void oracle_read_candidates(void* st, int32_t* counts, int32_t* lists) {
  State& s = *static_cast<State*>(st);
  std::memcpy(counts, s.ncand.data(), s.ncand.size() * sizeof(int32_t));
  std::memcpy(lists, s.cand.data(), s.cand.size() * sizeof(int32_t));
}

void oracle_body_stats(void* st, pbdr_body_stats* out) { body_stats(*static_cast<State*>(st), out); }

int64_t oracle_num_slots(void* st) { return static_cast<State*>(st)->n; }
int oracle_tile_kp(void* st) { return static_cast<State*>(st)->kp; }
float oracle_cell_size(void* st) { return static_cast<State*>(st)->h; }

}  // extern "C"

// ---- component entry points for the golden / KAT tests ----------------------
extern "C" {

// plane7 = (px, py, pz, nx, ny, nz, mu) per plane.
void oracle_kat_ground(const float* x, const float* xinit, float r, int nplanes, const float* plane7,
                       float relax, float* out) {
  std::vector<Plane4> planes(static_cast<size_t>(nplanes));
  for (int k = 0; k < nplanes; ++k) {
    for (int c = 0; c < 3; ++c) {
      planes[k].p[c] = plane7[7 * k + c];
      planes[k].n[c] = plane7[7 * k + 3 + c];
    }
    planes[k].mu = plane7[7 * k + 6];
  }
  out[0] = out[1] = out[2] = 0.0f;
  ground_delta(planes, relax, x, xinit, r, out);
}

void oracle_kat_pp(const float* xi, float wi, int64_t i, const float* xj, float wj, int64_t j,
                   float rr, float relax, float* out) {
  out[0] = out[1] = out[2] = 0.0f;
  pp_delta(xi, wi, i, xj, wj, j, rr, relax, out);
}

// One body iteration with given contact deltas; returns the error bits.
unsigned oracle_kat_body_iteration(int n, const float* x, const float* v, const float* m,
                                   const float* q0, const float* dc, const float* init,
                                   const float* anchor, float M, float dt, int incremental,
                                   int linfix, int angfix, float* xo, float* vo) {
  float rq[4] = {0.0f, 0.0f, 0.0f, 0.0f};
  BodyIn in{n, x, v, m, q0, dc, init, {anchor[0], anchor[1], anchor[2]}, rq, M, 1.0f / M, dt,
            1.0f / dt, incremental != 0, linfix != 0, angfix != 0};
  BodyOut out{xo, vo, {0, 0, 0}};
  body_iteration(in, out);
  return out.err;
}

// enforce_momentum on an asm state (positions are anchored at the origin).
unsigned oracle_kat_momentum(int n, const float* m, const float* xa, const float* va,
                             const float* Pb, const float* Lb, float dt, int linfix, int angfix,
                             float* xo, float* vo, double* axis) {
  float M = 0.0f;
  for (int q = 0; q < n; ++q) M = M + m[q];
  const float zero[3] = {0.0f, 0.0f, 0.0f};
  unsigned err = 0;
  momentum_fix(n, m, xa, va, xa, xa, zero, Pb, Lb, M, 1.0f / M, dt, linfix != 0, angfix != 0, xo,
               vo, err, axis);
  return err;
}

// Polar rotation of a row-major double matrix; returns 1 on success.
int oracle_polar(const double* a, double* r_out, double* q_out) {
  orc::M3 A;
  for (int i = 0; i < 9; ++i) A.a[i / 3][i % 3] = a[i];
  orc::M3 R;
  if (!orc::polar_rotation(A, R, q_out)) return 0;
  for (int i = 0; i < 9; ++i) r_out[i] = R.a[i / 3][i % 3];
  return 1;
}

// Warm-started polar (rq = previous rotation quaternion, zeros = none).
int oracle_polar_warm(const double* a, const float* rq, double* r_out, double* q_out) {
  orc::M3 A;
  for (int i = 0; i < 9; ++i) A.a[i / 3][i % 3] = a[i];
  orc::M3 R;
  if (!orc::polar_warm(A, rq, R, q_out)) return 0;
  for (int i = 0; i < 9; ++i) r_out[i] = R.a[i / 3][i % 3];
  return 1;
}

void oracle_sym_eigen(const double* a, double* ev, double* vecs) {
  orc::M3 A, V;
  for (int i = 0; i < 9; ++i) A.a[i / 3][i % 3] = a[i];
  orc::sym_eigen(A, ev, V);
  for (int i = 0; i < 9; ++i) vecs[i] = V.a[i / 3][i % 3];
}

// omega = pinv(I) dL; returns 0 or PBDR_DEVERR_RANK_DEFICIENT.
unsigned oracle_inertia_solve(const double* I9, const double* dL, double* w, double* axis) {
  orc::M3 I;
  for (int i = 0; i < 9; ++i) I.a[i / 3][i % 3] = I9[i];
  return orc::inertia_solve(I, dL, w, axis);
}

}  // extern "C"

// ---- pack_mesh restatement (geometry.cpp:73-195) ------------------------------
// Test infrastructure: checks the GPU pack_mesh; pinned against the reference's
// own pack_mesh (oracle/_ref) in tests/test_mesh.py.
namespace {
namespace mesh {
struct V {
  double x, y, z;
};
inline V sub(V a, V b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline double dot(V a, V b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline V cross(V a, V b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
inline double norm(V v) { return std::sqrt(dot(v, v)); }

// splitmix64 as rng.hpp:10-29 (seed + golden gamma, next_unit = (u64 >> 11) * 2^-53).
inline void unit3(uint64_t seed, double out[3]) {
  uint64_t s = seed + 0x9E3779B97F4A7C15ull;
  for (int k = 0; k < 3; ++k) {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z = z ^ (z >> 31);
    out[k] = static_cast<double>(z >> 11) * 0x1.0p-53;
  }
}

// 0 miss, 1 hit, 2 ambiguous (edge/grazing band 1e-9, geometry.cpp:77-104)
int ray_tri(V o, V d, V a, V b, V c) {
  const V e1 = sub(b, a), e2 = sub(c, a);
  const V pv = cross(d, e2);
  const double det = dot(e1, pv);
  const double scale = norm(e1) * norm(e2);
  if (std::abs(det) <= 1e-9 * std::max(scale, 1e-12)) {
    const V n = cross(e1, e2);
    const double nn = norm(n);
    if (nn <= 1e-12) return 0;
    const V u = {n.x / nn, n.y / nn, n.z / nn};
    return std::abs(dot(sub(o, a), u)) <= 1e-9 * std::max(1.0, norm(sub(o, a))) ? 2 : 0;
  }
  const double inv = 1.0 / det;
  const V tv = sub(o, a);
  const double u = dot(tv, pv) * inv;
  const V qv = cross(tv, e1);
  const double v = dot(d, qv) * inv;
  const double t = dot(e2, qv) * inv;
  if (u < -1e-9 || v < -1e-9 || u + v > 1.0 + 1e-9) return 0;
  if (t < -1e-9) return 0;
  if (u <= 1e-9 || v <= 1e-9 || u + v >= 1.0 - 1e-9 || t <= 1e-9) return 2;
  return 1;
}
}  // namespace mesh
}  // namespace

extern "C" int oracle_pack_mesh(const double* verts, int nv, const int* tris, int nt, double radius, double* centers,
                                long cap, long* count, long* candidates, long* ambiguous) {
  using mesh::V;
  if (!(radius > 0.0)) return 9;
  for (long k = 0; k < 3L * nt; ++k)
    if (tris[k] < 0 || tris[k] >= nv) return 9;
  V mn = {verts[0], verts[1], verts[2]}, mx = mn;
  for (int i = 0; i < nv; ++i) {
    mn.x = std::min(mn.x, verts[3 * i]); mx.x = std::max(mx.x, verts[3 * i]);
    mn.y = std::min(mn.y, verts[3 * i + 1]); mx.y = std::max(mx.y, verts[3 * i + 1]);
    mn.z = std::min(mn.z, verts[3 * i + 2]); mx.z = std::max(mx.z, verts[3 * i + 2]);
  }
  const double pitch = 2.0 * radius;
  const int nx = static_cast<int>(std::floor((mx.x - mn.x) / pitch + 1e-12));
  const int ny = static_cast<int>(std::floor((mx.y - mn.y) / pitch + 1e-12));
  const int nz = static_cast<int>(std::floor((mx.z - mn.z) / pitch + 1e-12));
  if (nx < 1 || ny < 1 || nz < 1) return 3;
  V dirs[8];
  for (int a = 0; a < 8; ++a) {
    V d = {0.577350269, 0.577350269, 0.577350269};
    if (a > 0) {
      double u[3];
      mesh::unit3(0x5EEDull + static_cast<uint64_t>(a), u);
      d.x += -0.3 + (0.3 - -0.3) * u[0];
      d.y += -0.3 + (0.3 - -0.3) * u[1];
      d.z += -0.3 + (0.3 - -0.3) * u[2];
    }
    const double n = mesh::norm(d);
    dirs[a] = n > 0.0 ? V{d.x / n, d.y / n, d.z / n} : V{0, 0, 0};
  }
  const long total = static_cast<long>(nx) * ny * nz;
  std::vector<uint8_t> inside(total, 0), amb(total, 0);
#pragma omp parallel for schedule(dynamic, 64)
  for (long i = 0; i < total; ++i) {
    const int iz = static_cast<int>(i % nz), iy = static_cast<int>((i / nz) % ny), ix = static_cast<int>(i / (static_cast<long>(nz) * ny));
    const V p = {mn.x + radius + ix * pitch, mn.y + radius + iy * pitch, mn.z + radius + iz * pitch};
    bool resolved = false;
    for (int a = 0; a < 8 && !resolved; ++a) {
      long crossings = 0;
      bool bad = false;
      for (int t = 0; t < nt && !bad; ++t) {
        const int* T = &tris[3 * t];
        const V A = {verts[3 * T[0]], verts[3 * T[0] + 1], verts[3 * T[0] + 2]};
        const V B = {verts[3 * T[1]], verts[3 * T[1] + 1], verts[3 * T[1] + 2]};
        const V Cc = {verts[3 * T[2]], verts[3 * T[2] + 1], verts[3 * T[2] + 2]};
        const int h = mesh::ray_tri(p, dirs[a], A, B, Cc);
        if (h == 1) ++crossings;
        if (h == 2) bad = true;
      }
      if (!bad) {
        resolved = true;
        inside[i] = (crossings % 2) == 1;
      }
    }
    amb[i] = !resolved;
  }
  long c = 0, am = 0;
  for (long i = 0; i < total; ++i) {
    am += amb[i];
    if (!inside[i]) continue;
    if (centers && c < cap) {
      const int iz = static_cast<int>(i % nz), iy = static_cast<int>((i / nz) % ny), ix = static_cast<int>(i / (static_cast<long>(nz) * ny));
      centers[3 * c] = mn.x + radius + ix * pitch;
      centers[3 * c + 1] = mn.y + radius + iy * pitch;
      centers[3 * c + 2] = mn.z + radius + iz * pitch;
    }
    ++c;
  }
  *count = c;
  *candidates = total;
  *ambiguous = am;
  return c == 0 ? 3 : 0;
}
