// TEST INFRASTRUCTURE ONLY. Never linked into the product library.
//
// extern "C" shim over the reference's own shipped math/body/geometry code
// (/root/reference/proj/src/{math,body,geometry}.cpp), compiled in place by
// oracle/Makefile into oracle/_ref/libpbdr_ref.so. It lets the Python tests
// and tests/golden/make_golden.py evaluate the reference's functions on fixed
// inputs, which pins the oracle's restatement of the same numerics
// (oracle/pbdr_oracle.cpp) and the product's host-side scene construction.
//
// Only the reference's public declarations are used:
//   math.hpp:149-164 (inverse/sym_eigen/invert_spd/pseudo_invert_spd),
//   math.hpp:224-239 (polar_decompose, geodesic_angle_deg, unwrapped_angle_deg),
//   body.hpp:37-66 (make_body, compute_com/inertia/momentum, extract_pose,
//   distribute_wrench), geometry.hpp:41-46 (pack_box, pack_rod), rng.hpp:10-29.
#include <cstdint>
#include <cstring>
#include <vector>

#include "pbdr/body.hpp"
#include "pbdr/errors.hpp"
#include "pbdr/geometry.hpp"
#include "pbdr/math.hpp"
#include "pbdr/rng.hpp"

using namespace pbdr;

namespace {

Mat3 load_m(const double* a) {
  Mat3 m;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) m.m[i][j] = a[3 * i + j];
  return m;
}

void store_m(const Mat3& m, double* a) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) a[3 * i + j] = m.m[i][j];
}

std::vector<Particle> make_particles(int n, const double* pos, const double* vel,
                                     const double* inv_mass) {
  std::vector<Particle> ps(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) {
    ps[i].position = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
    if (vel) ps[i].velocity = {vel[3 * i], vel[3 * i + 1], vel[3 * i + 2]};
    ps[i].inv_mass = inv_mass[i];
    ps[i].body_id = 0;
  }
  return ps;
}

std::vector<int> iota(int n) {
  std::vector<int> v(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) v[i] = i;
  return v;
}

}  // namespace

extern "C" {

// Status: 0 ok, 1 DegenerateConfigError, 2 RankDeficientError, 9 other Error.
#define REF_GUARD(...)                                                  \
  try {                                                                  \
    __VA_ARGS__;                                                              \
  } catch (const RankDeficientError& e) {                                \
    if (axis_out) {                                                      \
      axis_out[0] = e.axis_x; axis_out[1] = e.axis_y; axis_out[2] = e.axis_z; \
    }                                                                    \
    return 2;                                                            \
  } catch (const DegenerateConfigError&) {                               \
    return 1;                                                            \
  } catch (const Error&) {                                               \
    return 9;                                                            \
  }                                                                      \
  return 0;

void ref_rng_u64(uint64_t seed, int count, uint64_t* out) {
  Rng r(seed);
  for (int i = 0; i < count; ++i) out[i] = r.next_u64();
}

void ref_rng_unit(uint64_t seed, int count, double* out) {
  Rng r(seed);
  for (int i = 0; i < count; ++i) out[i] = r.next_unit();
}

int ref_pack_box(double hx, double hy, double hz, int n, double* centers, double* radius) {
  SpherePacking p = pack_box({hx, hy, hz}, n);
  for (size_t i = 0; i < p.centers.size(); ++i) {
    centers[3 * i] = p.centers[i].x;
    centers[3 * i + 1] = p.centers[i].y;
    centers[3 * i + 2] = p.centers[i].z;
  }
  *radius = p.radius;
  return static_cast<int>(p.centers.size());
}

// pack_mesh (geometry.cpp:151-195): returns the status (0 ok, 3 EmptyPackingError,
// 9 other Error); centers in grid order.
int ref_pack_mesh(const double* verts, int nv, const int* tris, int nt, double radius, double* centers,
                  long cap, long* count, long* candidates, long* ambiguous) {
  TriMesh m;
  for (int i = 0; i < nv; ++i) m.vertices.push_back({verts[3 * i], verts[3 * i + 1], verts[3 * i + 2]});
  for (int t = 0; t < nt; ++t) m.triangles.push_back({tris[3 * t], tris[3 * t + 1], tris[3 * t + 2]});
  try {
    SpherePacking p = pack_mesh(m, radius);
    *count = static_cast<long>(p.centers.size());
    *candidates = p.candidate_count;
    *ambiguous = p.ambiguous_count;
    for (size_t i = 0; i < p.centers.size() && static_cast<long>(i) < cap; ++i) {
      centers[3 * i] = p.centers[i].x;
      centers[3 * i + 1] = p.centers[i].y;
      centers[3 * i + 2] = p.centers[i].z;
    }
  } catch (const EmptyPackingError&) {
    return 3;
  } catch (const Error&) {
    return 9;
  }
  return 0;
}

int ref_polar(const double* a, double* r_out, double* s_out, double* q_out, double det_tol) {
  double* axis_out = nullptr;
  REF_GUARD({
    PolarResult pr = polar_decompose(load_m(a), det_tol);
    store_m(pr.rotation.to_matrix(), r_out);
    store_m(pr.stretch, s_out);
    q_out[0] = pr.rotation.w; q_out[1] = pr.rotation.x;
    q_out[2] = pr.rotation.y; q_out[3] = pr.rotation.z;
  })
}

int ref_sym_eigen(const double* a, double* values, double* vectors) {
  double* axis_out = nullptr;
  REF_GUARD({
    Mat3 v;
    sym_eigen(load_m(a), values, v);
    store_m(v, vectors);
  })
}

int ref_invert_spd(const double* a, double* out, double* axis_out) {
  REF_GUARD({ store_m(invert_spd(load_m(a)), out); })
}

int ref_pseudo_invert_spd(const double* a, double* out, int* rank, double* null_axis) {
  double* axis_out = nullptr;
  REF_GUARD({
    SpdPseudoInverse p = pseudo_invert_spd(load_m(a));
    store_m(p.pinv, out);
    *rank = p.rank;
    null_axis[0] = p.null_axis.x; null_axis[1] = p.null_axis.y; null_axis[2] = p.null_axis.z;
  })
}

int ref_inverse(const double* a, double* out) {
  double* axis_out = nullptr;
  REF_GUARD({ store_m(inverse(load_m(a)), out); })
}

// Rest pose = pos; returns com, inertia, P, L (about com) and the collinear flag.
int ref_body_props(int n, const double* pos, const double* vel, const double* inv_mass,
                   double* com, double* inertia, double* lin, double* ang, int* collinear,
                   double* rest_axis) {
  double* axis_out = nullptr;
  REF_GUARD({
    std::vector<Particle> ps = make_particles(n, pos, vel, inv_mass);
    Body b = make_body(ps, iota(n));
    Vec3 c = compute_com(b, ps);
    com[0] = c.x; com[1] = c.y; com[2] = c.z;
    store_m(compute_inertia(b, ps), inertia);
    MomentumState m = compute_momentum(b, ps);
    lin[0] = m.linear.x; lin[1] = m.linear.y; lin[2] = m.linear.z;
    ang[0] = m.angular.x; ang[1] = m.angular.y; ang[2] = m.angular.z;
    *collinear = b.collinear ? 1 : 0;
    rest_axis[0] = b.rest_axis.x; rest_axis[1] = b.rest_axis.y; rest_axis[2] = b.rest_axis.z;
  })
}

// Body made at rest_pos; pose extracted at cur_pos.
int ref_extract_pose(int n, const double* rest_pos, const double* cur_pos,
                     const double* inv_mass, double* com, double* quat) {
  double* axis_out = nullptr;
  REF_GUARD({
    std::vector<Particle> ps = make_particles(n, rest_pos, nullptr, inv_mass);
    Body b = make_body(ps, iota(n));
    for (int i = 0; i < n; ++i)
      ps[i].position = {cur_pos[3 * i], cur_pos[3 * i + 1], cur_pos[3 * i + 2]};
    Pose p = extract_pose(b, ps);
    com[0] = p.com.x; com[1] = p.com.y; com[2] = p.com.z;
    quat[0] = p.orientation.w; quat[1] = p.orientation.x;
    quat[2] = p.orientation.y; quat[3] = p.orientation.z;
  })
}

int ref_distribute_wrench(int n, const double* pos, const double* inv_mass, const double* force,
                          const double* torque, double* forces_out, double* axis_out) {
  REF_GUARD({
    std::vector<Particle> ps = make_particles(n, pos, nullptr, inv_mass);
    Body b = make_body(ps, iota(n));
    std::vector<Vec3> f = distribute_wrench(b, ps, {force[0], force[1], force[2]},
                                            {torque[0], torque[1], torque[2]});
    for (int i = 0; i < n; ++i) {
      forces_out[3 * i] = f[i].x; forces_out[3 * i + 1] = f[i].y; forces_out[3 * i + 2] = f[i].z;
    }
  })
}

double ref_geodesic_deg(const double* qa, const double* qb) {
  return geodesic_angle_deg(Rotation(qa[0], qa[1], qa[2], qa[3]),
                            Rotation(qb[0], qb[1], qb[2], qb[3]));
}

double ref_unwrapped_deg(const double* qa, const double* qb) {
  return unwrapped_angle_deg(Rotation(qa[0], qa[1], qa[2], qa[3]),
                             Rotation(qb[0], qb[1], qb[2], qb[3]));
}

void ref_quat_to_matrix(const double* q, double* m) {
  store_m(Rotation(q[0], q[1], q[2], q[3]).to_matrix(), m);
}

void ref_matrix_to_quat(const double* m, double* q) {
  Rotation r = Rotation::from_matrix(load_m(m));
  q[0] = r.w; q[1] = r.x; q[2] = r.y; q[3] = r.z;
}

}  // extern "C"
