// Host fp64 helpers behind include/pbdr/body.hpp, scene.hpp and the packing
// part of geometry.hpp: the reference's body module (proj/include/pbdr/
// body.hpp:38-65, semantics of proj/src/body.cpp), SolverConfig / Scene
// validation and add_packed_body (scene.hpp:30-82), pack_box / pack_rod
// (geometry.hpp:41-46). Used by callers of the drop-in to build scenes and to
// measure trajectories; the device computes per-body statistics itself.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "pbdr/body.hpp"
#include "pbdr/geometry.hpp"
#include "pbdr/scene.hpp"
#include "pbdr_gpu.h"

namespace pbdr {

namespace {

double mass_of(const Particle& p) {
  if (!(p.inv_mass > 0)) throw Error("pinned particles are not supported in rigid bodies");
  return 1.0 / p.inv_mass;
}

const Particle& member(const std::vector<Particle>& ps, int i) {
  if (i < 0 || static_cast<size_t>(i) >= ps.size()) throw Error("body particle index out of range");
  return ps[static_cast<size_t>(i)];
}

// Mass-weighted mean of the members (and the total mass).
Vec3 weighted_mean(const std::vector<Particle>& ps, const std::vector<int>& idx, double* total) {
  double M = 0;
  Vec3 s{0, 0, 0};
  for (const int i : idx) {
    const Particle& p = member(ps, i);
    const double m = mass_of(p);
    M += m;
    s += p.position * m;
  }
  if (total) *total = M;
  return s / M;
}

// Shortest-arc rotation taking direction `a` onto direction `b`.
Rotation shortest_arc(const Vec3& a, const Vec3& b) {
  const Vec3 u = normalized(a), v = normalized(b);
  const Vec3 axis = cross(u, v);
  const double s = norm(axis), c = dot(u, v);
  if (s > 1e-15) return Rotation::axis_angle(axis, std::atan2(s, c));
  if (c > 0) return Rotation();
  // Opposite directions: half a turn about any axis normal to u.
  const Vec3 helper = std::fabs(u.x) < 0.9 ? Vec3{1, 0, 0} : Vec3{0, 1, 0};
  return Rotation::axis_angle(cross(u, helper), M_PI);
}

}  // namespace

Body make_body(const std::vector<Particle>& particles, const std::vector<int>& indices) {
  if (indices.empty()) throw Error("make_body: empty particle set");
  Body b;
  b.particle_indices = indices;
  b.rest_com = weighted_mean(particles, indices, &b.total_mass);
  Mat3 second;  // sum m q q^T of the rest offsets
  b.rest_offsets.reserve(indices.size());
  for (const int i : indices) {
    const Particle& p = member(particles, i);
    const Vec3 q = p.position - b.rest_com;
    b.rest_offsets.push_back(q);
    second += Mat3::outer(q, q) * mass_of(p);
  }
  double ev[3];
  Mat3 V;
  sym_eigen(second, ev, V);
  if (ev[1] <= 1e-8 * std::max(ev[2], 1e-300)) {  // one non-negligible extent: a chain
    b.collinear = true;
    b.rest_axis = normalized(Vec3{V.m[0][2], V.m[1][2], V.m[2][2]});
  }
  return b;
}

Vec3 compute_com(const Body& body, const std::vector<Particle>& particles) {
  return weighted_mean(particles, body.particle_indices, nullptr);
}

Mat3 compute_inertia(const Body& body, const std::vector<Particle>& particles) {
  const Vec3 c = compute_com(body, particles);
  Mat3 I;
  for (const int i : body.particle_indices) {
    const Particle& p = member(particles, i);
    const Vec3 r = p.position - c;
    I += (Mat3::identity() * norm2(r) - Mat3::outer(r, r)) * mass_of(p);
  }
  return I;
}

MomentumState compute_momentum(const Body& body, const std::vector<Particle>& particles) {
  MomentumState s;
  s.com = compute_com(body, particles);
  for (const int i : body.particle_indices) {
    const Particle& p = member(particles, i);
    const Vec3 mv = p.velocity * mass_of(p);
    s.linear += mv;
    s.angular += cross(p.position - s.com, mv);
  }
  return s;
}

Pose extract_pose(const Body& body, const std::vector<Particle>& particles) {
  Pose pose;
  pose.com = compute_com(body, particles);
  Mat3 apq;  // sum m (x - com) q0^T
  for (size_t k = 0; k < body.particle_indices.size(); ++k) {
    const Particle& p = member(particles, body.particle_indices[k]);
    apq += Mat3::outer(p.position - pose.com, body.rest_offsets.at(k)) * mass_of(p);
  }
  if (body.collinear) {
    const Vec3 heading = apq * body.rest_axis;
    if (!(norm(heading) > 1e-15)) throw DegenerateConfigError("extract_pose: collapsed chain");
    pose.orientation = shortest_arc(body.rest_axis, heading);
  } else {
    pose.orientation = polar_decompose(apq).rotation;
  }
  return pose;
}

std::vector<Vec3> distribute_wrench(const Body& body, const std::vector<Particle>& particles, const Vec3& force,
                                    const Vec3& torque) {
  const Vec3 c = compute_com(body, particles);
  Vec3 alpha{0, 0, 0};
  if (norm2(torque) > 0) {
    const SpdPseudoInverse pi = pseudo_invert_spd(compute_inertia(body, particles));
    if (pi.rank < 3 && std::fabs(dot(torque, pi.null_axis)) > 1e-12)
      throw RankDeficientError("torque requested about a singular inertia axis", pi.null_axis.x, pi.null_axis.y,
                               pi.null_axis.z);
    alpha = pi.pinv * torque;
  }
  std::vector<Vec3> f;
  f.reserve(body.particle_indices.size());
  for (const int i : body.particle_indices) {
    const Particle& p = member(particles, i);
    const double m = mass_of(p);
    f.push_back(force * (m / body.total_mass) + cross(alpha, p.position - c) * m);
  }
  return f;
}

// ---- scene.hpp -------------------------------------------------------------
void SolverConfig::validate() const {
  if (!(frame_rate > 0) || !std::isfinite(frame_rate)) throw ConfigError("frame_rate", "must be > 0");
  if (substeps < 1) throw ConfigError("substeps", "must be >= 1");
  if (solver_iterations < 1) throw ConfigError("solver_iterations", "must be >= 1");
  if (!std::isfinite(gravity)) throw ConfigError("gravity", "must be finite");
}

namespace {
void check_plane(const Plane& p, const std::string& key) {
  if (std::fabs(norm(p.normal) - 1.0) > 1e-9) throw ConfigError(key + ".normal", "must be unit length");
  if (!(p.friction >= 0)) throw ConfigError(key + ".friction", "must be >= 0");
}
}  // namespace

void Scene::validate() const {
  check_plane(ground, "ground");
  for (size_t w = 0; w < walls.size(); ++w) check_plane(walls[w], "walls[" + std::to_string(w) + "]");
  if (!programs.empty() && programs.size() != bodies.size())
    throw ConfigError("programs", "must be parallel to bodies");
  if (!body_scene.empty() && body_scene.size() != bodies.size())
    throw ConfigError("body_scene", "must be parallel to bodies");
  if (!(contact_relaxation >= 0)) throw ConfigError("contact_relaxation", "must be >= 0");
}

int add_packed_body(Scene& scene, const std::vector<Vec3>& centers, double radius, double total_mass,
                    const Rotation& rotate, const Vec3& translate, double jitter, uint64_t seed) {
  if (centers.empty()) throw EmptyPackingError("add_packed_body: empty packing");
  if (!(total_mass > 0)) throw ConfigError("total_mass", "must be > 0");
  const int id = static_cast<int>(scene.bodies.size());
  const double inv_mass = static_cast<double>(centers.size()) / total_mass;
  // Rng(seed).next_in(-jitter, jitter) per axis: splitmix64 of rng.hpp:10-29.
  uint64_t state = seed + 0x9E3779B97F4A7C15ull;
  auto unit = [&state]() {
    state += 0x9E3779B97F4A7C15ull;
    uint64_t z = state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    return static_cast<double>(z >> 11) * 0x1.0p-53;
  };
  std::vector<int> idx;
  idx.reserve(centers.size());
  for (const Vec3& c : centers) {
    Particle p;
    p.position = rotate.rotate(c) + translate;
    if (jitter > 0) {
      const double jx = -jitter + 2 * jitter * unit();
      const double jy = -jitter + 2 * jitter * unit();
      const double jz = -jitter + 2 * jitter * unit();
      p.position += Vec3{jx, jy, jz};
    }
    p.inv_mass = inv_mass;
    p.radius = radius;
    p.body_id = id;
    idx.push_back(static_cast<int>(scene.particles.size()));
    scene.particles.push_back(p);
  }
  scene.bodies.push_back(make_body(scene.particles, idx));
  if (!scene.programs.empty()) scene.programs.emplace_back();
  if (!scene.body_scene.empty()) scene.body_scene.push_back(0);
  return id;
}

// ---- geometry.hpp (packing) ------------------------------------------------------
BoundingBox TriMesh::bounds() const {
  BoundingBox bb;
  if (vertices.empty()) return bb;
  bb.min = bb.max = vertices.front();
  for (const Vec3& v : vertices) {
    bb.min = {std::min(bb.min.x, v.x), std::min(bb.min.y, v.y), std::min(bb.min.z, v.z)};
    bb.max = {std::max(bb.max.x, v.x), std::max(bb.max.y, v.y), std::max(bb.max.z, v.z)};
  }
  return bb;
}

void TriMesh::validate() const {
  const long n = static_cast<long>(vertices.size());
  for (const auto& t : triangles)
    for (const int k : t)
      if (k < 0 || k >= n) throw Error("mesh triangle index out of range");
}

SpherePacking pack_box(const Vec3& half_extents, int n_per_axis) {
  SpherePacking p;
  p.centers.resize(static_cast<size_t>(std::max(n_per_axis, 0)) * n_per_axis * n_per_axis);
  const int st = pbdr_pack_box(half_extents.x, half_extents.y, half_extents.z, n_per_axis,
                               p.centers.empty() ? nullptr : &p.centers[0].x, &p.radius);
  if (st != PBDR_OK) throw Error(pbdr_last_error());
  char buf[128];
  std::snprintf(buf, sizeof buf, "box(h=%.9g,%.9g,%.9g,n=%d)", half_extents.x, half_extents.y, half_extents.z,
                n_per_axis);
  p.source = buf;
  return p;
}

SpherePacking pack_rod(double length, double radius) {
  if (!(radius > 0)) throw Error("pack_rod: radius must be positive");
  if (length < 2 * radius) throw Error("pack_rod: length must be >= sphere diameter");
  const double pitch = 2 * radius;
  const int count = static_cast<int>(std::floor(length / pitch + 1e-9));
  SpherePacking p;
  p.radius = radius;
  for (int k = 0; k < count; ++k) p.centers.push_back({pitch * (k - 0.5 * (count - 1)), 0.0, 0.0});
  char buf[96];
  std::snprintf(buf, sizeof buf, "rod(L=%.9g,r=%.9g)", length, radius);
  p.source = buf;
  return p;
}

}  // namespace pbdr
