// Implementation of the C++ drop-in layer (include/pbdr/pbdr_b200.hpp) on top
// of the C-ABI. Conversions only: all simulation work runs in the CUDA kernels.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "pbdr/pbdr_b200.hpp"

namespace pbdr {

void throw_last_error(int status) {
  const std::string msg = pbdr_last_error();
  double axis[3] = {0, 0, 0};
  int64_t frame = -1;
  int32_t body = -1;
  pbdr_last_error_payload(axis, &frame, &body);
  switch (status) {
    case PBDR_ERR_DEGENERATE: throw DegenerateConfigError(msg);
    case PBDR_ERR_RANK_DEFICIENT: throw RankDeficientError(msg, axis[0], axis[1], axis[2]);
    case PBDR_ERR_EMPTY_PACKING: throw EmptyPackingError(msg);
    case PBDR_ERR_INVALID_MOMENT: throw InvalidMomentError(msg);
    case PBDR_ERR_CONFIG: throw ConfigError(pbdr_last_error_key(), msg);
    case PBDR_ERR_SIMULATION: throw SimulationError(msg, static_cast<long>(frame));
    default: throw Error(msg);
  }
}

static void check(int status) {
  if (status != PBDR_OK) throw_last_error(status);
}

namespace {

// Largest/middle eigenvalue test for a chain-like rest shape (body.cpp:39-46
// semantics): collinear when the middle principal second moment is negligible.
void collinearity(const std::vector<Vec3>& q, const std::vector<double>& m, Body& b) {
  double S[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  for (size_t k = 0; k < q.size(); ++k) {
    const double v[3] = {q[k].x, q[k].y, q[k].z};
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) S[i][j] += m[k] * v[i] * v[j];
  }
  double V[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  for (int sweep = 0; sweep < 32; ++sweep) {
    const double off = std::fabs(S[0][1]) + std::fabs(S[0][2]) + std::fabs(S[1][2]);
    if (off <= 1e-15 * (std::fabs(S[0][0]) + std::fabs(S[1][1]) + std::fabs(S[2][2]) + 1e-300)) break;
    for (int p = 0; p < 2; ++p)
      for (int r = p + 1; r < 3; ++r) {
        if (S[p][r] == 0.0) continue;
        const double th = (S[r][r] - S[p][p]) / (2 * S[p][r]);
        const double t = (th >= 0 ? 1.0 : -1.0) / (std::fabs(th) + std::sqrt(th * th + 1));
        const double c = 1 / std::sqrt(t * t + 1), s = t * c;
        for (int k = 0; k < 3; ++k) {
          const double a = S[k][p], bb = S[k][r];
          S[k][p] = c * a - s * bb;
          S[k][r] = s * a + c * bb;
        }
        for (int k = 0; k < 3; ++k) {
          const double a = S[p][k], bb = S[r][k];
          S[p][k] = c * a - s * bb;
          S[r][k] = s * a + c * bb;
        }
        for (int k = 0; k < 3; ++k) {
          const double a = V[k][p], bb = V[k][r];
          V[k][p] = c * a - s * bb;
          V[k][r] = s * a + c * bb;
        }
      }
  }
  int idx[3] = {0, 1, 2};
  std::sort(idx, idx + 3, [&](int a, int c) { return S[a][a] < S[c][c]; });
  const double mid = S[idx[1]][idx[1]], top = S[idx[2]][idx[2]];
  if (mid <= 1e-8 * std::max(top, 1e-300)) {
    b.collinear = true;
    const int k = idx[2];
    const double n = std::sqrt(V[0][k] * V[0][k] + V[1][k] * V[1][k] + V[2][k] * V[2][k]);
    b.rest_axis = {V[0][k] / n, V[1][k] / n, V[2][k] / n};
  }
}

struct Flat {
  std::vector<double> pos, vel, inv_mass, radius, rest, mass, com;
  std::vector<int32_t> body_id, indices, scene;
  std::vector<int64_t> offsets;
  std::vector<pbdr_force_program> programs;
  std::vector<pbdr_plane> walls;
  pbdr_scene_desc desc{};
};

pbdr_plane to_c(const Plane& p) {
  pbdr_plane c{};
  c.point[0] = p.point.x; c.point[1] = p.point.y; c.point[2] = p.point.z;
  c.normal[0] = p.normal.x; c.normal[1] = p.normal.y; c.normal[2] = p.normal.z;
  c.friction = p.friction;
  return c;
}

void flatten(const Scene& s, Flat& f) {
  const size_t n = s.particles.size();
  f.pos.resize(3 * n);
  f.vel.resize(3 * n);
  f.inv_mass.resize(n);
  f.radius.resize(n);
  f.body_id.resize(n);
  for (size_t i = 0; i < n; ++i) {
    const Particle& p = s.particles[i];
    f.pos[3 * i] = p.position.x; f.pos[3 * i + 1] = p.position.y; f.pos[3 * i + 2] = p.position.z;
    f.vel[3 * i] = p.velocity.x; f.vel[3 * i + 1] = p.velocity.y; f.vel[3 * i + 2] = p.velocity.z;
    f.inv_mass[i] = p.inv_mass;
    f.radius[i] = p.radius;
    f.body_id[i] = p.body_id;
  }
  f.offsets.assign(1, 0);
  for (const Body& b : s.bodies) {
    for (size_t k = 0; k < b.particle_indices.size(); ++k) {
      f.indices.push_back(b.particle_indices[k]);
      const Vec3 q = k < b.rest_offsets.size() ? b.rest_offsets[k] : Vec3{};
      f.rest.insert(f.rest.end(), {q.x, q.y, q.z});
    }
    f.offsets.push_back(static_cast<int64_t>(f.indices.size()));
    f.mass.push_back(b.total_mass);
    f.com.insert(f.com.end(), {b.rest_com.x, b.rest_com.y, b.rest_com.z});
  }
  for (const ForceProgram& p : s.programs) {
    pbdr_force_program c{};
    c.force[0] = p.force.x; c.force[1] = p.force.y; c.force[2] = p.force.z;
    c.torque[0] = p.torque.x; c.torque[1] = p.torque.y; c.torque[2] = p.torque.z;
    c.t_start = p.t_start;
    c.t_stop = p.t_stop;
    c.gravity_exempt = p.gravity_exempt ? 1 : 0;
    f.programs.push_back(c);
  }
  for (const Plane& w : s.walls) f.walls.push_back(to_c(w));
  f.scene = s.body_scene;
  pbdr_scene_desc& d = f.desc;
  d.num_particles = static_cast<int64_t>(n);
  d.position = f.pos.data();
  d.velocity = f.vel.data();
  d.inv_mass = f.inv_mass.data();
  d.radius = f.radius.data();
  d.body_id = f.body_id.data();
  d.num_bodies = static_cast<int32_t>(s.bodies.size());
  d.body_offsets = f.offsets.data();
  d.body_indices = f.indices.data();
  d.rest_offsets = f.rest.data();
  d.total_mass = f.mass.data();
  d.rest_com = f.com.data();
  d.programs = f.programs.size() == s.bodies.size() && !f.programs.empty() ? f.programs.data() : nullptr;
  d.ground = to_c(s.ground);
  d.has_ground = s.has_ground ? 1 : 0;
  d.contact_relaxation = s.contact_relaxation;
  d.num_walls = static_cast<int32_t>(f.walls.size());
  d.walls = f.walls.empty() ? nullptr : f.walls.data();
  d.body_scene = f.scene.size() == s.bodies.size() && !f.scene.empty() ? f.scene.data() : nullptr;
}

pbdr_solver_cfg to_c(const SolverConfig& c) {
  pbdr_solver_cfg o{};
  o.frame_rate = c.frame_rate;
  o.substeps = c.substeps;
  o.solver_iterations = c.solver_iterations;
  o.precision = c.precision == Precision::kSingle ? PBDR_PRECISION_SINGLE : PBDR_PRECISION_DOUBLE;
  o.velocity_update =
      c.velocity_update == VelocityUpdate::kIncremental ? PBDR_VELOCITY_INCREMENTAL : PBDR_VELOCITY_LEGACY;
  o.linear_momentum_fix = c.linear_momentum_fix ? 1 : 0;
  o.angular_momentum_fix = c.angular_momentum_fix ? 1 : 0;
  o.momentum_frequency = c.momentum_frequency == MomentumFrequency::kPerIteration
                             ? PBDR_MOMENTUM_PER_ITERATION
                             : PBDR_MOMENTUM_PER_SUBSTEP;
  o.backend = c.backend == Backend::kSerial ? PBDR_BACKEND_SERIAL : PBDR_BACKEND_PARALLEL;
  o.gravity = c.gravity;
  return o;
}

}  // namespace

Body make_body(const std::vector<Particle>& particles, const std::vector<int>& indices) {
  if (indices.empty()) throw Error("make_body: empty particle set");
  Body b;
  b.particle_indices = indices;
  double mass = 0;
  Vec3 wsum{0, 0, 0};
  std::vector<double> m;
  m.reserve(indices.size());
  for (int i : indices) {
    const Particle& p = particles.at(static_cast<size_t>(i));
    if (!(p.inv_mass > 0)) throw Error("pinned particles are not supported in rigid bodies");
    const double mi = 1.0 / p.inv_mass;
    m.push_back(mi);
    mass += mi;
    wsum += p.position * mi;
  }
  b.total_mass = mass;
  b.rest_com = wsum / mass;
  for (int i : indices) b.rest_offsets.push_back(particles[static_cast<size_t>(i)].position - b.rest_com);
  collinearity(b.rest_offsets, m, b);
  return b;
}

SpherePacking pack_mesh(const TriMesh& mesh, double radius, int device) {
  std::vector<double> v;
  v.reserve(3 * mesh.vertices.size());
  for (const Vec3& p : mesh.vertices) {
    v.push_back(p.x);
    v.push_back(p.y);
    v.push_back(p.z);
  }
  std::vector<int32_t> t;
  t.reserve(3 * mesh.triangles.size());
  for (const auto& tri : mesh.triangles)
    for (int k = 0; k < 3; ++k) t.push_back(tri[k]);
  int64_t count = 0, cand = 0, amb = 0;
  check(pbdr_pack_mesh(v.data(), static_cast<int32_t>(mesh.vertices.size()), t.data(),
                       static_cast<int32_t>(mesh.triangles.size()), radius, device, nullptr, 0, &count, &cand, &amb));
  std::vector<double> c(3 * static_cast<size_t>(count));
  check(pbdr_pack_mesh(v.data(), static_cast<int32_t>(mesh.vertices.size()), t.data(),
                       static_cast<int32_t>(mesh.triangles.size()), radius, device, c.data(), count, &count, &cand,
                       &amb));
  SpherePacking p;
  p.radius = radius;
  p.candidate_count = static_cast<long>(cand);
  p.ambiguous_count = static_cast<long>(amb);
  for (int64_t i = 0; i < count; ++i) p.centers.push_back({c[3 * i], c[3 * i + 1], c[3 * i + 2]});
  return p;
}

int add_packed_body(Scene& scene, const std::vector<Vec3>& centers, double radius,
                    double total_mass, const Rotation& rotate, const Vec3& translate,
                    double jitter, uint64_t seed) {
  if (centers.empty()) throw EmptyPackingError("add_packed_body: empty packing");
  if (!(total_mass > 0)) throw ConfigError("total_mass", "must be > 0");
  const int id = static_cast<int>(scene.bodies.size());
  const double inv_mass = static_cast<double>(centers.size()) / total_mass;
  uint64_t state = seed + 0x9E3779B97F4A7C15ull;  // splitmix64 (rng.hpp:10-29)
  auto unit = [&]() {
    state += 0x9E3779B97F4A7C15ull;
    uint64_t z = state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z = z ^ (z >> 31);
    return static_cast<double>(z >> 11) * (1.0 / 9007199254740992.0);
  };
  std::vector<int> idx;
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

void SolverConfig::validate() const {
  if (!(frame_rate > 0)) throw ConfigError("frame_rate", "must be > 0");
  if (substeps < 1) throw ConfigError("substeps", "must be >= 1");
  if (solver_iterations < 1) throw ConfigError("solver_iterations", "must be >= 1");
}

void Scene::validate() const {
  const double nn = std::sqrt(ground.normal.x * ground.normal.x + ground.normal.y * ground.normal.y +
                              ground.normal.z * ground.normal.z);
  if (std::fabs(nn - 1.0) > 1e-9) throw ConfigError("ground.normal", "must be unit length");
  if (ground.friction < 0) throw ConfigError("ground.friction", "must be >= 0");
  if (!programs.empty() && programs.size() != bodies.size())
    throw ConfigError("programs", "must be parallel to bodies");
}

Solver::Solver(const Scene& scene, const SolverConfig& cfg, int device) {
  scene.validate();
  cfg.validate();
  Flat f;
  flatten(scene, f);
  const pbdr_solver_cfg c = to_c(cfg);
  check(pbdr_gpu_create(&f.desc, &c, device, &h_));
}

Solver::~Solver() { pbdr_gpu_destroy(h_); }

void Solver::step(long substeps) { check(pbdr_gpu_step(h_, substeps)); }
void Solver::step_frames(long frames) { check(pbdr_gpu_step_frames(h_, frames)); }

void Solver::download(Scene& scene) const {
  const size_t n = scene.particles.size();
  std::vector<double> p(3 * n), v(3 * n);
  check(pbdr_gpu_read_particles(h_, p.data(), v.data()));
  for (size_t i = 0; i < n; ++i) {
    scene.particles[i].position = {p[3 * i], p[3 * i + 1], p[3 * i + 2]};
    scene.particles[i].velocity = {v[3 * i], v[3 * i + 1], v[3 * i + 2]};
  }
}

void Solver::upload(const Scene& scene) {
  const size_t n = scene.particles.size();
  std::vector<double> p(3 * n), v(3 * n);
  for (size_t i = 0; i < n; ++i) {
    const Particle& q = scene.particles[i];
    p[3 * i] = q.position.x; p[3 * i + 1] = q.position.y; p[3 * i + 2] = q.position.z;
    v[3 * i] = q.velocity.x; v[3 * i + 1] = q.velocity.y; v[3 * i + 2] = q.velocity.z;
  }
  check(pbdr_gpu_write_particles(h_, p.data(), v.data()));
}

std::vector<pbdr_body_stats> Solver::body_stats() const {
  pbdr_info in{};
  check(pbdr_gpu_info(h_, &in));
  std::vector<pbdr_body_stats> out(static_cast<size_t>(in.num_bodies));
  check(pbdr_gpu_read_bodies(h_, out.data()));
  return out;
}

pbdr_info Solver::info() const {
  pbdr_info in{};
  check(pbdr_gpu_info(h_, &in));
  return in;
}

void step(Scene& scene, const SolverConfig& cfg) {
  Solver s(scene, cfg, 0);
  s.step(1);
  s.download(scene);
}

}  // namespace pbdr
