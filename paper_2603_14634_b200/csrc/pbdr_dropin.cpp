// Implementation of the C++ drop-in's solver layer (include/pbdr/solver.hpp,
// pack_mesh of geometry.hpp) on top of the C-ABI. Conversions only: all
// simulation work runs in the CUDA kernels. The host helpers (math, body,
// scene set-up) live in libpbdr_host.so (csrc/pbdr_hostmath.cpp, pbdr_body.cpp).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "pbdr/pbdr_b200.hpp"

namespace pbdr {

void throw_last_error(int status) {
  // The C-ABI message is already formatted like the reference's what()
  // strings; the exception constructors add the key prefix / frame suffix
  // again, so they get the bare message.
  std::string msg = pbdr_last_error();
  double axis[3] = {0, 0, 0};
  int64_t frame = -1;
  int32_t body = -1;
  pbdr_last_error_payload(axis, &frame, &body);
  switch (status) {
    case PBDR_ERR_DEGENERATE: throw DegenerateConfigError(msg);
    case PBDR_ERR_RANK_DEFICIENT: throw RankDeficientError(msg, axis[0], axis[1], axis[2]);
    case PBDR_ERR_EMPTY_PACKING: throw EmptyPackingError(msg);
    case PBDR_ERR_INVALID_MOMENT: throw InvalidMomentError(msg);
    case PBDR_ERR_CONFIG: {
      const std::string key = pbdr_last_error_key();
      const std::string prefix = "config key '" + key + "': ";
      if (msg.compare(0, prefix.size(), prefix) == 0) msg.erase(0, prefix.size());
      throw ConfigError(key, msg);
    }
    case PBDR_ERR_SIMULATION: {
      const std::string suffix = " (frame " + std::to_string(frame) + ")";
      if (msg.size() >= suffix.size() && msg.compare(msg.size() - suffix.size(), suffix.size(), suffix) == 0)
        msg.erase(msg.size() - suffix.size());
      throw SimulationError(msg, static_cast<long>(frame));
    }
    default: throw Error(msg);
  }
}

static void check(int status) {
  if (status != PBDR_OK) throw_last_error(status);
}

namespace {

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

Solver::Solver(const Scene& scene, const SolverConfig& cfg, int device) : dt_(cfg.dt()) {
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

namespace {

void pack_state(const Scene& scene, std::vector<double>& p, std::vector<double>& v) {
  const size_t n = scene.particles.size();
  p.resize(3 * n);
  v.resize(3 * n);
  for (size_t i = 0; i < n; ++i) {
    const Particle& q = scene.particles[i];
    p[3 * i] = q.position.x; p[3 * i + 1] = q.position.y; p[3 * i + 2] = q.position.z;
    v[3 * i] = q.velocity.x; v[3 * i + 1] = q.velocity.y; v[3 * i + 2] = q.velocity.z;
  }
}

void unpack_state(Scene& scene, const std::vector<double>& p, const std::vector<double>& v) {
  for (size_t i = 0; i < scene.particles.size(); ++i) {
    scene.particles[i].position = {p[3 * i], p[3 * i + 1], p[3 * i + 2]};
    scene.particles[i].velocity = {v[3 * i], v[3 * i + 1], v[3 * i + 2]};
  }
}

}  // namespace

void Solver::download(Scene& scene) const {
  std::vector<double> p(3 * scene.particles.size()), v(p.size());
  check(pbdr_gpu_read_particles(h_, p.data(), v.data()));
  unpack_state(scene, p, v);
}

void Solver::upload(const Scene& scene) {
  std::vector<double> p, v;
  pack_state(scene, p, v);
  check(pbdr_gpu_write_particles(h_, p.data(), v.data()));
}

void Solver::set_time(double t) {
  if (!(t >= 0)) throw ConfigError("time", "must be >= 0");
  check(pbdr_gpu_set_time(h_, static_cast<int64_t>(std::llround(t / dt_))));
}

double Solver::time() const {
  int64_t k = 0;
  check(pbdr_gpu_get_time(h_, &k));
  return static_cast<double>(k) * dt_;
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

namespace {

// FNV-1a over raw bytes: fingerprints of the scene's static part (bodies,
// masses, radii, programs, planes, config) and of the state step() wrote back.
struct Fnv {
  uint64_t h = 1469598103934665603ull;
  void add(const void* data, size_t bytes) {
    const unsigned char* b = static_cast<const unsigned char*>(data);
    for (size_t i = 0; i < bytes; ++i) h = (h ^ b[i]) * 1099511628211ull;
  }
  template <typename T>
  void pod(const T& x) { add(&x, sizeof x); }
};

uint64_t static_fingerprint(const Scene& s, const SolverConfig& c) {
  Fnv f;
  const pbdr_solver_cfg cc = to_c(c);
  f.pod(cc);
  const uint64_t n = s.particles.size(), nb = s.bodies.size();
  f.pod(n);
  f.pod(nb);
  for (const Particle& p : s.particles) {
    f.pod(p.inv_mass);
    f.pod(p.radius);
    f.pod(p.body_id);
  }
  for (const Body& b : s.bodies) {
    f.add(b.particle_indices.data(), sizeof(int) * b.particle_indices.size());
    f.add(b.rest_offsets.data(), sizeof(Vec3) * b.rest_offsets.size());
    f.pod(b.total_mass);
    f.pod(b.rest_com);
  }
  for (const ForceProgram& p : s.programs) {
    f.pod(p.force);
    f.pod(p.torque);
    f.pod(p.t_start);
    f.pod(p.t_stop);
    f.pod(p.gravity_exempt);
  }
  const pbdr_plane g = to_c(s.ground);
  f.pod(g);
  f.pod(s.has_ground);
  f.pod(s.contact_relaxation);
  for (const Plane& w : s.walls) {
    const pbdr_plane pw = to_c(w);
    f.pod(pw);
  }
  f.add(s.body_scene.data(), sizeof(int) * s.body_scene.size());
  return f.h;
}

uint64_t state_fingerprint(const std::vector<double>& p, const std::vector<double>& v) {
  Fnv f;
  f.add(p.data(), sizeof(double) * p.size());
  f.add(v.data(), sizeof(double) * v.size());
  return f.h;
}

// One cached device handle per thread for the stateless step().
struct StepCache {
  const Scene* scene = nullptr;
  uint64_t statics = 0;
  uint64_t written = 0;  // fingerprint of the state the last call wrote back
  std::unique_ptr<Solver> solver;
};
thread_local StepCache g_step;

}  // namespace

void step(Scene& scene, const SolverConfig& cfg, double t) {
  StepCache& c = g_step;
  const uint64_t statics = static_fingerprint(scene, cfg);
  std::vector<double> p, v;
  pack_state(scene, p, v);
  const bool same_scene = c.solver && c.scene == &scene && c.statics == statics;
  if (!same_scene) {
    c.solver.reset();  // free the previous scene's device memory first
    c.solver = std::make_unique<Solver>(scene, cfg, 0);
    c.scene = &scene;
    c.statics = statics;
    if (t > 0) c.solver->set_time(t);
  } else if (t >= 0 || state_fingerprint(p, v) != c.written) {
    // A new state (or an explicit clock): the step of a fresh handle on it.
    c.solver->upload(scene);
    c.solver->set_time(t >= 0 ? t : 0.0);
  }  // else: continue from the device state and clock this call left
  c.written = 0;
  try {
    c.solver->step(1);
  } catch (...) {
    c.solver.reset();  // a failed step leaves the device error record set
    c.scene = nullptr;
    throw;
  }
  c.solver->download(scene);
  pack_state(scene, p, v);
  c.written = state_fingerprint(p, v);
}

}  // namespace pbdr
