// C++ drop-in API test driver: exercises pbdr::Scene / SolverConfig / step()
// / Solver the way the reference's own solver tests would (SPEC.md:326-334
// worked examples), through the B200 C-ABI. Run by tests/test_dropin_cpp.py on
// a GPU box; exits non-zero on the first failure.
#include <cmath>
#include <algorithm>
#include <cstdio>
#include <string>
#include <vector>

// The reference's own include paths (proj/include/pbdr/...), unchanged.
#include "pbdr/body.hpp"
#include "pbdr/errors.hpp"
#include "pbdr/math.hpp"
#include "pbdr/scene.hpp"
#include "pbdr/solver.hpp"

namespace {

int failures = 0;

#define EXPECT(cond, ...)                    \
  do {                                       \
    if (!(cond)) {                           \
      std::printf("FAIL %s:%d: ", __FILE__, __LINE__); \
      std::printf(__VA_ARGS__);              \
      std::printf("\n");                     \
      ++failures;                            \
    }                                        \
  } while (0)

std::vector<pbdr::Vec3> lattice(int n, double r) {
  std::vector<pbdr::Vec3> c;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      for (int k = 0; k < n; ++k)
        c.push_back({(i - 0.5 * (n - 1)) * 2 * r, (j - 0.5 * (n - 1)) * 2 * r, (k - 0.5 * (n - 1)) * 2 * r});
  return c;
}

pbdr::Vec3 com_of(const pbdr::Scene& s) {
  pbdr::Vec3 c{0, 0, 0};
  double m = 0;
  for (const auto& p : s.particles) {
    c += p.position * (1.0 / p.inv_mass);
    m += 1.0 / p.inv_mass;
  }
  return c / m;
}

// free body, no gravity, v0 = (1,0,0), 100 steps of dt = 1 ms ->
// com displaced 0.1 m along x.
void free_flight() {
  pbdr::Scene s;
  s.has_ground = false;
  pbdr::add_packed_body(s, lattice(4, 0.025), 0.025, 4.0, pbdr::Rotation(), {0, 0, 1}, 0.0, 0);
  for (auto& p : s.particles) p.velocity = {1, 0, 0};
  pbdr::SolverConfig cfg;  // 100 Hz x 10 substeps -> dt = 1 ms
  cfg.gravity = 0.0;
  const pbdr::Vec3 c0 = com_of(s);
  pbdr::Solver solver(s, cfg);
  solver.step(100);
  solver.download(s);
  const pbdr::Vec3 c1 = com_of(s);
  EXPECT(std::fabs((c1.x - c0.x) - 0.1) < 1e-5, "free flight dx = %.9g", c1.x - c0.x);
  EXPECT(std::fabs(c1.y - c0.y) < 1e-6 && std::fabs(c1.z - c0.z) < 1e-6, "free flight drift");
  const auto st = solver.body_stats();
  EXPECT(std::fabs(st[0].linear[0] - 4.0) < 1e-4, "P_x = %.9g", st[0].linear[0]);
}

// with all dX = 0, V_{i+1} = V~ in incremental mode. A translating
// rigid body has dX = 0 up to fp32 rounding of the shape-matching goal, so the
// velocity is unchanged to within rounding / dt.
void zero_delta_velocity() {
  pbdr::Scene s;
  s.has_ground = false;
  pbdr::add_packed_body(s, lattice(3, 0.05), 0.05, 1.0, pbdr::Rotation(), {0, 0, 0}, 0.0, 0);
  for (auto& p : s.particles) p.velocity = {0.25, -0.5, 0.125};
  pbdr::SolverConfig cfg;
  cfg.gravity = 0.0;
  pbdr::step(s, cfg);
  double worst = 0;
  for (const auto& p : s.particles)
    worst = std::max({worst, std::fabs(p.velocity.x - 0.25), std::fabs(p.velocity.y + 0.5),
                      std::fabs(p.velocity.z - 0.125)});
  EXPECT(worst < 1e-4, "incremental update must return V~ when dX = 0 (|dv| = %.3g)", worst);
}

// Resting box on the ground: com stays put (SPEC.md:333 statics, short run).
void resting_box() {
  pbdr::Scene s;
  s.ground.friction = 0.4;
  pbdr::add_packed_body(s, lattice(4, 0.025), 0.025, 4.0, pbdr::Rotation(), {0, 0, 0.1}, 0.0, 0);
  pbdr::SolverConfig cfg;
  const pbdr::Vec3 c0 = com_of(s);
  pbdr::Solver solver(s, cfg);
  solver.step_frames(100);
  solver.download(s);
  const pbdr::Vec3 c1 = com_of(s);
  const double d = std::sqrt((c1.x - c0.x) * (c1.x - c0.x) + (c1.y - c0.y) * (c1.y - c0.y) +
                             (c1.z - c0.z) * (c1.z - c0.z));
  EXPECT(d < 1e-3, "resting box drift %.3g m", d);
}

void config_errors() {
  pbdr::Scene s;
  pbdr::add_packed_body(s, lattice(2, 0.05), 0.05, 1.0, pbdr::Rotation(), {0, 0, 1}, 0.0, 0);
  pbdr::SolverConfig cfg;
  cfg.precision = pbdr::Precision::kDouble;
  bool threw = false;
  try {
    pbdr::Solver solver(s, cfg);
  } catch (const pbdr::ConfigError& e) {
    threw = e.key_path == "precision";
  }
  EXPECT(threw, "kDouble must raise ConfigError('precision')");
}

// step(scene, cfg) -> scene at t + dt. Stateless calls carry the
// clock: a force window [10 dt, 11 dt) opens on the 11th consecutive call,
// exactly as in a resident Solver; an explicit t starts the clock there.
void stateless_step_carries_time() {
  pbdr::SolverConfig cfg;
  cfg.gravity = 0.0;
  const double dt = cfg.dt();
  auto make = [&]() {
    pbdr::Scene s;
    s.has_ground = false;
    pbdr::add_packed_body(s, lattice(3, 0.05), 0.05, 1.0, pbdr::Rotation(), {0, 0, 1}, 0.0, 0);
    s.programs.resize(1);
    s.programs[0].force = {2.0, 0, 0};
    s.programs[0].t_start = 10 * dt;
    s.programs[0].t_stop = 11 * dt;
    return s;
  };
  pbdr::Scene a = make();
  for (int k = 0; k < 12; ++k) pbdr::step(a, cfg);
  const pbdr::MomentumState ma = pbdr::compute_momentum(a.bodies[0], a.particles);
  EXPECT(std::fabs(ma.linear.x - 2.0 * dt) < 1e-6, "window applied once: P_x = %.9g", ma.linear.x);
  pbdr::Scene b = make();
  pbdr::Solver solver(b, cfg);
  solver.step(12);
  solver.download(b);
  double worst = 0;
  for (size_t i = 0; i < a.particles.size(); ++i)
    worst = std::max(worst, pbdr::norm(a.particles[i].position - b.particles[i].position));
  EXPECT(worst == 0.0, "12 stateless steps == Solver::step(12) bit for bit (max |dx| %.3g)", worst);
  EXPECT(std::fabs(solver.time() - 12 * dt) < 1e-12, "Solver::time %.9g", solver.time());
  pbdr::Scene c = make();
  pbdr::step(c, cfg, 10 * dt);  // explicit clock: the window is open for this step
  const pbdr::MomentumState mc = pbdr::compute_momentum(c.bodies[0], c.particles);
  EXPECT(std::fabs(mc.linear.x - 2.0 * dt) < 1e-6, "explicit t: P_x = %.9g", mc.linear.x);
}

// errors.hpp:32-44 message formats through the C-ABI.
void error_formats() {
  pbdr::Scene s;
  s.has_ground = false;
  pbdr::add_packed_body(s, lattice(2, 0.05), 0.05, 1.0, pbdr::Rotation(), {0, 0, 1}, 0.0, 0);
  pbdr::SolverConfig cfg;
  cfg.precision = pbdr::Precision::kDouble;
  try {
    pbdr::Solver solver(s, cfg);
    EXPECT(false, "expected ConfigError");
  } catch (const pbdr::ConfigError& e) {
    const std::string w = e.what();
    EXPECT(w.rfind("config key 'precision': ", 0) == 0 && w.find("config key", 5) == std::string::npos,
           "ConfigError what() = %s", e.what());
  }
  // A NaN velocity: SimulationError "... (frame 0)" exactly once.
  pbdr::Scene n;
  n.has_ground = false;
  pbdr::add_packed_body(n, lattice(3, 0.05), 0.05, 1.0, pbdr::Rotation(), {0, 0, 1}, 0.0, 0);
  n.particles[3].velocity.x = std::nan("");
  try {
    pbdr::step(n, pbdr::SolverConfig{});
    EXPECT(false, "expected SimulationError");
  } catch (const pbdr::SimulationError& e) {
    const std::string w = e.what();
    EXPECT(e.frame_index == 0 && w.size() > 10 && w.compare(w.size() - 10, 10, " (frame 0)") == 0 &&
               w.find("(frame", 0) == w.rfind("(frame"),
           "SimulationError what() = %s", e.what());
  }
}

// body.hpp helpers on a host scene (pinned against the reference's compiled
// code in tests/test_dropin_headers.py): a cube rotated by R reports R.
void host_helpers() {
  pbdr::Scene s;
  pbdr::add_packed_body(s, lattice(4, 0.025), 0.025, 4.0, pbdr::Rotation(), {0, 0, 1}, 0.0, 0);
  const pbdr::Rotation R = pbdr::Rotation::axis_angle({1, 2, 3}, 0.7);
  std::vector<pbdr::Particle> moved = s.particles;
  for (auto& p : moved) p.position = R.rotate(p.position - pbdr::Vec3{0, 0, 1}) + pbdr::Vec3{1, 2, 3};
  const pbdr::Pose pose = pbdr::extract_pose(s.bodies[0], moved);
  EXPECT(pbdr::geodesic_angle_deg(pose.orientation, R) < 1e-6, "pose angle");
  EXPECT(pbdr::norm(pose.com - pbdr::Vec3{1, 2, 3}) < 1e-12, "pose com");
  const pbdr::Mat3 I = pbdr::compute_inertia(s.bodies[0], s.particles);
  EXPECT(std::fabs(I(0, 0) - 0.025) < 1e-12, "I_xx = %.12g (SPEC.md: 0.025)", I(0, 0));
  const auto f = pbdr::distribute_wrench(s.bodies[0], s.particles, {1, 0, 0}, {0, 0, 0.5});
  pbdr::Vec3 F{0, 0, 0}, T{0, 0, 0};
  const pbdr::Vec3 c = pbdr::compute_com(s.bodies[0], s.particles);
  for (size_t k = 0; k < f.size(); ++k) {
    F += f[k];
    T += pbdr::cross(s.particles[k].position - c, f[k]);
  }
  EXPECT(pbdr::norm(F - pbdr::Vec3{1, 0, 0}) < 1e-12 && pbdr::norm(T - pbdr::Vec3{0, 0, 0.5}) < 1e-12,
         "wrench sums");
}

}  // namespace

int main() {
  try {
    free_flight();
    zero_delta_velocity();
    resting_box();
    config_errors();
    stateless_step_carries_time();
    error_formats();
    host_helpers();
  } catch (const pbdr::Error& e) {
    std::printf("FAIL: uncaught pbdr::Error: %s\n", e.what());
    return 2;
  }
  if (failures == 0) std::printf("test_dropin: all passed\n");
  return failures == 0 ? 0 : 1;
}
