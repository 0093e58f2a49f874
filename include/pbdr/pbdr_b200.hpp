// C++ drop-in layer for the reference's solver-facing API, backed by the B200
// C-ABI (include/pbdr_gpu.h).
//
// A user of the reference library (namespace pbdr) finds the same type names,
// fields and defaults here:
//   Particle, Body, MomentumState ............ proj/include/pbdr/body.hpp:11-36
//   Precision, VelocityUpdate, Backend,
//   MomentumFrequency, SolverConfig(pbd/pbdr),
//   Plane, ForceProgram, Scene,
//   add_packed_body .......................... proj/include/pbdr/scene.hpp:12-82
//   Error hierarchy .......................... proj/include/pbdr/errors.hpp:8-44
//   make_body ................................ proj/include/pbdr/body.hpp:40
// plus the step() the reference only specifies in prose and
// a stateful Solver that keeps the scene resident on the GPU between calls.
// The reference headers themselves cannot be included as shipped
// (math.hpp:199 does not compile), so this header is self-contained; it keeps
// only the small part of the math module the scene API needs (Vec3, Rotation).
//
// Extensions, all default-empty so a reference Scene maps 1:1:
//   Scene::walls       extra planes after the ground (config 3's container)
//   Scene::body_scene  independent-scene id per body (config 4's batches)
#pragma once

#include <cmath>
#include <cstdint>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <array>
#include <vector>

#include "pbdr_gpu.h"

namespace pbdr {

// ---- errors (errors.hpp:8-44) ------------------------------------------------
struct Error : std::runtime_error {
  explicit Error(const std::string& m) : std::runtime_error(m) {}
};
struct DegenerateConfigError : Error {
  explicit DegenerateConfigError(const std::string& m) : Error(m) {}
};
struct RankDeficientError : Error {
  RankDeficientError(const std::string& m, double ax, double ay, double az)
      : Error(m), axis_x(ax), axis_y(ay), axis_z(az) {}
  double axis_x, axis_y, axis_z;
};
struct EmptyPackingError : Error {
  explicit EmptyPackingError(const std::string& m) : Error(m) {}
};
struct InvalidMomentError : Error {
  explicit InvalidMomentError(const std::string& m) : Error(m) {}
};
struct ConfigError : Error {
  ConfigError(const std::string& key, const std::string& m) : Error(m), key_path(key) {}
  std::string key_path;
};
struct SimulationError : Error {
  SimulationError(const std::string& m, long frame) : Error(m), frame_index(frame) {}
  long frame_index;
};

// ---- minimal math (math.hpp Vec3T<double>, Rotation) ----------------------
struct Vec3 {
  double x = 0, y = 0, z = 0;
  Vec3() = default;
  Vec3(double a, double b, double c) : x(a), y(b), z(c) {}
  Vec3 operator+(const Vec3& o) const { return {x + o.x, y + o.y, z + o.z}; }
  Vec3 operator-(const Vec3& o) const { return {x - o.x, y - o.y, z - o.z}; }
  Vec3 operator*(double s) const { return {x * s, y * s, z * s}; }
  Vec3 operator/(double s) const { return {x / s, y / s, z / s}; }
  Vec3& operator+=(const Vec3& o) { x += o.x; y += o.y; z += o.z; return *this; }
};

// Unit quaternion (w, x, y, z), Hamilton convention.
struct Rotation {
  double w = 1, x = 0, y = 0, z = 0;
  Rotation() = default;
  Rotation(double w_, double x_, double y_, double z_) : w(w_), x(x_), y(y_), z(z_) {}
  static Rotation axis_angle(const Vec3& axis, double angle) {
    const double n = std::sqrt(axis.x * axis.x + axis.y * axis.y + axis.z * axis.z);
    const double s = std::sin(0.5 * angle) / (n > 0 ? n : 1.0);
    return {std::cos(0.5 * angle), axis.x * s, axis.y * s, axis.z * s};
  }
  Vec3 rotate(const Vec3& v) const {
    const double r00 = 1 - 2 * (y * y + z * z), r01 = 2 * (x * y - w * z), r02 = 2 * (x * z + w * y);
    const double r10 = 2 * (x * y + w * z), r11 = 1 - 2 * (x * x + z * z), r12 = 2 * (y * z - w * x);
    const double r20 = 2 * (x * z - w * y), r21 = 2 * (y * z + w * x), r22 = 1 - 2 * (x * x + y * y);
    return {r00 * v.x + r01 * v.y + r02 * v.z, r10 * v.x + r11 * v.y + r12 * v.z,
            r20 * v.x + r21 * v.y + r22 * v.z};
  }
};

// ---- body.hpp ----------------------------------------------------------------
struct Particle {
  Vec3 position;
  Vec3 velocity;
  double inv_mass = 1.0;
  double radius = 0.0;
  int body_id = -1;
};

struct Body {
  std::vector<int> particle_indices;
  std::vector<Vec3> rest_offsets;
  double total_mass = 0.0;
  Vec3 rest_com;
  bool collinear = false;
  Vec3 rest_axis{1, 0, 0};
};

struct MomentumState {
  Vec3 linear;
  Vec3 angular;
  Vec3 com;
};

// Rest pose = current positions of `indices` (body.cpp:16-48 semantics).
Body make_body(const std::vector<Particle>& particles, const std::vector<int>& indices);

// ---- scene.hpp -----------------------------------------------------------------
enum class Precision { kSingle, kDouble };
enum class VelocityUpdate { kLegacy, kIncremental };
enum class Backend { kSerial, kParallel };
enum class MomentumFrequency { kPerIteration, kPerSubstep };

struct SolverConfig {
  double frame_rate = 100.0;
  int substeps = 10;
  int solver_iterations = 10;
  Precision precision = Precision::kSingle;
  VelocityUpdate velocity_update = VelocityUpdate::kIncremental;
  bool linear_momentum_fix = true;
  bool angular_momentum_fix = true;
  MomentumFrequency momentum_frequency = MomentumFrequency::kPerIteration;
  double gravity = 9.81;
  Backend backend = Backend::kParallel;

  double dt() const { return 1.0 / (frame_rate * substeps); }
  void validate() const;
  static SolverConfig pbd() {
    SolverConfig c;
    c.velocity_update = VelocityUpdate::kLegacy;
    c.linear_momentum_fix = false;
    c.angular_momentum_fix = false;
    return c;
  }
  static SolverConfig pbdr() { return SolverConfig{}; }
};

struct Plane {
  Vec3 point{0, 0, 0};
  Vec3 normal{0, 0, 1};
  double friction = 0.0;
};

struct ForceProgram {
  Vec3 force{0, 0, 0};
  Vec3 torque{0, 0, 0};
  double t_start = 0.0;
  double t_stop = std::numeric_limits<double>::infinity();
  bool gravity_exempt = false;
  bool active(double t) const { return t >= t_start && t < t_stop; }
};

struct Scene {
  std::vector<Particle> particles;
  std::vector<Body> bodies;
  std::vector<ForceProgram> programs;  // parallel to bodies (may be empty)
  Plane ground;
  bool has_ground = true;
  double contact_relaxation = 1.0;
  std::vector<Plane> walls;      // extension
  std::vector<int> body_scene;   // extension
  void validate() const;
};

int add_packed_body(Scene& scene, const std::vector<Vec3>& centers, double radius,
                    double total_mass, const Rotation& rotate, const Vec3& translate,
                    double jitter, uint64_t seed);

// ---- Mesh packing (geometry.hpp:19-57) ------------------------------------------
struct TriMesh {
  std::vector<Vec3> vertices;
  std::vector<std::array<int, 3>> triangles;
};

struct SpherePacking {
  std::vector<Vec3> centers;
  double radius = 0;
  long ambiguous_count = 0;  // grid samples whose inside test stayed ambiguous
  long candidate_count = 0;  // grid samples tested
  size_t size() const { return centers.size(); }
};

// pack_mesh (geometry.cpp:151-195) on the GPU: grid points inside the closed
// mesh by ray-crossing parity, bit-identical to the reference's fp64 test.
SpherePacking pack_mesh(const TriMesh& mesh, double radius, int device = 0);

// ---- step ---------------------------------------------------
// Advances the scene by one substep dt = cfg.dt() on the GPU (device 0) and
// writes the new particle state back into `scene`. Stateless: uploads and
// downloads every call. Use Solver to keep the scene resident.
void step(Scene& scene, const SolverConfig& cfg);

// Device-resident solver: one scene on one B200, one CUDA stream.
class Solver {
 public:
  Solver(const Scene& scene, const SolverConfig& cfg, int device = 0);
  ~Solver();
  Solver(const Solver&) = delete;
  Solver& operator=(const Solver&) = delete;

  void step(long substeps = 1);       // substeps of dt
  void step_frames(long frames);      // frames * cfg.substeps substeps, CUDA-graph replay
  void download(Scene& scene) const;  // particle positions / velocities
  void upload(const Scene& scene);
  // Per-body com, orientation (rest-relative), P, L (trajectory hook).
  std::vector<pbdr_body_stats> body_stats() const;
  pbdr_info info() const;

 private:
  pbdr_handle* h_ = nullptr;
};

// Rethrows the last C-ABI failure as the matching pbdr exception.
[[noreturn]] void throw_last_error(int status);

}  // namespace pbdr
