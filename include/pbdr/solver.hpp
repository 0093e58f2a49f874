// pbdr/solver.hpp -- the step of the PBD-R substep loop on a B200, for the
// reference's scene API (pbdr/scene.hpp). The reference ships no solver
// header (proj/src/solver.cpp is absent, CMakeLists.txt:20); the operation is
// specified as step(scene, config) -> scene at t + dt.
#pragma once

#include <vector>

#include "pbdr/scene.hpp"
#include "pbdr_gpu.h"

namespace pbdr {

// Advances `scene` by one substep dt = cfg.dt() on device 0 and writes the new
// particle state back. `t` is the simulation time at the start of the step
// (ForceProgram windows, the frame index of SimulationError); t < 0 (the
// default) carries it: consecutive calls on the same Scene that continue from
// the state the previous call wrote back run on the previous call's device
// state and clock (t += dt, warm-started polar kept -- identical to
// Solver::step); any other call starts a fresh state at t = 0 or the given t.
// The device handle is cached per thread and re-used while the scene's
// bodies, masses and programs are unchanged.
void step(Scene& scene, const SolverConfig& cfg, double t = -1.0);

// Device-resident solver: one scene on one B200, one CUDA stream.
class Solver {
 public:
  Solver(const Scene& scene, const SolverConfig& cfg, int device = 0);
  ~Solver();
  Solver(const Solver&) = delete;
  Solver& operator=(const Solver&) = delete;

  void step(long substeps = 1);       // substeps of dt
  void step_frames(long frames);      // frames * cfg.substeps substeps, CUDA-graph replay
  void download(Scene& scene) const;  // particle positions / velocities (fp64, caller order)
  void upload(const Scene& scene);    // the same, into the device (re-anchors, cold polar)
  void set_time(double t);            // simulation time (rounded to a substep index)
  double time() const;
  // Per-body com, orientation (rest-relative), P, L (trajectory hook).
  std::vector<pbdr_body_stats> body_stats() const;
  pbdr_info info() const;

 private:
  pbdr_handle* h_ = nullptr;
  double dt_ = 0.0;
};

// Rethrows the last C-ABI failure as the matching pbdr exception.
[[noreturn]] void throw_last_error(int status);

}  // namespace pbdr
