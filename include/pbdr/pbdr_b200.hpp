// C++ drop-in for the reference's solver-facing API, backed by the B200 C-ABI
// (include/pbdr_gpu.h). The reference's own include paths are provided, so a
// caller's `#include "pbdr/scene.hpp"` (or body.hpp, math.hpp, errors.hpp,
// geometry.hpp) compiles unchanged against this tree:
//   pbdr/errors.hpp ..... proj/include/pbdr/errors.hpp:8-44
//   pbdr/math.hpp ....... proj/include/pbdr/math.hpp:14-294
//   pbdr/body.hpp ....... proj/include/pbdr/body.hpp:11-66
//   pbdr/scene.hpp ...... proj/include/pbdr/scene.hpp:12-82
//   pbdr/geometry.hpp ... proj/include/pbdr/geometry.hpp:12-57 (packing part)
//   pbdr/solver.hpp ..... step() of SPEC.md:326-334 and the resident Solver
// This umbrella header includes all of them.
#pragma once

#include "pbdr/body.hpp"
#include "pbdr/errors.hpp"
#include "pbdr/geometry.hpp"
#include "pbdr/math.hpp"
#include "pbdr/scene.hpp"
#include "pbdr/solver.hpp"
