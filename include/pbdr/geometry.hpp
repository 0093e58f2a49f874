// pbdr/geometry.hpp -- the scene-construction part of the reference's
// geometry module (proj/include/pbdr/geometry.hpp:12-57): bounding box, mesh,
// sphere packing, pack_box, pack_rod and pack_mesh (the last one on the GPU,
// bit-identical inside flags to the reference's fp64 ray-parity test). OBJ /
// CSV file I/O and the standalone point_in_mesh are not provided (DESIGN.md
// section 9: outside the substep loop).
#pragma once

#include <array>
#include <string>
#include <vector>

#include "pbdr/math.hpp"

namespace pbdr {

struct BoundingBox {
  Vec3 min{0, 0, 0};
  Vec3 max{0, 0, 0};
  Vec3 extent() const { return max - min; }
  double diagonal() const { return norm(extent()); }
};

struct TriMesh {
  std::vector<Vec3> vertices;
  std::vector<std::array<int, 3>> triangles;
  BoundingBox bounds() const;
  void validate() const;  // Error on an out-of-range index
};

struct SpherePacking {
  std::vector<Vec3> centers;
  double radius = 0;
  std::string source;
  long ambiguous_count = 0;  // grid samples whose inside test stayed ambiguous
  long candidate_count = 0;  // grid samples tested
  size_t size() const { return centers.size(); }
};

// n^3 centres filling the box, z fastest; radius = half the smallest spacing.
SpherePacking pack_box(const Vec3& half_extents, int n_per_axis);
// Touching spheres along +x, centred on the origin (remainder dropped).
SpherePacking pack_rod(double length, double radius);
// Grid points (pitch 2 radius over the bounding box) inside the closed mesh,
// one GPU thread per candidate. EmptyPackingError when none is inside.
SpherePacking pack_mesh(const TriMesh& mesh, double radius, int device = 0);

}  // namespace pbdr
