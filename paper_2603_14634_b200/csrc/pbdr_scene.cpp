// Host-side scene construction for the five BASELINE.json configs.
//
// Semantics follow the reference's scene-building API, re-implemented here:
//   * splitmix64 draws mapped to doubles with fixed bit arithmetic
//     (proj/include/pbdr/rng.hpp:10-29);
//   * pack_box lattices with the z index fastest (proj/src/geometry.cpp:32-55);
//   * add_packed_body placement: uniform particle mass M/N, rotate then
//     translate, rest pose recorded from the placed pose (scene.hpp:76-82,
//     body.cpp:16-48: total mass, mass-weighted rest com, rest offsets).
// Config readings (masses, layouts, jitters) are pinned in DESIGN.md section
// "Workloads" (SURVEY.md Appendix B lists the open choices).
//
// Everything here is host-only and deterministic: the oracle, the tests and
// bench.py all build their inputs through pbdr_scene_generate().
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <new>
#include <string>
#include <unordered_map>
#include <vector>

#include "pbdr_gpu.h"
#include "pbdr_internal.h"

namespace pbdr_host {

namespace {

struct SplitMix {
  uint64_t s;
  explicit SplitMix(uint64_t seed) : s(seed + 0x9E3779B97F4A7C15ull) {}
  uint64_t u64() {
    s += 0x9E3779B97F4A7C15ull;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double unit() { return static_cast<double>(u64() >> 11) * (1.0 / 9007199254740992.0); }
  double uniform(double lo, double hi) { return lo + (hi - lo) * unit(); }
};

struct V3 {
  double x, y, z;
};
inline V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 scl(V3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
inline double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline V3 crs(V3 a, V3 b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}

// Rotation matrix (row-major) of a unit quaternion (w, x, y, z), Hamilton.
struct Rot {
  double m[3][3];
  V3 apply(V3 v) const {
    return {m[0][0] * v.x + m[0][1] * v.y + m[0][2] * v.z,
            m[1][0] * v.x + m[1][1] * v.y + m[1][2] * v.z,
            m[2][0] * v.x + m[2][1] * v.y + m[2][2] * v.z};
  }
  V3 col(int c) const { return {m[0][c], m[1][c], m[2][c]}; }
};

Rot rot_from_quat(double w, double x, double y, double z) {
  Rot r;
  r.m[0][0] = 1 - 2 * (y * y + z * z);
  r.m[0][1] = 2 * (x * y - w * z);
  r.m[0][2] = 2 * (x * z + w * y);
  r.m[1][0] = 2 * (x * y + w * z);
  r.m[1][1] = 1 - 2 * (x * x + z * z);
  r.m[1][2] = 2 * (y * z - w * x);
  r.m[2][0] = 2 * (x * z - w * y);
  r.m[2][1] = 2 * (y * z + w * x);
  r.m[2][2] = 1 - 2 * (x * x + y * y);
  return r;
}

// Shoemake's uniform random rotation from three next_unit() draws (pinned
// order u1, u2, u3).
Rot uniform_rotation(SplitMix& rng) {
  const double u1 = rng.unit(), u2 = rng.unit(), u3 = rng.unit();
  const double a = std::sqrt(1.0 - u1), b = std::sqrt(u1);
  const double t2 = 2.0 * M_PI * u2, t3 = 2.0 * M_PI * u3;
  return rot_from_quat(b * std::cos(t3), a * std::sin(t2), a * std::cos(t2), b * std::sin(t3));
}

V3 uniform_box(SplitMix& rng, double lo, double hi) {
  const double x = rng.uniform(lo, hi);
  const double y = rng.uniform(lo, hi);
  const double z = rng.uniform(lo, hi);
  return {x, y, z};
}

// pack_box lattice (geometry.cpp:32-55 semantics): per-axis spacing
// s = h * (2/n), centres -h + (i + 0.5) s with the z index fastest, radius
// half the smallest spacing (returned through `radius`).
std::vector<V3> lattice_box(double hx, double hy, double hz, int nx, int ny, int nz, double* radius) {
  std::vector<V3> c;
  c.reserve(static_cast<size_t>(nx) * ny * nz);
  const double sx = hx * (2.0 / nx), sy = hy * (2.0 / ny), sz = hz * (2.0 / nz);
  for (int i = 0; i < nx; ++i)
    for (int j = 0; j < ny; ++j)
      for (int k = 0; k < nz; ++k)
        c.push_back({-hx + (i + 0.5) * sx, -hy + (j + 0.5) * sy, -hz + (k + 0.5) * sz});
  if (radius) *radius = 0.5 * std::min(sx, std::min(sy, sz));
  return c;
}

// Voxelised sphere: lattice points (i, j, k) with i^2 + j^2 + k^2 <= R^2, pitch 2r.
std::vector<V3> lattice_sphere(int R, double r) {
  std::vector<V3> c;
  const double p = 2.0 * r;
  for (int i = -R; i <= R; ++i)
    for (int j = -R; j <= R; ++j)
      for (int k = -R; k <= R; ++k)
        if (i * i + j * j + k * k <= R * R) c.push_back({i * p, j * p, k * p});
  return c;
}

// Conservative body shape for the non-overlap test at generation time.
struct Hull {
  V3 c;
  Rot R;
  V3 half;        // box half extents of the particle surfaces (box) ...
  double radius;  // ... or sphere radius (sphere); also bounding radius
  bool is_box;
};

bool hulls_overlap(const Hull& a, const Hull& b) {
  const V3 d = sub(b.c, a.c);
  const double dist2 = dot(d, d);
  const double rr = a.radius + b.radius;
  if (dist2 >= rr * rr) return false;
  if (!a.is_box && !b.is_box) return true;
  if (a.is_box && b.is_box) {
    // Separating-axis test over the 15 OBB axes.
    V3 axes[15];
    int na = 0;
    for (int i = 0; i < 3; ++i) axes[na++] = a.R.col(i);
    for (int i = 0; i < 3; ++i) axes[na++] = b.R.col(i);
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        V3 ax = crs(a.R.col(i), b.R.col(j));
        if (dot(ax, ax) > 1e-12) axes[na++] = ax;
      }
    const double ha[3] = {a.half.x, a.half.y, a.half.z};
    const double hb[3] = {b.half.x, b.half.y, b.half.z};
    for (int k = 0; k < na; ++k) {
      const V3 ax = axes[k];
      double pa = 0, pb = 0;
      for (int i = 0; i < 3; ++i) {
        pa += ha[i] * std::fabs(dot(a.R.col(i), ax));
        pb += hb[i] * std::fabs(dot(b.R.col(i), ax));
      }
      if (std::fabs(dot(d, ax)) > pa + pb) return false;
    }
    return true;
  }
  // Box vs sphere: closest point of the box to the sphere centre.
  const Hull& box = a.is_box ? a : b;
  const Hull& sph = a.is_box ? b : a;
  const V3 rel = sub(sph.c, box.c);
  const double h[3] = {box.half.x, box.half.y, box.half.z};
  double dd = 0;
  for (int i = 0; i < 3; ++i) {
    const double t = dot(rel, box.R.col(i));
    const double e = std::fabs(t) - h[i];
    if (e > 0) dd += e * e;
  }
  return dd < sph.radius * sph.radius;
}

// Buckets hulls on a coarse grid so overlap tests only touch nearby bodies.
struct HullGrid {
  double cell;
  std::unordered_map<uint64_t, std::vector<int>> buckets;
  std::vector<Hull> hulls;
  explicit HullGrid(double c) : cell(c) {}
  static uint64_t key(int64_t x, int64_t y, int64_t z) {
    return (static_cast<uint64_t>(x & 0x1FFFFF) << 42) | (static_cast<uint64_t>(y & 0x1FFFFF) << 21) |
           static_cast<uint64_t>(z & 0x1FFFFF);
  }
  bool overlaps(const Hull& h) const {
    const int64_t cx = static_cast<int64_t>(std::floor(h.c.x / cell));
    const int64_t cy = static_cast<int64_t>(std::floor(h.c.y / cell));
    const int64_t cz = static_cast<int64_t>(std::floor(h.c.z / cell));
    for (int64_t dz = -1; dz <= 1; ++dz)
      for (int64_t dy = -1; dy <= 1; ++dy)
        for (int64_t dx = -1; dx <= 1; ++dx) {
          auto it = buckets.find(key(cx + dx, cy + dy, cz + dz));
          if (it == buckets.end()) continue;
          for (int idx : it->second)
            if (hulls_overlap(h, hulls[idx])) return true;
        }
    return false;
  }
  void insert(const Hull& h) {
    const int64_t cx = static_cast<int64_t>(std::floor(h.c.x / cell));
    const int64_t cy = static_cast<int64_t>(std::floor(h.c.y / cell));
    const int64_t cz = static_cast<int64_t>(std::floor(h.c.z / cell));
    buckets[key(cx, cy, cz)].push_back(static_cast<int>(hulls.size()));
    hulls.push_back(h);
  }
};

Hull box_hull(V3 c, const Rot& R, int nx, int ny, int nz, double r) {
  Hull h;
  h.c = c;
  h.R = R;
  h.half = {nx * r, ny * r, nz * r};  // particle centres at +-(n-1)r, plus radius
  h.radius = std::sqrt(dot(h.half, h.half));
  h.is_box = true;
  return h;
}


}  // namespace

// Appends one rigid body: particles at R*centre + t with uniform mass M/N and
// velocity v + w x (x - t); rest pose recorded from the placed pose.
static void add_body(GeneratedScene& s, const std::vector<V3>& centres, double radius,
                     double total_mass, const Rot& R, V3 t, V3 v, V3 w, int scene_id) {
  const int64_t n = static_cast<int64_t>(centres.size());
  const int32_t body = static_cast<int32_t>(s.total_mass.size());
  const double inv_mass = static_cast<double>(n) / total_mass;
  const int64_t first = s.num_particles();
  for (int64_t k = 0; k < n; ++k) {
    const V3 arm = R.apply(centres[static_cast<size_t>(k)]);
    const V3 x = add(arm, t);
    const V3 vel = add(v, crs(w, arm));
    s.position.insert(s.position.end(), {x.x, x.y, x.z});
    s.velocity.insert(s.velocity.end(), {vel.x, vel.y, vel.z});
    s.inv_mass.push_back(inv_mass);
    s.radius.push_back(radius);
    s.body_id.push_back(body);
    s.body_indices.push_back(static_cast<int32_t>(first + k));
  }
  // make_body semantics: sequential mass and mass-weighted com, then offsets.
  double mass = 0, wx = 0, wy = 0, wz = 0;
  for (int64_t k = 0; k < n; ++k) {
    const double m = 1.0 / s.inv_mass[static_cast<size_t>(first + k)];
    mass += m;
    wx += s.position[3 * (first + k)] * m;
    wy += s.position[3 * (first + k) + 1] * m;
    wz += s.position[3 * (first + k) + 2] * m;
  }
  const V3 com = {wx / mass, wy / mass, wz / mass};
  for (int64_t k = 0; k < n; ++k) {
    s.rest_offsets.push_back(s.position[3 * (first + k)] - com.x);
    s.rest_offsets.push_back(s.position[3 * (first + k) + 1] - com.y);
    s.rest_offsets.push_back(s.position[3 * (first + k) + 2] - com.z);
  }
  s.total_mass.push_back(mass);
  s.rest_com.insert(s.rest_com.end(), {com.x, com.y, com.z});
  s.body_offsets.push_back(static_cast<int64_t>(s.body_indices.size()));
  s.body_scene.push_back(scene_id);
}

static pbdr_plane make_plane(V3 p, V3 n, double mu) {
  pbdr_plane pl;
  pl.point[0] = p.x; pl.point[1] = p.y; pl.point[2] = p.z;
  pl.normal[0] = n.x; pl.normal[1] = n.y; pl.normal[2] = n.z;
  pl.friction = mu;
  return pl;
}

static void default_cfg(pbdr_solver_cfg& c) {
  c.frame_rate = 240.0;  // "dt = 1/240 s, 10 substeps" (BASELINE.json configs)
  c.substeps = 10;
  c.solver_iterations = 10;
  c.precision = PBDR_PRECISION_SINGLE;
  c.velocity_update = PBDR_VELOCITY_INCREMENTAL;
  c.linear_momentum_fix = 1;
  c.angular_momentum_fix = 1;
  c.momentum_frequency = PBDR_MOMENTUM_PER_ITERATION;
  c.backend = PBDR_BACKEND_PARALLEL;
  c.gravity = 9.81;
}

// Config 1: one 8x8x8 cube, r = 0.01, 1 kg, com at z = 0.5, seeded orientation,
// v ~ U[-1,1]^3, w ~ U[-2,2]^3.
static void gen_c1(GeneratedScene& s, uint64_t seed) {
  SplitMix rng(seed);
  double r = 0.01;
  const std::vector<V3> lat = lattice_box(0.08, 0.08, 0.08, 8, 8, 8, &r);
  const Rot R = uniform_rotation(rng);
  const V3 v = uniform_box(rng, -1.0, 1.0);
  const V3 w = uniform_box(rng, -2.0, 2.0);
  add_body(s, lat, r, 1.0, R, {0, 0, 0.5}, v, w, 0);
  s.frames = 1000;
}

// Places `count` copies of cubes on a grid, resampling jitter + orientation on
// overlap (up to 256 attempts, then the last draw is kept and counted).
struct CubeGridSpec {
  int gx, gy, gz;
  double pitch;
  V3 origin;  // centre of grid cell (0,0,0)
  double jitter;
  int n;       // particles per axis
  double mass;
  double vmax; // linear velocity U[-vmax, vmax]^3
  double wmax; // angular velocity U[-wmax, wmax]^3 (0 = none)
  double max_tilt = 0.0;  // > 0: rotation by angle U[0, max_tilt] about a uniform axis
  bool x_major = false;   // body order: x slowest (x-slabs are contiguous body ranges)
};

// Rotation by angle U[0, max_angle] about a uniformly distributed axis (three
// draws: axis z, axis azimuth, angle).
Rot bounded_rotation(SplitMix& rng, double max_angle) {
  const double z = 2.0 * rng.unit() - 1.0;
  const double phi = 2.0 * M_PI * rng.unit();
  const double ang = max_angle * rng.unit();
  const double s = std::sqrt(std::max(0.0, 1.0 - z * z));
  const double ax = s * std::cos(phi), ay = s * std::sin(phi), az = z;
  const double h = 0.5 * ang, sh = std::sin(h);
  return rot_from_quat(std::cos(h), ax * sh, ay * sh, az * sh);
}

// Cubes t in [t_first, t_end) of the grid (t_end < 0: all). Each cube draws
// a fixed number of values unless its placement is resampled (never for the
// bounded-tilt grids of config 5, which are overlap-free by construction), so
// a sub-range starts from the stream skipped ahead by that many draws;
// `resamples` counts the placements that needed more than one attempt.
static int64_t gen_cube_grid(GeneratedScene& s, SplitMix& rng, const CubeGridSpec& g, int scene_id,
                             int64_t t_first = 0, int64_t t_end = -1, int64_t* resamples = nullptr) {
  double r = 0.01;
  const double h = g.n * 0.01;  // half extent: 0.06 for 6^3, 0.08 for 8^3
  const double hh = g.n == 6 ? 0.06 : (g.n == 8 ? 0.08 : h);
  const std::vector<V3> lat = lattice_box(hh, hh, hh, g.n, g.n, g.n, &r);
  HullGrid grid(0.5);
  int64_t forced = 0;
  const int64_t cells = static_cast<int64_t>(g.gx) * g.gy * g.gz;
  if (t_end < 0 || t_end > cells) t_end = cells;
  for (int64_t t = t_first; t < t_end; ++t) {
      int i, j, k;
      if (g.x_major) {
        k = static_cast<int>(t % g.gz);
        j = static_cast<int>((t / g.gz) % g.gy);
        i = static_cast<int>(t / (static_cast<int64_t>(g.gz) * g.gy));
      } else {
        i = static_cast<int>(t % g.gx);
        j = static_cast<int>((t / g.gx) % g.gy);
        k = static_cast<int>(t / (static_cast<int64_t>(g.gx) * g.gy));
      }
      {
        const V3 base = {g.origin.x + g.pitch * i, g.origin.y + g.pitch * j, g.origin.z + g.pitch * k};
        Rot R{};
        V3 c{};
        bool ok = false;
        for (int attempt = 0; attempt < 256 && !ok; ++attempt) {
          const V3 jit = g.jitter > 0 ? uniform_box(rng, -g.jitter, g.jitter) : V3{0, 0, 0};
          R = g.max_tilt > 0 ? bounded_rotation(rng, g.max_tilt) : uniform_rotation(rng);
          c = add(base, jit);
          ok = !grid.overlaps(box_hull(c, R, g.n, g.n, g.n, r));
          if (!ok && resamples) ++*resamples;
        }
        if (!ok) ++forced;
        grid.insert(box_hull(c, R, g.n, g.n, g.n, r));
        const V3 v = uniform_box(rng, -g.vmax, g.vmax);
        const V3 w = g.wmax > 0 ? uniform_box(rng, -g.wmax, g.wmax) : V3{0, 0, 0};
        add_body(s, lat, r, g.mass, R, c, v, w, scene_id);
      }
  }
  return forced;
}

// Config 2: 64 cubes 6^3 (0.5 kg) on a 4x4x4 grid of pitch 0.2, lowest layer at
// z = 0.2, jitter U[-0.02,0.02]^3, v ~ U[-0.5,0.5]^3.
static void gen_c2(GeneratedScene& s, uint64_t seed) {
  SplitMix rng(seed);
  CubeGridSpec g{4, 4, 4, 0.2, {-0.3, -0.3, 0.2}, 0.02, 6, 0.5, 0.5, 0.0};
  s.forced_overlaps = gen_cube_grid(s, rng, g, 0);
  s.frames = 1000;
}

// Config 3: `nb` bodies (default 8192) in a 4 m x 4 m walled container. Even
// bodies are boxes with per-axis counts U{3..10}, odd bodies voxelised spheres
// of radius U{3..6} particles; density U[500,2000] kg/m^3 with particle mass
// rho*(2r)^3. Drop slots: 11 x 11 per layer, pitch 0.35 m, lowest layer at
// z = 0.2, jitter U[-0.005,0.005]^3, seeded orientations, zero velocity.
static void gen_c3(GeneratedScene& s, uint64_t seed, int64_t nb) {
  SplitMix rng(seed);
  const double r = 0.01;
  const double pitch = 0.35;
  const int per_row = 11;
  for (int64_t b = 0; b < nb; ++b) {
    std::vector<V3> lat;
    if (b % 2 == 0) {
      const int nx = 3 + static_cast<int>(rng.u64() % 8);
      const int ny = 3 + static_cast<int>(rng.u64() % 8);
      const int nz = 3 + static_cast<int>(rng.u64() % 8);
      double rb = r;
      lat = lattice_box(nx * r, ny * r, nz * r, nx, ny, nz, &rb);
    } else {
      const int R = 3 + static_cast<int>(rng.u64() % 4);
      lat = lattice_sphere(R, r);
    }
    const double rho = rng.uniform(500.0, 2000.0);
    const double mass = rho * (8.0 * r * r * r) * static_cast<double>(lat.size());
    const int64_t layer = b / (per_row * per_row);
    const int64_t iy = (b / per_row) % per_row;
    const int64_t ix = b % per_row;
    const V3 base = {-1.75 + pitch * ix, -1.75 + pitch * iy, 0.2 + pitch * layer};
    const V3 jit = uniform_box(rng, -0.005, 0.005);
    const Rot R = uniform_rotation(rng);
    add_body(s, lat, r, mass, R, add(base, jit), {0, 0, 0}, {0, 0, 0}, 0);
  }
  s.walls.push_back(make_plane({-2, 0, 0}, {1, 0, 0}, 0.5));
  s.walls.push_back(make_plane({2, 0, 0}, {-1, 0, 0}, 0.5));
  s.walls.push_back(make_plane({0, -2, 0}, {0, 1, 0}, 0.5));
  s.walls.push_back(make_plane({0, 2, 0}, {0, -1, 0}, 0.5));
  s.frames = 500;
}

// Config 4: `ns` independent scenes (default 4096), scene k seeded seed + k,
// each 16 cubes 6^3 (0.5 kg) on a 4x4 grid of pitch 0.2 at z = 0.5 drawn as in
// config 1 (orientation, v ~ U[-1,1]^3, w ~ U[-2,2]^3).
static void gen_c4(GeneratedScene& s, uint64_t seed, int64_t ns, int64_t first_scene) {
  int64_t forced = 0;
  for (int64_t k = first_scene; k < first_scene + ns; ++k) {
    SplitMix rng(seed + static_cast<uint64_t>(k));
    CubeGridSpec g{4, 4, 1, 0.2, {-0.3, -0.3, 0.5}, 0.0, 6, 0.5, 1.0, 2.0};
    forced += gen_cube_grid(s, rng, g, static_cast<int>(k));
  }
  s.forced_overlaps = forced;
  s.frames = 200;
}

// Config 5: gx*gx*(gx/2) cubes 8^3 (1 kg; default gx = 64 -> 131,072 cubes) on a
// jittered grid of pitch 0.2, lowest layer at z = 0.2, v ~ U[-0.5,0.5]^3.
// "Seeded orientations": 8^3 cubes (half-diagonal 0.139 m incl. radius) cannot
// take uniformly random orientations at pitch 0.2 without overlapping, so the
// orientation is a seeded tilt of U[0, 0.07] rad about a uniform axis and the
// jitter is U[-0.01,0.01]^3 -- together provably overlap-free.
// Bodies are numbered x-major, so an x-slab (slab.py) is a contiguous range of
// bodies and slots up to migrations.
static void gen_c5(GeneratedScene& s, uint64_t seed, int64_t gx) {
  SplitMix rng(seed);
  const int g = static_cast<int>(gx);
  const double half = 0.5 * 0.2 * (g - 1);
  CubeGridSpec spec{g, g, std::max(1, g / 2), 0.2, {-half, -half, 0.2}, 0.01, 8, 1.0, 0.5, 0.0, 0.07, true};
  s.forced_overlaps = gen_cube_grid(s, rng, spec, 0, 0, -1, &s.resamples);
  s.frames = 100;
}

// Config 5's cubes in the x-columns [x_first, x_first + x_count) of a
// gx * gy * gz grid (centred in x and y like gen_c5; gx = gy = 64, gz = 32 is
// BASELINE config 5): the rank-local scene of an x-slab decomposition. Bodies
// keep the global x-major order, so local body k is global body
// x_first * gy * gz + k, and the cubes are bit-identical to the global
// generation's (the stream is skipped ahead by the 9 draws of every cube
// before the range -- valid because no placement is ever resampled; checked
// by tests/test_slab_native.py against the whole grid).
static void gen_c5_slab(GeneratedScene& s, uint64_t seed, int64_t gx, int64_t gy, int64_t gz, int64_t x_first,
                        int64_t x_count) {
  SplitMix rng(seed);
  constexpr uint64_t kDrawsPerCube = 9;  // jitter 3, bounded tilt 3, velocity 3
  const int64_t per_col = gy * gz;
  rng.s += kDrawsPerCube * static_cast<uint64_t>(x_first * per_col) * 0x9E3779B97F4A7C15ull;
  CubeGridSpec spec{static_cast<int>(gx), static_cast<int>(gy), static_cast<int>(gz), 0.2,
                    {-0.5 * 0.2 * static_cast<double>(gx - 1), -0.5 * 0.2 * static_cast<double>(gy - 1), 0.2},
                    0.01, 8, 1.0, 0.5, 0.0, 0.07, true};
  s.forced_overlaps = gen_cube_grid(s, rng, spec, 0, x_first * per_col, (x_first + x_count) * per_col,
                                    &s.resamples);
  s.frames = 100;
}

struct SplitMixPublic : SplitMix {
  explicit SplitMixPublic(uint64_t seed) : SplitMix(seed) {}
};

GeneratedScene* generate(int config_id, uint64_t seed, int64_t scale) {
  GeneratedScene* s = new GeneratedScene();
  default_cfg(s->cfg);
  s->has_ground = 1;
  s->ground = make_plane({0, 0, 0}, {0, 0, 1}, 0.5);
  s->contact_relaxation = 1.0;
  s->body_offsets.push_back(0);
  switch (config_id) {
    case 1: gen_c1(*s, seed); break;
    case 2: gen_c2(*s, seed); break;
    case 3: gen_c3(*s, seed, scale > 0 ? scale : 8192); break;
    case 4: gen_c4(*s, seed, scale > 0 ? scale : 4096, 0); break;
    case 5: gen_c5(*s, seed, scale > 0 ? scale : 64); break;
    default: delete s; return nullptr;
  }
  return s;
}

GeneratedScene* generate_c5_slab(uint64_t seed, int64_t gx, int64_t gy, int64_t gz, int64_t x_first,
                                 int64_t x_count) {
  GeneratedScene* s = new GeneratedScene();
  default_cfg(s->cfg);
  s->has_ground = 1;
  s->ground = make_plane({0, 0, 0}, {0, 0, 1}, 0.5);
  s->contact_relaxation = 1.0;
  s->body_offsets.push_back(0);
  gen_c5_slab(*s, seed, gx, gy, gz, x_first, x_count);
  return s;
}

GeneratedScene* generate_c4_shard(uint64_t seed, int64_t scenes, int64_t first_scene) {
  GeneratedScene* s = new GeneratedScene();
  default_cfg(s->cfg);
  s->has_ground = 1;
  s->ground = make_plane({0, 0, 0}, {0, 0, 1}, 0.5);
  s->contact_relaxation = 1.0;
  s->body_offsets.push_back(0);
  gen_c4(*s, seed, scenes, first_scene);
  return s;
}

void view(const GeneratedScene& s, pbdr_scene_desc& d) {
  std::memset(&d, 0, sizeof d);
  d.num_particles = s.num_particles();
  d.position = s.position.data();
  d.velocity = s.velocity.data();
  d.inv_mass = s.inv_mass.data();
  d.radius = s.radius.data();
  d.body_id = s.body_id.data();
  d.num_bodies = static_cast<int32_t>(s.total_mass.size());
  d.body_offsets = s.body_offsets.data();
  d.body_indices = s.body_indices.data();
  d.rest_offsets = s.rest_offsets.data();
  d.total_mass = s.total_mass.data();
  d.rest_com = s.rest_com.data();
  d.programs = s.programs.empty() ? nullptr : s.programs.data();
  d.ground = s.ground;
  d.has_ground = s.has_ground;
  d.contact_relaxation = s.contact_relaxation;
  d.num_walls = static_cast<int32_t>(s.walls.size());
  d.walls = s.walls.empty() ? nullptr : s.walls.data();
  d.body_scene = s.body_scene.data();
}

}  // namespace pbdr_host

extern "C" {

struct pbdr_generated_scene {
  pbdr_host::GeneratedScene* s;
};

int pbdr_scene_generate(int config_id, uint64_t seed, int64_t scale, pbdr_generated_scene** out) {
  if (!out) return PBDR_ERR_GENERIC;
  *out = nullptr;
  try {
    pbdr_host::GeneratedScene* s = pbdr_host::generate(config_id, seed, scale);
    if (!s) return pbdr_host::set_config_error("config_id", "must be 1..5");
    *out = new pbdr_generated_scene{s};
    return PBDR_OK;
  } catch (const std::bad_alloc&) {
    return pbdr_host::set_error(PBDR_ERR_GENERIC, "scene generation: out of host memory");
  }
}

int pbdr_scene_generate_c4_shard(uint64_t seed, int64_t scenes, int64_t first_scene,
                                 pbdr_generated_scene** out) {
  if (!out) return PBDR_ERR_GENERIC;
  try {
    *out = new pbdr_generated_scene{pbdr_host::generate_c4_shard(seed, scenes, first_scene)};
    return PBDR_OK;
  } catch (const std::bad_alloc&) {
    return pbdr_host::set_error(PBDR_ERR_GENERIC, "scene generation: out of host memory");
  }
}

int pbdr_scene_generate_c5_slab(uint64_t seed, int64_t gx, int64_t gy, int64_t gz, int64_t x_first,
                                int64_t x_count, pbdr_generated_scene** out) {
  if (!out) return pbdr_host::set_error(PBDR_ERR_GENERIC, "null output");
  *out = nullptr;
  if (gx < 1 || gy < 1 || gz < 1 || x_first < 0 || x_count < 1 || x_first + x_count > gx)
    return pbdr_host::set_config_error("slab", "column range outside the grid");
  pbdr_generated_scene* g = new (std::nothrow) pbdr_generated_scene();
  if (!g) return pbdr_host::set_error(PBDR_ERR_GENERIC, "out of host memory");
  g->s = pbdr_host::generate_c5_slab(seed, gx, gy, gz, x_first, x_count);
  *out = g;
  return PBDR_OK;
}

int64_t pbdr_scene_resamples(const pbdr_generated_scene* g) { return g && g->s ? g->s->resamples : 0; }

int pbdr_scene_view(const pbdr_generated_scene* g, pbdr_scene_desc* desc, pbdr_solver_cfg* cfg) {
  if (!g || !g->s) return PBDR_ERR_GENERIC;
  if (desc) pbdr_host::view(*g->s, *desc);
  if (cfg) *cfg = g->s->cfg;
  return PBDR_OK;
}

int64_t pbdr_scene_frames(const pbdr_generated_scene* g) { return g && g->s ? g->s->frames : 0; }
int64_t pbdr_scene_forced_overlaps(const pbdr_generated_scene* g) {
  return g && g->s ? g->s->forced_overlaps : 0;
}

int pbdr_pack_box(double hx, double hy, double hz, int n, double* centers, double* radius) {
  if (n < 1) return pbdr_host::set_error(PBDR_ERR_GENERIC, "pack_box: n_per_axis must be >= 1");
  if (!(hx > 0 && hy > 0 && hz > 0))
    return pbdr_host::set_error(PBDR_ERR_GENERIC, "pack_box: half extents must be positive");
  const double sx = hx * (2.0 / n), sy = hy * (2.0 / n), sz = hz * (2.0 / n);
  int64_t k = 0;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      for (int l = 0; l < n; ++l, ++k) {
        centers[3 * k] = -hx + (i + 0.5) * sx;
        centers[3 * k + 1] = -hy + (j + 0.5) * sy;
        centers[3 * k + 2] = -hz + (l + 0.5) * sz;
      }
  *radius = 0.5 * std::min(sx, std::min(sy, sz));
  return PBDR_OK;
}

void pbdr_rng_u64(uint64_t seed, int count, uint64_t* out) {
  pbdr_host::SplitMixPublic r(seed);
  for (int i = 0; i < count; ++i) out[i] = r.u64();
}

void pbdr_rng_unit(uint64_t seed, int count, double* out) {
  pbdr_host::SplitMixPublic r(seed);
  for (int i = 0; i < count; ++i) out[i] = r.unit();
}

void pbdr_scene_free(pbdr_generated_scene* g) {
  if (!g) return;
  delete g->s;
  delete g;
}

}  // extern "C"
