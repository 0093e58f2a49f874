// GPU pack_mesh: sphere packing of a closed triangle mesh by ray-crossing
// parity (reference geometry.cpp:73-195:
// ray_triangle, jittered_direction, point_in_mesh, pack_mesh).
//
// The candidates are the reference's grid (x slowest, z fastest, centres at
// bb.min + radius + i * 2 radius); each is tested by one thread against every
// triangle, the triangles streamed through shared memory in tiles. The
// Moller-Trumbore test and its ambiguity band are the reference's fp64 code,
// operation for operation (IEEE add/mul/div/sqrt, no contraction: the library
// builds with --fmad=false), so the inside / ambiguous flags are the
// reference's bit for bit; an ambiguous ray is re-cast along the next of the
// eight fixed jittered directions, which the host derives from the same
// splitmix64 sequence (Rng(0x5EED + attempt)). The host gathers the inside
// candidates in grid order, so the packing is deterministic.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "pbdr_gpu.h"
#include "pbdr_internal.h"

namespace pbdr_dev {
namespace {

constexpr int kMeshThreads = 128;
constexpr int kTriTile = 128;
constexpr int kAttempts = 8;

struct D3v {
  double x, y, z;
};
__device__ __forceinline__ D3v sub(D3v a, D3v b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ double dot(D3v a, D3v b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ D3v cross(D3v a, D3v b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__device__ __forceinline__ double norm(D3v v) { return sqrt(dot(v, v)); }

enum : int { kMiss = 0, kHit = 1, kAmbiguous = 2 };

// geometry.cpp:77-104, same operations in the same order.
__device__ int ray_triangle(D3v orig, D3v dir, D3v a, D3v b, D3v c) {
  const double kEps = 1e-12;
  const D3v e1 = sub(b, a);
  const D3v e2 = sub(c, a);
  const D3v pv = cross(dir, e2);
  const double det = dot(e1, pv);
  const double scale = norm(e1) * norm(e2);
  if (fabs(det) <= 1e-9 * fmax(scale, kEps)) {
    const D3v n = cross(e1, e2);
    const double nn = norm(n);
    if (nn <= kEps) return kMiss;
    const D3v nu = {n.x / nn, n.y / nn, n.z / nn};
    const double d = fabs(dot(sub(orig, a), nu));
    return d <= 1e-9 * fmax(1.0, norm(sub(orig, a))) ? kAmbiguous : kMiss;
  }
  const double inv = 1.0 / det;
  const D3v tv = sub(orig, a);
  const double u = dot(tv, pv) * inv;
  const D3v qv = cross(tv, e1);
  const double v = dot(dir, qv) * inv;
  const double t = dot(e2, qv) * inv;
  const double kBand = 1e-9;
  if (u < -kBand || v < -kBand || u + v > 1.0 + kBand) return kMiss;
  if (t < -kBand) return kMiss;
  if (u <= kBand || v <= kBand || u + v >= 1.0 - kBand || t <= kBand) return kAmbiguous;
  return kHit;
}

struct MeshArgs {
  const double* tri;  // 9 doubles per triangle (a, b, c)
  int ntri;
  const double* dirs;  // 3 * kAttempts
  double x0, y0, z0, pitch;
  int nx, ny, nz;
  uint8_t* flags;  // bit 0 inside, bit 1 ambiguous
};

__global__ void __launch_bounds__(kMeshThreads) k_pack_mesh(MeshArgs A) {
  __shared__ double s_tri[kTriTile * 9];
  const int64_t total = static_cast<int64_t>(A.nx) * A.ny * A.nz;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool valid = i < total;
  D3v p = {0.0, 0.0, 0.0};
  if (valid) {
    const int iz = static_cast<int>(i % A.nz);
    const int iy = static_cast<int>((i / A.nz) % A.ny);
    const int ix = static_cast<int>(i / (static_cast<int64_t>(A.nz) * A.ny));
    p = {A.x0 + ix * A.pitch, A.y0 + iy * A.pitch, A.z0 + iz * A.pitch};
  }
  bool resolved = !valid, inside = false;
  for (int attempt = 0; attempt < kAttempts; ++attempt) {
    if (!__syncthreads_or(!resolved)) break;
    const D3v dir = {A.dirs[3 * attempt], A.dirs[3 * attempt + 1], A.dirs[3 * attempt + 2]};
    long crossings = 0;
    bool bad = false;
    for (int t0 = 0; t0 < A.ntri; t0 += kTriTile) {
      const int nt = min(kTriTile, A.ntri - t0);
      __syncthreads();
      for (int k = threadIdx.x; k < nt * 9; k += blockDim.x) s_tri[k] = A.tri[static_cast<int64_t>(t0) * 9 + k];
      __syncthreads();
      if (resolved || bad) continue;
      for (int k = 0; k < nt && !bad; ++k) {
        const double* T = &s_tri[9 * k];
        const int h = ray_triangle(p, dir, {T[0], T[1], T[2]}, {T[3], T[4], T[5]}, {T[6], T[7], T[8]});
        if (h == kHit) ++crossings;
        else if (h == kAmbiguous) bad = true;
      }
    }
    if (!resolved && !bad) {
      resolved = true;
      inside = (crossings % 2) == 1;
    }
  }
  if (valid) A.flags[i] = static_cast<uint8_t>((inside ? 1 : 0) | (resolved ? 0 : 2));
}

}  // namespace
}  // namespace pbdr_dev

extern "C" {

int pbdr_pack_mesh(const double* vertices, int32_t num_vertices, const int32_t* triangles, int32_t num_triangles,
                   double radius, int device, double* centers, int64_t capacity, int64_t* count,
                   int64_t* candidates, int64_t* ambiguous) {
  using pbdr_host::set_error;
  pbdr_host::clear_error();
  if (!vertices || !triangles || !count) return set_error(PBDR_ERR_GENERIC, "pack_mesh: null argument");
  if (!(radius > 0.0)) return set_error(PBDR_ERR_GENERIC, "pack_mesh: radius must be positive");
  if (num_vertices <= 0 || num_triangles <= 0) return set_error(PBDR_ERR_GENERIC, "pack_mesh: empty mesh");
  for (int64_t k = 0; k < 3 * static_cast<int64_t>(num_triangles); ++k)
    if (triangles[k] < 0 || triangles[k] >= num_vertices)
      return set_error(PBDR_ERR_GENERIC, "mesh triangle index out of range");
  // Bounds and grid exactly as TriMesh::bounds / pack_mesh (geometry.cpp:13-23, 153-169).
  double mn[3] = {vertices[0], vertices[1], vertices[2]}, mx[3] = {vertices[0], vertices[1], vertices[2]};
  for (int v = 0; v < num_vertices; ++v)
    for (int c = 0; c < 3; ++c) {
      mn[c] = std::min(mn[c], vertices[3 * v + c]);
      mx[c] = std::max(mx[c], vertices[3 * v + c]);
    }
  const double pitch = 2.0 * radius;
  int nn[3];
  for (int c = 0; c < 3; ++c) nn[c] = static_cast<int>(std::floor((mx[c] - mn[c]) / pitch + 1e-12));
  if (nn[0] < 1 || nn[1] < 1 || nn[2] < 1)
    return set_error(PBDR_ERR_EMPTY_PACKING, "pack_mesh: radius too large for the mesh bounding box");
  const int64_t total = static_cast<int64_t>(nn[0]) * nn[1] * nn[2];
  // jittered_direction (geometry.cpp:106-116): attempt 0 canonical, then Rng(0x5EED + attempt).
  double dirs[3 * pbdr_dev::kAttempts];
  for (int a = 0; a < pbdr_dev::kAttempts; ++a) {
    double d[3] = {0.577350269, 0.577350269, 0.577350269};
    if (a > 0) {
      double u[3];
      pbdr_rng_unit(0x5EEDull + static_cast<uint64_t>(a), 3, u);
      for (int c = 0; c < 3; ++c) d[c] += -0.3 + (0.3 - -0.3) * u[c];
    }
    const double n = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    for (int c = 0; c < 3; ++c) dirs[3 * a + c] = n > 0.0 ? d[c] / n : 0.0;
  }
  std::vector<double> tri(9 * static_cast<size_t>(num_triangles));
  for (int t = 0; t < num_triangles; ++t)
    for (int k = 0; k < 3; ++k)
      for (int c = 0; c < 3; ++c) tri[9 * t + 3 * k + c] = vertices[3 * triangles[3 * t + k] + c];

  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return set_error(PBDR_ERR_CUDA, "no CUDA device available (pack_mesh has no CPU fallback)");
  if (device < 0 || device >= ndev) return pbdr_host::set_config_error("device", "out of range");
  cudaSetDevice(device);
  double *d_tri = nullptr, *d_dirs = nullptr;
  uint8_t* d_flags = nullptr;
  std::vector<uint8_t> flags(static_cast<size_t>(total));
  cudaError_t e = cudaMalloc(&d_tri, sizeof(double) * tri.size());
  if (e == cudaSuccess) e = cudaMalloc(&d_dirs, sizeof dirs);
  if (e == cudaSuccess) e = cudaMalloc(&d_flags, static_cast<size_t>(total));
  if (e == cudaSuccess) e = cudaMemcpy(d_tri, tri.data(), sizeof(double) * tri.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d_dirs, dirs, sizeof dirs, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    pbdr_dev::MeshArgs a{};
    a.tri = d_tri;
    a.ntri = num_triangles;
    a.dirs = d_dirs;
    a.x0 = mn[0] + radius;
    a.y0 = mn[1] + radius;
    a.z0 = mn[2] + radius;
    a.pitch = pitch;
    a.nx = nn[0];
    a.ny = nn[1];
    a.nz = nn[2];
    a.flags = d_flags;
    const unsigned blocks = static_cast<unsigned>((total + pbdr_dev::kMeshThreads - 1) / pbdr_dev::kMeshThreads);
    pbdr_dev::k_pack_mesh<<<blocks, pbdr_dev::kMeshThreads>>>(a);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpy(flags.data(), d_flags, static_cast<size_t>(total), cudaMemcpyDeviceToHost);
  cudaFree(d_tri);
  cudaFree(d_dirs);
  cudaFree(d_flags);
  if (e != cudaSuccess) return set_error(PBDR_ERR_CUDA, std::string("pack_mesh: ") + cudaGetErrorString(e));

  int64_t inside = 0, amb = 0;
  for (int64_t i = 0; i < total; ++i) {
    if (flags[i] & 2) ++amb;
    if (!(flags[i] & 1)) continue;
    if (centers && inside < capacity) {
      const int iz = static_cast<int>(i % nn[2]);
      const int iy = static_cast<int>((i / nn[2]) % nn[1]);
      const int ix = static_cast<int>(i / (static_cast<int64_t>(nn[2]) * nn[1]));
      centers[3 * inside] = (mn[0] + radius) + ix * pitch;
      centers[3 * inside + 1] = (mn[1] + radius) + iy * pitch;
      centers[3 * inside + 2] = (mn[2] + radius) + iz * pitch;
    }
    ++inside;
  }
  *count = inside;
  if (candidates) *candidates = total;
  if (ambiguous) *ambiguous = amb;
  if (inside == 0) return set_error(PBDR_ERR_EMPTY_PACKING, "pack_mesh: no grid point lies inside the mesh");
  if (centers && inside > capacity) return set_error(PBDR_ERR_GENERIC, "pack_mesh: centers capacity too small");
  return PBDR_OK;
}

}  // extern "C"
