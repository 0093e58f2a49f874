// How many Newton iterations the pinned polar takes, and single-lane latency
// of IEEE reciprocal variants on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
#include "pbdr_mat3.cuh"
using namespace pbdr_dev;

__device__ int polar_count(const float Af[9]) {
  D3 X;
  for (int i = 0; i < 9; ++i) X.a[i / 3][i % 3] = Af[i];
  bool scaled = true;
  int it = 0;
  for (; it < 64; ++it) {
    const double d = d3_det(X);
    const D3 inv = d3_adj_inverse(X, d);
    double g = 1.0, ig = 1.0;
    if (scaled) {
      const float xn = (float)d3_norm1_inf(X), in = (float)d3_norm1_inf(inv);
      const float gf = sqrtf(sqrtf(in / xn));
      g = gf; ig = 1.0f / gf;
    }
    double dd = 0, ff = 0;
    for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) {
      double nx = 0.5 * (g * X.a[i][j] + inv.a[j][i] * ig);
      dd += (nx - X.a[i][j]) * (nx - X.a[i][j]); ff += nx * nx; X.a[i][j] = nx;
    }
    if (dd <= 1e-18 * ff || (!scaled && dd <= 1e-9 * ff)) break;
    scaled = dd > 1e-4 * ff;
  }
  return it + 1;
}

__global__ void k(const float* A, int* its, long long* cyc, double* io) {
  its[0] = polar_count(A);
  its[1] = polar_count(A + 9);
  double x = io[1];
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 64; ++i) x = __drcp_rn(x) + 0.25;
  long long t1 = clock64();
  io[2] = x;
  float f = (float)io[1];
  long long t2 = clock64();
#pragma unroll 1
  for (int i = 0; i < 64; ++i) f = __frcp_rn(f) + 0.25f;
  long long t3 = clock64();
  io[3] = f;
  cyc[0] = (t1 - t0) / 64;
  cyc[1] = (t3 - t2) / 64;
}

int main() {
  // C4-like cube (isotropic) and C3-like box 3x10x10 second moments, slightly rotated.
  float hA[18] = {1.2e-3f, 3e-6f, -2e-6f, -3e-6f, 1.2e-3f, 1e-6f, 2e-6f, -1e-6f, 1.2e-3f,
                  1.0e-5f, 3e-7f, -2e-7f, -3e-7f, 1.1e-4f, 1e-7f, 2e-7f, -1e-7f, 1.1e-4f};
  double hio[4] = {0, 1.7, 0, 0};
  float* A; int* its; long long* c; double* io;
  cudaMalloc(&A, 72); cudaMalloc(&its, 8); cudaMalloc(&c, 16); cudaMalloc(&io, 32);
  cudaMemcpy(A, hA, 72, cudaMemcpyHostToDevice);
  cudaMemcpy(io, hio, 32, cudaMemcpyHostToDevice);
  for (int r = 0; r < 3; ++r) k<<<1, 1>>>(A, its, c, io);
  int hi[2]; long long hc[2];
  cudaMemcpy(hi, its, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(hc, c, 16, cudaMemcpyDeviceToHost);
  printf("newton iterations: cube %d, 3x10x10 box %d | drcp_rn+add %lld cyc | frcp_rn+add %lld cyc\n", hi[0], hi[1], hc[0], hc[1]);
}
