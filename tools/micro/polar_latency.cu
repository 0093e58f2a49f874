// Microbenchmark: single-lane latency of the per-body fp64 math on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
#include "pbdr_mat3.cuh"

using namespace pbdr_dev;

__global__ void k(const float* A, float* R, long long* cyc, double* io) {
  double q[4];
  float Rf[9];
  long long t0 = clock64();
  bool ok = polar_rotation_f(A, Rf, q);
  long long t1 = clock64();
  double x = io[1];
  float f = static_cast<float>(io[2]);
  __syncwarp();
  long long t2 = clock64();
#pragma unroll 1
  for (int i = 0; i < 64; ++i) x = 1.0 / x;
  io[3] = x;
  long long t3 = clock64();
#pragma unroll 1
  for (int i = 0; i < 64; ++i) x = sqrt(x) + 0.5;
  io[4] = x;
  long long t4 = clock64();
#pragma unroll 1
  for (int i = 0; i < 64; ++i) x = x * 1.0000001 + 1e-9;
  io[5] = x;
  long long t5 = clock64();
#pragma unroll 1
  for (int i = 0; i < 64; ++i) f = 1.0f / f;
  io[6] = f;
  long long t6 = clock64();
#pragma unroll 1
  for (int i = 0; i < 64; ++i) f = sqrtf(f) + 0.5f;
  io[7] = f;
  long long t7 = clock64();
  cyc[0] = t1 - t0; cyc[1] = (t3 - t2) / 64; cyc[2] = (t4 - t3) / 64; cyc[3] = (t5 - t4) / 64;
  cyc[4] = (t6 - t5) / 64; cyc[5] = (t7 - t6) / 64;
  for (int i = 0; i < 9; ++i) R[i] = Rf[i];
  io[0] = (ok ? 1 : 0) + q[0];
}

int main() {
  float hA[9] = {1e-3f, 2e-5f, -3e-5f, 1e-5f, 1.1e-3f, 4e-5f, -2e-5f, 3e-5f, 0.9e-3f};
  double hio[8] = {0, 1.7, 1.3, 0, 0, 0, 0, 0};
  float *A, *R; long long* c; double* io;
  cudaMalloc(&A, 36); cudaMalloc(&R, 36); cudaMalloc(&c, 64); cudaMalloc(&io, 64);
  cudaMemcpy(A, hA, 36, cudaMemcpyHostToDevice);
  cudaMemcpy(io, hio, 64, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 3; ++rep) k<<<1, 1>>>(A, R, c, io);
  long long hc[6];
  cudaMemcpy(hc, c, sizeof hc, cudaMemcpyDeviceToHost);
  printf("polar %lld cyc | ddiv %lld | dsqrt+dadd %lld | dfma-chain(mul+add) %lld | fdiv %lld | fsqrt+fadd %lld\n",
         hc[0], hc[1], hc[2], hc[3], hc[4], hc[5]);
  return 0;
}
