// Microbenchmark: single-lane latency of the warm-started polar and the
// inertia solve (the per-body math of k_iteration) on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
#include "pbdr_mat3.cuh"

using namespace pbdr_dev;

__global__ void k(const float* A, const float* rq, const float* If, const float* dL, long long* cyc, float* out) {
  double q[4];
  float Rf[9];
  float a[9], r[4], I6[6], l[3];
  for (int i = 0; i < 9; ++i) a[i] = A[i];
  for (int i = 0; i < 4; ++i) r[i] = rq[i];
  for (int i = 0; i < 6; ++i) I6[i] = If[i];
  for (int i = 0; i < 3; ++i) l[i] = dL[i];
  __syncwarp();
  long long t0 = clock64();
  bool ok = polar_warm_f(a, r, Rf, q);
  long long t1 = clock64();
  float om[3];
  double nax[3];
  unsigned e = inertia_solve_f(I6, l, om, nax);
  long long t2 = clock64();
  cyc[0] = t1 - t0;
  cyc[1] = t2 - t1;
  for (int i = 0; i < 9; ++i) out[i] = Rf[i];
  out[9] = ok + e + om[0] + om[1] + om[2];
}

int main() {
  // A = R(theta about z) * diag(s) with a small stretch; rq = R tilted by `tilt`.
  const double th = 0.3;
  float hA[9] = {(float)(1e-3 * cos(th)), (float)(-1.1e-3 * sin(th)), 0.f,
                 (float)(1e-3 * sin(th)), (float)(1.1e-3 * cos(th)), 0.f, 0.f, 0.f, 0.9e-3f};
  float hI[6] = {0.02f, 0.021f, 0.019f, 1e-4f, -2e-4f, 5e-5f};
  float hL[3] = {1e-3f, -2e-3f, 5e-4f};
  float *A, *rq, *I, *L, *o; long long* c;
  cudaMalloc(&A, 36); cudaMalloc(&rq, 16); cudaMalloc(&I, 24); cudaMalloc(&L, 12); cudaMalloc(&o, 64);
  cudaMalloc(&c, 16);
  cudaMemcpy(A, hA, 36, cudaMemcpyHostToDevice);
  cudaMemcpy(I, hI, 24, cudaMemcpyHostToDevice);
  cudaMemcpy(L, hL, 12, cudaMemcpyHostToDevice);
  const double tilts[4] = {-1, 1e-6, 1e-4, 1e-2};
  for (double tilt : tilts) {
    float hq[4] = {0, 0, 0, 0};
    if (tilt >= 0) {
      const double a = 0.5 * (th + tilt);
      hq[0] = (float)cos(a); hq[3] = (float)sin(a);
    }
    cudaMemcpy(rq, hq, 16, cudaMemcpyHostToDevice);
    for (int rep = 0; rep < 3; ++rep) k<<<1, 1>>>(A, rq, I, L, c, o);
    long long hc[2];
    cudaMemcpy(hc, c, sizeof hc, cudaMemcpyDeviceToHost);
    printf("tilt %-8g polar_warm %lld cyc | inertia_solve %lld cyc\n", tilt, hc[0], hc[1]);
  }
  return 0;
}
