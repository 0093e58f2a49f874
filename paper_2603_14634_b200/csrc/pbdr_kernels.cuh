// Device kernels of the PBD-R substep loop (sm_100a). See pbdr_kernels.cu.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "pbdr_pinned.h"

namespace pbdr_dev {

struct Planes {
  int count;
  float p[PBDR_MAX_PLANES][3];
  float n[PBDR_MAX_PLANES][3];
  float mu[PBDR_MAX_PLANES];
};

// Device error record: bits (atomicOr), first body (atomicMin), first substep
// (atomicMin), null axis of the first rank-deficient body.
struct DevError {
  unsigned bits;
  int body;
  long long substep;
  double axis[3];
};

struct BodyProgram {  // ForceProgram (scene.hpp:53-61), fp32 force + window
  float fx, fy, fz;
  int flags;  // bit0: has program, bit1: gravity exempt
  double t_start, t_stop;
};

struct IntegrateArgs {
  float4* pos;         // in: X (substep start), out: X~ (predicted)
  float4* vel;         // in: V, out: V~
  float4* init;        // out: X_init
  const int* body_of;
  const int* body_scene;
  const BodyProgram* programs;  // per body
  const float2* body_mass;      // (M, 1/M)
  uint32_t* keys;
  uint32_t* vals;
  const long long* substep_counter;
  int64_t n;
  float dt, gravity, inv_h;
  double dt_d;
  uint32_t mask;
};

struct RangesArgs {
  const uint32_t* keys;  // sorted
  const uint32_t* vals;  // sorted slots
  const int* body_of;
  uint32_t* cell_start;
  uint32_t* cell_end;
  int* sorted_body;
  long long* substep_counter;
  int64_t n;
};

struct NeighbourArgs {
  const float4* pos;  // X~
  const float4* rest;
  const int* body_of;
  const int* body_scene;
  const uint32_t* cell_start;
  const uint32_t* cell_end;
  const int* sorted_body;
  const uint32_t* sorted_vals;
  int* ncand;
  int* cand_j;     // slot-major: [k * n + i]
  float* cand_rr;  // slot-major
  DevError* err;
  const long long* substep_counter;
  int64_t n;
  float inv_h, h2;
  uint32_t mask;
};

struct IterArgs {
  const float4* pos_in;  // X_i snapshot (also gathered for neighbours)
  float4* pos_out;       // X_{i+1}
  float4* vel;           // V_i -> V_{i+1} (own particles only)
  const float4* rest;    // (q0, radius)
  const float4* init;    // X_init
  const int* ncand;
  const int* cand_j;
  const float* cand_rr;
  float4* anchor;        // per body (xyz)
  const int2* warp_desc; // per CTA warp: (body, warp index within body) or (-1, 0)
  const int4* body_desc; // (start, n, W, first warp in CTA)
  const float2* body_mass;
  DevError* err;
  const long long* substep_counter;
  int64_t n;
  Planes planes;
  float dt, inv_dt, relax;
  int incremental, linfix, angfix;
};

struct StatsArgs {
  const float4* pos;
  const float4* vel;
  const float4* rest;
  const float4* anchor;
  const int2* warp_desc;
  const int4* body_desc;
  const float2* body_mass;
  double* out;  // 13 doubles per body: com[3], quat[4], P[3], L[3]
};

void launch_integrate(const IntegrateArgs& a, cudaStream_t s);
void launch_ranges(const RangesArgs& a, cudaStream_t s);
void launch_neighbours(const NeighbourArgs& a, cudaStream_t s);
void launch_iteration(const IterArgs& a, int ctas, cudaStream_t s);
void launch_stats(const StatsArgs& a, int ctas, cudaStream_t s);

}  // namespace pbdr_dev
