// Onesweep radix sort interface (see pbdr_sort.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace pbdr_dev {

// Kernel classes for the optional per-launch profiler (pbdr_gpu_profile_frames).
enum HookClass {
  kHookIntegrate = 0,
  kHookHistogram = 1,
  kHookOnesweep = 2,
  kHookRanges = 3,
  kHookNeighbours = 4,
  kHookIteration = 5,
  kHookMemset = 6,
  kHookBroadphase = 7,
};

// Called around every launch when profiling; null otherwise. `launches` is
// the number of kernels the bracketed region issued.
struct LaunchHook {
  virtual void before(int cls) = 0;
  virtual void after(int cls, int launches = 1) = 0;
  virtual ~LaunchHook() = default;
};

size_t sort_temp_bytes(int64_t n, int passes);

// Sorts keys[0]/vals[0] by the low `key_bits` bits. Returns the buffer index
// (0 or 1) that holds the sorted pairs. When n_dev is non-null the key count is
// read on the device (n is then the maximum, used for launch sizes).
int sort_pairs(uint32_t* keys[2], uint32_t* vals[2], int64_t n, int key_bits, void* temp,
               int sm_count, cudaStream_t stream, LaunchHook* hook, const long long* n_dev = nullptr);

}  // namespace pbdr_dev
