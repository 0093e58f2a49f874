// Onesweep LSD radix sort of (cell-hash key, particle slot) pairs for sm_100a.
//
// Part of the uniform-hash-grid neighbour search (north_star: "cell-key kernel,
// onesweep radix sort, and cell-range scan"). The reference's spatial hash
// exists only as prose; this is the B200 replacement for the
// CPU sort/counting-sort it implies.
//
// Structure (Merrill & Garland style single-pass digit-binning):
//   1. pbdr_sort_histogram: one read of all keys builds the 256-bin digit
//      histograms for every pass at once (smem atomics, then global atomics).
//   2. pbdr_sort_scan: exclusive scan of each pass's histogram -> digit bases.
//   3. pbdr_sort_onesweep (one launch per 8-bit digit): each CTA claims a tile
//      id from an atomic counter (so it only ever waits on tiles that are
//      already resident), ranks its 2048 keys stably with warp-level
//      match_any, publishes its per-digit counts, and resolves its global
//      offsets by decoupled look-back over the preceding tiles' status words,
//      then scatters keys and values through shared memory (digit-ordered
//      runs, coalesced global writes).
// The key count may live on the device (the broadphase-filtered particle list):
// kernels are launched for the maximum and read the actual count.
// Stability: within a tile keys are ranked in (warp, item, lane) order, which
// is their input order; tiles are in input order. So equal keys keep ascending
// particle slots, which the cell-range and neighbour kernels rely on.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "pbdr_sort.cuh"

namespace pbdr_dev {

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortItems = 8;
constexpr int kSortTile = kSortThreads * kSortItems;  // 2048 keys
constexpr int kRadix = 256;
constexpr uint32_t kFlagAgg = 1u << 30;
constexpr uint32_t kFlagIncl = 2u << 30;
constexpr uint32_t kValueMask = (1u << 30) - 1u;

__global__ void __launch_bounds__(kSortThreads)
pbdr_sort_histogram(const uint32_t* __restrict__ keys, int64_t n_max, const long long* n_dev, int passes,
                    uint32_t* __restrict__ hist /* passes*256 */) {
  const int64_t n = n_dev ? static_cast<int64_t>(*n_dev) : n_max;
  __shared__ uint32_t s_hist[4][kRadix];
  for (int i = threadIdx.x; i < 4 * kRadix; i += blockDim.x) (&s_hist[0][0])[i] = 0u;
  __syncthreads();
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t k = keys[i];
    for (int p = 0; p < passes; ++p) atomicAdd(&s_hist[p][(k >> (8 * p)) & 0xFFu], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * kRadix; i += blockDim.x) {
    const uint32_t c = (&s_hist[0][0])[i];
    if (c) atomicAdd(&hist[i], c);
  }
}

// One CTA of 256 threads; exclusive scan of each pass's 256 bins in place.
__global__ void __launch_bounds__(kRadix) pbdr_sort_scan(uint32_t* __restrict__ hist, int passes) {
  __shared__ uint32_t s[kRadix];
  for (int p = 0; p < passes; ++p) {
    const uint32_t v = hist[p * kRadix + threadIdx.x];
    s[threadIdx.x] = v;
    __syncthreads();
    // Hillis-Steele inclusive scan (integer: order-independent).
    for (int off = 1; off < kRadix; off <<= 1) {
      const uint32_t add = threadIdx.x >= off ? s[threadIdx.x - off] : 0u;
      __syncthreads();
      s[threadIdx.x] += add;
      __syncthreads();
    }
    hist[p * kRadix + threadIdx.x] = s[threadIdx.x] - v;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kSortThreads)
pbdr_sort_onesweep(const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
                   uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out, int64_t n_max,
                   const long long* n_dev, int shift, const uint32_t* __restrict__ digit_base,
                   uint32_t* __restrict__ status /* tiles*256 */,
                   uint32_t* __restrict__ tile_counter) {
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_warp_hist[kSortWarps][kRadix];
  __shared__ uint32_t s_digit_off[kRadix];   // global start of this tile's digit group
  __shared__ uint32_t s_tile_excl[kRadix];   // tile-local start of the digit group
  __shared__ uint32_t s_wsum[kSortWarps];
  __shared__ uint32_t s_keys[kSortTile];
  __shared__ uint32_t s_vals[kSortTile];

  const int64_t n = n_dev ? static_cast<int64_t>(*n_dev) : n_max;
  // Persistent: the grid is at most one wave; each CTA keeps claiming tiles
  // (in increasing order, so look-back only waits on running CTAs) until the
  // device-side count is covered.
  for (;;) {
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
  for (int i = threadIdx.x; i < kSortWarps * kRadix; i += kSortThreads) (&s_warp_hist[0][0])[i] = 0u;
  __syncthreads();

  const uint32_t tile = s_tile;
  if (static_cast<int64_t>(tile) * kSortTile >= n) return;  // block-uniform
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t lt_mask = (1u << lane) - 1u;
  const int64_t tile_base = static_cast<int64_t>(tile) * kSortTile;
  const int64_t base = tile_base + warp * (32 * kSortItems);

  uint32_t k[kSortItems], v[kSortItems], rank[kSortItems];
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const int64_t idx = base + i * 32 + lane;
    if (idx < n) {
      k[i] = keys_in[idx];
      v[i] = vals_in[idx];
    } else {
      k[i] = 0xFFFFFFFFu;
      v[i] = 0u;
    }
  }
  // Stable per-warp ranking, item-major (item i of every lane precedes item i+1).
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const int64_t idx = base + i * 32 + lane;
    const bool valid = idx < n;
    const uint32_t d = valid ? ((k[i] >> shift) & 0xFFu) : 0x100u;
    const uint32_t peers = __match_any_sync(0xFFFFFFFFu, d);
    uint32_t cnt = 0u;
    if (valid) cnt = s_warp_hist[warp][d];
    __syncwarp();
    rank[i] = cnt + __popc(peers & lt_mask);
    if (valid && (peers & lt_mask) == 0u) s_warp_hist[warp][d] = cnt + __popc(peers);
    __syncwarp();
  }
  __syncthreads();

  // Thread t owns digit t: exclusive prefix across warps, tile total.
  const int d = threadIdx.x;
  uint32_t tile_count = 0u;
#pragma unroll
  for (int w = 0; w < kSortWarps; ++w) {
    const uint32_t c = s_warp_hist[w][d];
    s_warp_hist[w][d] = tile_count;
    tile_count += c;
  }
  // Tile-local exclusive scan over the 256 digits (warp scan + warp totals).
  uint32_t incl = tile_count;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, off);
    if (lane >= off) incl += y;
  }
  if (lane == 31) s_wsum[warp] = incl;
  // Decoupled look-back over earlier tiles' per-digit status words.
  volatile uint32_t* st = status;
  uint32_t exclusive = 0u;
  if (tile == 0u) {
    st[d] = kFlagIncl | tile_count;
  } else {
    st[static_cast<size_t>(tile) * kRadix + d] = kFlagAgg | tile_count;
    int64_t t = static_cast<int64_t>(tile) - 1;
    while (true) {
      const uint32_t s = st[static_cast<size_t>(t) * kRadix + d];
      if ((s & ~kValueMask) == 0u) continue;  // not yet published
      exclusive += s & kValueMask;
      if (s & kFlagIncl) break;
      --t;
    }
    st[static_cast<size_t>(tile) * kRadix + d] = kFlagIncl | (exclusive + tile_count);
  }
  s_digit_off[d] = digit_base[d] + exclusive;
  __syncthreads();
  uint32_t wpre = 0u;
  for (int w = 0; w < warp; ++w) wpre += s_wsum[w];
  s_tile_excl[d] = wpre + incl - tile_count;
  __syncthreads();

  // Local scatter into digit order, then coalesced runs to global memory.
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const int64_t idx = base + i * 32 + lane;
    if (idx < n) {
      const uint32_t dd = (k[i] >> shift) & 0xFFu;
      const uint32_t lp = s_tile_excl[dd] + s_warp_hist[warp][dd] + rank[i];
      s_keys[lp] = k[i];
      s_vals[lp] = v[i];
    }
  }
  __syncthreads();
  const int64_t rem = n - tile_base;
  const int tile_n = rem < kSortTile ? static_cast<int>(rem) : kSortTile;
  for (int j = threadIdx.x; j < tile_n; j += kSortThreads) {
    const uint32_t kk = s_keys[j];
    const uint32_t dd = (kk >> shift) & 0xFFu;
    const uint32_t dst = s_digit_off[dd] + (static_cast<uint32_t>(j) - s_tile_excl[dd]);
    keys_out[dst] = kk;
    vals_out[dst] = s_vals[j];
  }
  __syncthreads();  // shared buffers are reused by the next tile
  }
}

// Zeroes the histograms, tile counters and the status words of the tiles the
// device-side count actually uses (instead of a memset sized for the maximum).
__global__ void __launch_bounds__(256)
pbdr_sort_zero(uint32_t* __restrict__ temp, int passes, int64_t tiles_max, int64_t n_max, const long long* n_dev) {
  const int64_t n = n_dev ? static_cast<int64_t>(*n_dev) : n_max;
  const int64_t need = (n + kSortTile - 1) / kSortTile + 1;
  const int64_t tiles = need < tiles_max ? need : tiles_max;
  const int64_t head = static_cast<int64_t>(passes) * kRadix + passes;  // hist + counters
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < head; i += stride) temp[i] = 0u;
  uint32_t* status = temp + head;
  const int64_t used = tiles * kRadix;
  for (int p = 0; p < passes; ++p)
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < used; i += stride)
      status[static_cast<int64_t>(p) * tiles_max * kRadix + i] = 0u;
}

size_t sort_temp_bytes(int64_t n, int passes) {
  const int64_t tiles = (n + kSortTile - 1) / kSortTile;
  return sizeof(uint32_t) * (static_cast<size_t>(passes) * kRadix      // hist
                             + static_cast<size_t>(passes)              // tile counters
                             + static_cast<size_t>(passes) * tiles * kRadix);  // status
}

int sort_pairs(uint32_t* keys[2], uint32_t* vals[2], int64_t n, int key_bits, void* temp,
               int sm_count, cudaStream_t stream, LaunchHook* hook, const long long* n_dev) {
  const int passes = (key_bits + 7) / 8;
  const int64_t tiles = (n + kSortTile - 1) / kSortTile;
  uint32_t* hist = static_cast<uint32_t*>(temp);
  uint32_t* counters = hist + passes * kRadix;
  uint32_t* status = counters + passes;
  const size_t bytes = sort_temp_bytes(n, passes);
  if (hook) hook->before(kHookMemset);
  if (n_dev) {
    pbdr_sort_zero<<<sm_count * 4, 256, 0, stream>>>(static_cast<uint32_t*>(temp), passes, tiles, n, n_dev);
  } else {
    cudaMemsetAsync(temp, 0, bytes, stream);
  }
  if (hook) hook->after(kHookMemset);
  if (hook) hook->before(kHookHistogram);
  const int hist_blocks = sm_count * 4;
  pbdr_sort_histogram<<<hist_blocks, kSortThreads, 0, stream>>>(keys[0], n, n_dev, passes, hist);
  pbdr_sort_scan<<<1, kRadix, 0, stream>>>(hist, passes);
  if (hook) hook->after(kHookHistogram, 2);
  int cur = 0;
  for (int p = 0; p < passes; ++p) {
    if (hook) hook->before(kHookOnesweep);
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(tiles, static_cast<int64_t>(sm_count) * 4));
    pbdr_sort_onesweep<<<grid, kSortThreads, 0, stream>>>(
        keys[cur], vals[cur], keys[cur ^ 1], vals[cur ^ 1], n, n_dev, 8 * p, hist + p * kRadix,
        status + static_cast<size_t>(p) * tiles * kRadix, counters + p);
    if (hook) hook->after(kHookOnesweep);
    cur ^= 1;
  }
  return cur;  // buffer index holding the sorted pairs
}

}  // namespace pbdr_dev
