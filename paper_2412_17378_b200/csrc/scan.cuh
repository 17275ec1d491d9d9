// scan.cuh — device-wide exclusive prefix sum (reduce-then-scan, 2 kernels).
// Used for compaction offsets, tiles-touched offsets, radix-sort digit
// offsets and tile ranges.  Items at index >= *d_count (when d_count is given)
// count as zero, so counts that live on the device need no host sync.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace bs {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;  // 2048

template <typename T>
__device__ __forceinline__ T warp_inclusive_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  return v;
}

// Block-wide exclusive scan of one value per thread; returns the block total
// in *total.  blockDim.x must be a multiple of 32, <= 1024.
template <typename T>
__device__ __forceinline__ T block_exclusive_scan(T v, T* total) {
  __shared__ T warp_sums[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  T inc = warp_inclusive_scan(v);
  if (lane == 31) warp_sums[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T s = lane < nwarps ? warp_sums[lane] : T(0);
    s = warp_inclusive_scan(s);
    warp_sums[lane] = s;
  }
  __syncthreads();
  const T warp_prefix = warp == 0 ? T(0) : warp_sums[warp - 1];
  *total = warp_sums[nwarps - 1];
  __syncthreads();
  return warp_prefix + inc - v;
}

template <typename T>
__device__ __forceinline__ T block_reduce_sum(T v) {
  __shared__ T red[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  T s = T(0);
  if (threadIdx.x == 0)
    for (int w = 0; w < nwarps; ++w) s += red[w];
  __syncthreads();
  return s;  // valid in thread 0
}

template <typename TIn, typename TOut>
__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(const TIn* __restrict__ in, int64_t n_cap,
                                                              const int32_t* __restrict__ d_count,
                                                              TOut* __restrict__ partials) {
  bs::pdl_wait();
  const int64_t n = d_count ? (int64_t)*d_count : n_cap;
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
  TOut s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const int64_t k = base + (int64_t)i * kScanThreads + threadIdx.x;
    if (k < n) s += (TOut)in[k];
  }
  s = block_reduce_sum(s);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

// partials[] holds each block's raw sum (k_scan_reduce); every block adds up
// the sums before it itself (at most a few hundred L2 reads — cheaper than a
// third, single-CTA launch), and the last block writes the grand total.
template <typename TIn, typename TOut>
__global__ void __launch_bounds__(kScanThreads) k_scan_downsweep(const TIn* __restrict__ in, int64_t n_cap,
                                                                 const int32_t* __restrict__ d_count,
                                                                 const TOut* __restrict__ partials,
                                                                 TOut* __restrict__ out, TOut* __restrict__ total_out) {
  bs::pdl_wait();
  __shared__ TOut s_prefix;
  {
    TOut p = 0;
    for (int64_t i = threadIdx.x; i < (int64_t)blockIdx.x; i += kScanThreads) p += partials[i];
    p = block_reduce_sum(p);
    if (threadIdx.x == 0) s_prefix = p;
  }
  const int64_t n = d_count ? (int64_t)*d_count : n_cap;
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
  // blocked arrangement: thread t owns items [t*8, t*8+8) of the tile
  TOut v[kScanItems];
  TOut local = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const int64_t k = base + (int64_t)threadIdx.x * kScanItems + i;
    v[i] = k < n ? (TOut)in[k] : TOut(0);
    local += v[i];
  }
  TOut tot;
  const TOut ex = block_exclusive_scan(local, &tot);  // (its barriers also publish s_prefix)
  TOut run = ex + s_prefix;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const int64_t k = base + (int64_t)threadIdx.x * kScanItems + i;
    if (k < n_cap) out[k] = run;
    run += v[i];
  }
  if (total_out && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) *total_out = s_prefix + tot;
}

inline int64_t scan_num_blocks(int64_t n_cap) { return (n_cap + kScanTile - 1) / kScanTile; }

// Small arrays (block counts, tile counts; <= 16 items per thread): one CTA, each
// thread a contiguous run of ceil(n / 1024) items — one launch instead of
// three.
constexpr int64_t kScanSingleMax = (int64_t)1 << 14;

template <typename TIn, typename TOut>
__global__ void __launch_bounds__(1024) k_scan_single(const TIn* __restrict__ in, TOut* __restrict__ out,
                                                      int64_t n_cap, const int32_t* __restrict__ d_count,
                                                      TOut* __restrict__ total_out) {
  bs::pdl_wait();
  const int64_t n = d_count ? min((int64_t)*d_count, n_cap) : n_cap;
  const int64_t per = (n_cap + 1023) / 1024;
  const int64_t b = (int64_t)threadIdx.x * per, e = min(b + per, n_cap);
  TOut local = 0;
  for (int64_t k = b; k < e; ++k) local += k < n ? (TOut)in[k] : TOut(0);
  TOut tot;
  TOut run = block_exclusive_scan(local, &tot);
  for (int64_t k = b; k < e; ++k) {
    const TOut v = k < n ? (TOut)in[k] : TOut(0);  // (read before the write: out may alias in)
    out[k] = run;
    run += v;
  }
  if (threadIdx.x == 0 && total_out) *total_out = tot;
}

// Workspace: partials[nb].  total (device) may be null.  out may alias in.
template <typename TIn, typename TOut>
inline cudaError_t exclusive_scan(const TIn* in, TOut* out, int64_t n_cap, const int32_t* d_count, TOut* partials,
                                  TOut* total, cudaStream_t st) {
  const int64_t nb = scan_num_blocks(n_cap);
  if (nb == 0) {
    if (total) return cudaMemsetAsync(total, 0, sizeof(TOut), st);
    return cudaSuccess;
  }
  if (n_cap <= kScanSingleMax) {
    bs::launch_pdl(k_scan_single<TIn, TOut>, 1, 1024, 0, st, in, out, n_cap, d_count, total);
    count_launches(1);
    return cudaPeekAtLastError();
  }
  bs::launch_pdl(k_scan_reduce<TIn, TOut>, (unsigned)nb, kScanThreads, 0, st, in, n_cap, d_count, partials);
  bs::launch_pdl(k_scan_downsweep<TIn, TOut>, (unsigned)nb, kScanThreads, 0, st, in, n_cap, d_count, partials, out, total);
  count_launches(2);
  return cudaPeekAtLastError();
}

}  // namespace bs
