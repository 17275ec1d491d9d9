// radix_sort.cuh — stable LSD radix sort of (u32 key, u32 value) pairs.
//
// Reduce-then-scan, 8-bit digits, 4096-item block tiles (8 warps x 512):
//   k_radix_hist    per-block digit histogram (warp-aggregated smem atomics),
//                   written digit-major: hist[d * nblocks + b]
//   exclusive_scan  over the 256 x nblocks histogram -> global digit offsets
//   k_radix_scatter stable block-local ranking (match.any per warp-round,
//                   warp-private running counters, cross-warp prefix), local
//                   reorder through shared memory, then coalesced runs out.
// Stability: inside a block, warp w owns the contiguous sub-range
// [w*512, w*512+512) processed in 16 ordered rounds of 32 lanes, and warps are
// ranked in index order — so equal digits keep input order, as LSD needs.
// The element count may live on the device (d_count): items at index >=
// *d_count are ignored, so no host sync is needed between pipeline stages.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "bs_common.cuh"
#include "scan.cuh"

namespace bs {

constexpr int kSortWarps = 8;
constexpr int kSortThreads = kSortWarps * 32;
constexpr int kSortRounds = 16;
constexpr int kSortPerWarp = kSortRounds * 32;            // 512
constexpr int kSortTile = kSortWarps * kSortPerWarp;      // 4096

inline int64_t radix_num_blocks(int64_t n_cap) { return (n_cap + kSortTile - 1) / kSortTile; }

static __global__ void __launch_bounds__(kSortThreads) k_radix_hist(const uint32_t* __restrict__ keys, int64_t n_cap,
                                                             const int32_t* __restrict__ d_count, int shift,
                                                             int64_t nb, uint32_t* __restrict__ hist) {
  __shared__ uint32_t cnt[256];
  const int64_t n = d_count ? (int64_t)*d_count : n_cap;
  cnt[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kSortTile;
  const int lane = threadIdx.x & 31;
#pragma unroll 4
  for (int i = 0; i < kSortTile / kSortThreads; ++i) {
    const int64_t k = base + (int64_t)i * kSortThreads + threadIdx.x;
    const bool valid = k < n;
    const uint32_t d = valid ? (__ldg(keys + k) >> shift) & 255u : 256u;
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    if (valid && lane == __ffs(peers) - 1) atomicAdd(&cnt[d], (uint32_t)__popc(peers));
  }
  __syncthreads();
  hist[(int64_t)threadIdx.x * nb + blockIdx.x] = cnt[threadIdx.x];
}

static __global__ void __launch_bounds__(kSortThreads) k_radix_scatter(const uint32_t* __restrict__ keys_in,
                                                                const uint32_t* __restrict__ vals_in,
                                                                uint32_t* __restrict__ keys_out,
                                                                uint32_t* __restrict__ vals_out, int64_t n_cap,
                                                                const int32_t* __restrict__ d_count, int shift,
                                                                int64_t nb, const uint32_t* __restrict__ offsets) {
  __shared__ uint32_t wcnt[kSortWarps][256];
  __shared__ uint32_t local_start[256];
  __shared__ uint32_t digit_base[256];
  __shared__ uint32_t skeys[kSortTile];
  __shared__ uint32_t svals[kSortTile];
  const int64_t n = d_count ? (int64_t)*d_count : n_cap;
  const int64_t base = (int64_t)blockIdx.x * kSortTile;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < kSortWarps * 256; i += kSortThreads) (&wcnt[0][0])[i] = 0;
  __syncthreads();

  uint32_t key[kSortRounds], val[kSortRounds], rank[kSortRounds];
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int r = 0; r < kSortRounds; ++r) {
    const int64_t k = base + warp * kSortPerWarp + r * 32 + lane;
    const bool valid = k < n;
    key[r] = valid ? keys_in[k] : 0u;
    val[r] = valid ? vals_in[k] : 0u;
    const uint32_t d = valid ? (key[r] >> shift) & 255u : 256u;
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    uint32_t before = 0;
    if (valid) before = wcnt[warp][d];
    __syncwarp();
    if (valid && lane == __ffs(peers) - 1) wcnt[warp][d] = before + __popc(peers);
    __syncwarp();
    rank[r] = before + __popc(peers & lt);
  }
  __syncthreads();
  // per digit: exclusive prefix across warps, block total, global base
  {
    const int d = tid;  // kSortThreads == 256
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) {
      const uint32_t c = wcnt[w][d];
      wcnt[w][d] = run;
      run += c;
    }
    uint32_t tot;
    const uint32_t ex = block_exclusive_scan<uint32_t>(run, &tot);
    local_start[d] = ex;
    digit_base[d] = offsets[(int64_t)d * nb + blockIdx.x];
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kSortRounds; ++r) {
    const int64_t k = base + warp * kSortPerWarp + r * 32 + lane;
    if (k < n) {
      const uint32_t d = (key[r] >> shift) & 255u;
      const uint32_t pos = local_start[d] + wcnt[warp][d] + rank[r];
      skeys[pos] = key[r];
      svals[pos] = val[r];
    }
  }
  __syncthreads();
  const int64_t rem = n - base;
  const int valid_items = rem >= kSortTile ? kSortTile : (rem > 0 ? (int)rem : 0);
  for (int i = tid; i < valid_items; i += kSortThreads) {
    const uint32_t kk = skeys[i];
    const uint32_t d = (kk >> shift) & 255u;
    const uint32_t dst = digit_base[d] + (uint32_t)i - local_start[d];
    keys_out[dst] = kk;
    vals_out[dst] = svals[i];
  }
}

struct RadixWs {
  uint32_t* hist;      // 256 * nb
  uint32_t* partials;  // scan partials
};

inline void radix_ws_size(WsSizer& s, int64_t n_cap) {
  const int64_t nb = radix_num_blocks(n_cap);
  s.take<uint32_t>((size_t)(256 * nb));
  s.take<uint32_t>((size_t)scan_num_blocks(256 * nb));
}
inline RadixWs radix_ws_take(WsCarver& c, int64_t n_cap) {
  const int64_t nb = radix_num_blocks(n_cap);
  RadixWs w;
  w.hist = c.take<uint32_t>((size_t)(256 * nb));
  w.partials = c.take<uint32_t>((size_t)scan_num_blocks(256 * nb));
  return w;
}

// Sorts bits [0, key_bits) of keys.  Ping-pongs between (k0,v0) and (k1,v1);
// *result_in_alt says which pair holds the output.
inline cudaError_t radix_sort_pairs(uint32_t* k0, uint32_t* v0, uint32_t* k1, uint32_t* v1, int64_t n_cap,
                                    const int32_t* d_count, int key_bits, const RadixWs& w, bool* result_in_alt,
                                    cudaStream_t st) {
  *result_in_alt = false;
  const int64_t nb = radix_num_blocks(n_cap);
  if (nb == 0 || key_bits <= 0) return cudaSuccess;
  uint32_t *ki = k0, *vi = v0, *ko = k1, *vo = v1;
  for (int shift = 0; shift < key_bits; shift += 8) {
    k_radix_hist<<<(unsigned)nb, kSortThreads, 0, st>>>(ki, n_cap, d_count, shift, nb, w.hist);
    cudaError_t e = exclusive_scan<uint32_t, uint32_t>(w.hist, w.hist, 256 * nb, nullptr, w.partials, nullptr, st);
    if (e != cudaSuccess) return e;
    k_radix_scatter<<<(unsigned)nb, kSortThreads, 0, st>>>(ki, vi, ko, vo, n_cap, d_count, shift, nb, w.hist);
    count_launches(2);
    uint32_t* t;
    t = ki; ki = ko; ko = t;
    t = vi; vi = vo; vo = t;
    *result_in_alt = !*result_in_alt;
  }
  return cudaPeekAtLastError();
}

}  // namespace bs
