// radix_sort.cuh — stable LSD radix sort of (u32 key, u32 value) pairs.
//
// Reduce-then-scan with balanced digit widths (ceil(bits/8) passes of
// <= 8 bits each: 13-bit tile ids sort as 7 + 6 bits, so every pass has fewer
// buckets and longer output runs) and 4096-item partitions (16 warps x 8
// rounds x 32 lanes):
//   k_radix_hist    per-partition digit histogram, warp-private smem counters
//                   (plain shared atomics), written digit-major
//                   hist[d * nblocks + b]
//   exclusive_scan  over the buckets x nblocks histogram -> global offsets
//   k_radix_scatter stable partition-local ranking (match.any per warp round,
//                   u16 warp running counters, cross-warp prefix), reorder
//                   through shared memory, coalesced runs out.
// Stability: warp w owns the contiguous sub-range [w*256, w*256+256) of the
// partition, processed in 8 ordered rounds, and warps are ranked in index
// order — equal digits keep input order, as LSD needs.
// (A decoupled-look-back single-pass variant was measured slower here: with
// ~600 co-resident partitions the prefix frontier advances only a few
// partitions per L2 round trip.)
// The element count may live on the device (d_count): items at index >=
// *d_count are ignored, so no host sync is needed between pipeline stages.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "bs_common.cuh"
#include "scan.cuh"

namespace bs {

constexpr int kSortWarps = 16;
constexpr int kSortThreads = kSortWarps * 32;             // 512
constexpr int kSortRounds = 8;
constexpr int kSortPerWarp = kSortRounds * 32;            // 256
constexpr int kSortTile = kSortWarps * kSortPerWarp;      // 4096
constexpr int kSortBuckets = 256;

inline int64_t radix_num_blocks(int64_t n_cap) { return (n_cap + kSortTile - 1) / kSortTile; }

static __global__ void __launch_bounds__(kSortThreads) k_radix_hist(const uint32_t* __restrict__ keys, int64_t n_cap,
                                                                    const int32_t* __restrict__ d_count, int shift,
                                                                    uint32_t mask, int64_t nb,
                                                                    uint32_t* __restrict__ hist) {
  bs::pdl_wait();
  __shared__ uint32_t cnt[kSortWarps][kSortBuckets];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < kSortWarps * kSortBuckets; i += kSortThreads) (&cnt[0][0])[i] = 0;
  __syncthreads();
  const int64_t n = d_count ? (int64_t)*d_count : n_cap;
  const int64_t base = (int64_t)blockIdx.x * kSortTile + warp * kSortPerWarp + lane;
  uint32_t k[kSortRounds];
#pragma unroll
  for (int r = 0; r < kSortRounds; ++r) k[r] = (base + r * 32 < n) ? __ldg(keys + base + r * 32) : 0u;
#pragma unroll
  for (int r = 0; r < kSortRounds; ++r)
    if (base + r * 32 < n) atomicAdd(&cnt[warp][(k[r] >> shift) & mask], 1u);
  __syncthreads();
  if (tid <= (int)mask) {
    uint32_t s = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) s += cnt[w][tid];
    hist[(int64_t)tid * nb + blockIdx.x] = s;
  }
}

// Optional payload of the LAST pass: out_a[dst] = in_a[value], out_b[dst] =
// in_b[value] (a gather by the sorted values, fused into the write-out).
struct RadixGather {
  const uint32_t* in_a;
  const uint2* in_b;
  uint32_t* out_a;
  uint2* out_b;
};

template <bool GATHER>
static __global__ void __launch_bounds__(kSortThreads) k_radix_scatter(const uint32_t* __restrict__ keys_in,
                                                                       const uint32_t* __restrict__ vals_in,
                                                                       uint32_t* __restrict__ keys_out,
                                                                       uint32_t* __restrict__ vals_out, int64_t n_cap,
                                                                       const int32_t* __restrict__ d_count, int shift,
                                                                       uint32_t mask, int64_t nb,
                                                                       const uint32_t* __restrict__ offsets,
                                                                       RadixGather gat) {
  bs::pdl_wait();
  __shared__ uint16_t wcnt[kSortWarps][kSortBuckets];
  __shared__ uint32_t local_start[kSortBuckets];
  __shared__ uint32_t digit_base[kSortBuckets];
  __shared__ uint32_t skeys[kSortTile];
  __shared__ uint32_t svals[kSortTile];
  const int64_t n = d_count ? (int64_t)*d_count : n_cap;
  const int64_t base = (int64_t)blockIdx.x * kSortTile;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < kSortWarps * kSortBuckets; i += kSortThreads) (&wcnt[0][0])[i] = 0;
  if (tid <= (int)mask) digit_base[tid] = offsets[(int64_t)tid * nb + blockIdx.x];
  __syncthreads();

  uint32_t key[kSortRounds], val[kSortRounds], rank[kSortRounds];
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int r = 0; r < kSortRounds; ++r) {
    const int64_t k = base + warp * kSortPerWarp + r * 32 + lane;
    const bool valid = k < n;
    key[r] = valid ? keys_in[k] : 0u;
    val[r] = valid ? vals_in[k] : 0u;
  }
  // all match.any results first (independent -> their latencies overlap),
  // then the short dependent chain through the warp's smem counters.  (A
  // one-ballot-per-digit-bit variant measured slower overall on B200.)
  uint32_t peers[kSortRounds];
#pragma unroll
  for (int r = 0; r < kSortRounds; ++r) {
    const bool valid = base + warp * kSortPerWarp + r * 32 + lane < n;
    peers[r] = __match_any_sync(0xffffffffu, valid ? (key[r] >> shift) & mask : 0x100u);
  }
#pragma unroll
  for (int r = 0; r < kSortRounds; ++r) {
    const bool valid = base + warp * kSortPerWarp + r * 32 + lane < n;
    const uint32_t d = (key[r] >> shift) & mask;
    uint32_t before = 0;
    if (valid) before = wcnt[warp][d];
    __syncwarp();
    if (valid && lane == __ffs(peers[r]) - 1) wcnt[warp][d] = (uint16_t)(before + __popc(peers[r]));
    __syncwarp();
    rank[r] = before + __popc(peers[r] & lt);
  }
  __syncthreads();
  {
    // per digit (threads 0..255): exclusive prefix across warps, then a
    // block-wide exclusive scan of the digit totals (threads >= 256 add 0)
    uint32_t run = 0;
    if (tid < kSortBuckets) {
#pragma unroll
      for (int w = 0; w < kSortWarps; ++w) {
        const uint32_t c = wcnt[w][tid];
        wcnt[w][tid] = (uint16_t)run;
        run += c;
      }
    }
    uint32_t tot;
    const uint32_t ex = block_exclusive_scan<uint32_t>(run, &tot);
    if (tid < kSortBuckets) local_start[tid] = ex;
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kSortRounds; ++r) {
    const int64_t k = base + warp * kSortPerWarp + r * 32 + lane;
    if (k < n) {
      const uint32_t d = (key[r] >> shift) & mask;
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
    const uint32_t d = (kk >> shift) & mask;
    const uint32_t dst = digit_base[d] + (uint32_t)i - local_start[d];
    const uint32_t v = svals[i];
    keys_out[dst] = kk;
    vals_out[dst] = v;
    if (GATHER) {
      gat.out_a[dst] = __ldg(gat.in_a + v);
      gat.out_b[dst] = __ldg(gat.in_b + v);
    }
  }
}

struct RadixWs {
  uint32_t* hist;      // 256 * nb
  uint32_t* partials;  // scan partials
};

template <typename C>
inline void radix_ws_layout(C& c, int64_t n_cap, RadixWs* w) {
  const int64_t nb = radix_num_blocks(n_cap);
  RadixWs tmp;
  RadixWs& o = w ? *w : tmp;
  o.hist = c.template take<uint32_t>((size_t)(kSortBuckets * nb));
  o.partials = c.template take<uint32_t>((size_t)scan_num_blocks(kSortBuckets * nb));
}

// Sorts bits [0, key_bits) of keys in ceil(key_bits/8) passes of balanced
// width.  Ping-pongs between (k0,v0) and (k1,v1); *result_in_alt says which
// pair holds the output.
inline cudaError_t radix_sort_pairs(uint32_t* k0, uint32_t* v0, uint32_t* k1, uint32_t* v1, int64_t n_cap,
                                    const int32_t* d_count, int key_bits, const RadixWs& w, bool* result_in_alt,
                                    cudaStream_t st, const RadixGather* gather = nullptr) {
  *result_in_alt = false;
  const int64_t nb = radix_num_blocks(n_cap);
  if (nb == 0 || key_bits <= 0) return cudaSuccess;
  const int passes = (key_bits + 7) / 8;
  uint32_t *ki = k0, *vi = v0, *ko = k1, *vo = v1;
  int shift = 0;
  for (int p = 0; p < passes; ++p) {
    const int bits = (key_bits - shift + (passes - p) - 1) / (passes - p);  // balanced split
    const uint32_t mask = (1u << bits) - 1u;
    const int64_t buckets = (int64_t)mask + 1;
    bs::launch_pdl(k_radix_hist, (unsigned)nb, kSortThreads, 0, st, ki, n_cap, d_count, shift, mask, nb, w.hist);
    cudaError_t e = exclusive_scan<uint32_t, uint32_t>(w.hist, w.hist, buckets * nb, nullptr, w.partials, nullptr, st);
    if (e != cudaSuccess) return e;
    if (gather && p == passes - 1)
      bs::launch_pdl(k_radix_scatter<true>, (unsigned)nb, kSortThreads, 0, st, ki, vi, ko, vo, n_cap, d_count, shift, mask, nb,
                                                                   w.hist, *gather);
    else
      bs::launch_pdl(k_radix_scatter<false>, (unsigned)nb, kSortThreads, 0, st, ki, vi, ko, vo, n_cap, d_count, shift, mask, nb,
                                                                    w.hist, RadixGather{});
    count_launches(2);
    uint32_t* t;
    t = ki; ki = ko; ko = t;
    t = vi; vi = vo; vo = t;
    *result_in_alt = !*result_in_alt;
    shift += bits;
  }
  return cudaPeekAtLastError();
}

}  // namespace bs
