// tile_stats.cu — P6: per-tile list lengths, TileHistogram summary and the
// LPT task order for the fine-grained queue (src/preprocess.cpp:117-136).
//
// counts[t] = end - start.  The LPT order (length descending, tile ascending)
// is a stable LSD radix sort of key = ~count; the same sorted array read
// backwards is the ascending order the reference's nearest-rank p50/p99 and
// min/max come from.  mean = (sum in double) / T — every partial sum of u32
// counts is an integer < 2^53, so any summation order gives the reference's
// std::accumulate bits.
#include <math.h>

#include "bs_common.cuh"
#include "radix_sort.cuh"
#include "scan.cuh"

namespace bs {

__global__ void k_counts(const uint32_t* __restrict__ ranges, int T, uint32_t* __restrict__ counts,
                         uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const uint32_t c = ranges[2 * t + 1] - ranges[2 * t];
  counts[t] = c;
  keys[t] = ~c;
  vals[t] = (uint32_t)t;
}

__global__ void __launch_bounds__(1024) k_stats_finish(const uint32_t* __restrict__ counts,
                                                       const uint32_t* __restrict__ desc_order, int T,
                                                       bs_tile_histogram* __restrict__ out) {
  unsigned long long sum = 0, nonempty = 0;
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    const uint32_t c = counts[t];
    sum += c;
    nonempty += c > 0;
  }
  sum = block_reduce_sum(sum);
  nonempty = block_reduce_sum(nonempty);
  if (threadIdx.x == 0) {
    bs_tile_histogram s;
    s.tiles = T;
    s.total = sum;
    s.nonempty = (int32_t)nonempty;
    if (T == 0) {
      s.min = s.max = s.p50 = s.p99 = 0;
      s.mean = 0.0;
    } else {
      auto asc = [&](long long k) { return counts[desc_order[T - 1 - k]]; };
      s.min = asc(0);
      s.max = asc(T - 1);
      s.mean = (double)sum / (double)T;
      auto rank = [&](double q) {
        long long k = (long long)ceil(q * (double)T);
        long long idx = k == 0 ? 0 : k - 1;
        if (idx > T - 1) idx = T - 1;
        return asc(idx);
      };
      s.p50 = rank(0.50);
      s.p99 = rank(0.99);
    }
    *out = s;
  }
}

template <typename C>
inline void stats_ws_layout(C& c, int64_t T, uint32_t** k0, uint32_t** v0, uint32_t** k1, uint32_t** v1,
                            uint32_t** counts, RadixWs* rw) {
  *k0 = c.template take<uint32_t>((size_t)T);
  *v0 = c.template take<uint32_t>((size_t)T);
  *k1 = c.template take<uint32_t>((size_t)T);
  *v1 = c.template take<uint32_t>((size_t)T);
  *counts = c.template take<uint32_t>((size_t)T);
  radix_ws_layout(c, T, rw);
}


}  // namespace bs

using namespace bs;

extern "C" size_t bs_tile_stats_workspace_bytes(int32_t tiles) {
  if (tiles < 0) return 0;
  WsSizer s;
  uint32_t *a, *b, *c, *d, *e;
  RadixWs rw;
  stats_ws_layout(s, tiles, &a, &b, &c, &d, &e, &rw);
  return s.off + 256;
}

extern "C" int bs_tile_stats(const uint32_t* tile_ranges, int32_t tiles, bs_tile_histogram* stats, uint32_t* counts,
                             uint32_t* task_order, void* ws, size_t ws_bytes, void* stream) {
  if (tiles < 0 || !stats || (tiles > 0 && !tile_ranges)) return BS_ERR_INVALID_ARGUMENT;
  if (!ws || ws_bytes < bs_tile_stats_workspace_bytes(tiles)) return BS_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  WsCarver c(ws, ws_bytes);
  uint32_t *k0, *v0, *k1, *v1, *cnt;
  RadixWs rw;
  stats_ws_layout(c, tiles, &k0, &v0, &k1, &v1, &cnt, &rw);
  if (tiles > 0) {
    k_counts<<<(tiles + 255) / 256, 256, 0, st>>>(tile_ranges, tiles, cnt, k0, v0);
    BS_LAUNCH_CHECK();
    bool alt = false;
    BS_CUDA_TRY(radix_sort_pairs(k0, v0, k1, v1, tiles, nullptr, 32, rw, &alt, st));
    const uint32_t* order = alt ? v1 : v0;
    if (counts) BS_CUDA_TRY(cudaMemcpyAsync(counts, cnt, sizeof(uint32_t) * tiles, cudaMemcpyDeviceToDevice, st));
    if (task_order) BS_CUDA_TRY(cudaMemcpyAsync(task_order, order, sizeof(uint32_t) * tiles, cudaMemcpyDeviceToDevice, st));
    k_stats_finish<<<1, 1024, 0, st>>>(cnt, order, tiles, stats);
  } else {
    k_stats_finish<<<1, 1024, 0, st>>>(cnt, nullptr, 0, stats);
  }
  BS_LAUNCH_CHECK();
  return BS_OK;
}
