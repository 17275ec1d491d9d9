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
  bs::pdl_wait();
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
  bs::pdl_wait();
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

// Frame-pipeline form (bs_tile_order): one CTA, counts -> sum / max / nonempty
// and a stable counting sort of the tiles by an eighth-octave length bucket,
// longest bucket first, tile id ascending inside a bucket.  Lengths within a
// bucket differ by < 9 %, which is all the LPT queue order needs.
constexpr int kOrderBuckets = 256;
constexpr int kOrderMaxTiles = 32768;

__device__ __forceinline__ uint32_t len_bucket(uint32_t c) {
  const uint32_t v = c + 1u;  // >= 1
  const uint32_t e = 31u - __clz(v);
  return e < 3u ? v : min(8u * e + ((v >> (e - 3u)) & 7u), (uint32_t)kOrderBuckets - 1u);
}

struct SelectOut {  // optional: the per-frame variant choice from the same statistics
  int32_t* variant;
  int pw, ph, sm_count;
};

__global__ void __launch_bounds__(1024) k_tile_order(const uint32_t* __restrict__ ranges, int T,
                                                     uint32_t* __restrict__ order_out,
                                                     bs_tile_histogram* __restrict__ out, SelectOut sel) {
  bs::pdl_wait();
  __shared__ uint32_t s_cnt[32][kOrderBuckets];  // (warp, bucket) counts, then bases
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < 32 * kOrderBuckets; i += 1024) (&s_cnt[0][0])[i] = 0;
  __syncthreads();
  const int per = (T + 31) / 32, t0 = warp * per, t1 = min(T, t0 + per);  // warp's contiguous tile range
  unsigned long long sum = 0, nonempty = 0;
  uint32_t mx = 0;
  for (int t = t0 + lane; t < t1; t += 32) {
    const uint32_t c = ranges[2 * t + 1] - ranges[2 * t];
    sum += c;
    nonempty += c > 0;
    mx = max(mx, c);
    atomicAdd(&s_cnt[warp][len_bucket(c)], 1u);
  }
  sum = block_reduce_sum(sum);
  nonempty = block_reduce_sum(nonempty);
  {
    __shared__ uint32_t s_max[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) s_max[warp] = mx;
    __syncthreads();
    if (tid == 0) {
      uint32_t m = 0;
      for (int w = 0; w < 32; ++w) m = max(m, s_max[w]);
      bs_tile_histogram s;
      s.tiles = T;
      s.total = sum;
      s.nonempty = (int32_t)nonempty;
      s.max = m;
      s.min = s.p50 = s.p99 = 0;  // order statistics: bs_tile_stats
      s.mean = T ? (double)sum / (double)T : 0.0;
      *out = s;
      if (sel.variant) *sel.variant = select_variant_formula(sum, m, T, sel.pw, sel.ph, sel.sm_count);
    }
  }
  // bases: buckets descending, warps ascending inside a bucket
  {
    const int b = kOrderBuckets - 1 - tid;  // threads 0..255 walk buckets high -> low
    uint32_t tot = 0;
    if (tid < kOrderBuckets)
      for (int w = 0; w < 32; ++w) tot += s_cnt[w][b];
    uint32_t all;
    const uint32_t start = block_exclusive_scan<uint32_t>(tid < kOrderBuckets ? tot : 0u, &all);
    if (tid < kOrderBuckets) {
      uint32_t run = start;
      for (int w = 0; w < 32; ++w) {
        const uint32_t c = s_cnt[w][b];
        s_cnt[w][b] = run;
        run += c;
      }
    }
  }
  __syncthreads();
  const uint32_t lt = lanemask_lt();
  for (int base = t0; base < t1; base += 32) {
    const int t = base + lane;
    const bool act = t < t1;
    const uint32_t bk = act ? len_bucket(ranges[2 * t + 1] - ranges[2 * t]) : 0xffffffffu;
    const uint32_t peers = __match_any_sync(0xffffffffu, bk);
    uint32_t pos = 0;
    if (act) {
      pos = s_cnt[warp][bk] + __popc(peers & lt);
      order_out[pos] = (uint32_t)t;
    }
    __syncwarp();
    if (act && (peers >> lane) == 1u) s_cnt[warp][bk] = pos + 1;
    __syncwarp();
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
    bs::launch_pdl(k_counts, (tiles + 255) / 256, 256, 0, st, tile_ranges, tiles, cnt, k0, v0);
    BS_LAUNCH_CHECK();
    bool alt = false;
    BS_CUDA_TRY(radix_sort_pairs(k0, v0, k1, v1, tiles, nullptr, 32, rw, &alt, st));
    const uint32_t* order = alt ? v1 : v0;
    if (counts) BS_CUDA_TRY(cudaMemcpyAsync(counts, cnt, sizeof(uint32_t) * tiles, cudaMemcpyDeviceToDevice, st));
    if (task_order) BS_CUDA_TRY(cudaMemcpyAsync(task_order, order, sizeof(uint32_t) * tiles, cudaMemcpyDeviceToDevice, st));
    bs::launch_pdl(k_stats_finish, 1, 1024, 0, st, cnt, order, tiles, stats);
  } else {
    bs::launch_pdl(k_stats_finish, 1, 1024, 0, st, cnt, nullptr, 0, stats);
  }
  BS_LAUNCH_CHECK();
  return BS_OK;
}

extern "C" int bs_tile_order(const uint32_t* tile_ranges, int32_t tiles, bs_tile_histogram* stats,
                             uint32_t* task_order, void* stream) {
  if (tiles < 0 || !stats || !task_order || (tiles > 0 && !tile_ranges)) return BS_ERR_INVALID_ARGUMENT;
  if (tiles > kOrderMaxTiles) return BS_ERR_UNSUPPORTED;
  bs::launch_pdl(k_tile_order, 1, 1024, 0, (cudaStream_t)stream, tile_ranges, tiles, task_order, stats,
                                                     SelectOut{nullptr, 0, 0, 0});
  BS_LAUNCH_CHECK();
  return BS_OK;
}

// bs_tile_order + bs_select_variant_device in one launch (the frame
// pipeline's auto mode): *variant <- the selector's choice on these stats.
extern "C" int bs_tile_order_select(const uint32_t* tile_ranges, int32_t tiles, bs_tile_histogram* stats,
                                    uint32_t* task_order, int32_t width, int32_t height, int32_t pw, int32_t ph,
                                    int32_t sm_count, int32_t* variant, void* stream) {
  if (tiles < 0 || !stats || !task_order || !variant || (tiles > 0 && !tile_ranges)) return BS_ERR_INVALID_ARGUMENT;
  if (width <= 0 || height <= 0 || pw <= 0 || ph <= 0) return BS_ERR_INVALID_ARGUMENT;
  if (tiles > kOrderMaxTiles) return BS_ERR_UNSUPPORTED;
  bs::launch_pdl(k_tile_order, 1, 1024, 0, (cudaStream_t)stream, tile_ranges, tiles, task_order, stats,
                                                     SelectOut{variant, pw, ph, sm_count});
  BS_LAUNCH_CHECK();
  return BS_OK;
}
