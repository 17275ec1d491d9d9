// binning.cu — P5: tile binning, bit-exact with src/preprocess.cpp:66-115.
//
// The reference sorts (tile, depth, index) triples with std::sort.  Here the
// same order comes from two stable LSD radix sorts (radix_sort.cuh):
//   1. the n visible splats by depth key (float bits, 4 x 8-bit passes) with
//      values in index order  -> (depth, index) order.  Splats that touch no
//      tile get key 0xffffffff and sink to the end (they emit nothing);
//   2. the K = sum(tiles touched) (tile, splat) instances, expanded in that
//      depth order, by tile id (ceil(log2 T) bits)  -> (tile, depth, index).
// Sorting N depth keys once instead of K 45-bit keys cuts sort traffic ~3x.
//
// Per-tile list lengths are known before any instance exists: every splat's
// tile rectangle adds +1/-1 corners to a (cols+1) x (rows+1) difference grid
// whose 2-D prefix sum is the tile histogram.  That gives the tile ranges
// (exclusive scan; empty tiles get [pos, pos) like the reference's range loop)
// without a boundary search over the K sorted instances.
// The expansion is load-balanced: each thread writes 16 consecutive instances
// (one smem search for the first, then a carry-walk over the rectangle).
#include <math.h>
#include <stdlib.h>

#include "bs_common.cuh"
#include "radix_sort.cuh"
#include "scan.cuh"
#include "tiles.cuh"

namespace bs {

// Per visible splat: tiles touched, packed rect (tx0 | ty0<<16, w | h<<16),
// depth sort key (non-touching -> 0xffffffff), value = index, and the four
// difference-grid corners of its rectangle.  SMEM_DIFF: the CTA accumulates
// the corners in a private shared-memory grid (grid-stride over splats) and
// flushes the non-zero cells once — clustered scenes put thousands of corners
// on the same few cells, which global atomics would serialise.
template <bool SMEM_DIFF>
__global__ void __launch_bounds__(256) k_bin_rect(const float4* __restrict__ xyab, const float4* __restrict__ cop,
                                                  const float4* __restrict__ rgbr, int64_t n_cap,
                                                  const int32_t* __restrict__ n_visible, Grid g,
                                                  uint32_t* __restrict__ touched, uint2* __restrict__ rects,
                                                  uint32_t* __restrict__ dkeys, uint32_t* __restrict__ dvals,
                                                  int* __restrict__ diff) {
  bs::pdl_wait();
  extern __shared__ int s_diff[];
  const int stride = g.cols + 1;
  const int cells = stride * (g.rows + 1);
  int* dd = SMEM_DIFF ? s_diff : diff;
  if (SMEM_DIFF) {
    for (int i = threadIdx.x; i < cells; i += blockDim.x) s_diff[i] = 0;
    __syncthreads();
  }
  const int64_t n = min((int64_t)*n_visible, n_cap);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 a = xyab[i];
    Rect r;
    uint32_t cnt = 0;
    uint2 pk = make_uint2(0u, 0u);
    if (tile_rect(a.x, a.y, rgbr[i].w, g, r)) {
      const uint32_t w = (uint32_t)(r.tx1 - r.tx0 + 1), h = (uint32_t)(r.ty1 - r.ty0 + 1);
      cnt = w * h;
      pk = make_uint2((uint32_t)r.tx0 | ((uint32_t)r.ty0 << 16), w | (h << 16));
      atomicAdd(&dd[r.ty0 * stride + r.tx0], 1);
      atomicAdd(&dd[r.ty0 * stride + r.tx1 + 1], -1);
      atomicAdd(&dd[(r.ty1 + 1) * stride + r.tx0], -1);
      atomicAdd(&dd[(r.ty1 + 1) * stride + r.tx1 + 1], 1);
    }
    touched[i] = cnt;
    rects[i] = pk;
    dkeys[i] = cnt ? float_sort_key(cop[i].w) : 0xffffffffu;
    dvals[i] = (uint32_t)i;
  }
  if (SMEM_DIFF) {
    __syncthreads();
    for (int i = threadIdx.x; i < cells; i += blockDim.x) {
      const int v = s_diff[i];
      if (v) atomicAdd(&diff[i], v);
    }
  }
}

// One CTA: 2-D inclusive prefix of the difference grid in shared memory ->
// per-tile counts.
__global__ void __launch_bounds__(1024) k_diff_scan(const int* __restrict__ diff, Grid g, uint32_t* __restrict__ counts) {
  bs::pdl_wait();
  extern __shared__ int s_grid[];
  const int stride = g.cols + 1, cells = stride * (g.rows + 1);
  for (int i = threadIdx.x; i < cells; i += blockDim.x) s_grid[i] = diff[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int r = warp; r < g.rows; r += nw) {  // rows: warp scans in 32-wide chunks
    int carry = 0;
    for (int x0 = 0; x0 < g.cols; x0 += 32) {
      const int x = x0 + lane;
      int v = x < g.cols ? s_grid[r * stride + x] : 0;
      v = warp_inclusive_scan(v) + carry;
      if (x < g.cols) s_grid[r * stride + x] = v;
      carry = __shfl_sync(0xffffffffu, v, 31);
    }
  }
  __syncthreads();
  for (int tx = threadIdx.x; tx < g.cols; tx += blockDim.x) {  // columns: sequential down rows
    int run = 0;
    for (int ty = 0; ty < g.rows; ++ty) {
      run += s_grid[ty * stride + tx];
      counts[ty * g.cols + tx] = (uint32_t)run;
    }
  }
}

// Fallback for grids beyond shared memory: row CTAs, then a thread per column.
__global__ void __launch_bounds__(256) k_diff_rows(int* __restrict__ diff, int stride) {
  bs::pdl_wait();
  int* row = diff + (size_t)blockIdx.x * stride;
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < stride; base += 256) {
    const int x = base + threadIdx.x;
    const int v = x < stride ? row[x] : 0;
    int tot;
    const int ex = block_exclusive_scan<int>(v, &tot);
    const int c = carry;
    if (x < stride) row[x] = c + ex + v;
    __syncthreads();
    if (threadIdx.x == 0) carry = c + tot;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) k_diff_cols(const int* __restrict__ diff, Grid g, uint32_t* __restrict__ counts) {
  bs::pdl_wait();
  const int tx = blockIdx.x * blockDim.x + threadIdx.x;
  if (tx >= g.cols) return;
  const int stride = g.cols + 1;
  int run = 0;
  for (int ty = 0; ty < g.rows; ++ty) {
    run += diff[ty * stride + tx];
    counts[ty * g.cols + tx] = (uint32_t)run;
  }
}

constexpr size_t kMaxDiffSmem = 200 * 1024;  // <= 227 KB opt-in

// Expansion: block b writes instances [b*4096, b*4096+4096); thread t the 16
// consecutive ones at b*4096 + 16t.  Every splat of the depth-sorted prefix
// emits >= 1 instance, so the window of 4097 offsets in smem always covers a
// block (thread 0 finds its start by binary search).  Each thread searches
// the window once, then walks its rectangle with a carry (no division after
// the first output) and stores 4 x uint4.
constexpr int kExpandItems = 4096;
constexpr int kExpandPer = 16;
constexpr int kExpandWin = kExpandItems + 1;

// block_j0[b] = the splat (depth order) whose instance range holds output
// b*4096: every splat marks the expansion blocks whose first output it owns.
__global__ void k_mark_starts(const uint64_t* __restrict__ offs, const uint32_t* __restrict__ touched_sorted,
                              int64_t n_cap, const int32_t* __restrict__ n_visible, uint32_t* __restrict__ block_j0) {
  bs::pdl_wait();
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n_cap || j >= *n_visible) return;
  const uint64_t lo = offs[j], hi = lo + touched_sorted[j];
  for (uint64_t b = (lo + kExpandItems - 1) / kExpandItems; b * kExpandItems < hi; ++b) block_j0[b] = (uint32_t)j;
}

__global__ void __launch_bounds__(256) k_expand(const uint64_t* __restrict__ offs, const uint32_t* __restrict__ order,
                                                const uint2* __restrict__ rects_sorted, int64_t n_cap,
                                                const int32_t* __restrict__ n_visible, int64_t K, int cols,
                                                const uint32_t* __restrict__ block_j0, uint32_t* __restrict__ keys,
                                                uint32_t* __restrict__ vals) {
  bs::pdl_wait();
  __shared__ uint64_t s_offs[kExpandWin + 1];
  const int tid = threadIdx.x;
  const int64_t o0 = (int64_t)blockIdx.x * kExpandItems;
  const int64_t n = min((int64_t)*n_visible, n_cap);
  const int64_t j0 = block_j0[blockIdx.x];
  const int win = (int)min((int64_t)kExpandWin, n - j0);
  for (int i = tid; i <= win; i += 256) s_offs[i] = (j0 + i < n) ? offs[j0 + i] : (uint64_t)K;
  __syncthreads();
  const int64_t ot = o0 + (int64_t)tid * kExpandPer;
  if (ot >= K) return;
  int lo = 0, hi = win;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (s_offs[mid] <= (uint64_t)ot) lo = mid;
    else hi = mid;
  }
  int i = lo;
  uint64_t next_off = s_offs[i + 1];
  uint2 rc = rects_sorted[j0 + i];
  uint32_t id = order[j0 + i];
  uint32_t w = rc.y & 0xffffu, tx0 = rc.x & 0xffffu;
  uint32_t m = (uint32_t)(ot - (int64_t)s_offs[i]);
  uint32_t tx = tx0 + m % w, ty = (rc.x >> 16) + m / w;
  uint32_t kk[kExpandPer], vv[kExpandPer];
  const int cnt = (int)min((int64_t)kExpandPer, K - ot);
#pragma unroll
  for (int q = 0; q < kExpandPer; ++q) {
    if (q < cnt) {
      const uint64_t o = (uint64_t)(ot + q);
      if (o >= next_off) {
        ++i;
        next_off = s_offs[i + 1];
        rc = rects_sorted[j0 + i];
        id = order[j0 + i];
        w = rc.y & 0xffffu;
        tx0 = rc.x & 0xffffu;
        tx = tx0;
        ty = rc.x >> 16;
      }
      kk[q] = ty * (uint32_t)cols + tx;
      vv[q] = id;
      if (++tx == tx0 + w) {
        tx = tx0;
        ++ty;
      }
    }
  }
  if (cnt == kExpandPer) {
    uint4* k4 = reinterpret_cast<uint4*>(keys + ot);
    uint4* v4 = reinterpret_cast<uint4*>(vals + ot);
#pragma unroll
    for (int q = 0; q < kExpandPer / 4; ++q) {
      k4[q] = make_uint4(kk[4 * q], kk[4 * q + 1], kk[4 * q + 2], kk[4 * q + 3]);
      v4[q] = make_uint4(vv[4 * q], vv[4 * q + 1], vv[4 * q + 2], vv[4 * q + 3]);
    }
  } else {
#pragma unroll
    for (int q = 0; q < kExpandPer; ++q)
      if (q < cnt) {
        keys[ot + q] = kk[q];
        vals[ot + q] = vv[q];
      }
  }
}

// ---------------------------------------------------------------------------
// Chunked counting scatter (default path; replaces expand + tile radix sort).
// The depth-sorted splats are cut into chunks of ~Q consecutive instances.
//   k_chunk_bounds  chunk c = splats [first[c], first[c+1]) (those whose first
//                   instance lies in [cQ, (c+1)Q)); first[nchunks] = number of
//                   splats that touch a tile (they precede the non-touching
//                   ones in depth-key order)
//   k_chunk_hist    per chunk, a shared-memory difference grid of its
//                   rectangles -> per-tile counts M[c][t]
//   k_chunk_scan    in place, M[c][t] <- starts[t] + sum_{c' < c} M[c'][t]
//   k_chunk_scatter per chunk, the offsets row in shared memory; warp w owns
//                   a band of tile rows (equal instance counts) and walks the
//                   chunk's splats in depth order, 32 instances per step; equal tiles
//                   inside a step are ranked by match.any (lane order = depth
//                   order), so every tile list is written in (depth, index)
//                   order directly — point_list is the final order without
//                   materialising or sorting K keys.
constexpr int kScWarps = 16;
constexpr int kScThreads = kScWarps * 32;
constexpr int kScMaxRows = 1024;                     // tile rows the row-band split supports
constexpr int64_t kScTableBytes = 40 * 1024;         // offsets-row slice per CTA (row bands beyond)
constexpr int64_t kMaxChunkMatrix = (int64_t)64 << 20;  // entries of M (256 MB)
constexpr int kMaxChunks = 4096;
constexpr size_t kMaxScatterSmem = 200 * 1024;           // offsets row (T u32) + warp buffers

// first[c] = lower_bound(offs[0, nt), c*q) for c < nchunks, first[nchunks] =
// nt (the touching splats).  Splat j marks the chunks whose first instance
// offset c*q falls in (offs[j-1], offs[j]]; the last touching splat also
// marks every chunk past its own offset.  One coalesced pass, no searches.
__global__ void k_chunk_bounds(const uint64_t* __restrict__ offs, const uint32_t* __restrict__ touched_sorted,
                               int64_t n_cap, const int32_t* __restrict__ n_visible, const uint64_t* __restrict__ kd,
                               int64_t k_cap, int nchunks, uint32_t* __restrict__ first) {
  bs::pdl_wait();
  const uint64_t K = *kd;
  if (K == 0 || K > (uint64_t)k_cap) return;  // nothing to do / point_list too small (bs_bin_sort_async)
  const int64_t q = (int64_t)((K + (uint64_t)nchunks - 1) / (uint64_t)nchunks);
  const int64_t n = min((int64_t)*n_visible, n_cap);
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n || touched_sorted[j] == 0) return;
  const uint64_t hi = offs[j];
  const int64_t c_lo = j == 0 ? 0 : (int64_t)((offs[j - 1] + (uint64_t)q) / (uint64_t)q);  // c*q > offs[j-1]
  const int64_t c_hi = (int64_t)(hi / (uint64_t)q);                                        // c*q <= offs[j]
  for (int64_t c = c_lo; c <= c_hi && c < nchunks; ++c) first[c] = (uint32_t)j;
  if (j + 1 == n || touched_sorted[j + 1] == 0) {
    for (int64_t c = c_hi + 1; c <= nchunks; ++c) first[c] = (uint32_t)(j + 1);
  }
}

// Also writes the chunk's per-row instance counts rowc[c][ty] (the scatter
// splits the rows among its warps by them).
__global__ void __launch_bounds__(kScThreads) k_chunk_hist(const uint2* __restrict__ rects_sorted,
                                                           const uint32_t* __restrict__ first, Grid g,
                                                           uint32_t* __restrict__ m, uint32_t* __restrict__ rowc,
                                                           const uint64_t* __restrict__ kd, int64_t k_cap) {
  bs::pdl_wait();
  if (*kd == 0 || *kd > (uint64_t)k_cap) return;
  extern __shared__ int s_grid[];
  const int stride = g.cols + 1, cells = stride * (g.rows + 1);
  int* s_rowd = s_grid + cells;  // rows + 1 (difference array of per-row counts)
  const int c = blockIdx.x, tid = threadIdx.x;
  for (int i = tid; i < cells + g.rows + 1; i += kScThreads) s_grid[i] = 0;
  __syncthreads();
  const uint32_t j0 = first[c], j1 = first[c + 1];
  for (uint32_t j = j0 + tid; j < j1; j += kScThreads) {
    const uint2 rc = rects_sorted[j];
    const int tx0 = rc.x & 0xffff, ty0 = rc.x >> 16;
    const int w = (int)(rc.y & 0xffff);
    const int tx1 = tx0 + w, ty1 = ty0 + (int)(rc.y >> 16);  // exclusive
    atomicAdd(&s_grid[ty0 * stride + tx0], 1);
    atomicAdd(&s_grid[ty0 * stride + tx1], -1);
    atomicAdd(&s_grid[ty1 * stride + tx0], -1);
    atomicAdd(&s_grid[ty1 * stride + tx1], 1);
    atomicAdd(&s_rowd[ty0], w);
    atomicAdd(&s_rowd[ty1], -w);
  }
  __syncthreads();
  if (tid < 32) {
    int carry = 0;
    for (int r0 = 0; r0 < g.rows; r0 += 32) {
      const int r = r0 + tid;
      int v = r < g.rows ? s_rowd[r] : 0;
      v = warp_inclusive_scan(v) + carry;
      if (r < g.rows) rowc[(int64_t)c * g.rows + r] = (uint32_t)v;
      carry = __shfl_sync(0xffffffffu, v, 31);
    }
  }
  const int lane = tid & 31, warp = tid >> 5;
  for (int r = warp; r < g.rows; r += kScWarps) {
    int carry = 0;
    for (int x0 = 0; x0 < g.cols; x0 += 32) {
      const int x = x0 + lane;
      int v = x < g.cols ? s_grid[r * stride + x] : 0;
      v = warp_inclusive_scan(v) + carry;
      if (x < g.cols) s_grid[r * stride + x] = v;
      carry = __shfl_sync(0xffffffffu, v, 31);
    }
  }
  __syncthreads();
  uint32_t* row = m + (int64_t)c * g.cols * g.rows;
  for (int tx = tid; tx < g.cols; tx += kScThreads) {
    int run = 0;
    for (int ty = 0; ty < g.rows; ++ty) {
      run += s_grid[ty * stride + tx];
      row[ty * g.cols + tx] = (uint32_t)run;
    }
  }
}

// CTA = 32 consecutive tiles (lane) x 32 warps (chunk segments): enough
// independent loads in flight to stream M at HBM rate.
constexpr int kCsSeg = 32;
__global__ void __launch_bounds__(kCsSeg * 32) k_chunk_scan(uint32_t* __restrict__ m,
                                                            const uint32_t* __restrict__ starts, int T, int nchunks,
                                                            const uint64_t* __restrict__ kd, int64_t k_cap) {
  bs::pdl_wait();
  if (*kd == 0 || *kd > (uint64_t)k_cap) return;
  __shared__ uint32_t s_part[kCsSeg][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = blockIdx.x * 32 + lane;
  const int c0 = (int)((int64_t)nchunks * warp / kCsSeg), c1 = (int)((int64_t)nchunks * (warp + 1) / kCsSeg);
  uint32_t sum = 0;
  if (t < T) {
#pragma unroll 4
    for (int c = c0; c < c1; ++c) sum += m[(int64_t)c * T + t];
  }
  s_part[warp][lane] = sum;
  __syncthreads();
  if (t >= T) return;
  uint32_t run = starts[t];
  for (int w = 0; w < warp; ++w) run += s_part[w][lane];
#pragma unroll 4
  for (int c = c0; c < c1; ++c) {
    const int64_t i = (int64_t)c * T + t;
    const uint32_t v = m[i];
    m[i] = run;
    run += v;
  }
}

__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_u32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// Per chunk: the offsets row in shared memory; the tile rows are split into
// kScWarps contiguous bands of about equal instance count (from the chunk's
// per-row counts), warp w owning band w.  Each warp walks the chunk's splats
// in depth order, keeps those whose rectangle meets its band (ballot
// compaction into a per-warp queue), and for every 32 queued splats lists
// their band tiles (row-major, tile | lane << 16) in a per-warp window and
// drains it 32 instances per step: equal tiles in a step are ranked by
// match.any (lane order = depth order), the highest peer advances the
// tile's offset.  Every tile list comes out in (depth, index) order.
struct ScQ {
  uint32_t rx, ry, id;  // packed rect (tx0 | ty0 << 16, w | h << 16) and splat id
};

__global__ void __launch_bounds__(kScThreads) k_chunk_scatter(const uint32_t* __restrict__ m,
                                                              const uint32_t* __restrict__ rowc,
                                                              const uint32_t* __restrict__ first,
                                                              const uint2* __restrict__ rects_sorted,
                                                              const uint32_t* __restrict__ order, int T, int cols,
                                                              int rows, uint32_t* __restrict__ point_list,
                                                              const uint64_t* __restrict__ kd, int64_t k_cap,
                                                              int band_rows) {
  bs::pdl_wait();
  if (*kd == 0 || *kd > (uint64_t)k_cap) return;
  extern __shared__ uint32_t s_off[];
  __shared__ ScQ s_q[kScWarps][64];
  __shared__ uint32_t s_rowp[kScMaxRows + 1];
  const int c = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // this CTA: tile rows [R0, R0 + nbr) of chunk c (grids whose offsets row
  // would not fit shared memory are split into row bands, blockIdx.y)
  const int R0 = blockIdx.y * band_rows, nbr = min(rows - R0, band_rows);
  const uint32_t* mrow = m + (int64_t)c * T + (int64_t)R0 * cols;
  for (int t = tid; t < nbr * cols; t += kScThreads) s_off[t] = mrow[t];
  if (warp == 0) {  // inclusive prefix of the chunk's per-row counts (this band)
    uint32_t carry = 0;
    if (lane == 0) s_rowp[0] = 0;
    for (int r0 = 0; r0 < nbr; r0 += 32) {
      const int r = r0 + lane;
      uint32_t v = r < nbr ? rowc[(int64_t)c * rows + R0 + r] : 0u;
      v = warp_inclusive_scan(v) + carry;
      if (r < nbr) s_rowp[r + 1] = v;
      carry = __shfl_sync(0xffffffffu, v, 31);
    }
  }
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(s_off) - 4u * (uint32_t)(R0 * cols);
  __syncthreads();
  // band of this warp: row r belongs to warp floor(kScWarps * mid(r) / total),
  // mid(r) = the row's middle instance (monotone in r -> contiguous bands)
  const int rows_b = nbr;
  const uint64_t total = s_rowp[rows_b];
  if (total == 0) return;
  // (a multiply by a per-CTA reciprocal instead of a 64-bit division: any
  // monotone owner function gives contiguous bands, and every warp of the
  // CTA evaluates the same one)
  const double own_scale = (double)kScWarps / (2.0 * (double)total);
  auto owner = [&](int r) -> int {
    const double mid2 = (double)s_rowp[r] + (double)s_rowp[r + 1];  // 2 * middle
    return min(kScWarps - 1, (int)(mid2 * own_scale));
  };
  auto band_start = [&](int w) -> int {  // first row whose owner >= w
    int lo = 0, hi = rows_b;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (owner(mid) < w) lo = mid + 1;
      else hi = mid;
    }
    return lo;
  };
  const uint32_t r0 = (uint32_t)(R0 + band_start(warp)), r1 = (uint32_t)(R0 + band_start(warp + 1));
  const uint32_t lt = lanemask_lt();
  const uint32_t j0 = first[c], j1 = first[c + 1];
  int qn = 0;  // queued splats (warp-uniform)

  // drain the first nq queue entries' band tiles, 32 instances per step:
  // instance f of the flat (splat, row, column) enumeration belongs to the
  // last lane whose exclusive count is <= f (window bitmask, below); its
  // row / column come from one float multiply by the lane's 1/w (exact:
  // f < 2^22).  Equal tiles inside a step are ranked by match.any (lane
  // order = depth order); the highest peer advances the tile's offset.
  auto flush32 = [&](int nq) {
    const ScQ q = s_q[warp][lane];
    int cnt = 0;
    uint32_t tb = 0, w = 1;
    if (lane < nq) {
      const uint32_t rx0 = q.rx & 0xffffu, ry0 = q.rx >> 16;
      w = q.ry & 0xffffu;
      const uint32_t ya = max(ry0, r0), yb = min(ry0 + (q.ry >> 16), r1);
      cnt = (int)((yb - ya) * w);
      tb = ya * (uint32_t)cols + rx0;
    }
    const float inv = __frcp_rn((float)w);
    const int incl = warp_inclusive_scan(cnt);
    const int excl = incl - cnt;
    const int tot = __shfl_sync(0xffffffffu, incl, 31);
    // instance f -> (tile, splat id); 0xffffffff tile past the end.  The
    // queued splats whose first instance falls inside the 32-instance window
    // [f0, f0 + 32) set one bit each (one redux.or): instance f0 + lane
    // belongs to the window's first splat plus the number of starts in
    // (f0, f0 + lane]; sb tracks the window's first splat.  (A 5-step
    // shuffle binary search over the exclusive counts measured 2.6 % slower.)
    int sb = 0;
    auto resolve = [&](int f0, uint32_t& tile, uint32_t& sid, bool& one) {
      const int k = excl - f0;
      const uint32_t m = __reduce_or_sync(0xffffffffu, (lane < nq && k >= 1 && k < 32) ? (1u << k) : 0u);
      one = m == 0u;  // the whole window is one splat's: its tiles are distinct
      const bool next_starts = __ballot_sync(0xffffffffu, lane < nq && k == 32) != 0u;
      const uint32_t upto = lane == 31 ? 0xffffffffu : ((2u << lane) - 1u);
      const int sl = sb + __popc(m & upto);
      sb += __popc(m) + (next_starts ? 1 : 0);
      const int f = f0 + lane;
      const int e0 = __shfl_sync(0xffffffffu, excl, sl);
      const uint32_t local = (uint32_t)(f - e0);
      const uint32_t ws = __shfl_sync(0xffffffffu, w, sl);
      const float iv = __shfl_sync(0xffffffffu, inv, sl);
      const uint32_t t0 = __shfl_sync(0xffffffffu, tb, sl);
      sid = __shfl_sync(0xffffffffu, q.id, sl);
      const uint32_t r = (uint32_t)(((float)local + 0.5f) * iv);
      tile = f < tot ? t0 + r * (uint32_t)cols + (local - r * ws) : 0xffffffffu;
    };
    // software-pipelined: the next step's resolve is independent of
    // this step's match / shared-memory chain, so their latencies overlap
    uint32_t tile, sid;
    bool one;
    resolve(0, tile, sid, one);
    for (int f0 = 0; f0 < tot; f0 += 32) {
      uint32_t ntile = 0xffffffffu, nsid = 0;
      bool none = false;
      if (f0 + 32 < tot) resolve(f0 + 32, ntile, nsid, none);
      const bool act = tile != 0xffffffffu;
      const uint32_t peers = one ? (1u << lane) : __match_any_sync(0xffffffffu, tile);
      const uint32_t a = sbase + 4u * tile;
      uint32_t pos = 0;
      if (act) {
        pos = lds_u32(a) + __popc(peers & lt);
        point_list[pos] = sid;
      }
      __syncwarp();
      if (act && (peers >> lane) == 1u) sts_u32(a, pos + 1);  // highest peer publishes
      __syncwarp();
      tile = ntile;
      sid = nsid;
      one = none;
    }
  };

  // each warp walks the chunk on its own (no CTA barrier couples the warps'
  // unequal flush work), the batch two ahead in flight
  uint2 rc1 = make_uint2(0u, 0u), rc2 = rc1;
  uint32_t id1 = 0, id2 = 0;
  if (j0 + lane < j1) {
    rc1 = rects_sorted[j0 + lane];
    id1 = order[j0 + lane];
  }
  if (j0 + 32 + lane < j1) {
    rc2 = rects_sorted[j0 + 32 + lane];
    id2 = order[j0 + 32 + lane];
  }
  for (uint32_t b = j0; b < j1; b += 32) {
    const ScQ e = ScQ{rc1.x, rc1.y, id1};
    const bool valid = b + lane < j1;
    rc1 = rc2;
    id1 = id2;
    if (b + 64 + lane < j1) {
      rc2 = rects_sorted[b + 64 + lane];
      id2 = order[b + 64 + lane];
    }
    const uint32_t ry0 = e.rx >> 16, rh = e.ry >> 16;
    const bool hit = valid && ry0 < r1 && ry0 + rh > r0;
    const uint32_t hm = __ballot_sync(0xffffffffu, hit);
    if (hit) s_q[warp][qn + __popc(hm & lt)] = e;
    qn += __popc(hm);
    __syncwarp();
    if (qn >= 32) {
      flush32(32);
      __syncwarp();
      qn -= 32;
      if (lane < qn) s_q[warp][lane] = s_q[warp][lane + 32];
      __syncwarp();
    }
  }
  if (qn > 0) flush32(qn);
}

// Tile ranges from the exclusive scan of the counts.  On a point_list
// overflow (kd > k_cap) every range is written empty so a render enqueued
// behind it reads nothing.
__global__ void k_ranges(const uint32_t* __restrict__ starts, const uint32_t* __restrict__ counts, int T,
                         uint32_t* __restrict__ ranges, const uint64_t* __restrict__ kd, int64_t k_cap) {
  bs::pdl_wait();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  if (kd && *kd > (uint64_t)k_cap) {
    ranges[2 * t] = ranges[2 * t + 1] = 0u;
    return;
  }
  const uint32_t s = starts[t];
  ranges[2 * t] = s;
  ranges[2 * t + 1] = s + counts[t];
}

inline Grid make_grid(int W, int H, int pw, int ph) {
  Grid g;
  g.W = W; g.H = H; g.pw = pw; g.ph = ph;
  g.cols = (W + pw - 1) / pw;
  g.rows = (H + ph - 1) / ph;
  return g;
}

inline int bits_for(int64_t values) {  // bits to represent 0..values-1
  int b = 0;
  while (b < 63 && ((int64_t)1 << b) < values) ++b;
  return b;
}

// Workspace layout shared by bs_bin_count and bs_bin_sort (same carve order;
// the k-sized tail is last so a count-phase carve is a prefix of it).
struct BinWs {
  uint32_t *touched, *dk0, *dv0, *dk1, *dv1, *touched_sorted;
  uint2 *rects, *rects_sorted;
  uint64_t* offs;
  uint64_t* offs_partials;
  RadixWs rws_n;
  int* diff;
  uint32_t *counts, *starts, *cpartials;
  uint32_t *tk0, *tv_alt, *tk1, *block_j0;
  RadixWs rws_k;
  uint32_t *chunk_first, *chunk_m, *chunk_rowc;
};

// The chunked counting scatter needs the per-chunk offsets row (T u32) and
// the difference grid in shared memory; BS_BIN_RADIX=1 forces the expand +
// tile radix sort path (A/B measurement, parity tests of both paths).
inline bool bin_chunked(const Grid& g) {
  static const int forced_radix = [] {
    const char* e = getenv("BS_BIN_RADIX");
    return (e && e[0] == '1') ? 1 : 0;
  }();
  return !forced_radix && g.rows <= kScMaxRows && (size_t)(g.cols + 32) * 4 <= (size_t)kScTableBytes &&
         sizeof(int) * (size_t)(g.cols + 1) * (g.rows + 1) <= kMaxDiffSmem;
}

inline int64_t max_chunks(const Grid& g) {
  const int64_t T = max((int64_t)1, (int64_t)g.cols * g.rows);
  return max((int64_t)1, min((int64_t)kMaxChunks, kMaxChunkMatrix / T));
}

template <typename C>
inline void bin_ws_layout(C& c, int64_t n_cap, const Grid& g, int64_t k_cap, BinWs* w) {
  BinWs tmp;
  BinWs& o = w ? *w : tmp;
  const int64_t T = (int64_t)g.cols * g.rows;
  o.touched = c.template take<uint32_t>((size_t)n_cap);
  o.dk0 = c.template take<uint32_t>((size_t)n_cap);
  o.dv0 = c.template take<uint32_t>((size_t)n_cap);
  o.dk1 = c.template take<uint32_t>((size_t)n_cap);
  o.dv1 = c.template take<uint32_t>((size_t)n_cap);
  o.touched_sorted = c.template take<uint32_t>((size_t)n_cap);
  o.rects = c.template take<uint2>((size_t)n_cap);
  o.rects_sorted = c.template take<uint2>((size_t)n_cap);
  o.offs = c.template take<uint64_t>((size_t)n_cap);
  o.offs_partials = c.template take<uint64_t>((size_t)scan_num_blocks(n_cap) + 1);
  radix_ws_layout(c, n_cap, &o.rws_n);
  o.diff = c.template take<int>((size_t)(g.cols + 1) * (g.rows + 1));
  o.counts = c.template take<uint32_t>((size_t)T);
  o.starts = c.template take<uint32_t>((size_t)T);
  o.cpartials = c.template take<uint32_t>((size_t)scan_num_blocks(T) + 1);
  if (bin_chunked(g)) {
    // chunked counting scatter: chunk bounds + the chunk x tile offsets matrix
    o.chunk_first = c.template take<uint32_t>((size_t)kMaxChunks + 1);
    o.chunk_m = c.template take<uint32_t>((size_t)(max_chunks(g) * T));
    o.chunk_rowc = c.template take<uint32_t>((size_t)(max_chunks(g) * g.rows));
    return;
  }
  o.tk0 = c.template take<uint32_t>((size_t)k_cap);
  o.tv_alt = c.template take<uint32_t>((size_t)k_cap);
  o.tk1 = c.template take<uint32_t>((size_t)k_cap);
  o.block_j0 = c.template take<uint32_t>((size_t)(k_cap / kExpandItems + 1));
  radix_ws_layout(c, k_cap, &o.rws_k);
}

// K to *k_total — device memory, or mapped pinned host memory (the frame
// pipeline reads K there without a D2H copy); total == null stores 0
__global__ void k_store_k(const uint64_t* __restrict__ total, int64_t* k_total) {
  bs::pdl_wait();
  *reinterpret_cast<volatile int64_t*>(k_total) = total ? (int64_t)*total : 0;
  __threadfence_system();
}

}  // namespace bs

using namespace bs;

extern "C" size_t bs_bin_workspace_bytes(int64_t n_cap, int32_t width, int32_t height, int32_t pw, int32_t ph,
                                         int64_t k_cap) {
  if (n_cap < 0 || width <= 0 || height <= 0 || pw <= 0 || ph <= 0 || k_cap < 0) return 0;
  const Grid g = make_grid(width, height, pw, ph);
  WsSizer s;
  bin_ws_layout(s, n_cap, g, k_cap, nullptr);
  return s.off + 256;
}

static int check_grid(int32_t W, int32_t H, int32_t pw, int32_t ph) {
  if (W <= 0 || H <= 0 || pw <= 0 || ph <= 0) return BS_ERR_INVALID_ARGUMENT;
  const int64_t cols = (W + pw - 1) / pw, rows = (H + ph - 1) / ph;
  if (cols > 65535 || rows > 65535 || cols * rows > (1 << 24)) return BS_ERR_UNSUPPORTED;
  return BS_OK;
}

// P5 count after the per-splat pass (k_bin_rect or the fused
// k_project_bin): depth sort, sorted rects, instance offsets, K, tile counts.
static int bin_count_tail(int64_t n_cap, const int32_t* n_visible, const Grid& gr, const BinWs& w, bool smem_diff,
                          size_t diff_bytes, int64_t* k_total, cudaStream_t st) {
  const int64_t T = (int64_t)gr.cols * gr.rows;
  if (n_cap > 0) {
    const unsigned nb = (unsigned)((n_cap + 255) / 256);
    (void)nb;
    bool alt = false;
    // the last pass also gathers (touched, rect) into depth order
    const RadixGather gat{w.touched, w.rects, w.touched_sorted, w.rects_sorted};
    BS_CUDA_TRY(radix_sort_pairs(w.dk0, w.dv0, w.dk1, w.dv1, n_cap, n_visible, 32, w.rws_n, &alt, st, &gat));
    uint64_t* total = w.offs_partials + scan_num_blocks(n_cap);
    BS_CUDA_TRY((exclusive_scan<uint32_t, uint64_t>(w.touched_sorted, w.offs, n_cap, n_visible, w.offs_partials,
                                                    total, st)));
    bs::launch_pdl(k_store_k, 1, 1, 0, st, total, k_total);
    BS_LAUNCH_CHECK();
  } else {
    bs::launch_pdl(k_store_k, 1, 1, 0, st, nullptr, k_total);
    BS_LAUNCH_CHECK();
  }
  // tile histogram from the difference grid -> counts, starts, digit counts
  if (smem_diff) {
    bs::launch_pdl(k_diff_scan, 1, 1024, diff_bytes, st, w.diff, gr, w.counts);
    BS_LAUNCH_CHECK();
  } else {
    bs::launch_pdl(k_diff_rows, (unsigned)(gr.rows + 1), 256, 0, st, w.diff, gr.cols + 1);
    BS_LAUNCH_CHECK();
    bs::launch_pdl(k_diff_cols, (unsigned)((gr.cols + 255) / 256), 256, 0, st, w.diff, gr, w.counts);
    BS_LAUNCH_CHECK();
  }
  BS_CUDA_TRY((exclusive_scan<uint32_t, uint32_t>(w.counts, w.starts, T, nullptr, w.cpartials, nullptr, st)));
  return BS_OK;
}

static bool g_diff_attr_set = false;

extern "C" int bs_bin_count(bs_splats g, int64_t n_cap, const int32_t* n_visible, int32_t width, int32_t height,
                            int32_t pw, int32_t ph, int64_t* k_total, void* ws, size_t ws_bytes, void* stream) {
  int s = check_grid(width, height, pw, ph);
  if (s) return s;
  if (n_cap < 0 || !n_visible || !k_total || (n_cap > 0 && (!g.xyab || !g.cop || !g.rgbr))) return BS_ERR_INVALID_ARGUMENT;
  if (n_cap >= (int64_t)1 << 30) return BS_ERR_CAPACITY;
  cudaStream_t st = (cudaStream_t)stream;
  const Grid gr = make_grid(width, height, pw, ph);
  if (!ws || ws_bytes < bs_bin_workspace_bytes(n_cap, width, height, pw, ph, 0)) return BS_ERR_WORKSPACE;
  WsCarver c(ws, ws_bytes);
  BinWs w;
  bin_ws_layout(c, n_cap, gr, 0, &w);
  BS_CUDA_TRY(cudaMemsetAsync(w.diff, 0, sizeof(int) * (size_t)(gr.cols + 1) * (gr.rows + 1), st));
  const size_t diff_bytes = sizeof(int) * (size_t)(gr.cols + 1) * (gr.rows + 1);
  const bool smem_diff = diff_bytes <= kMaxDiffSmem;
  if (smem_diff && !g_diff_attr_set) {
    BS_CUDA_TRY(cudaFuncSetAttribute(k_bin_rect<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxDiffSmem));
    BS_CUDA_TRY(cudaFuncSetAttribute(k_diff_scan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxDiffSmem));
    g_diff_attr_set = true;
  }
  if (n_cap > 0) {
    const unsigned nb = (unsigned)((n_cap + 255) / 256);
    const float4* xa = reinterpret_cast<const float4*>(g.xyab);
    const float4* xc = reinterpret_cast<const float4*>(g.cop);
    const float4* xr = reinterpret_cast<const float4*>(g.rgbr);
    if (smem_diff) {
      int dev = 0, sms = 148;
      BS_CUDA_TRY(cudaGetDevice(&dev));
      BS_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      const unsigned grid = (unsigned)min((int64_t)nb, (int64_t)sms * 2);
      bs::launch_pdl(k_bin_rect<true>, grid, 256, diff_bytes, st, xa, xc, xr, n_cap, n_visible, gr, w.touched, w.rects, w.dk0,
                                                      w.dv0, w.diff);
    } else {
      bs::launch_pdl(k_bin_rect<false>, nb, 256, 0, st, xa, xc, xr, n_cap, n_visible, gr, w.touched, w.rects, w.dk0, w.dv0,
                                            w.diff);
    }
    BS_LAUNCH_CHECK();
  }
  return bin_count_tail(n_cap, n_visible, gr, w, smem_diff, diff_bytes, k_total, st);
}

// P1-P4 + P5 count in one pass for the frame pipeline (see
// launch_project_bin): splats stay at their input index, counts[0] <- n
// (what the binning kernels read as the splat count), counts[1] <- visible
// splats.  bs_bin_sort / bs_bin_sort_async follow with n_cap = n and
// n_visible = counts.  Tile lists index the uncompacted splat arrays; their
// order equals the reference's (compaction is monotone).
extern "C" int bs_preprocess_bin_count(const bs_gaussian3d* g3d, int64_t n, const bs_camera* cam,
                                       const bs_camera* cam_dev, bs_splats out, int32_t* counts, int32_t width,
                                       int32_t height, int32_t pw, int32_t ph, int64_t* k_total, void* ws,
                                       size_t ws_bytes, void* stream) {
  int s = check_grid(width, height, pw, ph);
  if (s) return s;
  if (n < 0 || (!cam && !cam_dev) || !counts || !k_total || (n > 0 && (!g3d || !out.xyab || !out.cop || !out.rgbr)))
    return BS_ERR_INVALID_ARGUMENT;
  if (n >= (int64_t)1 << 30) return BS_ERR_CAPACITY;
  cudaStream_t st = (cudaStream_t)stream;
  const Grid gr = make_grid(width, height, pw, ph);
  if (!ws || ws_bytes < bs_bin_workspace_bytes(n, width, height, pw, ph, 0)) return BS_ERR_WORKSPACE;
  WsCarver c(ws, ws_bytes);
  BinWs w;
  bin_ws_layout(c, n, gr, 0, &w);
  const size_t diff_bytes = sizeof(int) * (size_t)(gr.cols + 1) * (gr.rows + 1);
  const bool smem_diff = diff_bytes <= kMaxDiffSmem;
  if (smem_diff && !g_diff_attr_set) {
    BS_CUDA_TRY(cudaFuncSetAttribute(k_bin_rect<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxDiffSmem));
    BS_CUDA_TRY(cudaFuncSetAttribute(k_diff_scan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxDiffSmem));
    g_diff_attr_set = true;
  }
  BS_CUDA_TRY(cudaMemsetAsync(w.diff, 0, diff_bytes, st));
  BS_CUDA_TRY(cudaMemsetAsync(counts, 0, 2 * sizeof(int32_t), st));
  if (n > 0)
    BS_CUDA_TRY(launch_project_bin(g3d, n, cam, cam_dev, gr, reinterpret_cast<float4*>(out.xyab),
                                   reinterpret_cast<float4*>(out.cop), reinterpret_cast<float4*>(out.rgbr), w.touched,
                                   w.rects, w.dk0, w.dv0, w.diff, diff_bytes, smem_diff, counts, st));
  return bin_count_tail(n, counts, gr, w, smem_diff, diff_bytes, k_total, st);
}

// ---------------------------------------------------------------------------
// Super-tile binning for the frame pipeline: the lists are built at
// 2pw x 2ph (about a third of the instances at C2 — the scatter is the
// dominant binning cost) and the render keeps, per pw x ph tile, the entries
// whose rectangle contains it (bs_render_forward_super).  The pw x ph list
// lengths (tile statistics, LPT order, selector) come from a second
// difference grid in the same projection pass.  Power-of-two patches only.
static bool pow2i(int v) { return v > 0 && (v & (v - 1)) == 0; }

extern "C" size_t bs_super_aux_bytes(int32_t width, int32_t height, int32_t pw, int32_t ph) {
  if (width <= 0 || height <= 0 || pw <= 0 || ph <= 0) return 0;
  const Grid g = make_grid(width, height, pw, ph);
  const int64_t T = (int64_t)g.cols * g.rows;
  WsSizer z;
  z.take<int>((size_t)(g.cols + 1) * (g.rows + 1));  // diff
  z.take<uint32_t>((size_t)T);                        // counts
  z.take<uint32_t>((size_t)T);                        // starts
  z.take<uint32_t>((size_t)scan_num_blocks(T) + 1);   // scan partials
  return z.off + 256;
}

extern "C" int bs_super_tile_lengths(void* aux, size_t aux_bytes, int32_t width, int32_t height, int32_t pw,
                                     int32_t ph, uint32_t* tile_ranges, void* stream);

extern "C" int bs_preprocess_bin_count_super(const bs_gaussian3d* g3d, int64_t n, const bs_camera* cam,
                                             const bs_camera* cam_dev, bs_splats out, int32_t* counts,
                                             int32_t width, int32_t height, int32_t pw, int32_t ph,
                                             int64_t* k_total, void* ws, size_t ws_bytes, uint32_t* tile_ranges,
                                             void* aux, size_t aux_bytes, void* stream) {
  if (!pow2i(pw) || !pow2i(ph) || pw > 16384 || ph > 16384) return BS_ERR_UNSUPPORTED;
  int s = check_grid(width, height, 2 * pw, 2 * ph);
  if (s) return s;
  if (n < 0 || (!cam && !cam_dev) || !counts || !k_total ||
      (n > 0 && (!g3d || !out.xyab || !out.cop || !out.rgbr)))
    return BS_ERR_INVALID_ARGUMENT;
  if (n >= (int64_t)1 << 30) return BS_ERR_CAPACITY;
  cudaStream_t st = (cudaStream_t)stream;
  const Grid gs = make_grid(width, height, 2 * pw, 2 * ph);
  const Grid gt = make_grid(width, height, pw, ph);
  const int64_t T = (int64_t)gt.cols * gt.rows;
  if (!ws || ws_bytes < bs_bin_workspace_bytes(n, width, height, 2 * pw, 2 * ph, 0)) return BS_ERR_WORKSPACE;
  if (!aux || aux_bytes < bs_super_aux_bytes(width, height, pw, ph)) return BS_ERR_WORKSPACE;
  WsCarver c(ws, ws_bytes);
  BinWs w;
  bin_ws_layout(c, n, gs, 0, &w);
  WsCarver ca(aux, aux_bytes);
  int* diff2 = ca.take<int>((size_t)(gt.cols + 1) * (gt.rows + 1));
  uint32_t* counts2 = ca.take<uint32_t>((size_t)T);
  uint32_t* starts2 = ca.take<uint32_t>((size_t)T);
  uint32_t* partials2 = ca.take<uint32_t>((size_t)scan_num_blocks(T) + 1);
  const size_t diff_bytes = sizeof(int) * (size_t)(gs.cols + 1) * (gs.rows + 1);
  const size_t diff2_bytes = sizeof(int) * (size_t)(gt.cols + 1) * (gt.rows + 1);
  const bool smem_diff = diff_bytes <= kMaxDiffSmem;
  if (!g_diff_attr_set) {
    BS_CUDA_TRY(cudaFuncSetAttribute(k_bin_rect<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxDiffSmem));
    BS_CUDA_TRY(cudaFuncSetAttribute(k_diff_scan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxDiffSmem));
    g_diff_attr_set = true;
  }
  BS_CUDA_TRY(cudaMemsetAsync(w.diff, 0, diff_bytes, st));
  BS_CUDA_TRY(cudaMemsetAsync(diff2, 0, diff2_bytes, st));
  BS_CUDA_TRY(cudaMemsetAsync(counts, 0, 2 * sizeof(int32_t), st));
  if (n > 0)
    BS_CUDA_TRY(launch_project_bin(g3d, n, cam, cam_dev, gs, reinterpret_cast<float4*>(out.xyab),
                                   reinterpret_cast<float4*>(out.cop), reinterpret_cast<float4*>(out.rgbr), w.touched,
                                   w.rects, w.dk0, w.dv0, w.diff, diff_bytes, smem_diff, counts, st, &gt, diff2));
  s = bin_count_tail(n, counts, gs, w, smem_diff, diff_bytes, k_total, st);
  if (s) return s;
  (void)counts2;
  (void)starts2;
  (void)partials2;
  return tile_ranges ? bs_super_tile_lengths(aux, aux_bytes, width, height, pw, ph, tile_ranges, stream) : BS_OK;
}

// The pw x ph list lengths of the last bs_preprocess_bin_count_super on this
// aux workspace -> tile_ranges (lengths exact; starts are the lists' offsets
// had they been materialised).  Call once per count (the difference grid is
// prefix-summed in place when it exceeds shared memory).
extern "C" int bs_super_tile_lengths(void* aux, size_t aux_bytes, int32_t width, int32_t height, int32_t pw,
                                     int32_t ph, uint32_t* tile_ranges, void* stream) {
  if (!aux || !tile_ranges || width <= 0 || height <= 0 || pw <= 0 || ph <= 0) return BS_ERR_INVALID_ARGUMENT;
  if (aux_bytes < bs_super_aux_bytes(width, height, pw, ph)) return BS_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  const Grid gt = make_grid(width, height, pw, ph);
  const int64_t T = (int64_t)gt.cols * gt.rows;
  WsCarver ca(aux, aux_bytes);
  int* diff2 = ca.take<int>((size_t)(gt.cols + 1) * (gt.rows + 1));
  uint32_t* counts2 = ca.take<uint32_t>((size_t)T);
  uint32_t* starts2 = ca.take<uint32_t>((size_t)T);
  uint32_t* partials2 = ca.take<uint32_t>((size_t)scan_num_blocks(T) + 1);
  const size_t diff2_bytes = sizeof(int) * (size_t)(gt.cols + 1) * (gt.rows + 1);
  if (!g_diff_attr_set) {
    BS_CUDA_TRY(cudaFuncSetAttribute(k_bin_rect<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxDiffSmem));
    BS_CUDA_TRY(cudaFuncSetAttribute(k_diff_scan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxDiffSmem));
    g_diff_attr_set = true;
  }
  if (diff2_bytes <= kMaxDiffSmem) {
    bs::launch_pdl(k_diff_scan, 1, 1024, diff2_bytes, st, diff2, gt, counts2);
    BS_LAUNCH_CHECK();
  } else {
    bs::launch_pdl(k_diff_rows, (unsigned)(gt.rows + 1), 256, 0, st, diff2, gt.cols + 1);
    BS_LAUNCH_CHECK();
    bs::launch_pdl(k_diff_cols, (unsigned)((gt.cols + 255) / 256), 256, 0, st, diff2, gt, counts2);
    BS_LAUNCH_CHECK();
  }
  BS_CUDA_TRY((exclusive_scan<uint32_t, uint32_t>(counts2, starts2, T, nullptr, partials2, nullptr, st)));
  bs::launch_pdl(k_ranges, (unsigned)((T + 255) / 256), 256, 0, st, starts2, counts2, (int)T, tile_ranges, nullptr, 0);
  BS_LAUNCH_CHECK();
  return BS_OK;
}

// k >= 0: K known on the host (bs_bin_sort).  k < 0: K only on the device
// (bs_bin_sort_async; chunked path only) and point_list holds k_cap entries.
static int bin_sort_impl(int64_t n_cap, const int32_t* n_visible, int32_t width, int32_t height, int32_t pw,
                         int32_t ph, int64_t k, int64_t k_cap, uint32_t* point_list, uint32_t* tile_ranges, void* ws,
                         size_t ws_bytes, cudaStream_t st) {
  const Grid gr = make_grid(width, height, pw, ph);
  const int64_t T = (int64_t)gr.cols * gr.rows;
  if (!ws || ws_bytes < bs_bin_workspace_bytes(n_cap, width, height, pw, ph, k < 0 ? 0 : k)) return BS_ERR_WORKSPACE;
  WsCarver c(ws, ws_bytes);
  BinWs w;
  bin_ws_layout(c, n_cap, gr, k < 0 ? 0 : k, &w);
  const uint64_t* kd = w.offs_partials + scan_num_blocks(n_cap);  // K, written by bs_bin_count's scan
  const bool chunked = bin_chunked(gr);
  if (k < 0 && !chunked) return BS_ERR_UNSUPPORTED;
  if ((k > 0 || k < 0) && chunked && k_cap > 0) {
    const uint32_t* order = w.dv0;  // depth order (4 passes end in dv0)
    static bool attr_set = false;
    if (!attr_set) {
      BS_CUDA_TRY(cudaFuncSetAttribute(k_chunk_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxDiffSmem));
      BS_CUDA_TRY(cudaFuncSetAttribute(k_chunk_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)kMaxScatterSmem));
      attr_set = true;
    }
    // offsets row per CTA: the whole grid, or row bands of <= kScTableBytes
    const int nbands = (int)min((int64_t)gr.rows, ((int64_t)T * 4 + kScTableBytes - 1) / kScTableBytes);
    const int band_rows = (gr.rows + nbands - 1) / nbands;
    const size_t off_bytes = sizeof(uint32_t) * (size_t)((band_rows * gr.cols + 31) & ~31);
    const size_t diff_bytes = sizeof(int) * (size_t)(gr.cols + 1) * (gr.rows + 1);
    int dev = 0, sms = 148, per_sm = 1;
    BS_CUDA_TRY(cudaGetDevice(&dev));
    BS_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    BS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_chunk_scatter, kScThreads, off_bytes));
    // one wave of chunks (more only for very large K), >= 4096 instances
    // each; sized from the capacity when K lives on the device (the chunk
    // length q = ceil(K / nch) is computed on the device)
    const int64_t kk = k < 0 ? k_cap : k;
    const int64_t slots = (int64_t)sms * max(1, per_sm);
    static const int64_t min_waves = [] {
      const char* e = getenv("BS_BIN_CHUNK_WAVES");  // tuning override
      return (int64_t)(e ? max(1, atoi(e)) : 1);
    }();
    // target instances per chunk: 2^18 (C2); large grids (4K: 32,400 tiles)
    // balance better with 2^17 (measured); BS_BIN_CHUNK_LOG2 overrides
    static const int env_log2 = [] {
      const char* e = getenv("BS_BIN_CHUNK_LOG2");
      return e ? atoi(e) : 0;
    }();
    const int64_t per_chunk = (int64_t)1 << (env_log2 ? env_log2 : (T > 16384 ? 17 : 18));
    const int64_t waves = max(min_waves, (kk + slots * per_chunk - 1) / (slots * per_chunk));
    const int64_t nch = max((int64_t)1, min(max_chunks(gr), min(max((int64_t)1, slots * waves / nbands),
                                                                 (kk + 4095) / 4096)));
    bs::launch_pdl(k_chunk_bounds, (unsigned)((n_cap + 255) / 256), 256, 0, st, w.offs, w.touched_sorted, n_cap, n_visible, kd,
                                                                   k_cap, (int)nch, w.chunk_first);
    BS_LAUNCH_CHECK();
    bs::launch_pdl(k_chunk_hist, (unsigned)nch, kScThreads, diff_bytes + sizeof(int) * (size_t)(gr.rows + 1), st, 
        w.rects_sorted, w.chunk_first, gr, w.chunk_m, w.chunk_rowc, kd, k_cap);
    BS_LAUNCH_CHECK();
    bs::launch_pdl(k_chunk_scan, (unsigned)((T + 31) / 32), kCsSeg * 32, 0, st, w.chunk_m, w.starts, (int)T, (int)nch, kd, k_cap);
    BS_LAUNCH_CHECK();
    bs::launch_pdl(k_chunk_scatter, dim3((unsigned)nch, (unsigned)nbands), kScThreads, off_bytes, st, 
        w.chunk_m, w.chunk_rowc, w.chunk_first, w.rects_sorted, order, (int)T, gr.cols, gr.rows, point_list, kd, k_cap,
        band_rows);
    BS_LAUNCH_CHECK();
  } else if (k > 0) {
    const uint32_t* order = w.dv0;  // depth order (4 passes end in dv0)
    const int bits = bits_for(T);
    bs::launch_pdl(k_mark_starts, (unsigned)((n_cap + 255) / 256), 256, 0, st, w.offs, w.touched_sorted, n_cap, n_visible,
                                                                 w.block_j0);
    BS_LAUNCH_CHECK();
    bs::launch_pdl(k_expand, (unsigned)((k + kExpandItems - 1) / kExpandItems), 256, 0, st, 
        w.offs, order, w.rects_sorted, n_cap, n_visible, k, gr.cols, w.block_j0, w.tk0, point_list);
    BS_LAUNCH_CHECK();
    bool alt = false;
    BS_CUDA_TRY(radix_sort_pairs(w.tk0, point_list, w.tk1, w.tv_alt, k, nullptr, bits, w.rws_k, &alt, st));
    if (alt) BS_CUDA_TRY(cudaMemcpyAsync(point_list, w.tv_alt, sizeof(uint32_t) * (size_t)k, cudaMemcpyDeviceToDevice, st));
  }
  bs::launch_pdl(k_ranges, (unsigned)((T + 255) / 256), 256, 0, st, w.starts, w.counts, (int)T, tile_ranges,
                                                        n_cap > 0 ? kd : nullptr, k < 0 ? k_cap : k);
  BS_LAUNCH_CHECK();
  return BS_OK;
}

extern "C" int bs_bin_sort(bs_splats g, int64_t n_cap, const int32_t* n_visible, int32_t width, int32_t height,
                           int32_t pw, int32_t ph, int64_t k, uint32_t* point_list, uint32_t* tile_ranges, void* ws,
                           size_t ws_bytes, void* stream) {
  (void)g;
  int s = check_grid(width, height, pw, ph);
  if (s) return s;
  if (n_cap < 0 || k < 0 || !n_visible || !tile_ranges || (k > 0 && !point_list)) return BS_ERR_INVALID_ARGUMENT;
  if (k >= (int64_t)1 << 30) return BS_ERR_CAPACITY;
  return bin_sort_impl(n_cap, n_visible, width, height, pw, ph, k, k, point_list, tile_ranges, ws, ws_bytes,
                       (cudaStream_t)stream);
}

extern "C" int bs_bin_sort_async(bs_splats g, int64_t n_cap, const int32_t* n_visible, int32_t width, int32_t height,
                                 int32_t pw, int32_t ph, int64_t k_cap, uint32_t* point_list, uint32_t* tile_ranges,
                                 void* ws, size_t ws_bytes, void* stream) {
  (void)g;
  int s = check_grid(width, height, pw, ph);
  if (s) return s;
  if (n_cap < 0 || k_cap < 0 || !n_visible || !tile_ranges || (k_cap > 0 && !point_list))
    return BS_ERR_INVALID_ARGUMENT;
  if (k_cap >= (int64_t)1 << 30) return BS_ERR_CAPACITY;
  return bin_sort_impl(n_cap, n_visible, width, height, pw, ph, -1, k_cap, point_list, tile_ranges, ws, ws_bytes,
                       (cudaStream_t)stream);
}

extern "C" int bs_bin_async_supported(int32_t width, int32_t height, int32_t pw, int32_t ph) {
  if (check_grid(width, height, pw, ph)) return 0;
  return bin_chunked(make_grid(width, height, pw, ph)) ? 1 : 0;
}
