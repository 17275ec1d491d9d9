// binning.cu — P5: tile binning, bit-exact with src/preprocess.cpp:66-115.
//
// The reference sorts (tile, depth, index) triples with std::sort.  Here the
// same order comes from two stable LSD radix sorts:
//   1. the n visible splats by depth key (float bits, 4 x 8-bit passes) with
//      values in index order  -> (depth, index) order;
//   2. the K = sum(tiles touched) (tile, splat) instances, duplicated in that
//      depth order, by tile id (ceil(log2 T) bits)  -> (tile, depth, index).
// Sorting N depth keys once instead of K 45-bit keys cuts sort traffic ~3x.
// Tile ranges come from key boundaries + an exclusive scan of per-tile counts,
// so empty tiles get [pos, pos) exactly like the reference's range loop.
#include <math.h>

#include "bs_common.cuh"
#include "radix_sort.cuh"
#include "scan.cuh"

namespace bs {

struct Grid {
  int W, H, pw, ph, cols, rows;
};

// static_cast<int>(float) with x86-64 cvttss2si semantics (out of range /
// NaN -> INT_MIN), the behaviour of the reference's casts on its platform.
__device__ __forceinline__ int x86_f2i(float f) {
  if (!(f > -2147483904.0f && f < 2147483648.0f)) return (int)0x80000000;
  return (int)f;
}

struct Rect {
  int tx0, tx1, ty0, ty1;
};

// src/preprocess.cpp:81-92.  Returns false when rejected / empty.
__device__ __forceinline__ bool tile_rect(float x, float y, float radius, const Grid& g, Rect& r) {
  const float rr = ceilf(radius);
  const float x0 = __fsub_rn(x, rr), x1 = __fadd_rn(x, rr);
  const float y0 = __fsub_rn(y, rr), y1 = __fadd_rn(y, rr);
  if (x1 < 0.0f || y1 < 0.0f || x0 >= (float)g.W || y0 >= (float)g.H) return false;
  r.tx0 = max(0, x86_f2i(floorf(__fdiv_rn(x0, (float)g.pw))));
  r.tx1 = min(g.cols - 1, x86_f2i(floorf(__fdiv_rn(x1, (float)g.pw))));
  r.ty0 = max(0, x86_f2i(floorf(__fdiv_rn(y0, (float)g.ph))));
  r.ty1 = min(g.rows - 1, x86_f2i(floorf(__fdiv_rn(y1, (float)g.ph))));
  return r.tx0 <= r.tx1 && r.ty0 <= r.ty1;
}

__global__ void k_bin_rect(const float4* __restrict__ xyab, const float4* __restrict__ cop,
                           const float4* __restrict__ rgbr, int64_t n_cap, const int32_t* __restrict__ n_visible,
                           Grid g, uint32_t* __restrict__ touched, uint32_t* __restrict__ dkeys,
                           uint32_t* __restrict__ dvals) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_cap) return;
  const int64_t n = *n_visible;
  if (i >= n) return;
  const float4 a = xyab[i];
  const float radius = rgbr[i].w;
  Rect r;
  uint32_t cnt = 0;
  if (tile_rect(a.x, a.y, radius, g, r)) cnt = (uint32_t)(r.tx1 - r.tx0 + 1) * (uint32_t)(r.ty1 - r.ty0 + 1);
  touched[i] = cnt;
  dkeys[i] = float_sort_key(cop[i].w);
  dvals[i] = (uint32_t)i;
}

__global__ void k_gather_touched(const uint32_t* __restrict__ order, const uint32_t* __restrict__ touched,
                                 int64_t n_cap, const int32_t* __restrict__ n_visible, uint32_t* __restrict__ out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n_cap || j >= *n_visible) return;
  out[j] = touched[order[j]];
}

// One thread per splat in depth order writes its rect's tile ids row-major
// (ty outer, tx inner — the reference's push_back order, irrelevant after the
// stable sort but kept) at offs[j].
__global__ void k_duplicate(const float4* __restrict__ xyab, const float4* __restrict__ rgbr,
                            const uint32_t* __restrict__ order, const uint64_t* __restrict__ offs, int64_t n_cap,
                            const int32_t* __restrict__ n_visible, Grid g, uint32_t* __restrict__ keys,
                            uint32_t* __restrict__ vals) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n_cap || j >= *n_visible) return;
  const uint32_t i = order[j];
  const float4 a = xyab[i];
  Rect r;
  if (!tile_rect(a.x, a.y, rgbr[i].w, g, r)) return;
  uint64_t o = offs[j];
  for (int ty = r.ty0; ty <= r.ty1; ++ty)
    for (int tx = r.tx0; tx <= r.tx1; ++tx) {
      keys[o] = (uint32_t)(ty * g.cols + tx);
      vals[o] = i;
      ++o;
    }
}

__global__ void k_tile_bounds(const uint32_t* __restrict__ keys, int64_t K, uint32_t* __restrict__ counts) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  const uint32_t t = keys[k];
  // count[t] = last+1 - first, assembled from the two boundary writers
  if (k == 0 || keys[k - 1] != t) atomicSub(&counts[t], (uint32_t)k);
  if (k == K - 1 || keys[k + 1] != t) atomicAdd(&counts[t], (uint32_t)(k + 1));
}

__global__ void k_ranges(const uint32_t* __restrict__ starts, const uint32_t* __restrict__ counts, int T,
                         uint32_t* __restrict__ ranges) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
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

// Workspace layout shared by bs_bin_count and bs_bin_sort (same carve order).
struct BinWs {
  // count phase (n-sized)
  uint32_t *touched, *dk0, *dv0, *dk1, *dv1, *touched_sorted;
  uint64_t* offs;
  uint64_t* offs_partials;
  RadixWs rws_n;
  // sort phase (k-sized)
  uint32_t *tk0, *tv0, *tk1;
  RadixWs rws_k;
  uint32_t *counts, *starts, *cpartials;
};

template <typename C>
inline void bin_ws_layout(C& c, int64_t n_cap, int64_t T, int64_t k_cap, BinWs* w) {
  BinWs tmp;
  BinWs& o = w ? *w : tmp;
  o.touched = (uint32_t*)c.template take<uint32_t>((size_t)n_cap);
  o.dk0 = (uint32_t*)c.template take<uint32_t>((size_t)n_cap);
  o.dv0 = (uint32_t*)c.template take<uint32_t>((size_t)n_cap);
  o.dk1 = (uint32_t*)c.template take<uint32_t>((size_t)n_cap);
  o.dv1 = (uint32_t*)c.template take<uint32_t>((size_t)n_cap);
  o.touched_sorted = (uint32_t*)c.template take<uint32_t>((size_t)n_cap);
  o.offs = (uint64_t*)c.template take<uint64_t>((size_t)n_cap);
  o.offs_partials = (uint64_t*)c.template take<uint64_t>((size_t)scan_num_blocks(n_cap) + 1);
  {
    const int64_t nb = radix_num_blocks(n_cap);
    o.rws_n.hist = (uint32_t*)c.template take<uint32_t>((size_t)(256 * nb));
    o.rws_n.partials = (uint32_t*)c.template take<uint32_t>((size_t)scan_num_blocks(256 * nb));
  }
  o.counts = (uint32_t*)c.template take<uint32_t>((size_t)T);
  o.starts = (uint32_t*)c.template take<uint32_t>((size_t)T);
  o.cpartials = (uint32_t*)c.template take<uint32_t>((size_t)scan_num_blocks(T) + 1);
  o.tk0 = (uint32_t*)c.template take<uint32_t>((size_t)k_cap);
  o.tv0 = (uint32_t*)c.template take<uint32_t>((size_t)k_cap);
  o.tk1 = (uint32_t*)c.template take<uint32_t>((size_t)k_cap);
  {
    const int64_t nb = radix_num_blocks(k_cap);
    o.rws_k.hist = (uint32_t*)c.template take<uint32_t>((size_t)(256 * nb));
    o.rws_k.partials = (uint32_t*)c.template take<uint32_t>((size_t)scan_num_blocks(256 * nb));
  }
}


__global__ void k_store_k(const uint64_t* __restrict__ total, int64_t* __restrict__ k_total) {
  *k_total = (int64_t)*total;
}

}  // namespace bs

using namespace bs;

extern "C" size_t bs_bin_workspace_bytes(int64_t n_cap, int32_t width, int32_t height, int32_t pw, int32_t ph,
                                         int64_t k_cap) {
  if (n_cap < 0 || width <= 0 || height <= 0 || pw <= 0 || ph <= 0 || k_cap < 0) return 0;
  const Grid g = make_grid(width, height, pw, ph);
  WsSizer s;
  bin_ws_layout(s, n_cap, (int64_t)g.cols * g.rows, k_cap, nullptr);
  return s.off + 256;
}

static int check_grid(int32_t W, int32_t H, int32_t pw, int32_t ph) {
  if (W <= 0 || H <= 0 || pw <= 0 || ph <= 0) return BS_ERR_INVALID_ARGUMENT;
  const int64_t T = (int64_t)((W + pw - 1) / pw) * ((H + ph - 1) / ph);
  if (T > (1 << 24)) return BS_ERR_UNSUPPORTED;
  return BS_OK;
}

extern "C" int bs_bin_count(bs_splats g, int64_t n_cap, const int32_t* n_visible, int32_t width, int32_t height,
                            int32_t pw, int32_t ph, int64_t* k_total, void* ws, size_t ws_bytes, void* stream) {
  int s = check_grid(width, height, pw, ph);
  if (s) return s;
  if (n_cap < 0 || !n_visible || !k_total || (n_cap > 0 && (!g.xyab || !g.cop || !g.rgbr))) return BS_ERR_INVALID_ARGUMENT;
  if (n_cap >= (int64_t)0x7fffffff) return BS_ERR_CAPACITY;
  cudaStream_t st = (cudaStream_t)stream;
  const Grid gr = make_grid(width, height, pw, ph);
  const int64_t T = (int64_t)gr.cols * gr.rows;
  if (!ws || ws_bytes < bs_bin_workspace_bytes(n_cap, width, height, pw, ph, 0)) return BS_ERR_WORKSPACE;
  WsCarver c(ws, ws_bytes);
  BinWs w;
  bin_ws_layout(c, n_cap, T, 0, &w);
  if (n_cap == 0) {
    BS_CUDA_TRY(cudaMemsetAsync(k_total, 0, sizeof(int64_t), st));
    return BS_OK;
  }
  const unsigned nb = (unsigned)((n_cap + 255) / 256);
  k_bin_rect<<<nb, 256, 0, st>>>(reinterpret_cast<const float4*>(g.xyab), reinterpret_cast<const float4*>(g.cop),
                                 reinterpret_cast<const float4*>(g.rgbr), n_cap, n_visible, gr, w.touched, w.dk0, w.dv0);
  BS_LAUNCH_CHECK();
  bool alt = false;
  BS_CUDA_TRY(radix_sort_pairs(w.dk0, w.dv0, w.dk1, w.dv1, n_cap, n_visible, 32, w.rws_n, &alt, st));
  const uint32_t* order = alt ? w.dv1 : w.dv0;
  k_gather_touched<<<nb, 256, 0, st>>>(order, w.touched, n_cap, n_visible, w.touched_sorted);
  BS_LAUNCH_CHECK();
  uint64_t* total = w.offs_partials + scan_num_blocks(n_cap);
  BS_CUDA_TRY((exclusive_scan<uint32_t, uint64_t>(w.touched_sorted, w.offs, n_cap, n_visible, w.offs_partials, total, st)));
  k_store_k<<<1, 1, 0, st>>>(total, k_total);
  BS_LAUNCH_CHECK();
  return BS_OK;
}

extern "C" int bs_bin_sort(bs_splats g, int64_t n_cap, const int32_t* n_visible, int32_t width, int32_t height,
                           int32_t pw, int32_t ph, int64_t k, uint32_t* point_list, uint32_t* tile_ranges, void* ws,
                           size_t ws_bytes, void* stream) {
  int s = check_grid(width, height, pw, ph);
  if (s) return s;
  if (n_cap < 0 || k < 0 || !n_visible || !tile_ranges || (k > 0 && !point_list)) return BS_ERR_INVALID_ARGUMENT;
  if (k > (int64_t)0xfffffffe) return BS_ERR_CAPACITY;
  cudaStream_t st = (cudaStream_t)stream;
  const Grid gr = make_grid(width, height, pw, ph);
  const int64_t T = (int64_t)gr.cols * gr.rows;
  if (!ws || ws_bytes < bs_bin_workspace_bytes(n_cap, width, height, pw, ph, k)) return BS_ERR_WORKSPACE;
  WsCarver c(ws, ws_bytes);
  BinWs w;
  // k_cap = the largest k this workspace can hold (same layout prefix)
  bin_ws_layout(c, n_cap, T, k, &w);
  BS_CUDA_TRY(cudaMemsetAsync(w.counts, 0, sizeof(uint32_t) * (size_t)T, st));
  if (k > 0) {
    // 4 passes of 8 bits leave the depth order back in dv0.
    const uint32_t* order = w.dv0;
    const unsigned nb = (unsigned)((n_cap + 255) / 256);
    // values go straight into point_list; (tk1, tv0) is the ping-pong pair
    k_duplicate<<<nb, 256, 0, st>>>(reinterpret_cast<const float4*>(g.xyab), reinterpret_cast<const float4*>(g.rgbr),
                                    order, w.offs, n_cap, n_visible, gr, w.tk0, point_list);
    BS_LAUNCH_CHECK();
    bool alt = false;
    uint32_t* tv_alt = w.tv0;
    BS_CUDA_TRY(radix_sort_pairs(w.tk0, point_list, w.tk1, tv_alt, k, nullptr, bits_for(T), w.rws_k, &alt, st));
    const uint32_t* sorted_keys = alt ? w.tk1 : w.tk0;
    if (alt) BS_CUDA_TRY(cudaMemcpyAsync(point_list, tv_alt, sizeof(uint32_t) * (size_t)k, cudaMemcpyDeviceToDevice, st));
    k_tile_bounds<<<(unsigned)((k + 255) / 256), 256, 0, st>>>(sorted_keys, k, w.counts);
    BS_LAUNCH_CHECK();
  }
  BS_CUDA_TRY((exclusive_scan<uint32_t, uint32_t>(w.counts, w.starts, T, nullptr, w.cpartials, nullptr, st)));
  k_ranges<<<(unsigned)((T + 255) / 256), 256, 0, st>>>(w.starts, w.counts, (int)T, tile_ranges);
  BS_LAUNCH_CHECK();
  return BS_OK;
}
