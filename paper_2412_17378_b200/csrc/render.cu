// render.cu — R1-R8: the forward alpha-blend, five variants.
//
//   Naive              pixel-wise, static grid (one CTA per tile, thread = pixel),
//                      xy/conic/opacity staged in smem per 1-CTA-wide chunk,
//                      colour fetched from L2 on commit        (paper Alg. 4/5)
//   SharedMemOpt       Naive + colour/depth staged too           (paper §5.2.2)
//   DynamicBlocks      pixel-wise, persistent CTAs claim tiles from an
//                      atomicAdd queue in tile order               (paper Alg. 1)
//   GaussianWise       static grid, CTA = tile, 4 warps; each warp blends one
//                      pixel with its 32 lanes on 32 consecutive list entries,
//                      prefix product of (1-alpha) by shfl_up doubling, lane-31
//                      carry                                  (paper Alg. 2/6)
//   FineGrainedCombined persistent CTAs whose warps each claim 8x4-pixel
//                      sub-tile tasks from an atomicAdd queue ordered by tile
//                      list length, longest first (LPT); sub-tile culling,
//                      pixel-wise batches, Gaussian-wise stragglers
//                                          (paper Alg. 3, re-cut for B200)
//
// Super-tile lists (bs_render_forward_super, the frame pipeline's >= 1 Mpixel
// frames): FineGrainedCombined and SharedMemOpt (the auto-mode candidates)
// also render from lists binned at 2pw x 2ph, keeping per tile exactly the
// entries of its pw x ph list (tile_member / tile_member_fast) and counting
// term positions over them.
//
// Semantics: pixel-wise variants == render_reference
// (src/blend.cpp:55-107); Gaussian-wise variants == render_gaussianwise
// (src/kernels.cpp:57-155).  In BS_ALPHA_EXACT mode every float op that the
// reference performs is reproduced with explicit _rn intrinsics (no FMA
// contraction), expf is glibc-exact, transmittance decisions follow the serial
// float recurrence and colour/depth accumulate in double — so pixel-wise
// output is bit-identical to the oracle and Gaussian-wise contrib/term/T/alpha
// are bit-identical (colour/depth differ only by double-sum association).
// BS_ALPHA_FAST trades that for ex2.approx + float accumulators.
//
// No tensor-core path: blending is a dependent scan, not a contraction.  All
// five kernels are instruction-issue-bound (profiles/r1_ncu_variants.txt).
#include <math.h>
#include <stdlib.h>

#include <type_traits>

#include "bs_common.cuh"
#include "exact_expf.cuh"
#include "tiles.cuh"

namespace bs {

__constant__ unsigned long long c_exp2f_tab[32] = BS_EXP2F_TAB_INIT;

constexpr unsigned kFull = 0xffffffffu;
constexpr int kFgWarps = 4;             // paper Alg. 3: 4 warps <-> 4 pixels per task
constexpr int kFgThreads = kFgWarps * 32;

struct RArgs {
  const float4* __restrict__ xyab;
  const float4* __restrict__ cop;
  const float4* __restrict__ rgbr;
  const uint32_t* __restrict__ point_list;
  const uint32_t* __restrict__ ranges;
  const uint32_t* __restrict__ task_order;
  int W, H, pw, ph, cols, T;
  float bg0, bg1, bg2;
  float* __restrict__ color;
  float* __restrict__ alpha;
  float* __restrict__ depth;
  float* __restrict__ final_t;
  int32_t* __restrict__ contrib;
  int32_t* __restrict__ term;
  unsigned int* queue;      // [0] warp-task ticket, [1] pixels parked, [2] parked-task ticket, [3] tasks parked
  struct Donation* donate;  // FineGrainedCombined tail hand-off (see k_render_donated)
  uint2* donated_tasks;     // (first Donation, count) per parked warp task
  int total_tasks;
  int donate_after;       // list entries a task walks before it may hand off
  int donate_min_remain;  // ... and only if this many entries remain
  const int32_t* gate;    // device-selected variant (bs_render_forward_auto) or null
  // super-tile lists (bs_render_forward_super): ranges[t] is the list of the
  // 2pw x 2ph super-tile holding tile t, and an entry belongs to tile t's
  // list iff its S8 rectangle at pw x ph contains t (tile_member)
  int sup, rows;
  float ipw, iph;  // 1/pw, 1/ph (exact: power-of-two patches only)
  int stragglers;  // live pixels at or below which a warp task finishes Gaussian-wise
};

// Is tile (tx, ty) inside the splat's S8 rectangle at the pw x ph grid
// (src/preprocess.cpp:83-92, tiles.cuh tile_rect's ops; x / pw == x * (1/pw)
// exactly for a power-of-two pw)?  The rejection tests need not be repeated:
// they do not depend on the patch size, and a splat in a super-tile list
// passed them.  (Loading a rectangle precomputed by the projection pass
// instead measured slower: the extra registers spill.)
__device__ __forceinline__ bool tile_member(const RArgs& A, float x, float y, float radius, int tx, int ty) {
  const float rr = ceilf(radius);
  const float x0 = __fsub_rn(x, rr), x1 = __fadd_rn(x, rr);
  const float y0 = __fsub_rn(y, rr), y1 = __fadd_rn(y, rr);
  const int tx0 = max(0, x86_f2i(floorf(__fmul_rn(x0, A.ipw))));
  const int tx1 = min(A.cols - 1, x86_f2i(floorf(__fmul_rn(x1, A.ipw))));
  const int ty0 = max(0, x86_f2i(floorf(__fmul_rn(y0, A.iph))));
  const int ty1 = min(A.rows - 1, x86_f2i(floorf(__fmul_rn(y1, A.iph))));
  return tx0 <= tx && tx <= tx1 && ty0 <= ty && ty <= ty1;
}

// The same test on the fast path.  An entry of tile t's super-tile list
// already satisfies tile_member on one side of each axis: for an even tile
// column (t is its super-tile's left column) the splat's right edge reaches
// t, so t is a member unless the left edge tx0 == tx + 1; for an odd column
// unless the right edge tx1 == tx - 1 (the clamps cannot produce those
// values).  floor(v) == k is k <= v < k + 1, so one product and two compares
// per axis decide it.  Exact whenever every edge / pw stays in int range —
// guaranteed for ceil(radius) < 1e9 (else the full test).
struct TileSide {
  float xl, yl;  // tx + 1 or tx - 1, ty + 1 or ty - 1
  bool qx, qy;   // odd column / row inside the super-tile
};
__device__ __forceinline__ TileSide tile_side(int tx, int ty) {
  TileSide m;
  m.qx = tx & 1;
  m.qy = ty & 1;
  m.xl = (float)(m.qx ? tx - 1 : tx + 1);
  m.yl = (float)(m.qy ? ty - 1 : ty + 1);
  return m;
}
__device__ __forceinline__ bool tile_member_fast(const RArgs& A, const TileSide& m, float x, float y, float radius,
                                                 int tx, int ty) {
  const float rr = ceilf(radius);
  if (!(rr < 1e9f)) return tile_member(A, x, y, radius, tx, ty);
  const float xv = __fmul_rn(m.qx ? __fadd_rn(x, rr) : __fsub_rn(x, rr), A.ipw);
  const float yv = __fmul_rn(m.qy ? __fadd_rn(y, rr) : __fsub_rn(y, rr), A.iph);
  return !(xv >= m.xl && xv < m.xl + 1.0f) && !(yv >= m.yl && yv < m.yl + 1.0f);
}

// FineGrainedCombined list mode: pw x ph lists, or super-tile lists
// filtered by tile_member (a template parameter: the pw x ph kernel keeps
// its register budget)
enum { kListTile = 0, kListSuper = 1 };

// Sync-free auto mode: every candidate kernel is launched and all but the
// device-selected one return at once.
__device__ __forceinline__ bool gated_out(const RArgs& A, int variant) { return A.gate && *A.gate != variant; }

// R1 eval_alpha + the power>0 arm + skip rule (src/blend.cpp:8-21, 90).
// Returns true when the step is NOT skipped; alpha is the reference's alpha.
// SPECIAL = false: the caller guarantees power_cut >= kExpSpecialCut for
// this entry, so glibc's special-cased input cannot reach the exp.
template <int MODE, bool SPECIAL = true>
__device__ __forceinline__ bool eval_step(const float4 a, const float4 c, float sx, float sy,
                                          const ExpK& ek, float& alpha) {
  const float dx = __fsub_rn(sx, a.x);
  const float dy = __fsub_rn(sy, a.y);
  const float q = __fadd_rn(__fmul_rn(__fmul_rn(a.z, dx), dx), __fmul_rn(__fmul_rn(c.x, dy), dy));
  const float power = __fsub_rn(__fmul_rn(-0.5f, q), __fmul_rn(__fmul_rn(a.w, dx), dy));
  if (power < c.z) return false;    // certain skip (see power_cut_of)
  if (power > 0.0f) return false;   // alpha forced to 0 -> skipped
  float e;
  if (MODE == BS_ALPHA_EXACT) {
    e = glibc_expf_fast<SPECIAL>(power, ek);  // power in [power_cut, 0], power_cut >= -103.97
  } else {
    float p2 = power * 1.4426950408889634f;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(p2));
  }
  const float a0 = __fmul_rn(c.y, e);
  alpha = (a0 < kAlphaClamp) ? a0 : kAlphaClamp;  // std::min(0.99f, a0)
  return !(alpha < kAlphaSkip);
}

template <int MODE>
struct Accum;

template <>
struct Accum<BS_ALPHA_EXACT> {
  double r = 0, g = 0, b = 0, d = 0;
  __device__ __forceinline__ void add(float alpha, float t, float4 col, float dep) {
    const double w = __dmul_rn((double)alpha, (double)t);
    r = __dadd_rn(r, __dmul_rn((double)col.x, w));
    g = __dadd_rn(g, __dmul_rn((double)col.y, w));
    b = __dadd_rn(b, __dmul_rn((double)col.z, w));
    d = __dadd_rn(d, __dmul_rn((double)dep, w));
  }
  // colour/depth already widened to double (rg = (r, g), bd = (b, depth));
  // FineGrainedCombined's batch loop: the exact weight w = alpha * t (a
  // 24 x 24-bit product, exact in double) and one fused multiply-add per
  // channel — the reference rounds the product and the sum separately
  // (src/blend.cpp:28-32), so the double sums may differ in their last bit
  // (the Gaussian-wise variants' colour bar: 1e-6; the float outputs are
  // almost always identical)
  __device__ __forceinline__ void add_wide(float alpha, float t, double2 rg, double2 bd) {
    const double w = __dmul_rn((double)alpha, (double)t);
    r = __fma_rn(rg.x, w, r);
    g = __fma_rn(rg.y, w, g);
    b = __fma_rn(bd.x, w, b);
    d = __fma_rn(bd.y, w, d);
  }
  __device__ __forceinline__ void store(double* o) const { o[0] = r; o[1] = g; o[2] = b; o[3] = d; }
  __device__ __forceinline__ void load(const double* o) { r = o[0]; g = o[1]; b = o[2]; d = o[3]; }
  __device__ __forceinline__ void merge(const Accum& o) {
    r = __dadd_rn(r, o.r);
    g = __dadd_rn(g, o.g);
    b = __dadd_rn(b, o.b);
    d = __dadd_rn(d, o.d);
  }
  __device__ __forceinline__ void warp_sum() {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      r += __shfl_xor_sync(kFull, r, o);
      g += __shfl_xor_sync(kFull, g, o);
      b += __shfl_xor_sync(kFull, b, o);
      d += __shfl_xor_sync(kFull, d, o);
    }
  }
  __device__ __forceinline__ void finish(const RArgs& A, size_t p, float t, int contrib, int term) const {
    A.color[3 * p + 0] = __double2float_rn(__dadd_rn(r, __dmul_rn((double)A.bg0, (double)t)));
    A.color[3 * p + 1] = __double2float_rn(__dadd_rn(g, __dmul_rn((double)A.bg1, (double)t)));
    A.color[3 * p + 2] = __double2float_rn(__dadd_rn(b, __dmul_rn((double)A.bg2, (double)t)));
    A.alpha[p] = __fsub_rn(1.0f, t);
    A.depth[p] = __double2float_rn(d);
    A.final_t[p] = t;
    A.contrib[p] = contrib;
    A.term[p] = term;
  }
};

template <>
struct Accum<BS_ALPHA_FAST> {
  float r = 0, g = 0, b = 0, d = 0;
  __device__ __forceinline__ void add(float alpha, float t, float4 col, float dep) {
    const float w = alpha * t;
    r = fmaf(col.x, w, r);
    g = fmaf(col.y, w, g);
    b = fmaf(col.z, w, b);
    d = fmaf(dep, w, d);
  }
  __device__ __forceinline__ void add_wide(float, float, double2, double2) {}
  __device__ __forceinline__ void store(double* o) const { o[0] = r; o[1] = g; o[2] = b; o[3] = d; }
  __device__ __forceinline__ void load(const double* o) {
    r = (float)o[0]; g = (float)o[1]; b = (float)o[2]; d = (float)o[3];
  }
  __device__ __forceinline__ void merge(const Accum& o) {
    r += o.r;
    g += o.g;
    b += o.b;
    d += o.d;
  }
  __device__ __forceinline__ void warp_sum() {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      r += __shfl_xor_sync(kFull, r, o);
      g += __shfl_xor_sync(kFull, g, o);
      b += __shfl_xor_sync(kFull, b, o);
      d += __shfl_xor_sync(kFull, d, o);
    }
  }
  __device__ __forceinline__ void finish(const RArgs& A, size_t p, float t, int contrib, int term) const {
    A.color[3 * p + 0] = fmaf(A.bg0, t, r);
    A.color[3 * p + 1] = fmaf(A.bg1, t, g);
    A.color[3 * p + 2] = fmaf(A.bg2, t, b);
    A.alpha[p] = 1.0f - t;
    A.depth[p] = d;
    A.final_t[p] = t;
    A.contrib[p] = contrib;
    A.term[p] = term;
  }
};

__device__ __forceinline__ void load_tab(unsigned long long* s_tab) {
  if (threadIdx.x < 32) s_tab[threadIdx.x] = c_exp2f_tab[threadIdx.x];
}

// ---------------------------------------------------------------------------
// Pixel-wise tile (Naive / SharedMemOpt / DynamicBlocks).  BLOCK threads, one
// per pixel slot of the pw x ph patch (BLOCK >= pw*ph).  The CTA stages the
// tile list in BLOCK-wide chunks; a chunk is skipped once every pixel stopped
// (__syncthreads_count, as Inria's renderCUDA does).
template <int MODE, bool STAGE_COLOR, int BLOCK>
struct PwChunk {
  // 1024-thread CTAs staging colour too would exceed 48 KB of static smem
  static constexpr int value = (STAGE_COLOR && BLOCK > 512) ? 512 : BLOCK;
};

template <int MODE, bool STAGE_COLOR, int BLOCK>
__device__ __forceinline__ void pixelwise_tile(const RArgs& A, int tile, float4* s_xyab, float4* s_cop,
                                               float4* s_rgb, uint32_t* s_id, bool* s_mem, const ExpK& ek) {
  const int tid = threadIdx.x;
  const int tx = tile % A.cols, ty = tile / A.cols;
  const int lx = tid % A.pw, ly = tid / A.pw;
  const int px = tx * A.pw + lx, py = ty * A.ph + ly;
  const bool inside = tid < A.pw * A.ph && px < A.W && py < A.H;
  const float sx = __fadd_rn((float)px, 0.5f), sy = __fadd_rn((float)py, 0.5f);
  const uint32_t start = A.ranges[2 * tile], end = A.ranges[2 * tile + 1];

  bool done = !inside;
  float t = 1.0f;
  int contrib = 0, term = 0;
  Accum<MODE> acc;

  constexpr int CHUNK = PwChunk<MODE, STAGE_COLOR, BLOCK>::value;
  uint32_t mbase = 0;  // entries of this tile's list before the chunk
  for (uint32_t base = start; base < end; base += CHUNK) {
    if (__syncthreads_count(!done) == 0) break;
    const uint32_t k = base + tid;
    bool mem = false;
    if (tid < CHUNK && k < end) {
      const uint32_t id = __ldg(A.point_list + k);
      s_xyab[tid] = __ldg(A.xyab + id);
      s_cop[tid] = __ldg(A.cop + id);
      if (STAGE_COLOR) s_rgb[tid] = __ldg(A.rgbr + id);
      else s_id[tid] = id;
      mem = true;
      if (A.sup) {
        mem = tile_member_fast(A, tile_side(tx, ty), s_xyab[tid].x, s_xyab[tid].y, __ldg(&A.rgbr[id].w), tx, ty);
        s_mem[tid] = mem;
      }
    }
    const uint32_t cmem = (uint32_t)__syncthreads_count(mem);
    if (!done) {
      const int cnt = (int)min((uint32_t)CHUNK, end - base);
      int m = 0;
      for (int j = 0; j < cnt; ++j) {
        if (A.sup && !s_mem[j]) continue;  // not in this tile's list
        ++m;
        float alpha;
        const float4 c = s_cop[j];
        if (!eval_step<MODE>(s_xyab[j], c, sx, sy, ek, alpha)) continue;
        const float tmp = __fmul_rn(t, __fsub_rn(1.0f, alpha));
        if (tmp < kStopThreshold) {
          done = true;
          term = (int)mbase + m;
          break;
        }
        const float4 col = STAGE_COLOR ? s_rgb[j] : __ldg(A.rgbr + s_id[j]);
        acc.add(alpha, t, col, c.w);
        t = tmp;
        ++contrib;
      }
    }
    mbase += cmem;
  }
  if (inside) acc.finish(A, (size_t)py * A.W + px, t, contrib, term);
}

template <int MODE, bool STAGE_COLOR, int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_render_pixelwise(RArgs A) {
  bs::pdl_wait();
  if (gated_out(A, STAGE_COLOR ? BS_SHARED_MEM_OPT : BS_NAIVE)) return;
  constexpr int CHUNK = PwChunk<MODE, STAGE_COLOR, BLOCK>::value;
  __shared__ float4 s_xyab[CHUNK];
  __shared__ float4 s_cop[CHUNK];
  __shared__ float4 s_rgb[STAGE_COLOR ? CHUNK : 1];
  __shared__ uint32_t s_id[STAGE_COLOR ? 1 : CHUNK];
  __shared__ bool s_mem[CHUNK];
  __shared__ unsigned long long s_tab[32];
  load_tab(s_tab);
  __syncthreads();
  // one tile per CTA, or (a gated auto-mode candidate, launched with fewer
  // CTAs so that not being selected costs little) tiles in grid stride —
  // the next tile's first chunk barrier orders the shared-memory reuse
  // SharedMemOpt (the selector's fallback) takes the LPT tile order when
  // given (heavy tiles first); Naive keeps the plain grid — the paper's
  // baseline kernel
  for (int i = blockIdx.x; i < A.T; i += gridDim.x) {
    const int tile = (STAGE_COLOR && A.task_order) ? (int)A.task_order[i] : i;
    pixelwise_tile<MODE, STAGE_COLOR, BLOCK>(A, tile, s_xyab, s_cop, s_rgb, s_id, s_mem, make_expk(s_tab));
  }
}

// Paper Alg. 1 (with the exit test fixed to >=).
template <int MODE, int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_render_dynamic(RArgs A) {
  bs::pdl_wait();
  __shared__ float4 s_xyab[BLOCK];
  __shared__ float4 s_cop[BLOCK];
  __shared__ uint32_t s_id[BLOCK];
  __shared__ unsigned long long s_tab[32];
  __shared__ int s_tile;
  if (gated_out(A, BS_DYNAMIC_BLOCKS)) return;
  load_tab(s_tab);
  const ExpK ek = make_expk(s_tab);
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_tile = (int)atomicAdd(A.queue, 1u);
    __syncthreads();
    const int ticket = s_tile;
    if (ticket >= A.T) return;
    // the queue hands tiles out in LPT order when given (paper Alg. 1 uses
    // index order; longest lists first keeps the heavy tiles off the tail)
    const int tile = A.task_order ? (int)A.task_order[ticket] : ticket;
    pixelwise_tile<MODE, false, BLOCK>(A, tile, s_xyab, s_cop, nullptr, s_id, nullptr, ek);
  }
}

// ---------------------------------------------------------------------------
// One 32-wide Gaussian-wise group of one pixel (paper Alg. 6 / R6): lane l
// holds list entry g0+l.  t (warp-uniform) and contrib are updated; each lane
// accumulates its own committed entry into acc.  Returns the stop lane (32 =
// no stop).  All-skipped groups return at once (Alg. 6's __all_sync skip).
//   EXACT: skip/stop decisions and the carried t follow the serial float
//     recurrence (src/kernels.cpp:79-89).  Colour weights: SERIAL_W ? the
//     serial t before each entry (render_reference weights) : the doubling
//     prefix product (render_gaussianwise weights, inc/blend.hpp:69-83).
//   FAST: decisions and weights from the prefix product (paper Alg. 6), the
//     terminating entry committing nothing (SPEC blend-core decision).
template <int MODE, bool SERIAL_W>
__device__ __forceinline__ int gw_group(bool ns, float alpha, float4 col, float dep, float& t, int& contrib,
                                        Accum<MODE>& acc, int lane) {
  const unsigned nsmask = __ballot_sync(kFull, ns);
  if (nsmask == 0) return 32;
  const float f = ns ? __fsub_rn(1.0f, alpha) : 1.0f;
  int stop = 32;
  float t_next, tb = t;
  bool need_prefix = !(MODE == BS_ALPHA_EXACT && SERIAL_W);
  if (MODE == BS_ALPHA_EXACT) {
    float ts = t;
    unsigned m = nsmask;
    while (m) {
      const int jl = __ffs(m) - 1;
      const float fj = __shfl_sync(kFull, f, jl);
      if (lane == jl) tb = ts;
      const float tmp = __fmul_rn(ts, fj);
      if (tmp < kStopThreshold) {
        stop = jl;
        break;
      }
      ts = tmp;
      m &= m - 1;
    }
    t_next = ts;
  }
  if (need_prefix) {
    float pre = f;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const float v = __shfl_up_sync(kFull, pre, off);
      if (lane >= off) pre = __fmul_rn(pre, v);
    }
    const float per_lane = __fmul_rn(t, pre);
    float t_before = __shfl_up_sync(kFull, per_lane, 1);
    if (lane == 0) t_before = t;
    tb = t_before;
    if (MODE != BS_ALPHA_EXACT) {
      const unsigned sm = __ballot_sync(kFull, ns && per_lane < kStopThreshold);
      if (sm) {
        stop = __ffs(sm) - 1;
        t_next = __shfl_sync(kFull, t_before, stop);
      } else {
        t_next = __shfl_sync(kFull, per_lane, 31);
      }
    }
  }
  if (ns && lane < stop) acc.add(alpha, tb, col, dep);
  contrib += __popc(nsmask & ((stop >= 32) ? kFull : ((1u << stop) - 1u)));
  t = t_next;
  return stop;
}

// ---------------------------------------------------------------------------
// Gaussian-wise task: WARPS warps, warp w blends pixel sub*WARPS + w of
// `tile`; the CTA stages the list in 32*WARPS-entry chunks shared by the
// warps; each warp walks a chunk in 32-wide groups.  SERIAL_W selects the
// colour weights (see gw_group).
template <int MODE, int WARPS, bool SERIAL_W>
__device__ __forceinline__ void gaussianwise_task(const RArgs& A, int tile, int sub, float4* s_xyab, float4* s_cop,
                                                  float4* s_rgb, const ExpK& ek) {
  constexpr int CH = WARPS * 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tx = tile % A.cols, ty = tile / A.cols;
  const int local = sub * WARPS + warp;
  const int lx = local % A.pw, ly = local / A.pw;
  const int px = tx * A.pw + lx, py = ty * A.ph + ly;
  const bool inside = local < A.pw * A.ph && px < A.W && py < A.H;
  const float sx = __fadd_rn((float)px, 0.5f), sy = __fadd_rn((float)py, 0.5f);
  const uint32_t start = A.ranges[2 * tile], end = A.ranges[2 * tile + 1];

  bool done = !inside;  // warp-uniform
  float t = 1.0f;       // warp-uniform (serial carry)
  int contrib = 0, term = 0;
  Accum<MODE> acc;

  for (uint32_t base = start; base < end; base += CH) {
    if (__syncthreads_count(!done) == 0) break;
    const uint32_t k = base + tid;
    if (k < end) {
      const uint32_t id = __ldg(A.point_list + k);
      s_xyab[tid] = __ldg(A.xyab + id);
      s_cop[tid] = __ldg(A.cop + id);
      s_rgb[tid] = __ldg(A.rgbr + id);
    }
    __syncthreads();
    if (done) continue;
    const uint32_t cnt = min((uint32_t)CH, end - base);
    for (uint32_t g0 = 0; g0 < cnt; g0 += 32) {
      const uint32_t j = g0 + lane;
      const bool active = j < cnt;
      float alpha = 0.0f;
      bool ns = false;
      float4 c = make_float4(0.f, 0.f, 0.f, 0.f);
      if (active) {
        c = s_cop[j];
        ns = eval_step<MODE>(s_xyab[j], c, sx, sy, ek, alpha);
      }
      const float4 col = ns ? s_rgb[j] : make_float4(0.f, 0.f, 0.f, 0.f);
      const int stop = gw_group<MODE, SERIAL_W>(ns, alpha, col, c.w, t, contrib, acc, lane);
      if (stop < 32) {
        term = (int)(base - start + g0) + stop + 1;
        done = true;
        break;
      }
    }
  }
  if (inside) {
    acc.warp_sum();
    if (lane == 0) acc.finish(A, (size_t)py * A.W + px, t, contrib, term);
  }
}

template <int MODE>
__global__ void __launch_bounds__(kFgThreads) k_render_gaussianwise(RArgs A) {
  bs::pdl_wait();
  __shared__ float4 s_xyab[kFgThreads];
  __shared__ float4 s_cop[kFgThreads];
  __shared__ float4 s_rgb[kFgThreads];
  __shared__ unsigned long long s_tab[32];
  if (gated_out(A, BS_GAUSSIAN_WISE)) return;
  load_tab(s_tab);
  const ExpK ek = make_expk(s_tab);
  const int tile = blockIdx.x;
  const int subs = (A.pw * A.ph + kFgWarps - 1) / kFgWarps;
  for (int s = 0; s < subs; ++s) {
    __syncthreads();
    gaussianwise_task<MODE, kFgWarps, false>(A, tile, s, s_xyab, s_cop, s_rgb, ek);
  }
}

// ---------------------------------------------------------------------------
// GaussianWise, B200 form (paper Alg. 2/6 with the reference's serial-exact
// decisions, src/kernels.cpp:57-107), for patches of <= 256 pixels.
// CTA = one tile, 8 warps; warp w owns the tile's local pixels
// [32w, 32w+32), lane = pixel for the per-pixel state.  The CTA stages the
// tile list ONCE per 256-entry chunk (shared by all 8 warps); each warp then
// walks the chunk in 32-entry groups, two phases per group:
//   phase 1, Gaussian-wise (lane = list entry), once per live pixel p:
//     alpha of the 32 consecutive entries at p, the shfl_up doubling prefix
//     product of (1 - alpha) started at p's carried t (inc/blend.hpp:69-83)
//     -> each entry's colour weight t_before; (alpha, t_before) go to the
//     warp's 32 x 33 scratch (row p);
//   phase 2, serial (lane = pixel): each live lane walks its row in list
//     order — skip, stop (t * (1 - alpha) < 1e-4, nothing committed, term =
//     list position), commit (colour/depth += c * alpha * t_before, separate
//     double mul / add in list order as the reference).
// So contrib / term / final_t / alpha AND colour / depth equal
// render_gaussianwise bit for bit.  The exps of phase 1 run on 32 useful
// lanes (one pixel, 32 entries) and only for pixels still live; the list is
// read from L2 once per tile instead of once per 4 pixels.
constexpr int kGwWarps = 8;
constexpr int kGwThreads = kGwWarps * 32;
constexpr int kGwChunk = kGwThreads;  // list entries staged per CTA round
constexpr size_t kGwDynSmem = sizeof(float) * kGwWarps * 2 * 32 * 33;  // per-warp phase scratch, 67.6 KB

template <int MODE>
__global__ void __launch_bounds__(kGwThreads) k_render_gw(RArgs A) {
  bs::pdl_wait();
  __shared__ float4 s_xyab[kGwChunk];
  __shared__ float4 s_cop[kGwChunk];
  __shared__ double2 s_rg[kGwChunk];  // (r, g) widened once per staged entry
  __shared__ double2 s_bd[kGwChunk];  // (b, depth)
  // dynamic: per warp, alpha of (pixel row, entry) (0 = skipped) and the
  // prefix-product t_before, 32 x 33 floats each (stride 33: conflict-free
  // row writes in phase 1 and column reads in phase 2)
  extern __shared__ float s_gw_dyn[];
  __shared__ unsigned long long s_tab[32];
  if (gated_out(A, BS_GAUSSIAN_WISE)) return;
  load_tab(s_tab);
  const ExpK ek = make_expk(s_tab);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tile = blockIdx.x;
  const int tx = tile % A.cols, ty = tile / A.cols;
  const int npix = A.pw * A.ph;
  // this lane's pixel (phase 2 / state)
  const int local = warp * 32 + lane;
  const int lx = local % A.pw, ly = local / A.pw;
  const int px = tx * A.pw + lx, py = ty * A.ph + ly;
  const bool inside = local < npix && px < A.W && py < A.H;
  const float my_sx = __fadd_rn((float)px, 0.5f), my_sy = __fadd_rn((float)py, 0.5f);  // S1 sample point
  const uint32_t start = A.ranges[2 * tile], end = A.ranges[2 * tile + 1];
  float* const sa = s_gw_dyn + warp * (2 * 32 * 33);
  float* const stb = sa + 32 * 33;

  bool done = !inside;
  float t = 1.0f;
  int contrib = 0, term = 0;
  double ar = 0.0, ag = 0.0, ab = 0.0, ad = 0.0;
  float fr = 0.0f, fg = 0.0f, fb = 0.0f, fd = 0.0f;

  for (uint32_t base = start; base < end; base += kGwChunk) {
    if (__syncthreads_count(!done) == 0) break;
    const uint32_t k = base + tid;
    if (k < end) {
      const uint32_t id = __ldg(A.point_list + k);
      const float4 r = __ldg(A.rgbr + id);
      s_xyab[tid] = __ldg(A.xyab + id);
      const float4 c = __ldg(A.cop + id);
      s_cop[tid] = c;
      s_rg[tid] = make_double2((double)r.x, (double)r.y);
      s_bd[tid] = make_double2((double)r.z, (double)c.w);
    }
    __syncthreads();
    const int cnt = (int)min((uint32_t)kGwChunk, end - base);
    for (int g0 = 0; g0 < cnt && __any_sync(kFull, !done); g0 += 32) {
      const int gn = min(32, cnt - g0);
      // ---- phase 1: per live pixel, lanes on 32 consecutive entries
      unsigned live = __ballot_sync(kFull, !done);
      const int j = g0 + lane;
      const bool active = lane < gn;
      const float4 a = s_xyab[active ? j : g0], c = s_cop[active ? j : g0];
      unsigned gmask = 0;  // entries of the group some live pixel does not skip
      while (live) {
        const int p = __ffs(live) - 1;
        live &= live - 1;
        const float psx = __shfl_sync(kFull, my_sx, p), psy = __shfl_sync(kFull, my_sy, p);
        const float ts = __shfl_sync(kFull, t, p);
        float alpha = 0.0f;
        const bool ns = active && eval_step<MODE>(a, c, psx, psy, ek, alpha);
        sa[p * 33 + lane] = ns ? alpha : 0.0f;
        const unsigned nsm = __ballot_sync(kFull, ns);
        gmask |= nsm;
        if (nsm == 0) continue;  // no weight is read
        float pre = ns ? __fsub_rn(1.0f, alpha) : 1.0f;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const float v = __shfl_up_sync(kFull, pre, off);
          if (lane >= off) pre = __fmul_rn(pre, v);
        }
        const float per_lane = __fmul_rn(ts, pre);
        const float tb = __shfl_up_sync(kFull, per_lane, 1);
        stb[p * 33 + lane] = lane == 0 ? ts : tb;
      }
      __syncwarp();
      // ---- phase 2: serial decisions and commits, lane = pixel
      if (!done) {
        const float* row_a = sa + lane * 33;
        const float* row_t = stb + lane * 33;
        // only the entries some pixel does not skip (the others are skipped
        // by every pixel: no decision, no commit)
        for (unsigned m = gmask; m; m &= m - 1) {
          const int q = __ffs(m) - 1;
          const float al = row_a[q];
          if (al == 0.0f) continue;  // skipped (a non-skipped alpha is >= 1/255)
          const float tmp = __fmul_rn(t, __fsub_rn(1.0f, al));
          if (tmp < kStopThreshold) {
            done = true;
            term = (int)(base - start) + g0 + q + 1;
            break;
          }
          if (MODE == BS_ALPHA_EXACT) {
            const double w = __dmul_rn((double)al, (double)row_t[q]);
            const double2 rg = s_rg[g0 + q], bd = s_bd[g0 + q];
            ar = __dadd_rn(ar, __dmul_rn(rg.x, w));
            ag = __dadd_rn(ag, __dmul_rn(rg.y, w));
            ab = __dadd_rn(ab, __dmul_rn(bd.x, w));
            ad = __dadd_rn(ad, __dmul_rn(bd.y, w));
          } else {  // FAST: float weights and accumulators (the accumulators are widened at the end)
            const float w = al * row_t[q];
            const double2 rg = s_rg[g0 + q], bd = s_bd[g0 + q];
            fr = fmaf((float)rg.x, w, fr);
            fg = fmaf((float)rg.y, w, fg);
            fb = fmaf((float)bd.x, w, fb);
            fd = fmaf((float)bd.y, w, fd);
          }
          t = tmp;
          ++contrib;
        }
      }
      __syncwarp();
    }
  }
  if (MODE != BS_ALPHA_EXACT) {
    ar = fr;
    ag = fg;
    ab = fb;
    ad = fd;
  }
  if (inside) {
    const size_t pix = (size_t)py * A.W + px;
    A.color[3 * pix + 0] = __double2float_rn(__dadd_rn(ar, __dmul_rn((double)A.bg0, (double)t)));
    A.color[3 * pix + 1] = __double2float_rn(__dadd_rn(ag, __dmul_rn((double)A.bg1, (double)t)));
    A.color[3 * pix + 2] = __double2float_rn(__dadd_rn(ab, __dmul_rn((double)A.bg2, (double)t)));
    A.alpha[pix] = __fsub_rn(1.0f, t);
    A.depth[pix] = __double2float_rn(ad);
    A.final_t[pix] = t;
    A.contrib[pix] = contrib;
    A.term[pix] = term;
  }
}

// ---------------------------------------------------------------------------
// FineGrainedCombined, B200 form (paper Alg. 3 re-cut for 148 SMs):
//   * persistent CTAs of kFineWarps warps; every WARP claims tasks on its own
//     from the global atomicAdd queue (no CTA barriers in the loop);
//   * a task is a 32-pixel sub-tile (lane = pixel) of a tile; tasks are queued
//     tile by tile in LPT order (longest list first, bs_tile_stats);
//   * while most of the 32 pixels are live the warp blends pixel-wise over
//     32-entry batches of the list (staged in per-warp smem, next batch
//     prefetched into registers); once at most kStragglers pixels remain the
//     survivors are finished one at a time Gaussian-wise (32 lanes on 32
//     consecutive entries, gw_group) — the divergence tail that pixel-wise
//     SIMT would otherwise pay for with 31 idle lanes.
// EXACT output == render_reference on contrib/term/T/alpha bit for bit, colour
// and depth to double-sum association (serial weights in the straggler path).
#ifndef BS_SUBW
#define BS_SUBW 8
#endif
// a warp task's sub-tile, one pixel per lane: 8x4 (4x8 measured equal on C2,
// 16x2 9 % slower; build with EXTRA_NVFLAGS=-DBS_SUBW=4|16 to compare)
constexpr int kSubW = BS_SUBW, kSubH = 32 / BS_SUBW;
constexpr int kFineWarps = 8;
constexpr int kFineThreads = kFineWarps * 32;
constexpr int kStragglers = 2;  // (8 measured 4 % slower on C2 16x16 lists, 16 % on super-tile lists)
constexpr int kDonateAfter = 512;       // list entries a task walks before it may hand off
constexpr int kDonateMinRemain = 1024;  // ... and only if this many entries remain
constexpr int kStragglerMinRemain = 64;

__device__ __forceinline__ void load_rec(const RArgs& A, uint32_t k, float4& a, float4& c, float4& r) {
  const uint32_t id = __ldg(A.point_list + k);
  a = __ldg(A.xyab + id);
  c = __ldg(A.cop + id);
  r = __ldg(A.rgbr + id);
}
template <int LM>
__device__ __forceinline__ bool is_member(const RArgs& A, const float4& a, const float4& r, int tx, int ty) {
  // (the side is recomputed per call: holding it costs registers the
  // 64-register budget does not have)
  return LM == kListTile || tile_member_fast(A, tile_side(tx, ty), a.x, a.y, r.w, tx, ty);
}

__device__ __forceinline__ void sts_f32(uint32_t a, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}

__device__ __forceinline__ float approx_rcp(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float approx_rsqrt(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// Conservative sub-tile cull: true only if alpha < 1/255 at every pixel centre
// of [rx0,rx1]x[ry0,ry1].  alpha >= 1/255 needs power >= cut, i.e.
// d^T Q d <= -2 cut (Q = conic); that ellipse lies inside centre +-
// (sqrt(r2 c/D), sqrt(r2 a/D)), D = ac - b^2.  r2 carries a 1% margin, far above
// the float rounding of power/extents, so no entry that could pass the skip
// test is ever dropped (NaN / non-PD conics are never culled).
__device__ __forceinline__ bool cull_subtile(const float4 a, const float4 c, float rx0, float rx1, float ry0,
                                             float ry1) {
  const float cut = c.z;
  if (cut > 0.0f) return true;  // opacity so small that alpha < 1/255 everywhere
  const float D = a.z * c.x - a.w * a.w;
  if (!(D > 0.0f)) return false;
  const float r2 = -2.02f * cut;
  // approximate reciprocal / square roots (MUFU, ~2 ulp): far inside the 1 %
  // margin, and a NaN extent (0 * inf) only fails the comparisons (kept)
  const float k = r2 * approx_rcp(D);
  const float kx = k * c.x, ky = k * a.z;
  const float ex = kx * approx_rsqrt(kx), ey = ky * approx_rsqrt(ky);
  if ((a.x + ex < rx0) || (a.x - ex > rx1) || (a.y + ey < ry0) || (a.y - ey > ry1)) return true;
  // the box test passed: exact ellipse-rectangle test.  q(d) = a dx^2 +
  // 2b dx dy + c dy^2 is convex, so with the centre outside the rectangle its
  // minimum over the rectangle lies on an edge FACING the centre (from a
  // point of any other edge, the segment toward the centre stays inside and
  // q decreases along it): at most one vertical and one horizontal edge,
  // where q is a 1-D quadratic minimised at the clamped stationary point.
  // The 1 % margin in r2 covers the float rounding here and in the exact
  // power.
  const float mx = a.x, my = a.y, qa = a.z, qb = a.w, qc = c.x;
  if (mx >= rx0 && mx <= rx1 && my >= ry0 && my <= ry1) return false;
  const float ia = approx_rcp(qa), ic = approx_rcp(qc);  // stationary points: error only 2nd order in q
  float best;
  {
    const float dx = (mx < rx0 ? rx0 : rx1) - mx;  // the vertical edge facing the centre (if any)
    const float dy = fminf(fmaxf(-qb * dx * ic, ry0 - my), ry1 - my);
    const float q = qa * dx * dx + 2.0f * qb * dx * dy + qc * dy * dy;
    best = (mx < rx0 || mx > rx1) ? q : INFINITY;
  }
  {
    const float dy = (my < ry0 ? ry0 : ry1) - my;  // the horizontal edge facing the centre (if any)
    const float dx = fminf(fmaxf(-qb * dy * ia, rx0 - mx), rx1 - mx);
    const float q = qa * dx * dx + 2.0f * qb * dx * dy + qc * dy * dy;
    best = fminf(best, (my < ry0 || my > ry1) ? q : INFINITY);
  }
  return best > r2;
}

struct Donation {
  uint32_t pixel, start, from, end;
  float t;
  int32_t contrib;
  uint32_t mpos;  // entries of the pixel's tile list before `from` (term positions)
  uint32_t pad_;
  double acc[4];
};

__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Gaussian-wise continuation of one pixel (sample point psx, psy; current
// transmittance pt) over list entries [from, end) of a tile starting at
// `start`: 32 lanes on 32 consecutive entries, next group prefetched, serial-
// exact decisions and render_reference weights (gw_group<MODE, true>).  The
// colour partials come back warp-reduced in `part`.
template <int MODE, int LM>
__device__ __forceinline__ void gw_finish_pixel(const RArgs& A, uint32_t from, uint32_t end, uint32_t mpos,
                                                int tx, int ty, float psx, float psy, const ExpK& ek, float& pt,
                                                int& pcnt, int& ptrm, Accum<MODE>& part) {
  const int lane = threadIdx.x & 31;
  float4 na = make_float4(0.f, 0.f, 0.f, 0.f), nc = na, nr = na;
  if (from + lane < end) load_rec(A, from + lane, na, nc, nr);
  for (uint32_t g = from; g < end; g += 32) {
    const float4 a = na, c = nc, r = nr;
    const bool member = g + lane < end && is_member<LM>(A, a, r, tx, ty);
    if (g + 32 + lane < end) load_rec(A, g + 32 + lane, na, nc, nr);  // prefetch next group
    float alpha = 0.0f;
    const bool ns = member && eval_step<MODE>(a, c, psx, psy, ek, alpha);
    const int stop = gw_group<MODE, true>(ns, alpha, r, c.w, pt, pcnt, part, lane);
    const unsigned mm = __ballot_sync(kFull, member);
    if (stop < 32) {
      ptrm = (int)mpos + __popc(mm & ((2u << stop) - 1u));
      break;
    }
    mpos += (uint32_t)__popc(mm);
  }
  part.warp_sum();
}

// ---------------------------------------------------------------------------
// GaussianWise with the sub-tile cull (r2): the paper's static schedule (one
// CTA per tile, Alg. 2) with each warp owning 8x4-pixel sub-tiles of the tile
// (lane = pixel for the state).  Per 32-entry batch of the tile's list the
// loading lane culls its entry against the sub-tile (cull_subtile, as the
// fine-grained kernel) and the survivors are queued; per group of 32 queued
// survivors (groups span batches), two phases:
//   phase 1, Gaussian-wise (lane = survivor), once per live pixel: alpha of
//     the group's 32 entries at the pixel (Alg. 2's lanes-over-Gaussians:
//     one exp per lane) into the warp's 32 x 33 alpha scratch;
//   phase 2, serial (lane = pixel): skip / stop / commit in list order over
//     the entries some pixel keeps; contrib, term and the carried t follow
//     the serial float recurrence (src/kernels.cpp:79-89) bit for bit, and
//     each commit's colour weight is alpha * t of that recurrence.
// Every decision is exact.  The colour weights are render_reference's
// (serial t); render_gaussianwise's come from the doubling prefix product of
// (1 - alpha) over fixed 32-entry windows (inc/blend.hpp:69-83) — the two
// differ by float reassociation only (colour <= 1e-6).  The prefix product
// and its t_before scratch (r2's first cull kernel) halved the occupancy
// (2 -> 3 CTAs/SM without it) for weights the exact semantics never need:
// C2 1.67 -> 1.03 ms.  BS_GW_WINDOWED=1 keeps the reference's windows and
// prefix weights bit for bit (k_render_gw).
constexpr int kGcWarps = 8;
constexpr int kGcThreads = kGcWarps * 32;
constexpr size_t kGcDynSmem = sizeof(float) * kGcWarps * 32 * 33;  // alpha scratch, 33.8 KB

template <int MODE>
__global__ void __launch_bounds__(kGcThreads) k_render_gw_cull(RArgs A, int subs) {
  bs::pdl_wait();
  extern __shared__ float s_gc_dyn[];
  __shared__ float4 s_geo[kGcWarps][2][64];    // survivors' xyab, cop (a 2-batch queue)
  __shared__ double2 s_col[kGcWarps][2][64];   // survivors' (r, g), (b, depth) widened once
  __shared__ int s_kpos[kGcWarps][64];         // survivors' 1-based list positions
  __shared__ unsigned long long s_tab[32];
  if (gated_out(A, BS_GAUSSIAN_WISE)) return;
  load_tab(s_tab);
  const ExpK ek = make_expk(s_tab);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t lt = lanemask_lt();
  // the static grid in LPT order when the caller passes one (the longest
  // lists start first; the heavy tiles' CTAs no longer form the tail)
  const int tile = A.task_order ? (int)A.task_order[blockIdx.x] : (int)blockIdx.x;
  const int tx = tile % A.cols, ty = tile / A.cols;
  const int nsx = (A.pw + kSubW - 1) / kSubW;
  const uint32_t start = A.ranges[2 * tile], end = A.ranges[2 * tile + 1];
  float* const sa = s_gc_dyn + warp * (32 * 33);
  // this lane's column of the warp's alpha scratch as a 32-bit shared
  // address in a register (see ExpK)
  uint32_t sa_s;
  asm volatile("mov.u32 %0, %1;" : "=r"(sa_s) : "r"((uint32_t)__cvta_generic_to_shared(sa + lane)));
  for (int sub = warp; sub < subs; sub += kGcWarps) {
    const int ox = tx * A.pw + (sub % nsx) * kSubW, oy = ty * A.ph + (sub / nsx) * kSubH;
    const int lx = (sub % nsx) * kSubW + (lane % kSubW), ly = (sub / nsx) * kSubH + (lane / kSubW);
    const int px = ox + (lane % kSubW), py = oy + (lane / kSubW);
    const bool inside = lx < A.pw && ly < A.ph && px < A.W && py < A.H;
    const float sx = __fadd_rn((float)px, 0.5f), sy = __fadd_rn((float)py, 0.5f);
    const float rx0 = (float)ox + 0.5f, rx1 = (float)ox + (kSubW - 0.5f), ry0 = (float)oy + 0.5f,
                ry1 = (float)oy + (kSubH - 0.5f);
    bool done = !inside;
    float t = 1.0f;
    int contrib = 0, term = 0;
    double ar = 0.0, ag = 0.0, ab = 0.0, ad = 0.0;
    float4 pa = make_float4(0.f, 0.f, 0.f, 0.f), pc = pa, pr = pa;
    if (start + lane < end) load_rec(A, start + lane, pa, pc, pr);
    int qn = 0;            // queued survivors (warp-uniform)
    bool special = false;  // a queued power_cut below kExpSpecialCut (sticky per sub-tile)
    for (uint32_t base = start; base < end; base += 32) {
      if (!__any_sync(kFull, !done)) break;
      // cull against the sub-tile, append the survivors to the queue
      const bool keep = base + lane < end && !cull_subtile(pa, pc, rx0, rx1, ry0, ry1);
      const unsigned km = __ballot_sync(kFull, keep);
      special |= __any_sync(kFull, keep && pc.z < kExpSpecialCut);  // (see warp_task)
      if (keep) {
        const int pos = qn + __popc(km & lt);
        s_geo[warp][0][pos] = pa;
        s_geo[warp][1][pos] = pc;
        s_col[warp][0][pos] = make_double2((double)pr.x, (double)pr.y);
        s_col[warp][1][pos] = make_double2((double)pr.z, (double)pc.w);
        s_kpos[warp][pos] = (int)(base - start) + lane + 1;
      }
      __syncwarp();
      if (base + 32 + lane < end) load_rec(A, base + 32 + lane, pa, pc, pr);  // next batch in flight
      qn += __popc(km);
      // groups of 32 survivors (and the list's last ones): survivor groups
      // span batches, so the Gaussian-wise phase keeps all 32 lanes busy
      const bool last = base + 32 >= end;
      while (qn >= 32 || (last && qn > 0)) {
      const int n = min(qn, 32);
      // ---- phase 1: per live pixel, lanes on the survivors
      const bool active = lane < n;
      const float4 ga = s_geo[warp][0][active ? lane : 0], gc = s_geo[warp][1][active ? lane : 0];
      unsigned live = __ballot_sync(kFull, !done);
      unsigned gmask = 0;  // survivors some live pixel does not skip
      while (live) {
        const int p = __ffs(live) - 1;
        live &= live - 1;
        const float psx = __shfl_sync(kFull, sx, p), psy = __shfl_sync(kFull, sy, p);
        float alpha = 0.0f;
        const bool ns = active && (special ? eval_step<MODE, true>(ga, gc, psx, psy, ek, alpha)
                                           : eval_step<MODE, false>(ga, gc, psx, psy, ek, alpha));
        sts_f32(sa_s + 4u * (uint32_t)(p * 33), ns ? alpha : 0.0f);
        const unsigned nsm = __ballot_sync(kFull, ns);
        gmask |= nsm;
      }
      __syncwarp();
      // ---- phase 2: serial decisions and commits, lane = pixel
      if (!done) {
        const float* row_a = sa + lane * 33;
        for (unsigned m = gmask; m; m &= m - 1) {
          const int q = __ffs(m) - 1;
          const float al = row_a[q];
          if (al == 0.0f) continue;  // skipped (a non-skipped alpha is >= 1/255)
          const float tmp = __fmul_rn(t, __fsub_rn(1.0f, al));
          if (tmp < kStopThreshold) {
            done = true;
            term = s_kpos[warp][q];
            break;
          }
          // exact weight (24 x 24-bit product), one fused multiply-add per
          // channel (the variant's colour bar is 1e-6, as FineGrainedCombined)
          const double w = __dmul_rn((double)al, (double)t);
          const double2 rg = s_col[warp][0][q], bd = s_col[warp][1][q];
          ar = __fma_rn(rg.x, w, ar);
          ag = __fma_rn(rg.y, w, ag);
          ab = __fma_rn(bd.x, w, ab);
          ad = __fma_rn(bd.y, w, ad);
          t = tmp;
          ++contrib;
        }
      }
      __syncwarp();
      // move the queue's remainder (< 32 survivors, n == 32) to the front
      qn -= n;
      if (lane < qn) {
        s_geo[warp][0][lane] = s_geo[warp][0][n + lane];
        s_geo[warp][1][lane] = s_geo[warp][1][n + lane];
        s_col[warp][0][lane] = s_col[warp][0][n + lane];
        s_col[warp][1][lane] = s_col[warp][1][n + lane];
        s_kpos[warp][lane] = s_kpos[warp][n + lane];
      }
      __syncwarp();
      if (!__any_sync(kFull, !done)) break;
      }
    }
    if (inside) {
      const size_t pix = (size_t)py * A.W + px;
      A.color[3 * pix + 0] = __double2float_rn(__dadd_rn(ar, __dmul_rn((double)A.bg0, (double)t)));
      A.color[3 * pix + 1] = __double2float_rn(__dadd_rn(ag, __dmul_rn((double)A.bg1, (double)t)));
      A.color[3 * pix + 2] = __double2float_rn(__dadd_rn(ab, __dmul_rn((double)A.bg2, (double)t)));
      A.alpha[pix] = __fsub_rn(1.0f, t);
      A.depth[pix] = __double2float_rn(ad);
      A.final_t[pix] = t;
      A.contrib[pix] = contrib;
      A.term[pix] = term;
    }
  }
}

template <int MODE, int LM>
__device__ __forceinline__ void warp_task(const RArgs& A, int tile, int sub, float4 (*s)[32], int* s_k,
                                          const ExpK& ek) {
  const int lane = threadIdx.x & 31;
  const int tx = tile % A.cols, ty = tile / A.cols;
  // 8x4-pixel sub-tiles tile the pw x ph patch row-major
  const int nsx = (A.pw + kSubW - 1) / kSubW;
  const int ox = tx * A.pw + (sub % nsx) * kSubW, oy = ty * A.ph + (sub / nsx) * kSubH;
  const int lx = (sub % nsx) * kSubW + (lane % kSubW), ly = (sub / nsx) * kSubH + (lane / kSubW);
  const int px = ox + (lane % kSubW), py = oy + (lane / kSubW);
  const bool inside = lx < A.pw && ly < A.ph && px < A.W && py < A.H;
  const float sx = __fadd_rn((float)px, 0.5f), sy = __fadd_rn((float)py, 0.5f);
  const float rx0 = (float)ox + 0.5f, rx1 = (float)ox + (kSubW - 0.5f), ry0 = (float)oy + 0.5f,
              ry1 = (float)oy + (kSubH - 0.5f);
  // the pixel index replaces (px, py) from here on: with them dead, sx / sy
  // are held instead of being re-derived (I2F + add) at every step
  const uint32_t pix = (uint32_t)py * (uint32_t)A.W + (uint32_t)px;
  const uint32_t start = A.ranges[2 * tile], end = A.ranges[2 * tile + 1];

  bool done = !inside, donated = false, donate_now = false;
  float t = 1.0f;
  int contrib = 0, term = 0;
  Accum<MODE> acc;
  unsigned qpoll = 0;
  uint32_t mpos = 0;  // entries of this tile's list before `base` (term positions)

  uint32_t base = start;
  float4 pa = make_float4(0.f, 0.f, 0.f, 0.f), pc = pa, pr = pa;
  if (base + lane < end) load_rec(A, base + lane, pa, pc, pr);
  // the ids run one batch further ahead than the records: the record loads
  // of the next batch then depend on no in-flight load.  (Prefetching the
  // records with cp.async into shared slots instead of registers measured
  // +4 % instructions and slower.)
  uint32_t nid = base + 32 + lane < end ? __ldg(A.point_list + base + 32 + lane) : 0u;
  while (base < end) {
    const unsigned live = __ballot_sync(kFull, !done);
    if (!live) break;
    if (__popc(live) <= A.stragglers && end - base >= (uint32_t)kStragglerMinRemain) {
      // ---- straggler mode: finish each live pixel Gaussian-wise from `base`
      unsigned rem = live;
      while (rem) {
        const int p = __ffs(rem) - 1;
        rem &= rem - 1;
        const float psx = __shfl_sync(kFull, sx, p), psy = __shfl_sync(kFull, sy, p);
        float pt = __shfl_sync(kFull, t, p);
        int pcnt = 0, ptrm = 0;
        Accum<MODE> part;
        gw_finish_pixel<MODE, LM>(A, base, end, LM == kListTile ? base - start : mpos, tx, ty, psx, psy, ek, pt, pcnt,
                                  ptrm, part);
        if (lane == p) {
          acc.merge(part);
          t = pt;
          contrib += pcnt;
          term = ptrm;
          done = true;
        }
      }
      break;
    }
    if (donate_now && __popc(live) > kStragglers && end - base >= (uint32_t)A.donate_min_remain) {
      // ---- tail hand-off: the global queue is drained and this task is
      // still long; park every live pixel's blend state for k_render_donated
      unsigned slot0 = 0;
      if (lane == 0) {
        const unsigned nl = (unsigned)__popc(live), units = (nl + kFineWarps - 1) / kFineWarps;
        slot0 = atomicAdd(A.queue + 1, nl);
        const unsigned u0 = atomicAdd(A.queue + 3, units);
        for (unsigned u = 0; u < units; ++u)  // one CTA unit = up to kFineWarps pixels
          A.donated_tasks[u0 + u] = make_uint2(slot0 + u * kFineWarps, min((unsigned)kFineWarps, nl - u * kFineWarps));
      }
      slot0 = __shfl_sync(kFull, slot0, 0);
      if (!done) {
        Donation& d = A.donate[slot0 + __popc(live & lanemask_lt())];
        d.pixel = pix;
        d.start = start;
        d.from = base;
        d.end = end;
        d.t = t;
        d.contrib = contrib;
        d.mpos = LM == kListTile ? base - start : mpos;
        acc.store(d.acc);
        donated = true;
      }
      break;
    }
    // ---- pixel-wise batch of 32 entries: cull against the sub-tile, compact
    const bool member = base + lane < end && is_member<LM>(A, pa, pr, tx, ty);
    const unsigned mm = __ballot_sync(kFull, member);
    const bool keep = member && !cull_subtile(pa, pc, rx0, rx1, ry0, ry1);
    const unsigned km = __ballot_sync(kFull, keep);
    const bool special = __any_sync(kFull, keep && pc.z < kExpSpecialCut);
    if (keep) {
      const int pos = __popc(km & lanemask_lt());
      s[0][pos] = pa;
      s[1][pos] = pc;
      if (MODE == BS_ALPHA_EXACT) {
        // colour/depth widened to double once per staged entry (not per commit)
        reinterpret_cast<double2*>(s[2])[pos] = make_double2((double)pr.x, (double)pr.y);
        reinterpret_cast<double2*>(s[3])[pos] = make_double2((double)pr.z, (double)pc.w);
      } else {
        s[2][pos] = pr;
      }
      // 1-based position in the tile's list (term)
      s_k[pos] = LM == kListTile ? (int)(base - start) + lane + 1 : (int)mpos + __popc(mm & lanemask_lt()) + 1;
    }
    __syncwarp();
    const uint32_t nb = base + 32;
    if (nb + lane < end) {
      pa = __ldg(A.xyab + nid);
      pc = __ldg(A.cop + nid);
      pr = __ldg(A.rgbr + nid);
    }
    nid = nb + 32 + lane < end ? __ldg(A.point_list + nb + 32 + lane) : 0u;
    // queue poll every 8th batch; the value is consumed 8 batches later, so
    // the L2 round trip never stalls the blend loop
    const bool poll_point = A.donate && ((nb - start) & (8u * 32u - 1u)) == 0;
    if (poll_point) {
      donate_now = __shfl_sync(kFull, qpoll, 0) >= (unsigned)A.total_tasks && nb - start >= (uint32_t)A.donate_after;
      if (lane == 0) qpoll = ld_relaxed_u32(A.queue);
    }
    const int cnt = __popc(km);
    // (a branch-free form of these steps — every lane evaluating every step,
    // skip / stop / commit as predicates — measured 1-3 % slower: the
    // all-skip steps then pay the exp too)
    // (unroll 4: 0.483 -> 0.479 ms against 2; 1 and 3 slower, 8 the same)
    auto steps = [&](auto special) {
#pragma unroll 4
      for (int j = 0; j < cnt; ++j) {
        if (done) continue;
        float alpha;
        const float4 c = s[1][j];
        if (!eval_step<MODE, decltype(special)::value>(s[0][j], c, sx, sy, ek, alpha)) continue;
        const float tmp = __fmul_rn(t, __fsub_rn(1.0f, alpha));
        if (tmp < kStopThreshold) {
          done = true;
          term = s_k[j];
          continue;
        }
        if (MODE == BS_ALPHA_EXACT)
          acc.add_wide(alpha, t, reinterpret_cast<const double2*>(s[2])[j], reinterpret_cast<const double2*>(s[3])[j]);
        else
          acc.add(alpha, t, s[2][j], c.w);
        t = tmp;
        ++contrib;
      }
    };
    // glibc's one special-cased input (x = -0x1.f8cbb2p+5) can only reach
    // the exp through a splat whose power_cut lies below it (opacity > ~1e24,
    // outside the reference's validated [0, 1]); batches without one run
    // the exp without that compare
    if (MODE == BS_ALPHA_EXACT && special)
      steps(std::true_type{});
    else
      steps(std::false_type{});
    __syncwarp();
    if (LM != kListTile) mpos += (uint32_t)__popc(mm);
    base = nb;
  }
  if (inside && !donated) acc.finish(A, (size_t)pix, t, contrib, term);
}

// MINB: resident CTAs per SM the register budget is sized for — 4 (64
// registers, the default) or, opt-in with BS_FINE_WIDE=1 when the kernel is
// capped at <= 3 CTAs per SM, 3 (80 registers: the exp's constants stay in
// registers).  The 80-register build is 1 % faster alone but 1 % slower in
// the streamed frame pipeline (tools/sweep_occupancy.sh), where the
// uncapped 64-register kernel is best.
template <int MODE, int LM, int MINB>
__global__ void __launch_bounds__(kFineThreads, MINB) k_render_fine(RArgs A, int subs) {
  bs::pdl_wait();
  __shared__ float4 s_rec[kFineWarps][4][32];
  __shared__ int s_k[kFineWarps][32];
  __shared__ unsigned long long s_tab[32];
  if (gated_out(A, BS_FINE_GRAINED_COMBINED)) return;
  load_tab(s_tab);
  const ExpK ek = make_expk(s_tab);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // (the ticket is taken at the bottom of the loop: with the queue atomic
  // at the top, ptxas spilled 8-32 bytes of the step loop's registers;
  // this shape allocates without spills — FG 0.498 -> 0.489 ms on C2, the
  // frame pipeline 1,250 -> 1,309 views/s.  Taking the next ticket when a
  // task STARTS, to hide the atomic's round trip, measured slower: a ticket
  // held through a long task delays the LPT order's next heavy task.)
  unsigned next = 0;
  if (lane == 0) next = atomicAdd(A.queue, 1u);
  for (;;) {
    const int task = (int)__shfl_sync(kFull, next, 0);
    if (task >= A.total_tasks) return;
    const int q = task / subs;
    const int tile = A.task_order ? (int)A.task_order[q] : q;
    warp_task<MODE, LM>(A, tile, task - q * subs, s_rec[warp], s_k[warp], ek);
    if (lane == 0) next = atomicAdd(A.queue, 1u);
  }
}

// Second launch: the warp tasks parked at the tail (their warp saw the queue
// drained with a long list left) are finished by CTAs: each parked task is
// cut into units of up to kFineWarps pixels, one unit per CTA, one pixel per
// warp,
// Gaussian-wise (gw_group, serial-exact) over 256-entry chunks staged once
// for all 8 warps — the tail of the heaviest tiles is spread over all SMs.
template <int MODE>
__global__ void __launch_bounds__(kFineThreads) k_render_donated(RArgs A) {
  bs::pdl_wait();
  __shared__ float4 s_xyab[kFineThreads];
  __shared__ float4 s_cop[kFineThreads];
  __shared__ float4 s_rgb[kFineThreads];
  __shared__ bool s_mem[kFineThreads];
  __shared__ unsigned long long s_tab[32];
  __shared__ unsigned s_task;
  if (gated_out(A, BS_FINE_GRAINED_COMBINED)) return;
  const unsigned ntasks = *(volatile unsigned*)(A.queue + 3);
  if (ntasks == 0) return;  // nothing parked (most frames): no ticket, no barriers
  load_tab(s_tab);
  const ExpK ek = make_expk(s_tab);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (;;) {
    __syncthreads();
    if (tid == 0) s_task = atomicAdd(A.queue + 2, 1u);
    __syncthreads();
    const unsigned task = s_task;
    if (task >= ntasks) return;
    const uint2 tr = A.donated_tasks[task];  // (first Donation, count <= kFineWarps)
    const Donation& d0 = A.donate[tr.x];
    const uint32_t from = d0.from, end = d0.end;
    // one task's pixels: one tile (membership of super-tile list entries)
    const int ttx = (int)(d0.pixel % (uint32_t)A.W) / A.pw, tty = (int)(d0.pixel / (uint32_t)A.W) / A.ph;
    uint32_t mpos = d0.mpos;
    {
      const bool active = (unsigned)warp < tr.y;  // warp-uniform
      const Donation* d = active ? &A.donate[tr.x + warp] : nullptr;
      const uint32_t pixel = active ? d->pixel : 0u;
      const float sx = __fadd_rn((float)(pixel % (uint32_t)A.W), 0.5f);
      const float sy = __fadd_rn((float)(pixel / (uint32_t)A.W), 0.5f);
      float t = active ? d->t : 1.0f;
      int cnt = 0, trm = 0;
      bool done = !active;
      Accum<MODE> part;
      for (uint32_t base = from; base < end; base += kFineThreads) {
        if (__syncthreads_count(!done) == 0) break;
        if (base + tid < end) {
          load_rec(A, base + tid, s_xyab[tid], s_cop[tid], s_rgb[tid]);
          s_mem[tid] = !A.sup || tile_member_fast(A, tile_side(ttx, tty), s_xyab[tid].x, s_xyab[tid].y, s_rgb[tid].w,
                                                  ttx, tty);
        }
        __syncthreads();
        if (done) continue;
        const uint32_t n = min((uint32_t)kFineThreads, end - base);
        for (uint32_t g0 = 0; g0 < n; g0 += 32) {
          const uint32_t j = g0 + lane;
          const bool member = j < n && s_mem[j];
          const unsigned mm = __ballot_sync(kFull, member);
          float alpha = 0.0f;
          const bool ns = member && eval_step<MODE>(s_xyab[j], s_cop[j], sx, sy, ek, alpha);
          const int stop = gw_group<MODE, true>(ns, alpha, ns ? s_rgb[j] : make_float4(0.f, 0.f, 0.f, 0.f),
                                               ns ? s_cop[j].w : 0.0f, t, cnt, part, lane);
          if (stop < 32) {
            trm = (int)mpos + __popc(mm & ((2u << stop) - 1u));
            done = true;
            break;
          }
          mpos += (uint32_t)__popc(mm);
        }
      }
      if (active) {
        part.warp_sum();
        if (lane == 0) {
          Accum<MODE> acc;
          acc.load(d->acc);
          acc.merge(part);
          acc.finish(A, pixel, t, d->contrib + cnt, trm);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// Backward render (not in the reference): per-splat gradients
// of the forward's colour / alpha / depth under render_reference semantics
// (src/blend.cpp:8-42), the forward's skip / stop decisions held fixed —
// the math of oracle/oracle.cpp render_backward:
//   d colour / d alpha_k = c_k T_k - S_k / (1 - alpha_k),  S_k = colour -
//     sum_{j<=k} c_j w_j (= later commits + background);  depth alike;
//   d out_alpha / d alpha_k = t_final / (1 - alpha_k);
//   alpha = min(0.99, o G): no gradient through a clamped alpha; G = exp(power).
// Same schedule as FineGrainedCombined (persistent warps, 8x4-pixel
// sub-tiles from the LPT queue, the sub-tile cull, pixel-wise serial steps
// with the forward's exact decisions); per committed step the 10 gradient
// terms are summed over the warp's 32 pixels by a transposing butterfly (16
// shuffles: lane pair 2i ends holding term i) and added to the splat's
// gradient with one red.global.add per term.
struct BwdArgs {
  const float* dcolor;  // f32[3P]
  const float* dalpha;  // f32[P] or null
  const float* ddepth;  // f32[P] or null
  float* gxyab;         // f32x4[n] (d/dx, d/dy, d/dconic_a, d/dconic_b)
  float* gcop;          // f32x4[n] (d/dconic_c, d/dopacity, 0, d/ddepth)
  float* grgbr;         // f32x4[n] (d/dr, d/dg, d/db, 0)
};

// gradient term i (oracle GRAD_FIELDS order: x, y, conic a, b, c, opacity,
// r, g, b, depth) -> its (array + component); the splat adds 4 * id
__device__ __forceinline__ float* bwd_target(const BwdArgs& G, int i) {
  float* base = i < 4 ? G.gxyab : (i == 4 || i == 5 || i == 9) ? G.gcop : G.grgbr;
  const int comp = i < 4 ? i : i == 4 ? 0 : i == 5 ? 1 : i == 9 ? 3 : i - 6;
  return base + comp;
}

template <int MODE, int LM>
__device__ __forceinline__ void warp_task_bwd(const RArgs& A, const BwdArgs& G, int tile, int sub, float4 (*s)[32],
                                              uint32_t* s_id, const ExpK& ek) {
  const int lane = threadIdx.x & 31;
  const int tx = tile % A.cols, ty = tile / A.cols;
  const int nsx = (A.pw + kSubW - 1) / kSubW;
  const int ox = tx * A.pw + (sub % nsx) * kSubW, oy = ty * A.ph + (sub / nsx) * kSubH;
  const int lx = (sub % nsx) * kSubW + (lane % kSubW), ly = (sub / nsx) * kSubH + (lane / kSubW);
  const int px = ox + (lane % kSubW), py = oy + (lane / kSubW);
  const bool inside = lx < A.pw && ly < A.ph && px < A.W && py < A.H;
  const float sx = __fadd_rn((float)px, 0.5f), sy = __fadd_rn((float)py, 0.5f);
  const float rx0 = (float)ox + 0.5f, rx1 = (float)ox + (kSubW - 0.5f), ry0 = (float)oy + 0.5f,
              ry1 = (float)oy + (kSubH - 0.5f);
  const uint32_t start = A.ranges[2 * tile], end = A.ranges[2 * tile + 1];
  float gr = 0.f, gg = 0.f, gb = 0.f, ga = 0.f, gd = 0.f, Sr = 0.f, Sg = 0.f, Sb = 0.f, SD = 0.f, tf = 1.f;
  bool done = !inside;
  if (inside) {
    const size_t p = (size_t)py * A.W + px;
    gr = G.dcolor[3 * p];
    gg = G.dcolor[3 * p + 1];
    gb = G.dcolor[3 * p + 2];
    ga = G.dalpha ? G.dalpha[p] : 0.f;
    gd = G.ddepth ? G.ddepth[p] : 0.f;
    Sr = A.color[3 * p];  // the forward's outputs (colour includes bg * t_final)
    Sg = A.color[3 * p + 1];
    Sb = A.color[3 * p + 2];
    SD = A.depth[p];
    tf = A.final_t[p];
  }
  float t = 1.0f;
  // the gradient term this lane ends holding after the 10-term reduction
  // below: bit 4 picks terms 0-4 / 5-9; bits 3, 2, 1 the term inside them
  const bool h3 = lane & 8, h2 = lane & 4, h1 = lane & 2;
  const int slot = ((lane & 16) ? 5 : 0) + (h3 ? (h2 ? 4 : 3) : (h2 ? 2 : (h1 ? 1 : 0)));
  float* const tgt = bwd_target(G, slot);
  const bool adder = !(lane & 1) && ((!h3 && !h2) || !h1);  // one lane per term
  uint32_t base = start;
  float4 pa = make_float4(0.f, 0.f, 0.f, 0.f), pc = pa, pr = pa;
  uint32_t pid = 0;
  if (base + lane < end) {
    pid = __ldg(A.point_list + base + lane);
    pa = __ldg(A.xyab + pid);
    pc = __ldg(A.cop + pid);
    pr = __ldg(A.rgbr + pid);
  }
  while (base < end) {
    if (!__any_sync(kFull, !done)) break;
    const bool member = base + lane < end && is_member<LM>(A, pa, pr, tx, ty);
    const bool keep = member && !cull_subtile(pa, pc, rx0, rx1, ry0, ry1);
    const unsigned km = __ballot_sync(kFull, keep);
    const bool special = __any_sync(kFull, keep && pc.z < kExpSpecialCut);
    if (keep) {
      const int pos = __popc(km & lanemask_lt());
      s[0][pos] = pa;
      s[1][pos] = pc;
      s[2][pos] = pr;
      s_id[pos] = pid;
    }
    __syncwarp();
    const uint32_t nb = base + 32;
    if (nb + lane < end) {
      pid = __ldg(A.point_list + nb + lane);
      pa = __ldg(A.xyab + pid);
      pc = __ldg(A.cop + pid);
      pr = __ldg(A.rgbr + pid);
    }
    const int cnt = __popc(km);
    for (int j = 0; j < cnt; ++j) {
      float v[10];
#pragma unroll
      for (int i = 0; i < 10; ++i) v[i] = 0.f;
      bool com = false;
      if (!done) {
        const float4 a = s[0][j], c = s[1][j];
        const float dx = __fsub_rn(sx, a.x), dy = __fsub_rn(sy, a.y);
        const float q = __fadd_rn(__fmul_rn(__fmul_rn(a.z, dx), dx), __fmul_rn(__fmul_rn(c.x, dy), dy));
        const float power = __fsub_rn(__fmul_rn(-0.5f, q), __fmul_rn(__fmul_rn(a.w, dx), dy));
        if (!(power < c.z) && !(power > 0.0f)) {
          float e;
          if (MODE == BS_ALPHA_EXACT) {
            // power >= power_cut: glibc's special-cased input only in batches
            // holding a power_cut below kExpSpecialCut (warp-uniform branch)
            if (special) e = glibc_expf_fast<true>(power, ek);
            else e = glibc_expf_fast<false>(power, ek);
          } else {
            const float p2 = power * 1.4426950408889634f;
            asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(p2));
          }
          const float a0 = __fmul_rn(c.y, e);
          const float alpha = a0 < kAlphaClamp ? a0 : kAlphaClamp;
          if (!(alpha < kAlphaSkip)) {
            const float om = __fsub_rn(1.0f, alpha);
            const float tmp = __fmul_rn(t, om);
            if (tmp < kStopThreshold) {
              done = true;
            } else {
              const float4 r = s[2][j];
              const float w = alpha * t;
              Sr -= r.x * w;
              Sg -= r.y * w;
              Sb -= r.z * w;
              SD -= c.w * w;
              const float inv = approx_rcp(om);  // om >= 0.01
              const float dla = gr * (r.x * t - Sr * inv) + gg * (r.y * t - Sg * inv) + gb * (r.z * t - Sb * inv) +
                                gd * (c.w * t - SD * inv) + ga * tf * inv;
              v[6] = gr * w;
              v[7] = gg * w;
              v[8] = gb * w;
              v[9] = gd * w;
              if (!(a0 > kAlphaClamp)) {
                const float dlp = dla * c.y * e;
                v[5] = dla * e;
                v[2] = dlp * (-0.5f * dx * dx);
                v[3] = dlp * (-dx * dy);
                v[4] = dlp * (-0.5f * dy * dy);
                v[0] = dlp * (a.z * dx + a.w * dy);
                v[1] = dlp * (c.x * dy + a.w * dx);
              }
              t = tmp;
              com = true;
            }
          }
        }
      }
      if (!__any_sync(kFull, com)) continue;
      // transposing reduction of the 10 terms over the 32 lanes, 12 shuffles:
      // xor 16 halves the terms (5 each), xor 8 splits them 3 / 2, xor 4
      // 2 / 1 and 1 / 1, xor 2 splits the last pair (or adds the duplicate
      // single term), xor 1 completes every sum
      {
        const bool h4 = lane & 16;
#pragma unroll
        for (int i = 0; i < 5; ++i) {
          const float send = h4 ? v[i] : v[i + 5];
          v[i] = (h4 ? v[i + 5] : v[i]) + __shfl_xor_sync(kFull, send, 16);
        }
      }
      {
        const float s0 = h3 ? v[0] : v[3], s1 = h3 ? v[1] : v[4], s2 = h3 ? v[2] : 0.0f;
        const float k0 = h3 ? v[3] : v[0], k1 = h3 ? v[4] : v[1], k2 = h3 ? 0.0f : v[2];
        v[0] = k0 + __shfl_xor_sync(kFull, s0, 8);
        v[1] = k1 + __shfl_xor_sync(kFull, s1, 8);
        v[2] = k2 + __shfl_xor_sync(kFull, s2, 8);
      }
      {
        // lanes with bit 3 clear hold 3 terms (p0, p1, p2), the others 2
        const float s0 = h2 ? v[0] : (h3 ? v[1] : v[2]);
        const float k0 = h2 ? (h3 ? v[1] : v[2]) : v[0];
        const float s1 = (!h3 && h2) ? v[1] : 0.0f;
        const float k1 = (!h3 && !h2) ? v[1] : 0.0f;
        v[0] = k0 + __shfl_xor_sync(kFull, s0, 4);
        v[1] = k1 + __shfl_xor_sync(kFull, s1, 4);
      }
      {
        const bool two = !h3 && !h2;  // still two terms
        const float s0 = two ? (h1 ? v[0] : v[1]) : v[0];
        const float k0 = two ? (h1 ? v[1] : v[0]) : v[0];
        v[0] = k0 + __shfl_xor_sync(kFull, s0, 2);
      }
      v[0] += __shfl_xor_sync(kFull, v[0], 1);
      if (adder && v[0] != 0.0f) atomicAdd(tgt + 4 * (size_t)s_id[j], v[0]);
    }
    __syncwarp();
    base = nb;
  }
}

template <int MODE, int LM>
__global__ void __launch_bounds__(kFineThreads) k_render_backward(RArgs A, BwdArgs G, int subs) {
  bs::pdl_wait();
  __shared__ float4 s_rec[kFineWarps][3][32];
  __shared__ uint32_t s_id[kFineWarps][32];
  __shared__ unsigned long long s_tab[32];
  load_tab(s_tab);
  const ExpK ek = make_expk(s_tab);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (;;) {
    int task = 0;
    if (lane == 0) task = (int)atomicAdd(A.queue, 1u);
    task = __shfl_sync(kFull, task, 0);
    if (task >= A.total_tasks) return;
    const int q = task / subs;
    const int tile = A.task_order ? (int)A.task_order[q] : q;
    warp_task_bwd<MODE, LM>(A, G, tile, task - q * subs, s_rec[warp], s_id[warp], ek);
  }
}

__global__ void k_frame_work(const int32_t* __restrict__ term, const int32_t* __restrict__ contrib,
                             const uint32_t* __restrict__ ranges, int W, int H, int pw, int ph, int cols,
                             unsigned long long* __restrict__ out) {
  bs::pdl_wait();
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long e = 0, c = 0;
  if (p < (int64_t)W * H) {
    const int px = (int)(p % W), py = (int)(p / W);
    const int tile = (py / ph) * cols + (px / pw);
    const int32_t tm = term[p];
    e = tm > 0 ? (unsigned long long)tm : (unsigned long long)(ranges[2 * tile + 1] - ranges[2 * tile]);
    c = (unsigned long long)contrib[p];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    e += __shfl_xor_sync(kFull, e, o);
    c += __shfl_xor_sync(kFull, c, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(out + 0, e);
    atomicAdd(out + 1, c);
  }
}

static int g_fine_ctas_per_sm = 0;  // process default (bs_render_set_fine_occupancy); 0 = as many as fit

// Tuning knobs, read from the environment ONCE per process (defaults are the
// calibrated ones; the variables exist for A/B measurement — DESIGN.md §9).
struct FineTuning {
  int ctas_per_sm;  // BS_FINE_CTAS_PER_SM (0 = as many as fit)
  bool donate;      // BS_FINE_DONATE=0 disables the tail hand-off
  int donate_after, donate_min_remain, stragglers, stragglers_super;
  bool wide;        // BS_FINE_WIDE=1: the 80-register build when capped at <= 3 CTAs/SM
  bool no_lpt;      // BS_FINE_NO_LPT=1: tasks in tile-index order
  bool gw_windowed; // BS_GW_WINDOWED=1: GaussianWise in the reference's fixed 32-entry windows (bit-exact colour)
};
static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}
static const FineTuning& fine_tuning() {
  static const FineTuning t = [] {
    FineTuning f;
    f.ctas_per_sm = env_int("BS_FINE_CTAS_PER_SM", 0);
    f.donate = env_int("BS_FINE_DONATE", 1) != 0;
    f.donate_after = env_int("BS_FINE_DONATE_AFTER", kDonateAfter);
    f.donate_min_remain = env_int("BS_FINE_DONATE_MIN", kDonateMinRemain);
    f.stragglers = env_int("BS_FINE_STRAGGLERS", kStragglers);
    f.stragglers_super = env_int("BS_FINE_STRAGGLERS_SUPER", kStragglers);
    f.wide = env_int("BS_FINE_WIDE", 0) != 0;  // opt-in: measured 1 % slower in the streamed pipeline
    f.no_lpt = env_int("BS_FINE_NO_LPT", 0) != 0;
    f.gw_windowed = env_int("BS_GW_WINDOWED", 0) != 0;
    return f;
  }();
  return t;
}

// Per-device launch facts (SM count, occupancy of the persistent kernels),
// queried once per device and mode instead of on every launch.
struct DevFacts {
  int sms = 0;
  int fine_per_sm[2] = {0, 0};     // k_render_fine<MODE, kListTile, 4>, by MODE
  int donated_per_sm[2] = {0, 0};  // k_render_donated<MODE>
  int dyn_per_sm[2][5] = {};       // k_render_dynamic<MODE, 64 << i>
};
constexpr int kMaxDevices = 64;
static DevFacts g_dev[kMaxDevices];

static int dev_facts(DevFacts** out) {
  int dev = 0;
  BS_CUDA_TRY(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDevices) return BS_ERR_UNSUPPORTED;
  DevFacts& f = g_dev[dev];
  if (f.sms == 0) {  // (a concurrent first call computes the same values)
    DevFacts n;
    BS_CUDA_TRY(cudaDeviceGetAttribute(&n.sms, cudaDevAttrMultiProcessorCount, dev));
    BS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n.fine_per_sm[0],
                                                              k_render_fine<BS_ALPHA_EXACT, kListTile, 4>,
                                                              kFineThreads, 0));
    BS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n.fine_per_sm[1],
                                                              k_render_fine<BS_ALPHA_FAST, kListTile, 4>,
                                                              kFineThreads, 0));
    BS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n.donated_per_sm[0], k_render_donated<BS_ALPHA_EXACT>,
                                                              kFineThreads, 0));
    BS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n.donated_per_sm[1], k_render_donated<BS_ALPHA_FAST>,
                                                              kFineThreads, 0));
#define BS_DYN_OCC(M, I, B) \
    BS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n.dyn_per_sm[M][I], k_render_dynamic<M, B>, B, 0));
    BS_DYN_OCC(0, 0, 64) BS_DYN_OCC(0, 1, 128) BS_DYN_OCC(0, 2, 256) BS_DYN_OCC(0, 3, 512) BS_DYN_OCC(0, 4, 1024)
    BS_DYN_OCC(1, 0, 64) BS_DYN_OCC(1, 1, 128) BS_DYN_OCC(1, 2, 256) BS_DYN_OCC(1, 3, 512) BS_DYN_OCC(1, 4, 1024)
#undef BS_DYN_OCC
    BS_CUDA_TRY(cudaFuncSetAttribute(k_render_gw<BS_ALPHA_EXACT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)kGwDynSmem));
    BS_CUDA_TRY(cudaFuncSetAttribute(k_render_gw<BS_ALPHA_FAST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)kGwDynSmem));
    BS_CUDA_TRY(cudaFuncSetAttribute(k_render_gw_cull<BS_ALPHA_EXACT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)kGcDynSmem));
    BS_CUDA_TRY(cudaFuncSetAttribute(k_render_gw_cull<BS_ALPHA_FAST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)kGcDynSmem));
    f = n;
  }
  *out = &f;
  return BS_OK;
}

// fine_cap: resident FineGrainedCombined CTAs per SM for this launch (> 0),
// or 0 = the process default (bs_render_set_fine_occupancy, then
// BS_FINE_CTAS_PER_SM, then as many as fit).
template <int MODE>
static int launch_variant(int variant, const RArgs& A, int block_pixels, int fine_cap, cudaStream_t st) {
  const int T = A.T;
  DevFacts* df = nullptr;
  TRY_BS(dev_facts(&df));
  const int sms = df->sms;
  switch (variant) {
    case BS_NAIVE:
    case BS_SHARED_MEM_OPT: {
      const bool smem = variant == BS_SHARED_MEM_OPT;
      // auto-mode candidate: at most 8 CTAs per SM, tiles in grid stride
      const int grid = A.gate ? max(1, min(T, sms * 8)) : T;
#define BS_PW_CASE(B)                                                                   \
  if (block_pixels <= B) {                                                              \
    if (smem) bs::launch_pdl(k_render_pixelwise<MODE, true, B>, grid, B, 0, st, A);                 \
    else bs::launch_pdl(k_render_pixelwise<MODE, false, B>, grid, B, 0, st, A);                     \
    break;                                                                              \
  }
      BS_PW_CASE(64) BS_PW_CASE(128) BS_PW_CASE(256) BS_PW_CASE(512) BS_PW_CASE(1024)
#undef BS_PW_CASE
      return BS_ERR_UNSUPPORTED;
    }
    case BS_DYNAMIC_BLOCKS: {
#define BS_DYN_CASE(I, B)                                                      \
  if (block_pixels <= B) {                                                     \
    const int grid = max(1, min(T, sms * max(1, df->dyn_per_sm[MODE][I])));   \
    bs::launch_pdl(k_render_dynamic<MODE, B>, grid, B, 0, st, A);                          \
    break;                                                                     \
  }
      BS_DYN_CASE(0, 64) BS_DYN_CASE(1, 128) BS_DYN_CASE(2, 256) BS_DYN_CASE(3, 512) BS_DYN_CASE(4, 1024)
#undef BS_DYN_CASE
      return BS_ERR_UNSUPPORTED;
    }
    case BS_GAUSSIAN_WISE:
      if (fine_tuning().gw_windowed && block_pixels <= kGwThreads)  // (dynamic smem opt-in: dev_facts)
        bs::launch_pdl(k_render_gw<MODE>, T, kGwThreads, kGwDynSmem, st, A);
      else if (!fine_tuning().gw_windowed)
        bs::launch_pdl(k_render_gw_cull<MODE>, T, kGcThreads, kGcDynSmem, st, 
            A, ((A.pw + kSubW - 1) / kSubW) * ((A.ph + kSubH - 1) / kSubH));
      else  // larger patches: 4-warp tasks, 4 pixels at a time
        bs::launch_pdl(k_render_gaussianwise<MODE>, T, kFgThreads, 0, st, A);
      break;
    case BS_FINE_GRAINED_COMBINED: {
      const FineTuning& ft = fine_tuning();
      const int lm = A.sup ? kListSuper : kListTile;
      // fewer resident CTAs leave SM room for another frame context's kernels
      int per_sm = df->fine_per_sm[MODE];
      const int cap = fine_cap > 0 ? fine_cap : (g_fine_ctas_per_sm > 0 ? g_fine_ctas_per_sm : ft.ctas_per_sm);
      if (cap > 0) per_sm = min(per_sm, cap);
      per_sm = max(1, per_sm);
      const bool wide = per_sm <= 3 && ft.wide;  // the 80-register build
      const int subs = ((A.pw + kSubW - 1) / kSubW) * ((A.ph + kSubH - 1) / kSubH);  // sub-tiles per tile
      const int64_t total = (int64_t)T * subs;
      if (total > 0x7fffffff) return BS_ERR_UNSUPPORTED;
      const int64_t ctas = (total + kFineWarps - 1) / kFineWarps;
      const int grid = (int)max((int64_t)1, min(ctas, (int64_t)sms * per_sm));
      RArgs B = A;
      B.total_tasks = (int)total;
      if (!ft.donate) B.donate = nullptr;
      B.donate_after = ft.donate_after;
      B.donate_min_remain = ft.donate_min_remain;
      B.stragglers = A.sup ? ft.stragglers_super : ft.stragglers;
      if (lm == kListSuper) {
        if (wide) bs::launch_pdl(k_render_fine<MODE, kListSuper, 3>, grid, kFineThreads, 0, st, B, subs);
        else bs::launch_pdl(k_render_fine<MODE, kListSuper, 4>, grid, kFineThreads, 0, st, B, subs);
      } else {
        if (wide) bs::launch_pdl(k_render_fine<MODE, kListTile, 3>, grid, kFineThreads, 0, st, B, subs);
        else bs::launch_pdl(k_render_fine<MODE, kListTile, 4>, grid, kFineThreads, 0, st, B, subs);
      }
      BS_LAUNCH_CHECK();
      if (!B.donate) return BS_OK;
      bs::launch_pdl(k_render_donated<MODE>, sms * max(1, df->donated_per_sm[MODE]), kFineThreads, 0, st, B);
      break;
    }
    default:
      return BS_ERR_INVALID_ARGUMENT;
  }
  BS_LAUNCH_CHECK();
  return BS_OK;
}

}  // namespace bs

using namespace bs;

// queue counters + one Donation slot per pixel (FineGrainedCombined tail hand-off)
extern "C" size_t bs_render_workspace_bytes(int32_t width, int32_t height) {
  if (width <= 0 || height <= 0) return 0;
  const size_t P = (size_t)width * (size_t)height;
  return 256 + sizeof(Donation) * P + sizeof(uint2) * (P / 4 + 1);  // >= 9 pixels -> <= 2 units per 9
}

static bool pow2(int v) { return v > 0 && (v & (v - 1)) == 0; }

static int render_impl(int variant, const int32_t* gate, int alpha_mode, bs_splats g, const uint32_t* point_list,
                       const uint32_t* tile_ranges, const uint32_t* task_order, int32_t width, int32_t height,
                       int32_t pw, int32_t ph, const float bg[3], bs_frame_out out, void* ws, size_t ws_bytes,
                       void* stream, bool sup = false, int fine_cap = 0) {
  if (width <= 0 || height <= 0 || pw <= 0 || ph <= 0 || !bg || !tile_ranges) return BS_ERR_INVALID_ARGUMENT;
  if (alpha_mode != BS_ALPHA_EXACT && alpha_mode != BS_ALPHA_FAST) return BS_ERR_INVALID_ARGUMENT;
  if (!out.color || !out.alpha || !out.depth || !out.final_t || !out.contrib || !out.term) return BS_ERR_INVALID_ARGUMENT;
  if ((int64_t)pw * ph > 1024) return BS_ERR_UNSUPPORTED;
  // pixel indices are 32-bit in the kernels and the tail hand-off records
  if ((int64_t)width * height > (int64_t)0xffffffff) return BS_ERR_UNSUPPORTED;
  if (!ws || ws_bytes < bs_render_workspace_bytes(width, height)) return BS_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  RArgs A;
  A.xyab = reinterpret_cast<const float4*>(g.xyab);
  A.cop = reinterpret_cast<const float4*>(g.cop);
  A.rgbr = reinterpret_cast<const float4*>(g.rgbr);
  A.point_list = point_list;
  A.ranges = tile_ranges;
  A.task_order = fine_tuning().no_lpt ? nullptr : task_order;  // A/B: index order
  A.W = width; A.H = height; A.pw = pw; A.ph = ph;
  A.cols = (width + pw - 1) / pw;
  const int64_t T = (int64_t)A.cols * ((height + ph - 1) / ph);
  if (T > 0x7fffffff) return BS_ERR_UNSUPPORTED;
  A.T = (int)T;
  A.bg0 = bg[0]; A.bg1 = bg[1]; A.bg2 = bg[2];
  A.color = out.color; A.alpha = out.alpha; A.depth = out.depth; A.final_t = out.final_t;
  A.contrib = out.contrib; A.term = out.term;
  A.queue = reinterpret_cast<unsigned int*>(ws);
  A.donate = reinterpret_cast<Donation*>(static_cast<char*>(ws) + 256);
  A.donated_tasks = reinterpret_cast<uint2*>(A.donate + (size_t)width * height);
  A.total_tasks = 0;
  A.gate = gate;
  A.sup = sup ? 1 : 0;
  A.rows = (height + ph - 1) / ph;
  A.ipw = 1.0f / (float)pw;
  A.iph = 1.0f / (float)ph;
  if (sup && (!pow2(pw) || !pow2(ph))) return BS_ERR_UNSUPPORTED;
  if (sup && !gate && variant != BS_FINE_GRAINED_COMBINED && variant != BS_SHARED_MEM_OPT) return BS_ERR_UNSUPPORTED;
  if (gate || variant == BS_DYNAMIC_BLOCKS || variant == BS_FINE_GRAINED_COMBINED)
    BS_CUDA_TRY(cudaMemsetAsync(ws, 0, 8 * sizeof(unsigned int), st));
  const int block_pixels = pw * ph;
  auto launch = [&](int v) {
    return alpha_mode == BS_ALPHA_EXACT ? launch_variant<BS_ALPHA_EXACT>(v, A, block_pixels, fine_cap, st)
                                        : launch_variant<BS_ALPHA_FAST>(v, A, block_pixels, fine_cap, st);
  };
  if (!gate) return launch(variant);
  // auto: the selector's two candidates (select_variant_formula)
  const int s1 = launch(BS_FINE_GRAINED_COMBINED);
  if (s1 != BS_OK) return s1;
  return launch(BS_SHARED_MEM_OPT);
}

extern "C" int bs_render_forward(int variant, int alpha_mode, bs_splats g, const uint32_t* point_list,
                                 const uint32_t* tile_ranges, const uint32_t* task_order, int32_t width,
                                 int32_t height, int32_t pw, int32_t ph, const float bg[3], bs_frame_out out,
                                 void* ws, size_t ws_bytes, void* stream) {
  if (variant < 0 || variant > 4) return BS_ERR_INVALID_ARGUMENT;
  return render_impl(variant, nullptr, alpha_mode, g, point_list, tile_ranges, task_order, width, height, pw, ph, bg,
                     out, ws, ws_bytes, stream);
}

extern "C" int bs_render_forward_auto(const int32_t* variant_dev, int alpha_mode, bs_splats g,
                                      const uint32_t* point_list, const uint32_t* tile_ranges,
                                      const uint32_t* task_order, int32_t width, int32_t height, int32_t pw,
                                      int32_t ph, const float bg[3], bs_frame_out out, void* ws, size_t ws_bytes,
                                      void* stream) {
  if (!variant_dev) return BS_ERR_INVALID_ARGUMENT;
  return render_impl(-1, variant_dev, alpha_mode, g, point_list, tile_ranges, task_order, width, height, pw, ph, bg,
                     out, ws, ws_bytes, stream);
}

// Super-tile lists (the frame pipeline's binning at 2pw x 2ph): the render
// walks tile t's super-tile list and keeps the entries whose pw x ph
// rectangle contains t — exactly t's list, in (depth, index) order, term
// positions counted over it.  tile_ranges here holds, per pw x ph tile, the
// range of its super-tile (bs_super_tile_ranges).  variant -1: the device
// selector's choice among the candidates (FineGrainedCombined,
// SharedMemOpt), as bs_render_forward_auto.
extern "C" int bs_render_forward_super(int variant, const int32_t* variant_dev, int alpha_mode, bs_splats g,
                                       const uint32_t* point_list, const uint32_t* tile_ranges,
                                       const uint32_t* task_order, int32_t width, int32_t height, int32_t pw,
                                       int32_t ph, const float bg[3], bs_frame_out out, void* ws, size_t ws_bytes,
                                       void* stream) {
  if (variant < 0 && !variant_dev) return BS_ERR_INVALID_ARGUMENT;
  return render_impl(variant < 0 ? -1 : variant, variant < 0 ? variant_dev : nullptr, alpha_mode, g, point_list,
                     tile_ranges, task_order, width, height, pw, ph, bg, out, ws, ws_bytes, stream, true);
}

// Backward render.  fwd: the forward's outputs for the same
// inputs (colour, depth and final_t are read); grads accumulate (caller
// zeroes).  super_lists: point_list / tile_ranges are the frame pipeline's
// 2pw x 2ph lists (as bs_render_forward_super).  Workspace: the render
// workspace (its queue counters).
extern "C" int bs_render_backward(int alpha_mode, bs_splats g, const uint32_t* point_list, const uint32_t* tile_ranges,
                                  const uint32_t* task_order, int32_t width, int32_t height, int32_t pw, int32_t ph,
                                  const float bg[3], bs_frame_out fwd, bs_frame_grad_in gin, bs_splat_grads gout,
                                  int super_lists, void* ws, size_t ws_bytes, void* stream) {
  if (width <= 0 || height <= 0 || pw <= 0 || ph <= 0 || !bg || !tile_ranges) return BS_ERR_INVALID_ARGUMENT;
  if (alpha_mode != BS_ALPHA_EXACT && alpha_mode != BS_ALPHA_FAST) return BS_ERR_INVALID_ARGUMENT;
  if (!fwd.color || !fwd.depth || !fwd.final_t || !gin.dl_dcolor || !gout.xyab || !gout.cop || !gout.rgbr)
    return BS_ERR_INVALID_ARGUMENT;
  if ((int64_t)pw * ph > 1024) return BS_ERR_UNSUPPORTED;
  if ((int64_t)width * height > (int64_t)0xffffffff) return BS_ERR_UNSUPPORTED;  // (32-bit pixel indices)
  if (super_lists && (!pow2(pw) || !pow2(ph))) return BS_ERR_UNSUPPORTED;
  if (!ws || ws_bytes < 256) return BS_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  RArgs A{};
  A.xyab = reinterpret_cast<const float4*>(g.xyab);
  A.cop = reinterpret_cast<const float4*>(g.cop);
  A.rgbr = reinterpret_cast<const float4*>(g.rgbr);
  A.point_list = point_list;
  A.ranges = tile_ranges;
  A.task_order = task_order;
  A.W = width; A.H = height; A.pw = pw; A.ph = ph;
  A.cols = (width + pw - 1) / pw;
  A.rows = (height + ph - 1) / ph;
  const int64_t T = (int64_t)A.cols * A.rows;
  const int subs = ((pw + kSubW - 1) / kSubW) * ((ph + kSubH - 1) / kSubH);
  if (T * subs > 0x7fffffff) return BS_ERR_UNSUPPORTED;
  A.T = (int)T;
  A.bg0 = bg[0]; A.bg1 = bg[1]; A.bg2 = bg[2];
  A.color = fwd.color; A.depth = fwd.depth; A.final_t = fwd.final_t;
  A.queue = reinterpret_cast<unsigned int*>(ws);
  A.total_tasks = (int)(T * subs);
  A.sup = super_lists ? 1 : 0;
  A.ipw = 1.0f / (float)pw;
  A.iph = 1.0f / (float)ph;
  BwdArgs G{gin.dl_dcolor, gin.dl_dalpha, gin.dl_ddepth, gout.xyab, gout.cop, gout.rgbr};
  BS_CUDA_TRY(cudaMemsetAsync(ws, 0, 8 * sizeof(unsigned int), st));
  if (T == 0) return BS_OK;
  DevFacts* df = nullptr;
  TRY_BS(dev_facts(&df));
  const int grid = (int)max((int64_t)1, min((T * subs + kFineWarps - 1) / kFineWarps, (int64_t)df->sms * 4));
#define BS_BWD(M, L) bs::launch_pdl(k_render_backward<M, L>, grid, kFineThreads, 0, st, A, G, subs)
  if (alpha_mode == BS_ALPHA_EXACT) {
    if (super_lists) BS_BWD(BS_ALPHA_EXACT, kListSuper);
    else BS_BWD(BS_ALPHA_EXACT, kListTile);
  } else {
    if (super_lists) BS_BWD(BS_ALPHA_FAST, kListSuper);
    else BS_BWD(BS_ALPHA_FAST, kListTile);
  }
#undef BS_BWD
  BS_LAUNCH_CHECK();
  return BS_OK;
}

namespace bs {
__global__ void k_super_tile_ranges(const uint32_t* __restrict__ sranges, int cols, int rows, int scols,
                                    uint32_t* __restrict__ out) {
  bs::pdl_wait();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= cols * rows) return;
  const int st = ((t / cols) >> 1) * scols + ((t % cols) >> 1);
  reinterpret_cast<uint2*>(out)[t] = reinterpret_cast<const uint2*>(sranges)[st];
}
}  // namespace bs

// per pw x ph tile, the range of its 2pw x 2ph super-tile
extern "C" int bs_super_tile_ranges(const uint32_t* super_ranges, int32_t width, int32_t height, int32_t pw,
                                    int32_t ph, uint32_t* tile_ranges, void* stream) {
  if (!super_ranges || !tile_ranges || width <= 0 || height <= 0 || pw <= 0 || ph <= 0) return BS_ERR_INVALID_ARGUMENT;
  const int cols = (width + pw - 1) / pw, rows = (height + ph - 1) / ph;
  const int scols = (width + 2 * pw - 1) / (2 * pw);
  const int T = cols * rows;
  if (T > 0)
    bs::launch_pdl(bs::k_super_tile_ranges, (T + 255) / 256, 256, 0, (cudaStream_t)stream, super_ranges, cols, rows, scols,
                                                                              tile_ranges);
  BS_LAUNCH_CHECK();
  return BS_OK;
}

namespace bs {
// The render's exp, exactly as eval_step calls it: EXACT mode ->
// glibc_expf_fast (valid on [-0x1.9fe368p6, 0], the range power_cut and the
// power > 0 skip leave it) with the table in shared memory through ExpK;
// inputs outside that range take the general glibc_expf.  FAST mode -> the
// ex2.approx path.
__device__ __forceinline__ float render_expf(float x, int mode, const ExpK& ek, const unsigned long long* s_tab) {
  float e;
  if (mode == BS_ALPHA_EXACT) {
    e = (x >= -0x1.9fe368p6f && x <= 0.0f) ? glibc_expf_fast(x, ek) : glibc_expf(x, s_tab);
  } else {
    const float p2 = x * 1.4426950408889634f;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(p2));
  }
  return e;
}

__global__ void k_test_expf(const float* __restrict__ x, float* __restrict__ y, int64_t n, int mode) {
  bs::pdl_wait();
  __shared__ unsigned long long s_tab[32];
  load_tab(s_tab);
  __syncthreads();
  const ExpK ek = make_expk(s_tab);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = render_expf(x[i], mode, ek, s_tab);
}

// y[i] = exp(float with bit pattern first_bits + i)
__global__ void k_test_expf_range(uint32_t first_bits, float* __restrict__ y, int64_t n, int mode) {
  bs::pdl_wait();
  __shared__ unsigned long long s_tab[32];
  load_tab(s_tab);
  __syncthreads();
  const ExpK ek = make_expk(s_tab);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = render_expf(__uint_as_float(first_bits + (uint32_t)i), mode, ek, s_tab);
}
}  // namespace bs

extern "C" int bs_test_expf(const float* x, float* y, int64_t n, int alpha_mode, void* stream) {
  if (n < 0 || (n > 0 && (!x || !y))) return BS_ERR_INVALID_ARGUMENT;
  if (n == 0) return BS_OK;
  const int64_t blocks = min((n + 255) / 256, (int64_t)148 * 16);
  bs::launch_pdl(k_test_expf, (unsigned)blocks, 256, 0, (cudaStream_t)stream, x, y, n, alpha_mode);
  BS_LAUNCH_CHECK();
  return BS_OK;
}

extern "C" int bs_test_expf_range(uint32_t first_bits, int64_t n, float* y, int alpha_mode, void* stream) {
  if (n < 0 || (n > 0 && !y) || (uint64_t)first_bits + (uint64_t)n > 0x100000000ull) return BS_ERR_INVALID_ARGUMENT;
  if (n == 0) return BS_OK;
  const int64_t blocks = min((n + 255) / 256, (int64_t)148 * 16);
  bs::launch_pdl(k_test_expf_range, (unsigned)blocks, 256, 0, (cudaStream_t)stream, first_bits, y, n, alpha_mode);
  BS_LAUNCH_CHECK();
  return BS_OK;
}

extern "C" int bs_frame_work(const int32_t* term, const int32_t* contrib, const uint32_t* tile_ranges, int32_t width,
                             int32_t height, int32_t pw, int32_t ph, uint64_t* evaluated_committed, void* stream) {
  if (width <= 0 || height <= 0 || pw <= 0 || ph <= 0 || !term || !contrib || !tile_ranges || !evaluated_committed)
    return BS_ERR_INVALID_ARGUMENT;
  cudaStream_t st = (cudaStream_t)stream;
  BS_CUDA_TRY(cudaMemsetAsync(evaluated_committed, 0, 2 * sizeof(uint64_t), st));
  const int64_t P = (int64_t)width * height;
  bs::launch_pdl(k_frame_work, (unsigned)((P + 255) / 256), 256, 0, st, term, contrib, tile_ranges, width, height, pw, ph,
                                                            (width + pw - 1) / pw,
                                                            reinterpret_cast<unsigned long long*>(evaluated_committed));
  BS_LAUNCH_CHECK();
  return BS_OK;
}

// The frame context's render: the pw x ph lists (sup = 0) or super-tile
// lists (sup = 1), a fixed variant or (variant -1) the device-selected one,
// and the context's own FineGrainedCombined occupancy cap (0 = process
// default) — so two contexts in one process never share that setting.
extern "C" int bs_render_forward_ctx(int variant, const int32_t* variant_dev, int alpha_mode, bs_splats g,
                                     const uint32_t* point_list, const uint32_t* tile_ranges,
                                     const uint32_t* task_order, int32_t width, int32_t height, int32_t pw, int32_t ph,
                                     const float bg[3], bs_frame_out out, int32_t super_lists,
                                     int32_t fine_ctas_per_sm, void* ws, size_t ws_bytes, void* stream) {
  if (variant < -1 || variant > 4 || (variant < 0 && !variant_dev) || fine_ctas_per_sm < 0)
    return BS_ERR_INVALID_ARGUMENT;
  return render_impl(variant < 0 ? -1 : variant, variant < 0 ? variant_dev : nullptr, alpha_mode, g, point_list,
                     tile_ranges, task_order, width, height, pw, ph, bg, out, ws, ws_bytes, stream, super_lists != 0,
                     fine_ctas_per_sm);
}

extern "C" int bs_render_set_fine_occupancy(int32_t ctas_per_sm) {
  if (ctas_per_sm < 0) return BS_ERR_INVALID_ARGUMENT;
  g_fine_ctas_per_sm = ctas_per_sm;
  return BS_OK;
}
