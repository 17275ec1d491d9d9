// frame_context.cpp — host-buffer forward pipeline over the C-ABI.
//
// The drop-in for the reference's host call chain
//   project_all (src/preprocess.cpp:57) -> bin_tiles (:66) ->
//   tile_load_histogram (:117) -> run_kernel (src/kernels.cpp:268)
// on HOST data: one H2D copy of the Gaussians, the whole pipeline on the
// device (one stream, buffers that persist and grow), one D2H copy per
// requested output plane.  The only mid-frame sync is the 8-byte K readback
// needed to size point_list (the reference pipeline has the same data
// dependency).
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <vector>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>

#include "splatsim_b200.h"

namespace bs {
void count_launches(unsigned long long n);  // csrc/capi.cu: the library's kernel launch counter
}

constexpr int kStages = 6;  // preprocess, bin_count, k_readback, bin_sort, stats_select, render

struct bs_context {
  int alpha_mode = BS_ALPHA_EXACT;
  int32_t fine_ctas = 0;  // FineGrainedCombined CTAs per SM for this context (0 = process default)
  cudaStream_t stream = nullptr;
  int sm_count = 148;
  // device buffers
  void* g3d = nullptr;
  size_t g3d_bytes = 0;
  float4* splat[3] = {nullptr, nullptr, nullptr};
  int64_t splat_cap = 0;
  int32_t* n_visible = nullptr;
  int64_t* k_dev = nullptr;
  int64_t* k_host = nullptr;  // pinned
  void* pre_ws = nullptr;
  size_t pre_ws_bytes = 0;
  void* bin_ws = nullptr;
  size_t bin_ws_bytes = 0;
  int64_t bin_n = -1, bin_k = -1;
  int bin_key[4] = {0, 0, 0, 0};
  uint32_t* point_list = nullptr;
  int64_t pl_cap = 0;
  uint32_t* ranges = nullptr;  // binning-grid ranges (the 2pw x 2ph super-tiles in super mode)
  int64_t ranges_cap = 0;
  // super mode: pw x ph list lengths (stats, LPT order, selector, info) and
  // the per-tile super-tile ranges the render walks
  uint32_t* ranges16 = nullptr;
  int64_t ranges16_cap = 0;
  uint32_t* ranges_t = nullptr;
  int64_t ranges_t_cap = 0;
  void* aux_ws = nullptr;
  size_t aux_ws_bytes = 0;
  bool last_super = false;
  bool lengths16_done = false;  // ranges16 holds the last frame's pw x ph lengths
  void* stats_ws = nullptr;
  size_t stats_ws_bytes = 0;
  uint32_t* order = nullptr;
  int64_t order_cap = 0;
  bs_tile_histogram* stats_dev = nullptr;
  bs_tile_histogram* stats_host = nullptr;  // pinned
  void* render_ws = nullptr;
  size_t render_ws_bytes = 0;
  float* planes[4] = {nullptr, nullptr, nullptr, nullptr};
  int32_t* iplanes[2] = {nullptr, nullptr};
  int64_t pixel_cap = 0;
  uint64_t* work_dev = nullptr;
  uint64_t* work_host = nullptr;  // pinned
  int32_t* variant_dev = nullptr;
  int32_t* variant_host = nullptr;  // pinned
  cudaStream_t user_stream = nullptr;
  bool use_user_stream = false;
  // last frame (bs_context_last_info)
  int32_t last_variant = -1;  // host-known variant, -1 = device-selected
  int64_t last_k = 0;
  int last_W = 0, last_H = 0, last_pw = 0, last_ph = 0;
  int64_t last_n = 0;
  float last_bg[3] = {0, 0, 0};
  // per-stage timing (bs_context_enable_timing)
  bs_frame_out last_out{};
  bool timing = false;
  bool last_fused = false;  // last frame used bs_preprocess_bin_count (visible count in n_visible[1])
  // async mode (bs_context_set_async): point_list sized from a capacity, K
  // checked one call later; an overflowed frame is re-rendered then
  bool async_mode = false;
  static constexpr int kDepth = 2;  // frames the host may run ahead of their K check
  cudaEvent_t ev_k[kDepth] = {};
  struct Pending {
    const bs_gaussian3d* g3d = nullptr;
    int64_t n = 0;
    bs_camera cam{};
    int32_t pw = 0, ph = 0, variant = 0;
    float bg[3] = {0, 0, 0};
    bs_frame_out out{};
    int slot = 0;
    // the point_list capacity the frame was sorted into (for a graph replay:
    // the one baked in at capture) — its K is checked against this, not
    // against a capacity grown since
    int64_t cap = 0;
    // host-buffer pipeline (bs_render_frame_host_async): host planes the
    // frame's outputs go to (a re-render copies them again); io = -1 otherwise
    int io = -1;
    void* host_out[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  } pending[kDepth];
  int n_pending = 0, next_slot = 0;
  int64_t reruns = 0;
  int64_t pl_grows = 0;
  // CUDA-graph mode (bs_context_set_graphs): the async frame body captured
  // once per configuration and per K slot, replayed with the camera copied
  // into cam_dev from a pinned ring ahead of each launch
  bool graphs = false;
  uint64_t gen = 0;  // bumped by every (re)allocation: graphs bake pointers in
  struct GKey {
    const void* g3d = nullptr;
    int64_t n = -1;
    int32_t W = 0, H = 0, pw = 0, ph = 0, variant = 0;
    float bg[3] = {0, 0, 0};
    bs_frame_out out{};
    uint64_t gen = ~0ull;
    cudaStream_t st = nullptr;
    bool operator==(const GKey& o) const { return std::memcmp(this, &o, sizeof(GKey)) == 0; }
  } gkey;
  cudaGraphExec_t gexec[2] = {nullptr, nullptr};
  uint64_t gkernels[2] = {0, 0};  // kernel launches recorded in each graph
  int64_t gcap[2] = {0, 0};       // point_list capacity baked into each graph
  cudaStream_t cap_stream = nullptr;
  bs_camera* cam_dev = nullptr;
  bs_camera* cam_ring = nullptr;  // pinned, 4 slots
  int ring_i = 0;
  int64_t graph_launches = 0;
  // host-buffer pipeline: kIo input/output slots; H2D on st_h2d, D2H on
  // st_d2h, compute on the context stream — frame i+1's upload and frame i-1's
  // download overlap frame i's kernels
  static constexpr int kIo = 3;
  cudaStream_t st_h2d = nullptr, st_d2h = nullptr;
  void* io_g3d[kIo] = {nullptr, nullptr, nullptr};
  size_t io_g3d_bytes[kIo] = {0, 0, 0};
  void* io_out[kIo][6] = {};
  int64_t io_pixels = 0;
  cudaEvent_t ev_h2d[kIo] = {}, ev_comp[kIo] = {}, ev_d2h[kIo] = {};
  int io_next = 0;
  // bs_render_views_host (on the batch's first context): the scene's two
  // alternating device buffers, their upload and "all readers done" events
  void* batch_g3d[2] = {nullptr, nullptr};
  size_t batch_g3d_bytes[2] = {0, 0};
  cudaEvent_t ev_batch[2] = {}, ev_batch_done[2] = {};
  int batch_next = 0;
  cudaEvent_t ev_any = nullptr;  // this context's stream position (batch bookkeeping)
  // BS_PIPE_TRACE=1: per-frame H2D / compute / D2H event timeline, printed at sync
  std::vector<std::array<cudaEvent_t, 6>> trace;
  bool pl_calibrated = false;
  cudaEvent_t ev[kStages + 1] = {};
};

namespace {

uint64_t g_alloc_gen = 0;  // (re)allocations anywhere in a context -> graph keys change

int grow(void** p, size_t* cap, size_t need) {
  if (*p && *cap >= need) return BS_OK;
  ++g_alloc_gen;
  if (*p) cudaFree(*p);
  *p = nullptr;
  need = std::max<size_t>(need, 256);
  if (cudaMalloc(p, need) != cudaSuccess) {
    (void)cudaGetLastError();
    *cap = 0;
    return BS_ERR_CUDA;
  }
  *cap = need;
  return BS_OK;
}

template <typename T>
int grow_n(T** p, int64_t* cap, int64_t need, double slack = 1.0) {
  if (*p && *cap >= need) return BS_OK;
  const int64_t n = std::max<int64_t>(int64_t(double(need) * slack), 1);
  size_t bytes = 0;
  void* v = *p;
  size_t c = 0;
  int s = grow(&v, &c, size_t(n) * sizeof(T));
  (void)bytes;
  *p = static_cast<T*>(v);
  *cap = s == BS_OK ? n : 0;
  return s;
}

#define TRY(x)                 \
  do {                         \
    int _s = (x);              \
    if (_s != BS_OK) return _s; \
  } while (0)
// BS_DEBUG=1: name the failing CUDA call on stderr
bool debug_on() {
  static const bool on = [] {
    const char* e = getenv("BS_DEBUG");
    return e && e[0] == '1';
  }();
  return on;
}

#define CUTRY(x)                                                                                    \
  do {                                                                                              \
    const cudaError_t _e = (x);                                                                     \
    if (_e != cudaSuccess) {                                                                        \
      if (debug_on()) fprintf(stderr, "bs: %s failed: %s (%s:%d)\n", #x, cudaGetErrorString(_e),     \
                              __FILE__, __LINE__);                                                  \
      (void)cudaGetLastError();                                                                     \
      return BS_ERR_CUDA;                                                                           \
    }                                                                                               \
  } while (0)

}  // namespace

extern "C" int bs_context_create(bs_context** out, int alpha_mode) {
  if (!out || (alpha_mode != BS_ALPHA_EXACT && alpha_mode != BS_ALPHA_FAST)) return BS_ERR_INVALID_ARGUMENT;
  int32_t sms = 0;
  int s = bs_device_sm_count(&sms);
  if (s != BS_OK) return s;
  bs_context* c = new (std::nothrow) bs_context();
  if (!c) return BS_ERR_INVALID_ARGUMENT;
  c->alpha_mode = alpha_mode;
  c->sm_count = sms;
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMalloc(reinterpret_cast<void**>(&c->n_visible), 256) != cudaSuccess ||
      cudaMalloc(reinterpret_cast<void**>(&c->k_dev), 256) != cudaSuccess ||
      cudaMalloc(reinterpret_cast<void**>(&c->stats_dev), sizeof(bs_tile_histogram) + 256) != cudaSuccess ||
      cudaMalloc(reinterpret_cast<void**>(&c->work_dev), 256) != cudaSuccess ||
      cudaMalloc(reinterpret_cast<void**>(&c->variant_dev), 256) != cudaSuccess ||
      cudaMallocHost(reinterpret_cast<void**>(&c->variant_host), 256) != cudaSuccess ||
      cudaMallocHost(reinterpret_cast<void**>(&c->k_host), 256) != cudaSuccess ||
      cudaMallocHost(reinterpret_cast<void**>(&c->stats_host), sizeof(bs_tile_histogram) + 256) != cudaSuccess ||
      cudaMallocHost(reinterpret_cast<void**>(&c->work_host), 256) != cudaSuccess) {
    (void)cudaGetLastError();
    bs_context_destroy(c);
    return BS_ERR_CUDA;
  }
  // point_list grows through cudaMallocAsync: keep freed pool memory mapped so
  // a regrowth never goes back to the OS mid-run (tens of ms per remap)
  int dev = 0;
  cudaMemPool_t pool = nullptr;
  if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  (void)cudaGetLastError();
  *out = c;
  return BS_OK;
}

extern "C" int bs_context_destroy(bs_context* c) {
  if (!c) return BS_OK;
  if (c->stream) cudaStreamSynchronize(c->stream);
  void* dev[] = {c->g3d, c->splat[0], c->splat[1], c->splat[2], c->n_visible, c->k_dev, c->pre_ws, c->bin_ws,
                 c->point_list, c->ranges, c->stats_ws, c->order, c->stats_dev, c->render_ws, c->planes[0],
                 c->planes[1], c->planes[2], c->planes[3], c->iplanes[0], c->iplanes[1], c->work_dev,
                 c->variant_dev, c->ranges16, c->ranges_t, c->aux_ws};
  for (void* p : dev)
    if (p) cudaFree(p);
  if (c->k_host) cudaFreeHost(c->k_host);
  if (c->stats_host) cudaFreeHost(c->stats_host);
  if (c->work_host) cudaFreeHost(c->work_host);
  if (c->variant_host) cudaFreeHost(c->variant_host);
  for (cudaEvent_t e : c->ev)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : c->ev_k)
    if (e) cudaEventDestroy(e);
  for (cudaGraphExec_t& e : c->gexec)
    if (e) cudaGraphExecDestroy(e);
  for (int i = 0; i < bs_context::kIo; ++i) {
    if (c->io_g3d[i]) cudaFree(c->io_g3d[i]);
    for (void* q : c->io_out[i])
      if (q) cudaFree(q);
    for (cudaEvent_t e : {c->ev_h2d[i], c->ev_comp[i], c->ev_d2h[i]})
      if (e) cudaEventDestroy(e);
  }
  for (int b = 0; b < 2; ++b) {
    if (c->batch_g3d[b]) cudaFree(c->batch_g3d[b]);
    for (cudaEvent_t e : {c->ev_batch[b], c->ev_batch_done[b]})
      if (e) cudaEventDestroy(e);
  }
  if (c->ev_any) cudaEventDestroy(c->ev_any);
  if (c->st_h2d) cudaStreamSynchronize(c->st_h2d), cudaStreamDestroy(c->st_h2d);
  if (c->st_d2h) cudaStreamSynchronize(c->st_d2h), cudaStreamDestroy(c->st_d2h);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  if (c->cam_dev) cudaFree(c->cam_dev);
  if (c->cam_ring) cudaFreeHost(c->cam_ring);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return BS_OK;
}

extern "C" void* bs_context_stream(bs_context* c) {
  if (!c) return nullptr;
  return static_cast<void*>(c->use_user_stream ? c->user_stream : c->stream);
}

extern "C" int bs_context_enable_timing(bs_context* c, int32_t on) {
  if (!c) return BS_ERR_INVALID_ARGUMENT;
  if (on && !c->ev[0])
    for (cudaEvent_t& e : c->ev) CUTRY(cudaEventCreate(&e));
  c->timing = on != 0;
  return BS_OK;
}

extern "C" int bs_context_stage_ms(bs_context* c, float* ms, int32_t n) {
  if (!c || !ms || n < kStages || !c->timing) return BS_ERR_INVALID_ARGUMENT;
  CUTRY(cudaEventSynchronize(c->ev[kStages]));
  for (int i = 0; i < kStages; ++i) CUTRY(cudaEventElapsedTime(&ms[i], c->ev[i], c->ev[i + 1]));
  return BS_OK;
}

namespace {

int grow_pl_async(bs_context* c, int64_t cap, cudaStream_t st);

// The whole forward on device input, stream-ordered on the context stream.
// One host sync (the 8-byte K readback that sizes point_list); variant = -1
// selects on the device (bs_select_variant_device + bs_render_forward_auto),
// so no sync follows it.
int frame_device(bs_context* c, const bs_gaussian3d* g3d_dev, int64_t n, const bs_camera* cam, int32_t pw, int32_t ph,
                 int32_t variant, const float bg[3], bs_frame_out fo_in, cudaStream_t st, bool allow_async,
                 const bs_camera* cam_dev = nullptr, int capture_slot = -1) {
  const bool capturing = capture_slot >= 0;  // recording into a CUDA graph: no allocation, no pending entry
  const int32_t W = cam->width, H = cam->height;
  const int64_t cols = (W + pw - 1) / pw, rows = (H + ph - 1) / ph, T = cols * rows;
  const int64_t P = int64_t(W) * H;
  auto mark = [&](int i) {
    if (c->timing) cudaEventRecord(c->ev[i], st);
  };
  mark(0);
  // P1-P4
  if (n > c->splat_cap) {
    ++g_alloc_gen;
    for (auto& p : c->splat) {
      if (p) cudaFree(p);
      p = nullptr;
    }
    for (auto& p : c->splat) CUTRY(cudaMalloc(reinterpret_cast<void**>(&p), size_t(n) * sizeof(float4)));
    c->splat_cap = n;
  }
  bs_splats sp{reinterpret_cast<float*>(c->splat[0]), reinterpret_cast<float*>(c->splat[1]),
               reinterpret_cast<float*>(c->splat[2])};
  // default: projection fused with the per-splat binning pass
  // (bs_preprocess_bin_count, splats uncompacted); BS_NO_FUSED_PRE=1 runs
  // bs_preprocess (compacting) + bs_bin_count
  static const bool fused = [] {
    const char* e = getenv("BS_NO_FUSED_PRE");
    return !(e && *e == '1');
  }();
  c->last_fused = fused;
  if (!fused) {
    TRY(grow(&c->pre_ws, &c->pre_ws_bytes, bs_preprocess_workspace_bytes(n)));
    if (cam_dev)
      TRY(bs_preprocess_devcam(g3d_dev, n, cam_dev, sp, c->n_visible, c->pre_ws, c->pre_ws_bytes, st));
    else
      TRY(bs_preprocess(g3d_dev, n, cam, sp, c->n_visible, c->pre_ws, c->pre_ws_bytes, st));
  }
  mark(1);
  // super mode (default with the fused pass, power-of-two patches, and a
  // variant the super-list render supports): lists at 2pw x 2ph, the render
  // keeps each tile's members (bs_render_forward_super); BS_NO_SUPER=1 off
  static const bool super_env = [] {
    const char* e = getenv("BS_NO_SUPER");
    return !(e && *e == '1');
  }();
  auto pow2 = [](int v) { return v > 0 && (v & (v - 1)) == 0; };
  // (small frames keep the pw x ph lists: below ~1 Mpixel their scatter is
  // cheap and the longer super-tile walks cost more — C1 measured 10 % slower)
  const bool super = fused && super_env && pow2(pw) && pow2(ph) && 2 * pw <= 65535 && 2 * ph <= 65535 &&
                     int64_t(W) * H >= (int64_t(1) << 20) &&
                     (variant < 0 || variant == BS_FINE_GRAINED_COMBINED || variant == BS_SHARED_MEM_OPT);
  c->last_super = super;
  const int32_t bpw = super ? 2 * pw : pw, bph = super ? 2 * ph : ph;  // the binning grid's patch
  if (super) {
    TRY(grow(&c->aux_ws, &c->aux_ws_bytes, bs_super_aux_bytes(W, H, pw, ph)));
    TRY(grow_n(&c->ranges16, &c->ranges16_cap, 2 * T));
    TRY(grow_n(&c->ranges_t, &c->ranges_t_cap, 2 * T));
  }
  const bool async = allow_async && c->async_mode && bs_bin_async_supported(W, H, bpw, bph);
  // K slots: 0..kDepth-1 for async frames (checked later), kDepth for a
  // synchronous frame (read at once) — a synchronous frame never overwrites
  // the K of an async frame still pending
  const int slot = capturing ? capture_slot : (async ? c->next_slot : bs_context::kDepth);
  // K goes straight to its pinned host slot (mapped memory, written by the
  // count's last kernel): no copy that could queue behind another stream's
  // download on the copy engine
  int64_t* k_out = c->k_host + 1 + slot;
  auto count = [&]() -> int {
    if (super)
      return bs_preprocess_bin_count_super(g3d_dev, n, cam_dev ? nullptr : cam, cam_dev, sp, c->n_visible, W, H, pw,
                                           ph, k_out, c->bin_ws, c->bin_ws_bytes, nullptr, c->aux_ws,
                                           c->aux_ws_bytes, st);  // pw x ph lengths on demand (fill_info)
    if (fused)
      return bs_preprocess_bin_count(g3d_dev, n, cam_dev ? nullptr : cam, cam_dev, sp, c->n_visible, W, H, pw, ph,
                                     k_out, c->bin_ws, c->bin_ws_bytes, st);
    return bs_bin_count(sp, n, c->n_visible, W, H, pw, ph, k_out, c->bin_ws, c->bin_ws_bytes, st);
  };

  // P5 count (workspace keyed on n and the tile grid; k part grown below)
  const int key[4] = {W, H, bpw, bph};
  const bool same_grid = std::equal(key, key + 4, c->bin_key);
  if (!same_grid || n > c->bin_n || !c->bin_ws) {
    c->bin_n = std::max<int64_t>(n, c->bin_n);
    c->bin_k = std::max<int64_t>(c->bin_k, 0);
    std::copy(key, key + 4, c->bin_key);
    TRY(grow(&c->bin_ws, &c->bin_ws_bytes, bs_bin_workspace_bytes(c->bin_n, W, H, bpw, bph, c->bin_k)));
  }
  TRY(count());
  mark(2);

  if (async) {
    // no wait: sort into the current capacity; K is checked kDepth calls later
    if (!c->ev_k[slot]) CUTRY(cudaEventCreateWithFlags(&c->ev_k[slot], cudaEventDisableTiming));
    // in a capture the record must be an external event-record node, or the
    // event is only usable inside the capture (the host waits on it later)
    if (capturing)
      CUTRY(cudaEventRecordWithFlags(c->ev_k[slot], st, cudaEventRecordExternal));
    else
      CUTRY(cudaEventRecord(c->ev_k[slot], st));
    mark(3);
    if (!c->point_list) TRY(grow_pl_async(c, std::max<int64_t>(n, 1) * 64, st));  // 64 tiles / splat to start
    TRY(grow_n(&c->ranges, &c->ranges_cap, 2 * T));
    const int64_t kcap = std::min<int64_t>(c->pl_cap, (int64_t(1) << 30) - 1);
    TRY(bs_bin_sort_async(sp, n, c->n_visible, W, H, bpw, bph, kcap, c->point_list, c->ranges, c->bin_ws,
                          c->bin_ws_bytes, st));
    if (capturing) c->gcap[slot] = kcap;
    if (!capturing) {
    bs_context::Pending& q = c->pending[c->n_pending++];
    q.g3d = g3d_dev;
    q.n = n;
    q.cam = *cam;
    q.pw = pw;
    q.ph = ph;
    q.variant = variant;
    std::copy(bg, bg + 3, q.bg);
    q.out = fo_in;
    q.slot = slot;
    q.cap = kcap;
    q.io = -1;
    c->next_slot = (slot + 1) % bs_context::kDepth;
    }
  } else {
    CUTRY(cudaStreamSynchronize(st));
    const int64_t k = c->k_host[1 + bs_context::kDepth];
    if (k > c->bin_k && bs_bin_workspace_bytes(c->bin_n, W, H, bpw, bph, k) > c->bin_ws_bytes) {
      // the count state lives in the workspace: grow, then count again
      c->bin_k = int64_t(double(k) * 1.25) + 1024;
      void* fresh = nullptr;
      size_t fresh_bytes = 0;
      TRY(grow(&fresh, &fresh_bytes, bs_bin_workspace_bytes(c->bin_n, W, H, bpw, bph, c->bin_k)));
      if (c->bin_ws) cudaFree(c->bin_ws);
      c->bin_ws = fresh;
      c->bin_ws_bytes = fresh_bytes;
      TRY(count());
    }
    mark(3);
    if (k > c->pl_cap) TRY(grow_pl_async(c, int64_t(double(std::max<int64_t>(k, 1)) * 1.25), st));
    TRY(grow_n(&c->ranges, &c->ranges_cap, 2 * T));
    TRY(bs_bin_sort(sp, n, c->n_visible, W, H, bpw, bph, k, c->point_list, c->ranges, c->bin_ws, c->bin_ws_bytes,
                    st));
    c->last_k = k;
  }
  mark(4);

  // P6 + selection
  TRY(grow(&c->stats_ws, &c->stats_ws_bytes, bs_tile_stats_workspace_bytes(int32_t(T))));
  TRY(grow_n(&c->order, &c->order_cap, T));
  // LPT order by the lengths the render walks: in super mode each tile walks
  // its super-tile's list (ordering by the pw x ph lengths measured 2.5 %
  // slower); the pw x ph lengths themselves are computed on demand (fill_info)
  if (super) TRY(bs_super_tile_ranges(c->ranges, W, H, pw, ph, c->ranges_t, st));
  c->lengths16_done = false;
  const uint32_t* tranges = super ? c->ranges_t : c->ranges;
  if (T <= 32768 && variant < 0)  // LPT order + stats + the device selector, one launch
    TRY(bs_tile_order_select(tranges, int32_t(T), c->stats_dev, c->order, W, H, pw, ph, c->sm_count,
                             c->variant_dev, st));
  else if (T <= 32768)  // LPT order at eighth-octave granularity + the selector's inputs, one launch
    TRY(bs_tile_order(tranges, int32_t(T), c->stats_dev, c->order, st));
  else
    TRY(bs_tile_stats(tranges, int32_t(T), c->stats_dev, nullptr, c->order, c->stats_ws, c->stats_ws_bytes, st));
  if (variant < 0 && T > 32768)
    TRY(bs_select_variant_device(c->stats_dev, W, H, pw, ph, c->sm_count, c->variant_dev, st));
  mark(5);

  // R
  bs_frame_out fo = fo_in;
  if (!fo.color) {
    if (P > c->pixel_cap) {
      ++g_alloc_gen;
      for (auto& p : c->planes) {
        if (p) cudaFree(p);
        p = nullptr;
      }
      for (auto& p : c->iplanes) {
        if (p) cudaFree(p);
        p = nullptr;
      }
      CUTRY(cudaMalloc(reinterpret_cast<void**>(&c->planes[0]), size_t(P) * 3 * sizeof(float)));
      for (int i = 1; i < 4; ++i) CUTRY(cudaMalloc(reinterpret_cast<void**>(&c->planes[i]), size_t(P) * sizeof(float)));
      for (auto& p : c->iplanes) CUTRY(cudaMalloc(reinterpret_cast<void**>(&p), size_t(P) * sizeof(int32_t)));
      c->pixel_cap = P;
    }
    fo = bs_frame_out{c->planes[0], c->planes[1], c->planes[2], c->planes[3], c->iplanes[0], c->iplanes[1]};
  }
  TRY(grow(&c->render_ws, &c->render_ws_bytes, bs_render_workspace_bytes(W, H)));
  TRY(bs_render_forward_ctx(variant, c->variant_dev, c->alpha_mode, sp, c->point_list, super ? c->ranges_t : c->ranges,
                            c->order, W, H, pw, ph, bg, fo, super ? 1 : 0, c->fine_ctas, c->render_ws,
                            c->render_ws_bytes, st));
  mark(6);
  c->last_variant = variant;
  c->last_n = n;
  for (int i = 0; i < 3; ++i) c->last_bg[i] = bg[i];
  c->last_W = W;
  c->last_H = H;
  c->last_pw = pw;
  c->last_ph = ph;
  c->last_out = fo;
  return BS_OK;
}

// point_list growth without a device-wide sync: stream-ordered free of the
// old buffer (after every frame already enqueued on st) and allocation of the
// new one (cudaFreeAsync / cudaMallocAsync on the default pool).
int grow_pl_async(bs_context* c, int64_t cap, cudaStream_t st) {
  if (cap <= c->pl_cap) return BS_OK;
  ++c->pl_grows;
  ++g_alloc_gen;
  if (c->point_list) CUTRY(cudaFreeAsync(c->point_list, st));
  c->point_list = nullptr;
  c->pl_cap = 0;
  void* p = nullptr;
  CUTRY(cudaMallocAsync(&p, size_t(cap) * sizeof(uint32_t), st));
  c->point_list = static_cast<uint32_t*>(p);
  c->pl_cap = cap;
  return BS_OK;
}

// Async mode: wait for the oldest pending frame's K (its binning, not its
// render).  If it overflowed the point_list capacity: grow it and render that
// frame and every newer pending one again, in order, synchronously (same
// inputs; stream order puts them after the first tries, so shared outputs end
// with the newest frame).  keep = pending frames that may stay unchecked.
int download_planes(bs_context* c, const bs_context::Pending& p, cudaStream_t st) {
  const size_t P = size_t(p.cam.width) * size_t(p.cam.height);
  const size_t bytes[6] = {P * 12, P * 4, P * 4, P * 4, P * 4, P * 4};
  for (int k = 0; k < 6; ++k)
    if (p.host_out[k]) CUTRY(cudaMemcpyAsync(p.host_out[k], c->io_out[p.io][k], bytes[k], cudaMemcpyDeviceToHost, st));
  return BS_OK;
}

int verify_pending(bs_context* c, cudaStream_t st, int keep = 0) {
  while (c->n_pending > keep) {
    const bs_context::Pending p0 = c->pending[0];
    CUTRY(cudaEventSynchronize(c->ev_k[p0.slot]));
    const int64_t k = c->k_host[1 + p0.slot];
    c->last_k = k;
    if (k <= p0.cap) {  // (p0.cap <= pl_cap: the capacity only grows)
      // keep >= 50 % headroom over every K seen, growing to 3x: a regrowth
      // maps new memory (a multi-ms stall), so it must be rare — HBM is not
      // (the first checked frame calibrates the capacity to 3x its K at once)
      if (!c->pl_calibrated || double(k) * 1.5 > double(c->pl_cap))
        TRY(grow_pl_async(c, int64_t(double(k) * 3.0) + 1024, st));
      c->pl_calibrated = true;
      for (int i = 1; i < c->n_pending; ++i) c->pending[i - 1] = c->pending[i];
      --c->n_pending;
      continue;
    }
    bs_context::Pending redo[bs_context::kDepth];
    const int nr = c->n_pending;
    std::copy(c->pending, c->pending + nr, redo);
    c->n_pending = 0;
    TRY(grow_pl_async(c, int64_t(double(k) * 3.0) + 1024, st));
    c->pl_calibrated = true;
    for (int i = 0; i < nr; ++i) {
      ++c->reruns;
      const bs_context::Pending& p = redo[i];
      TRY(frame_device(c, p.g3d, p.n, &p.cam, p.pw, p.ph, p.variant, p.bg, p.out, st, false));
      if (p.io >= 0) {  // host pipeline: the first download carried the overflowed frame
        CUTRY(cudaStreamSynchronize(c->st_d2h));
        TRY(download_planes(c, p, st));
        CUTRY(cudaStreamSynchronize(st));
      }
    }
  }
  return BS_OK;
}

int fill_info(bs_context* c, cudaStream_t st, bs_frame_info* info) {
  TRY(verify_pending(c, st));
  if (!c->last_out.term) return BS_ERR_INVALID_ARGUMENT;
  if (c->last_super && !c->lengths16_done) {  // the last frame's pw x ph list lengths, from its difference grid
    TRY(bs_super_tile_lengths(c->aux_ws, c->aux_ws_bytes, c->last_W, c->last_H, c->last_pw, c->last_ph, c->ranges16,
                              st));
    c->lengths16_done = true;
  }
  const uint32_t* tranges = c->last_super ? c->ranges16 : c->ranges;  // pw x ph list lengths
  TRY(bs_frame_work(c->last_out.term, c->last_out.contrib, tranges, c->last_W, c->last_H, c->last_pw, c->last_ph,
                    c->work_dev, st));
  // full tile_load_histogram (order statistics too) on request only
  const int32_t T = int32_t(((c->last_W + c->last_pw - 1) / c->last_pw) * ((c->last_H + c->last_ph - 1) / c->last_ph));
  TRY(bs_tile_stats(tranges, T, c->stats_dev, nullptr, nullptr, c->stats_ws, c->stats_ws_bytes, st));
  CUTRY(cudaMemcpyAsync(c->stats_host, c->stats_dev, sizeof(bs_tile_histogram), cudaMemcpyDeviceToHost, st));
  CUTRY(cudaMemcpyAsync(c->work_host, c->work_dev, 2 * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
  if (c->last_variant < 0)
    CUTRY(cudaMemcpyAsync(c->variant_host, c->variant_dev, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  int32_t nv = 0;
  CUTRY(cudaMemcpyAsync(c->variant_host + 1, c->n_visible + (c->last_fused ? 1 : 0), sizeof(int32_t),
                        cudaMemcpyDeviceToHost, st));
  CUTRY(cudaStreamSynchronize(st));
  nv = c->variant_host[1];
  info->variant = c->last_variant < 0 ? c->variant_host[0] : c->last_variant;
  info->n_visible = nv;
  info->k = c->last_super ? int64_t(c->stats_host->total) : c->last_k;  // pw x ph instances (not super-tile ones)
  info->stats = *c->stats_host;
  info->evaluated = c->work_host[0];
  info->committed = c->work_host[1];
  return BS_OK;
}

bs_context::GKey graph_key(const bs_gaussian3d* g3d, int64_t n, const bs_camera* cam, int32_t pw, int32_t ph,
                           int32_t variant, const float bg[3], bs_frame_out out, cudaStream_t st) {
  bs_context::GKey k;
  std::memset(static_cast<void*>(&k), 0, sizeof(k));  // padding too: keys compare bytewise
  k.g3d = g3d;
  k.n = n;
  k.W = cam->width;
  k.H = cam->height;
  k.pw = pw;
  k.ph = ph;
  k.variant = variant;
  std::copy(bg, bg + 3, k.bg);
  k.out = out;
  k.gen = g_alloc_gen;
  k.st = st;
  return k;
}

// Graph mode: the first frame of a configuration runs normally (it sizes
// every buffer); later frames replay a captured graph of the same body (one
// per K slot), the camera copied to cam_dev from a pinned ring slot right
// before the launch (a slot is reused 4 frames later, when its copy has long
// run: at most kDepth frames are unverified).
int frame_graph(bs_context* c, const bs_gaussian3d* g3d, int64_t n, const bs_camera* cam, int32_t pw, int32_t ph,
                int32_t variant, const float bg[3], bs_frame_out out, cudaStream_t st) {
  if (!c->cam_dev) {
    CUTRY(cudaMalloc(reinterpret_cast<void**>(&c->cam_dev), sizeof(bs_camera)));
    CUTRY(cudaMallocHost(reinterpret_cast<void**>(&c->cam_ring), 4 * sizeof(bs_camera)));
    CUTRY(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
    ++g_alloc_gen;
  }
  bs_context::GKey k = graph_key(g3d, n, cam, pw, ph, variant, bg, out, st);
  if (!(k == c->gkey)) {
    for (cudaGraphExec_t& e : c->gexec)
      if (e) {
        cudaGraphExecDestroy(e);
        e = nullptr;
      }
    // a plain frame of the new configuration (allocations happen here)
    TRY(frame_device(c, g3d, n, cam, pw, ph, variant, bg, out, st, true));
    c->gkey = graph_key(g3d, n, cam, pw, ph, variant, bg, out, st);
    return BS_OK;
  }
  const int slot = c->next_slot;
  if (!c->gexec[slot]) {
    cudaGraph_t g = nullptr;
    const uint64_t l0 = bs_kernel_launches();
    CUTRY(cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeRelaxed));
    const int rc = frame_device(c, g3d, n, cam, pw, ph, variant, bg, out, c->cap_stream, true, c->cam_dev, slot);
    c->gkernels[slot] = bs_kernel_launches() - l0;
    const cudaError_t ec = cudaStreamEndCapture(c->cap_stream, &g);
    if (debug_on() && (rc != BS_OK || ec != cudaSuccess))
      fprintf(stderr, "bs: graph capture: body status %d, end capture %s\n", rc, cudaGetErrorString(ec));
    if (rc != BS_OK) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    CUTRY(ec);
    const cudaError_t ei = cudaGraphInstantiate(&c->gexec[slot], g, 0);
    cudaGraphDestroy(g);
    CUTRY(ei);
    if (!(graph_key(g3d, n, cam, pw, ph, variant, bg, out, st) == c->gkey)) return BS_ERR_CUDA;  // allocated in capture
  }
  bs_camera* ring = c->cam_ring + c->ring_i;
  c->ring_i = (c->ring_i + 1) % 4;
  *ring = *cam;
  CUTRY(cudaMemcpyAsync(c->cam_dev, ring, sizeof(bs_camera), cudaMemcpyHostToDevice, st));
  CUTRY(cudaGraphLaunch(c->gexec[slot], st));
  bs::count_launches(c->gkernels[slot]);  // every replay runs the graph's kernels
  ++c->graph_launches;
  bs_context::Pending& q = c->pending[c->n_pending++];
  q.g3d = g3d;
  q.n = n;
  q.cam = *cam;
  q.pw = pw;
  q.ph = ph;
  q.variant = variant;
  std::copy(bg, bg + 3, q.bg);
  q.out = out;
  q.slot = slot;
  q.cap = c->gcap[slot];
  q.io = -1;
  c->next_slot = (slot + 1) % bs_context::kDepth;
  c->last_variant = variant;
  c->lengths16_done = false;  // the replayed frame's pw x ph lengths are not computed yet
  return BS_OK;
}

}  // namespace

extern "C" int bs_render_frame_device(bs_context* c, const bs_gaussian3d* g3d_dev, int64_t n, const bs_camera* cam,
                                      int32_t pw, int32_t ph, int32_t variant, const float bg[3], bs_frame_out out,
                                      bs_frame_info* info) {
  if (!c || !cam || !bg || n < 0 || (n > 0 && !g3d_dev) || pw <= 0 || ph <= 0) return BS_ERR_INVALID_ARGUMENT;
  if (variant < -1 || variant > 4) return BS_ERR_INVALID_ARGUMENT;
  if (cam->width <= 0 || cam->height <= 0) return BS_ERR_INVALID_ARGUMENT;
  const bool own = !out.color && !out.alpha && !out.depth && !out.final_t && !out.contrib && !out.term;
  if (!own && (!out.color || !out.alpha || !out.depth || !out.final_t || !out.contrib || !out.term))
    return BS_ERR_INVALID_ARGUMENT;
  cudaStream_t st = static_cast<cudaStream_t>(bs_context_stream(c));
  TRY(verify_pending(c, st, bs_context::kDepth - 1));
  if (c->graphs && c->async_mode && !c->timing && !info && bs_bin_async_supported(cam->width, cam->height, pw, ph)) {
    TRY(frame_graph(c, g3d_dev, n, cam, pw, ph, variant, bg, out, st));
    return BS_OK;
  }
  TRY(frame_device(c, g3d_dev, n, cam, pw, ph, variant, bg, out, st, true));
  if (info) TRY(fill_info(c, st, info));
  return BS_OK;
}

extern "C" int bs_context_set_graphs(bs_context* c, int32_t on) {
  if (!c) return BS_ERR_INVALID_ARGUMENT;
  c->graphs = on != 0;
  return BS_OK;
}

extern "C" int bs_context_set_fine_occupancy(bs_context* c, int32_t ctas_per_sm) {
  if (!c || ctas_per_sm < 0) return BS_ERR_INVALID_ARGUMENT;
  if (c->fine_ctas != ctas_per_sm) ++g_alloc_gen;  // captured graphs bake the grid size in
  c->fine_ctas = ctas_per_sm;
  return BS_OK;
}

extern "C" int bs_context_graph_launches(bs_context* c, int64_t* launches) {
  if (!c || !launches) return BS_ERR_INVALID_ARGUMENT;
  *launches = c->graph_launches;
  return BS_OK;
}

extern "C" int bs_context_set_async(bs_context* c, int32_t on) {
  if (!c) return BS_ERR_INVALID_ARGUMENT;
  TRY(verify_pending(c, static_cast<cudaStream_t>(bs_context_stream(c))));
  c->async_mode = on != 0;
  return BS_OK;
}

extern "C" int bs_context_sync(bs_context* c, int64_t* reruns) {
  if (!c) return BS_ERR_INVALID_ARGUMENT;
  cudaStream_t st = static_cast<cudaStream_t>(bs_context_stream(c));
  TRY(verify_pending(c, st));
  CUTRY(cudaStreamSynchronize(st));
  if (c->st_h2d) CUTRY(cudaStreamSynchronize(c->st_h2d));
  if (c->st_d2h) CUTRY(cudaStreamSynchronize(c->st_d2h));
  if (!c->trace.empty()) {
    const cudaEvent_t t0 = c->trace[0][0];
    for (size_t i = 0; i < c->trace.size(); ++i) {
      float ms[6];
      for (int k = 0; k < 6; ++k) cudaEventElapsedTime(&ms[k], t0, c->trace[i][k]);
      fprintf(stderr, "frame %zu: h2d %.3f-%.3f  compute %.3f-%.3f  d2h %.3f-%.3f\n", i, ms[0], ms[1], ms[2], ms[3],
              ms[4], ms[5]);
    }
    for (auto& tv : c->trace)
      for (cudaEvent_t e : tv) cudaEventDestroy(e);
    c->trace.clear();
    (void)cudaGetLastError();
  }
  if (reruns) *reruns = c->reruns;
  return BS_OK;
}

extern "C" int bs_context_capacity(bs_context* c, int64_t* point_list_cap, int64_t* grows) {
  if (!c) return BS_ERR_INVALID_ARGUMENT;
  if (point_list_cap) *point_list_cap = c->pl_cap;
  if (grows) *grows = c->pl_grows;
  return BS_OK;
}

// Backward render of the context's last frame: its splats
// (at the input Gaussian index — the fused projection does not compact),
// lists (super-tile or pw x ph, as the frame used), LPT order and output
// planes.  Pending frames are verified first, so an overflowed frame has
// been rendered again and the lists are final.
extern "C" int bs_context_render_backward(bs_context* c, bs_frame_grad_in gin, bs_splat_grads gout) {
  if (!c || !gin.dl_dcolor || !gout.xyab || !gout.cop || !gout.rgbr) return BS_ERR_INVALID_ARGUMENT;
  if (c->last_W <= 0 || !c->last_out.color) return BS_ERR_INVALID_ARGUMENT;  // no frame yet
  if (!c->last_fused) return BS_ERR_UNSUPPORTED;  // compacted splats (BS_NO_FUSED_PRE=1)
  cudaStream_t st = static_cast<cudaStream_t>(bs_context_stream(c));
  TRY(verify_pending(c, st, 0));
  const bs_splats sp{reinterpret_cast<float*>(c->splat[0]), reinterpret_cast<float*>(c->splat[1]),
                     reinterpret_cast<float*>(c->splat[2])};
  return bs_render_backward(c->alpha_mode, sp, c->last_k > 0 ? c->point_list : nullptr,
                            c->last_super ? c->ranges_t : c->ranges, c->order, c->last_W, c->last_H, c->last_pw,
                            c->last_ph, c->last_bg, c->last_out, gin, gout, c->last_super ? 1 : 0, c->render_ws,
                            c->render_ws_bytes, st);
}

extern "C" int bs_context_last_info(bs_context* c, bs_frame_info* info) {
  if (!c || !info) return BS_ERR_INVALID_ARGUMENT;
  return fill_info(c, static_cast<cudaStream_t>(bs_context_stream(c)), info);
}

extern "C" int bs_render_frame_host(bs_context* c, const bs_gaussian3d* g3d, int64_t n, const bs_camera* cam,
                                    int32_t pw, int32_t ph, int32_t variant, const float bg[3], float* color,
                                    float* alpha, float* depth, float* final_t, int32_t* contrib, int32_t* term,
                                    bs_frame_info* info) {
  if (!c || !cam || !bg || n < 0 || (n > 0 && !g3d) || pw <= 0 || ph <= 0) return BS_ERR_INVALID_ARGUMENT;
  if (variant < -1 || variant > 4) return BS_ERR_INVALID_ARGUMENT;
  const int32_t W = cam->width, H = cam->height;
  if (W <= 0 || H <= 0) return BS_ERR_INVALID_ARGUMENT;
  cudaStream_t st = static_cast<cudaStream_t>(bs_context_stream(c));
  const int64_t P = int64_t(W) * H;
  TRY(grow(&c->g3d, &c->g3d_bytes, size_t(std::max<int64_t>(n, 1)) * sizeof(bs_gaussian3d)));
  if (n > 0) CUTRY(cudaMemcpyAsync(c->g3d, g3d, size_t(n) * sizeof(bs_gaussian3d), cudaMemcpyHostToDevice, st));
  TRY(verify_pending(c, st));
  TRY(frame_device(c, static_cast<const bs_gaussian3d*>(c->g3d), n, cam, pw, ph, variant, bg, bs_frame_out{}, st,
                   false));
  // D2H
  const size_t pb = size_t(P) * sizeof(float);
  if (color) CUTRY(cudaMemcpyAsync(color, c->planes[0], pb * 3, cudaMemcpyDeviceToHost, st));
  if (alpha) CUTRY(cudaMemcpyAsync(alpha, c->planes[1], pb, cudaMemcpyDeviceToHost, st));
  if (depth) CUTRY(cudaMemcpyAsync(depth, c->planes[2], pb, cudaMemcpyDeviceToHost, st));
  if (final_t) CUTRY(cudaMemcpyAsync(final_t, c->planes[3], pb, cudaMemcpyDeviceToHost, st));
  if (contrib) CUTRY(cudaMemcpyAsync(contrib, c->iplanes[0], pb, cudaMemcpyDeviceToHost, st));
  if (term) CUTRY(cudaMemcpyAsync(term, c->iplanes[1], pb, cudaMemcpyDeviceToHost, st));
  if (info) TRY(fill_info(c, st, info));
  CUTRY(cudaStreamSynchronize(st));
  return BS_OK;
}

// NULL selects the legacy default stream (what torch's default stream is),
// not the context's own stream — pass bs_context_stream()'s earlier value
// to go back to that one.
extern "C" int bs_context_set_stream(bs_context* c, void* stream) {
  if (!c) return BS_ERR_INVALID_ARGUMENT;
  TRY(verify_pending(c, static_cast<cudaStream_t>(bs_context_stream(c))));
  c->use_user_stream = static_cast<cudaStream_t>(stream) != c->stream;
  c->user_stream = static_cast<cudaStream_t>(stream);
  return BS_OK;
}

// Drops the pending K checks without waiting: for a caller that captured
// bs_render_frame_device into a CUDA graph (the captured call's check has no
// executed event to wait on).  The caller owns capacity safety from then on.
extern "C" int bs_context_drop_pending(bs_context* c) {
  if (!c) return BS_ERR_INVALID_ARGUMENT;
  c->n_pending = 0;
  return BS_OK;
}

// Pipelined host-buffer frames: upload (st_h2d), the async frame body
// (context stream), download (st_d2h), ordered by per-slot events so three
// frames are in flight.  Outputs are final after bs_context_sync.
namespace {
int ensure_io(bs_context* c) {
  if (c->st_h2d) return BS_OK;
  CUTRY(cudaEventCreateWithFlags(&c->ev_any, cudaEventDisableTiming));
  CUTRY(cudaStreamCreateWithFlags(&c->st_h2d, cudaStreamNonBlocking));
  CUTRY(cudaStreamCreateWithFlags(&c->st_d2h, cudaStreamNonBlocking));
  for (int i = 0; i < bs_context::kIo; ++i)
    for (cudaEvent_t* e : {&c->ev_h2d[i], &c->ev_comp[i], &c->ev_d2h[i]})
      CUTRY(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  return BS_OK;
}

// One pipelined frame.  g3d_dev == NULL: upload g3d_host into the I/O slot
// first (on st_h2d); else the scene is already on the device and the frame
// waits for scene_ready (an event on another context's upload stream).
int host_async_frame(bs_context* c, const bs_gaussian3d* g3d_host, const bs_gaussian3d* g3d_dev,
                     cudaEvent_t scene_ready, int64_t n, const bs_camera* cam, int32_t pw, int32_t ph,
                     int32_t variant, const float bg[3], void* const hs[6]) {
  const int32_t W = cam->width, H = cam->height;
  cudaStream_t st = static_cast<cudaStream_t>(bs_context_stream(c));
  TRY(ensure_io(c));
  const int io = c->io_next;
  c->io_next = (io + 1) % bs_context::kIo;
  const int64_t P = int64_t(W) * H;
  if (P > c->io_pixels || !c->io_out[io][0]) {  // (re)size every slot's planes
    CUTRY(cudaDeviceSynchronize());
    for (int i = 0; i < bs_context::kIo; ++i)
      for (int k = 0; k < 6; ++k) {
        if (c->io_out[i][k]) cudaFree(c->io_out[i][k]);
        CUTRY(cudaMalloc(&c->io_out[i][k], size_t(P) * (k == 0 ? 12 : 4)));
      }
    c->io_pixels = P;
    ++g_alloc_gen;
  }
  static const bool tracing = [] {
    const char* e = getenv("BS_PIPE_TRACE");
    return e && e[0] == '1';
  }();
  std::array<cudaEvent_t, 6> tev{};
  if (tracing)
    for (auto& e : tev) cudaEventCreate(&e);
  const bs_gaussian3d* gd = g3d_dev;
  if (!gd) {
    // upload into slot io once the frame that last read it is done
    CUTRY(cudaStreamWaitEvent(c->st_h2d, c->ev_comp[io], 0));
    if (c->io_g3d_bytes[io] < size_t(std::max<int64_t>(n, 1)) * sizeof(bs_gaussian3d)) {
      CUTRY(cudaStreamSynchronize(c->st_h2d));
      TRY(grow(&c->io_g3d[io], &c->io_g3d_bytes[io], size_t(std::max<int64_t>(n, 1)) * sizeof(bs_gaussian3d)));
    }
    if (tracing) cudaEventRecord(tev[0], c->st_h2d);
    if (n > 0)
      CUTRY(cudaMemcpyAsync(c->io_g3d[io], g3d_host, size_t(n) * sizeof(bs_gaussian3d), cudaMemcpyHostToDevice,
                            c->st_h2d));
    if (tracing) cudaEventRecord(tev[1], c->st_h2d);
    CUTRY(cudaEventRecord(c->ev_h2d[io], c->st_h2d));
    CUTRY(cudaStreamWaitEvent(st, c->ev_h2d[io], 0));
    gd = static_cast<const bs_gaussian3d*>(c->io_g3d[io]);
  } else if (scene_ready) {
    CUTRY(cudaStreamWaitEvent(st, scene_ready, 0));
  }
  // compute after the slot's previous download
  CUTRY(cudaStreamWaitEvent(st, c->ev_d2h[io], 0));
  TRY(verify_pending(c, st, bs_context::kDepth - 1));
  const bs_frame_out fo{static_cast<float*>(c->io_out[io][0]), static_cast<float*>(c->io_out[io][1]),
                        static_cast<float*>(c->io_out[io][2]), static_cast<float*>(c->io_out[io][3]),
                        static_cast<int32_t*>(c->io_out[io][4]), static_cast<int32_t*>(c->io_out[io][5])};
  if (tracing) cudaEventRecord(tev[2], st);
  TRY(frame_device(c, gd, n, cam, pw, ph, variant, bg, fo, st, true));
  if (tracing) cudaEventRecord(tev[3], st);
  bs_context::Pending& q = c->pending[c->n_pending - 1];  // the entry frame_device just queued
  q.io = io;
  std::copy(hs, hs + 6, q.host_out);
  CUTRY(cudaEventRecord(c->ev_comp[io], st));
  // download once computed
  CUTRY(cudaStreamWaitEvent(c->st_d2h, c->ev_comp[io], 0));
  if (tracing) cudaEventRecord(tev[4], c->st_d2h);
  TRY(download_planes(c, q, c->st_d2h));
  if (tracing) cudaEventRecord(tev[5], c->st_d2h);
  CUTRY(cudaEventRecord(c->ev_d2h[io], c->st_d2h));
  if (tracing) c->trace.push_back(tev);
  return BS_OK;
}
}  // namespace

extern "C" int bs_render_frame_host_async(bs_context* c, const bs_gaussian3d* g3d, int64_t n, const bs_camera* cam,
                                          int32_t pw, int32_t ph, int32_t variant, const float bg[3], float* color,
                                          float* alpha, float* depth, float* final_t, int32_t* contrib,
                                          int32_t* term) {
  if (!c || !cam || !bg || n < 0 || (n > 0 && !g3d) || pw <= 0 || ph <= 0) return BS_ERR_INVALID_ARGUMENT;
  if (variant < -1 || variant > 4) return BS_ERR_INVALID_ARGUMENT;
  const int32_t W = cam->width, H = cam->height;
  if (W <= 0 || H <= 0) return BS_ERR_INVALID_ARGUMENT;
  if (!c->async_mode || !bs_bin_async_supported(W, H, pw, ph)) {  // no pipeline: the synchronous form
    return bs_render_frame_host(c, g3d, n, cam, pw, ph, variant, bg, color, alpha, depth, final_t, contrib, term,
                                nullptr);
  }
  void* const hs[6] = {color, alpha, depth, final_t, contrib, term};
  return host_async_frame(c, g3d, nullptr, nullptr, n, cam, pw, ph, variant, bg, hs);
}

// A batch of views of ONE scene from host memory: the scene is uploaded
// once (on ctxs[0]'s upload stream, into one of two device buffers that
// alternate between calls), then view i = cams[view_ids[i]] renders on
// ctxs[i % nctx] (its async frame body) and its six planes are downloaded
// into host_out[6 i .. 6 i + 5] (color, alpha, depth, final_t, contrib,
// term; NULL skips a plane).  Outputs are final after bs_context_sync on
// every context.  Requires async mode on every context.
extern "C" int bs_render_views_host(bs_context* const* ctxs, int32_t nctx, const bs_gaussian3d* g3d_host, int64_t n,
                                    const bs_camera* cams, const int32_t* view_ids, int32_t count, int32_t pw,
                                    int32_t ph, int32_t variant, const float bg[3], void* const* host_out) {
  if (!ctxs || nctx <= 0 || !cams || !view_ids || count < 0 || !bg || !host_out || n < 0 || (n > 0 && !g3d_host))
    return BS_ERR_INVALID_ARGUMENT;
  if (pw <= 0 || ph <= 0 || variant < -1 || variant > 4) return BS_ERR_INVALID_ARGUMENT;
  for (int32_t k = 0; k < nctx; ++k)
    if (!ctxs[k] || !ctxs[k]->async_mode) return BS_ERR_INVALID_ARGUMENT;
  if (count == 0) return BS_OK;
  bs_context* c0 = ctxs[0];
  for (int32_t k = 0; k < nctx; ++k) TRY(ensure_io(ctxs[k]));
  if (!c0->ev_batch[0])
    for (auto* e : {&c0->ev_batch[0], &c0->ev_batch[1], &c0->ev_batch_done[0], &c0->ev_batch_done[1]})
      CUTRY(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  // Every earlier frame is verified first (a frame whose K overflowed is
  // rendered again now, reading its batch buffer), then the previous call's
  // buffer is marked free once all its readers — re-renders included — are
  // done.  (The host waits here for the previous call's last counts: one
  // short bubble per batch.)
  for (int32_t k = 0; k < nctx; ++k) TRY(verify_pending(ctxs[k], static_cast<cudaStream_t>(bs_context_stream(ctxs[k]))));
  const int b = c0->batch_next;
  c0->batch_next ^= 1;
  if (c0->batch_g3d[b ^ 1]) {
    for (int32_t k = 0; k < nctx; ++k) {
      CUTRY(cudaEventRecord(ctxs[k]->ev_any, static_cast<cudaStream_t>(bs_context_stream(ctxs[k]))));
      CUTRY(cudaStreamWaitEvent(c0->st_h2d, ctxs[k]->ev_any, 0));
    }
    CUTRY(cudaEventRecord(c0->ev_batch_done[b ^ 1], c0->st_h2d));
  }
  const size_t bytes = size_t(std::max<int64_t>(n, 1)) * sizeof(bs_gaussian3d);
  // the buffer's previous readers (the views of the call before last) are done
  CUTRY(cudaStreamWaitEvent(c0->st_h2d, c0->ev_batch_done[b], 0));
  if (c0->batch_g3d_bytes[b] < bytes) {
    CUTRY(cudaStreamSynchronize(c0->st_h2d));
    TRY(grow(&c0->batch_g3d[b], &c0->batch_g3d_bytes[b], bytes));
  }
  if (n > 0) CUTRY(cudaMemcpyAsync(c0->batch_g3d[b], g3d_host, size_t(n) * sizeof(bs_gaussian3d),
                                   cudaMemcpyHostToDevice, c0->st_h2d));
  CUTRY(cudaEventRecord(c0->ev_batch[b], c0->st_h2d));
  const bs_gaussian3d* gd = static_cast<const bs_gaussian3d*>(c0->batch_g3d[b]);
  for (int32_t i = 0; i < count; ++i) {
    bs_context* c = ctxs[i % nctx];
    const bs_camera& cam = cams[view_ids[i]];
    if (cam.width <= 0 || cam.height <= 0) return BS_ERR_INVALID_ARGUMENT;
    if (!bs_bin_async_supported(cam.width, cam.height, pw, ph)) return BS_ERR_UNSUPPORTED;
    TRY(host_async_frame(c, nullptr, gd, c0->ev_batch[b], n, &cam, pw, ph, variant, bg, host_out + 6 * size_t(i)));
  }
  return BS_OK;
}

// A batch of views across several contexts, round-robin, enqueued from one
// native loop (no per-view interpreter overhead): view i renders
// cams[view_ids[i]] on ctxs[i % nctx] into that context's own planes; with
// flush_bufs, a cudaMemsetAsync of flush_bytes on the context's stream
// precedes each view (an L2 flush when flush_bytes > L2).
extern "C" int bs_render_views(bs_context* const* ctxs, int32_t nctx, const bs_gaussian3d* g3d_dev, int64_t n,
                               const bs_camera* cams, const int32_t* view_ids, int32_t count, int32_t pw, int32_t ph,
                               int32_t variant, const float bg[3], void* const* flush_bufs, size_t flush_bytes) {
  if (!ctxs || nctx <= 0 || !cams || !view_ids || count < 0 || !bg) return BS_ERR_INVALID_ARGUMENT;
  for (int32_t i = 0; i < count; ++i) {
    bs_context* c = ctxs[i % nctx];
    if (!c) return BS_ERR_INVALID_ARGUMENT;
    if (flush_bufs && flush_bufs[i % nctx] && flush_bytes)
      CUTRY(cudaMemsetAsync(flush_bufs[i % nctx], 0, flush_bytes, static_cast<cudaStream_t>(bs_context_stream(c))));
    TRY(bs_render_frame_device(c, g3d_dev, n, &cams[view_ids[i]], pw, ph, variant, bg, bs_frame_out{}, nullptr));
  }
  return BS_OK;
}

// The context-owned output planes (written by frames rendered with an empty
// bs_frame_out, e.g. by bs_render_views); all NULL before the first such frame.
extern "C" int bs_context_frame(bs_context* c, bs_frame_out* out) {
  if (!c || !out) return BS_ERR_INVALID_ARGUMENT;
  *out = bs_frame_out{c->planes[0], c->planes[1], c->planes[2], c->planes[3], c->iplanes[0], c->iplanes[1]};
  return BS_OK;
}

// 1 when the context's last frame used super-tile lists (2pw x 2ph binning,
// bs_render_forward_super), 0 for pw x ph lists.
extern "C" int bs_context_list_mode(bs_context* c, int32_t* super_lists) {
  if (!c || !super_lists) return BS_ERR_INVALID_ARGUMENT;
  *super_lists = c->last_super ? 1 : 0;
  return BS_OK;
}
