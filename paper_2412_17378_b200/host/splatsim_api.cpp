// splatsim_api.cpp — the value-typed reference API (splatsim_b200.hpp) on top
// of the C-ABI.  Host vectors in, host vectors out; all compute on the GPU.
// Device buffers live in a per-thread context and grow on demand.
#include "splatsim_b200.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstring>
#include <fstream>
#include <numeric>
#include <sstream>

#include "splatsim_b200.h"

static_assert(sizeof(splatsim::Gaussian3D) == sizeof(bs_gaussian3d), "Gaussian3D layout");
static_assert(offsetof(splatsim::Gaussian3D, rotation) == offsetof(bs_gaussian3d, rot), "Gaussian3D layout");
static_assert(offsetof(splatsim::Gaussian3D, color) == offsetof(bs_gaussian3d, color), "Gaussian3D layout");
static_assert(sizeof(splatsim::Gaussian2D) == sizeof(bs_gaussian2d), "Gaussian2D layout");
static_assert(offsetof(splatsim::Gaussian2D, depth) == offsetof(bs_gaussian2d, depth), "Gaussian2D layout");

namespace splatsim {
namespace {

[[noreturn]] void raise(const char* where, int status) {
  std::string msg = std::string(where) + ": " + bs_status_string(status);
  if (status == BS_ERR_INVALID_ARGUMENT || status == BS_ERR_GRID_MISMATCH) throw std::invalid_argument(msg);
  if (status == BS_ERR_LOGIC) throw std::logic_error(msg);
  throw std::runtime_error(msg);
}

void ck(const char* where, int status) {
  if (status != BS_OK) raise(where, status);
}

void cu(const char* where, cudaError_t e) {
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    throw std::runtime_error(std::string(where) + ": " + cudaGetErrorString(e));
  }
}

// Growable device buffer.
struct DBuf {
  void* p = nullptr;
  size_t cap = 0;
  void* get(size_t bytes) {
    bytes = std::max<size_t>(bytes, 256);
    if (bytes > cap) {
      if (p) cudaFree(p);
      p = nullptr;
      cu("cudaMalloc", cudaMalloc(&p, bytes));
      cap = bytes;
    }
    return p;
  }
  ~DBuf() {
    if (p) cudaFree(p);
  }
};

struct Ctx {
  cudaStream_t st = nullptr;
  DBuf g3d, xyab, cop, rgbr, nvis, kdev, pre_ws, bin_ws, pl, ranges, stats_ws, order, hist, render_ws, g2d;
  DBuf dl, grads;  // render_backward: dL planes, per-splat gradients
  DBuf planes[6];
  DBuf flush;  // L2 flush buffer for time_kernel_ms (larger than the 126 MB L2)
  Ctx() { cu("cudaStreamCreate", cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking)); }
  ~Ctx() {
    if (st) cudaStreamDestroy(st);
  }
  void sync() { cu("cudaStreamSynchronize", cudaStreamSynchronize(st)); }
  bs_splats splats(int64_t n) {
    const size_t b = size_t(std::max<int64_t>(n, 1)) * 16;
    return bs_splats{static_cast<float*>(xyab.get(b)), static_cast<float*>(cop.get(b)), static_cast<float*>(rgbr.get(b))};
  }
};

Ctx& ctx() {
  thread_local Ctx c;
  return c;
}

AlphaMode g_mode = AlphaMode::Exact;

int grid_cols(int w, int pw) { return (w + pw - 1) / pw; }

bs_camera to_c(const Camera& c) {
  bs_camera o;
  std::memcpy(o.view, c.view_transform.data(), sizeof(o.view));
  o.focal[0] = c.focal[0];
  o.focal[1] = c.focal[1];
  o.width = c.width;
  o.height = c.height;
  return o;
}

// Uploads Gaussian2D to device splats (n entries).
bs_splats upload_g2d(Ctx& c, const std::vector<Gaussian2D>& g) {
  const int64_t n = int64_t(g.size());
  bs_splats s = c.splats(n);
  if (n) {
    void* d = c.g2d.get(size_t(n) * sizeof(bs_gaussian2d));
    cu("H2D g2d", cudaMemcpyAsync(d, g.data(), size_t(n) * sizeof(bs_gaussian2d), cudaMemcpyHostToDevice, c.st));
    ck("bs_splats_from_g2d", bs_splats_from_g2d(static_cast<bs_gaussian2d*>(d), n, s, c.st));
  }
  return s;
}

struct DeviceBinning {
  uint32_t* pl;
  uint32_t* ranges;
};

DeviceBinning upload_binning(Ctx& c, const TileBinning& b) {
  DeviceBinning d;
  d.pl = static_cast<uint32_t*>(c.pl.get(std::max<size_t>(b.point_list.size(), 1) * 4));
  d.ranges = static_cast<uint32_t*>(c.ranges.get(size_t(b.tile_count()) * 8));
  if (!b.point_list.empty())
    cu("H2D pl", cudaMemcpyAsync(d.pl, b.point_list.data(), b.point_list.size() * 4, cudaMemcpyHostToDevice, c.st));
  static_assert(sizeof(std::pair<uint32_t, uint32_t>) == 8, "range pair layout");
  if (b.tile_count() > 0)
    cu("H2D ranges", cudaMemcpyAsync(d.ranges, b.tile_ranges.data(), size_t(b.tile_count()) * 8,
                                     cudaMemcpyHostToDevice, c.st));
  return d;
}

// LPT order + stats for a device binning (order lives in c.order).
void device_stats(Ctx& c, const DeviceBinning& d, int T) {
  void* ws = c.stats_ws.get(bs_tile_stats_workspace_bytes(T));
  ck("bs_tile_stats", bs_tile_stats(d.ranges, T, static_cast<bs_tile_histogram*>(c.hist.get(sizeof(bs_tile_histogram))),
                                    nullptr, static_cast<uint32_t*>(c.order.get(size_t(std::max(T, 1)) * 4)), ws,
                                    bs_tile_stats_workspace_bytes(T), c.st));
}

bs_frame_out device_frame(Ctx& c, int64_t P) {
  const size_t pb = size_t(std::max<int64_t>(P, 1)) * 4;
  return bs_frame_out{static_cast<float*>(c.planes[0].get(pb * 3)), static_cast<float*>(c.planes[1].get(pb)),
                      static_cast<float*>(c.planes[2].get(pb)), static_cast<float*>(c.planes[3].get(pb)),
                      static_cast<int32_t*>(c.planes[4].get(pb)), static_cast<int32_t*>(c.planes[5].get(pb))};
}

int mode_c() { return g_mode == AlphaMode::Exact ? BS_ALPHA_EXACT : BS_ALPHA_FAST; }

void check_grid(const char* who, const TileBinning& b, int w, int h, int pw, int ph) {
  if (grid_cols(w, pw) != b.tile_cols || grid_cols(h, ph) != b.tile_rows)
    throw std::invalid_argument(std::string(who) + ": binning grid does not match image dims");
}

}  // namespace

// ---------------------------------------------------------------------------
std::string_view variant_name(KernelVariant v) { return bs_variant_name(static_cast<int>(v)); }

std::optional<KernelVariant> variant_from_name(std::string_view name) {
  const std::string s(name);
  const int v = bs_variant_from_name(s.c_str());
  if (v < 0) return std::nullopt;
  return static_cast<KernelVariant>(v);
}

Dispatch dispatch_for(KernelVariant v) {
  return (v == KernelVariant::DynamicBlocks || v == KernelVariant::FineGrainedCombined) ? Dispatch::Dynamic
                                                                                        : Dispatch::Static;
}

void set_alpha_mode(AlphaMode m) { g_mode = m; }
AlphaMode alpha_mode() { return g_mode; }

std::vector<Gaussian2D> project_all(const std::vector<Gaussian3D>& gaussians, const Camera& cam) {
  Ctx& c = ctx();
  const int64_t n = int64_t(gaussians.size());
  const bs_camera cc = to_c(cam);
  void* g = c.g3d.get(size_t(std::max<int64_t>(n, 1)) * sizeof(bs_gaussian3d));
  if (n) cu("H2D g3d", cudaMemcpyAsync(g, gaussians.data(), size_t(n) * sizeof(bs_gaussian3d), cudaMemcpyHostToDevice, c.st));
  bs_splats s = c.splats(n);
  const size_t wsb = bs_preprocess_workspace_bytes(n);
  int32_t* nv = static_cast<int32_t*>(c.nvis.get(4));
  ck("project_all", bs_preprocess(static_cast<bs_gaussian3d*>(g), n, &cc, s, nv, c.pre_ws.get(wsb), wsb, c.st));
  int32_t m = 0;
  cu("D2H n_visible", cudaMemcpyAsync(&m, nv, 4, cudaMemcpyDeviceToHost, c.st));
  c.sync();
  std::vector<Gaussian2D> out(size_t(std::max(m, 0)));
  if (m > 0) {
    void* d = c.g2d.get(size_t(m) * sizeof(bs_gaussian2d));
    ck("project_all", bs_splats_to_g2d(s, m, static_cast<bs_gaussian2d*>(d), c.st));
    cu("D2H g2d", cudaMemcpyAsync(out.data(), d, size_t(m) * sizeof(bs_gaussian2d), cudaMemcpyDeviceToHost, c.st));
    c.sync();
  }
  return out;
}

std::optional<Gaussian2D> project_gaussian(const Gaussian3D& g, const Camera& cam) {
  auto v = project_all(std::vector<Gaussian3D>{g}, cam);
  if (v.empty()) return std::nullopt;
  return v[0];
}

TileBinning bin_tiles(const std::vector<Gaussian2D>& gaussians, int width, int height, int patch_width,
                      int patch_height) {
  if (width <= 0 || height <= 0 || patch_width <= 0 || patch_height <= 0)
    throw std::invalid_argument("bin_tiles: dims and patch must be positive");
  Ctx& c = ctx();
  const int64_t n = int64_t(gaussians.size());
  bs_splats s = upload_g2d(c, gaussians);
  int32_t* nv = static_cast<int32_t*>(c.nvis.get(4));
  const int32_t n32 = int32_t(n);
  cu("H2D n", cudaMemcpyAsync(nv, &n32, 4, cudaMemcpyHostToDevice, c.st));
  TileBinning b;
  b.tile_cols = grid_cols(width, patch_width);
  b.tile_rows = grid_cols(height, patch_height);
  const int T = b.tile_count();
  size_t wsb = bs_bin_workspace_bytes(n, width, height, patch_width, patch_height, 0);
  int64_t* kd = static_cast<int64_t*>(c.kdev.get(8));
  ck("bin_tiles", bs_bin_count(s, n, nv, width, height, patch_width, patch_height, kd, c.bin_ws.get(wsb), wsb, c.st));
  int64_t k = 0;
  cu("D2H K", cudaMemcpyAsync(&k, kd, 8, cudaMemcpyDeviceToHost, c.st));
  c.sync();
  const size_t need = bs_bin_workspace_bytes(n, width, height, patch_width, patch_height, k);
  if (need > c.bin_ws.cap) {  // the count state lives in the workspace: regrow + recount
    DBuf fresh;
    fresh.get(need);
    std::swap(fresh.p, c.bin_ws.p);
    std::swap(fresh.cap, c.bin_ws.cap);
    ck("bin_tiles", bs_bin_count(s, n, nv, width, height, patch_width, patch_height, kd, c.bin_ws.p, c.bin_ws.cap, c.st));
  }
  uint32_t* pl = static_cast<uint32_t*>(c.pl.get(size_t(std::max<int64_t>(k, 1)) * 4));
  uint32_t* rg = static_cast<uint32_t*>(c.ranges.get(size_t(T) * 8));
  ck("bin_tiles", bs_bin_sort(s, n, nv, width, height, patch_width, patch_height, k, pl, rg, c.bin_ws.p, c.bin_ws.cap, c.st));
  b.point_list.resize(size_t(k));
  b.tile_ranges.resize(size_t(T));
  if (k) cu("D2H pl", cudaMemcpyAsync(b.point_list.data(), pl, size_t(k) * 4, cudaMemcpyDeviceToHost, c.st));
  if (T) cu("D2H ranges", cudaMemcpyAsync(b.tile_ranges.data(), rg, size_t(T) * 8, cudaMemcpyDeviceToHost, c.st));
  c.sync();
  return b;
}

TileHistogram tile_load_histogram(const TileBinning& binning) {
  Ctx& c = ctx();
  const int T = binning.tile_count();
  TileHistogram h;
  if (T <= 0) return h;
  TileBinning only_ranges;
  only_ranges.tile_cols = binning.tile_cols;
  only_ranges.tile_rows = binning.tile_rows;
  only_ranges.tile_ranges = binning.tile_ranges;
  DeviceBinning d = upload_binning(c, only_ranges);
  const size_t wsb = bs_tile_stats_workspace_bytes(T);
  uint32_t* counts = static_cast<uint32_t*>(c.order.get(size_t(T) * 4));
  auto* hd = static_cast<bs_tile_histogram*>(c.hist.get(sizeof(bs_tile_histogram)));
  ck("tile_load_histogram", bs_tile_stats(d.ranges, T, hd, counts, nullptr, c.stats_ws.get(wsb), wsb, c.st));
  bs_tile_histogram hs;
  h.counts.resize(size_t(T));
  cu("D2H counts", cudaMemcpyAsync(h.counts.data(), counts, size_t(T) * 4, cudaMemcpyDeviceToHost, c.st));
  cu("D2H hist", cudaMemcpyAsync(&hs, hd, sizeof(hs), cudaMemcpyDeviceToHost, c.st));
  c.sync();
  h.min = hs.min;
  h.max = hs.max;
  h.mean = hs.mean;
  h.p50 = hs.p50;
  h.p99 = hs.p99;
  return h;
}

std::string binning_csv(const TileBinning& binning, const std::string& config_comment) {
  std::ostringstream out;
  out << "# " << config_comment << "\n" << "tile_id,count\n";
  for (int t = 0; t < binning.tile_count(); ++t) out << t << ',' << binning.tile_size(t) << "\n";
  return out.str();
}

namespace {

RenderOutput render_on_device(Ctx& c, KernelVariant v, const TileBinning& b, const std::vector<Gaussian2D>& g,
                              int w, int h, int pw, int ph, const std::array<float, 3>& bg) {
  bs_splats s = upload_g2d(c, g);
  DeviceBinning d = upload_binning(c, b);
  device_stats(c, d, b.tile_count());
  const int64_t P = int64_t(w) * h;
  bs_frame_out fo = device_frame(c, P);
  const size_t rwb = bs_render_workspace_bytes(w, h);
  void* rws = c.render_ws.get(rwb);
  ck("run_kernel", bs_render_forward(static_cast<int>(v), mode_c(), s, d.pl, d.ranges,
                                     static_cast<uint32_t*>(c.order.p), w, h, pw, ph, bg.data(), fo, rws,
                                     rwb, c.st));
  RenderOutput o;
  o.width = w;
  o.height = h;
  o.color.resize(size_t(P) * 3);
  o.alpha.resize(size_t(P));
  o.depth.resize(size_t(P));
  o.final_t.resize(size_t(P));
  o.contrib.resize(size_t(P));
  o.term.resize(size_t(P));
  const size_t pb = size_t(P) * 4;
  cu("D2H", cudaMemcpyAsync(o.color.data(), fo.color, pb * 3, cudaMemcpyDeviceToHost, c.st));
  cu("D2H", cudaMemcpyAsync(o.alpha.data(), fo.alpha, pb, cudaMemcpyDeviceToHost, c.st));
  cu("D2H", cudaMemcpyAsync(o.depth.data(), fo.depth, pb, cudaMemcpyDeviceToHost, c.st));
  cu("D2H", cudaMemcpyAsync(o.final_t.data(), fo.final_t, pb, cudaMemcpyDeviceToHost, c.st));
  cu("D2H", cudaMemcpyAsync(o.contrib.data(), fo.contrib, pb, cudaMemcpyDeviceToHost, c.st));
  cu("D2H", cudaMemcpyAsync(o.term.data(), fo.term, pb, cudaMemcpyDeviceToHost, c.st));
  c.sync();
  return o;
}

}  // namespace

RenderOutput render_reference(const TileBinning& binning, const std::vector<Gaussian2D>& gaussians, int width,
                              int height, int patch_width, int patch_height, const std::array<float, 3>& background) {
  check_grid("render_reference", binning, width, height, patch_width, patch_height);
  return render_on_device(ctx(), KernelVariant::Naive, binning, gaussians, width, height, patch_width, patch_height,
                          background);
}

KernelRun run_kernel(KernelVariant variant, const TileBinning& binning, const std::vector<Gaussian2D>& gaussians,
                     int width, int height, int patch_width, int patch_height,
                     const std::array<float, 3>& background) {
  check_grid("run_kernel", binning, width, height, patch_width, patch_height);
  KernelRun run;
  run.output = render_on_device(ctx(), variant, binning, gaussians, width, height, patch_width, patch_height,
                                background);
  // per-tile work (src/kernels.cpp:283-298): consumed = term > 0 ? term : list_len, -1 outside the image
  const int cap = patch_width * patch_height;
  std::vector<TileWork> tiles(size_t(binning.tile_count()));
  for (int t = 0; t < binning.tile_count(); ++t) {
    TileWork& tw = tiles[size_t(t)];
    tw.list_len = binning.tile_size(t);
    tw.consumed.assign(size_t(cap), -1);
    const int ox = (t % binning.tile_cols) * patch_width, oy = (t / binning.tile_cols) * patch_height;
    for (int s = 0; s < cap; ++s) {
      const int px = ox + s % patch_width, py = oy + s / patch_width;
      if (px >= width || py >= height) continue;
      const int32_t tm = run.output.term[size_t(py) * width + px];
      tw.consumed[size_t(s)] = tm > 0 ? tm : tw.list_len;
    }
  }
  run.trace = trace_from_work(variant, tiles);
  return run;
}

std::vector<SplatGrad> render_backward(const TileBinning& binning, const std::vector<Gaussian2D>& gaussians,
                                       int width, int height, int patch_width, int patch_height,
                                       const std::array<float, 3>& background, const RenderOutput& forward,
                                       const std::vector<float>& dl_dcolor, const std::vector<float>& dl_dalpha,
                                       const std::vector<float>& dl_ddepth) {
  check_grid("render_backward", binning, width, height, patch_width, patch_height);
  const size_t P = size_t(width) * size_t(height);
  if (forward.width != width || forward.height != height || forward.color.size() != 3 * P ||
      forward.depth.size() != P || forward.final_t.size() != P)
    throw std::invalid_argument("render_backward: forward output does not match image dims");
  if (dl_dcolor.size() != 3 * P || (!dl_dalpha.empty() && dl_dalpha.size() != P) ||
      (!dl_ddepth.empty() && dl_ddepth.size() != P))
    throw std::invalid_argument("render_backward: gradient planes do not match image dims");
  Ctx& c = ctx();
  bs_splats s = upload_g2d(c, gaussians);
  DeviceBinning d = upload_binning(c, binning);
  bs_frame_out fo = device_frame(c, int64_t(P));
  cu("H2D fwd", cudaMemcpyAsync(fo.color, forward.color.data(), P * 12, cudaMemcpyHostToDevice, c.st));
  cu("H2D fwd", cudaMemcpyAsync(fo.depth, forward.depth.data(), P * 4, cudaMemcpyHostToDevice, c.st));
  cu("H2D fwd", cudaMemcpyAsync(fo.final_t, forward.final_t.data(), P * 4, cudaMemcpyHostToDevice, c.st));
  // dL planes (colour, alpha, depth) and the zeroed gradients, one buffer each
  float* dl = static_cast<float*>(c.dl.get(P * 20));
  cu("H2D dl", cudaMemcpyAsync(dl, dl_dcolor.data(), P * 12, cudaMemcpyHostToDevice, c.st));
  if (!dl_dalpha.empty())
    cu("H2D dl", cudaMemcpyAsync(dl + 3 * P, dl_dalpha.data(), P * 4, cudaMemcpyHostToDevice, c.st));
  if (!dl_ddepth.empty())
    cu("H2D dl", cudaMemcpyAsync(dl + 4 * P, dl_ddepth.data(), P * 4, cudaMemcpyHostToDevice, c.st));
  const size_t n = gaussians.size();
  const size_t gb = std::max<size_t>(n, 1) * 48;
  float* g = static_cast<float*>(c.grads.get(gb));
  cu("grads", cudaMemsetAsync(g, 0, gb, c.st));
  const size_t n4 = std::max<size_t>(n, 1) * 4;
  const bs_frame_grad_in gin{dl, dl_dalpha.empty() ? nullptr : dl + 3 * P, dl_ddepth.empty() ? nullptr : dl + 4 * P};
  const bs_splat_grads gout{g, g + n4, g + 2 * n4};
  const size_t rwb = bs_render_workspace_bytes(width, height);
  ck("render_backward", bs_render_backward(mode_c(), s, binning.point_list.empty() ? nullptr : d.pl, d.ranges,
                                           nullptr, width, height, patch_width, patch_height, background.data(), fo,
                                           gin, gout, 0, c.render_ws.get(rwb), rwb, c.st));
  std::vector<float> h(3 * n4);
  cu("D2H grads", cudaMemcpyAsync(h.data(), g, h.size() * 4, cudaMemcpyDeviceToHost, c.st));
  c.sync();
  std::vector<SplatGrad> out(n);
  for (size_t i = 0; i < n; ++i) {
    const float* x = &h[4 * i];
    const float* o = &h[n4 + 4 * i];
    const float* r = &h[2 * n4 + 4 * i];
    out[i].xy = {x[0], x[1]};
    out[i].conic = {x[2], x[3], o[0]};
    out[i].opacity = o[1];
    out[i].color = {r[0], r[1], r[2]};
    out[i].depth = o[3];
  }
  return out;
}

double time_kernel_ms(KernelVariant variant, const TileBinning& binning, const std::vector<Gaussian2D>& gaussians,
                      int width, int height, int patch_width, int patch_height, int repeats) {
  check_grid("time_kernel_ms", binning, width, height, patch_width, patch_height);
  Ctx& c = ctx();
  bs_splats s = upload_g2d(c, gaussians);
  DeviceBinning d = upload_binning(c, binning);
  device_stats(c, d, binning.tile_count());
  bs_frame_out fo = device_frame(c, int64_t(width) * height);
  const size_t rwb = bs_render_workspace_bytes(width, height);
  void* rws = c.render_ws.get(rwb);
  const float bg[3] = {0, 0, 0};
  // every timed launch starts from a flushed L2 (a 256 MiB write, outside
  // the timed interval), like the frames of a real view stream: warm-L2
  // repeats would favour the kernel whose lists happen to stay resident
  constexpr size_t kFlush = size_t(256) << 20;
  void* fl = c.flush.get(kFlush);
  const int reps = std::max(1, repeats);
  std::vector<cudaEvent_t> ev(2 * size_t(reps));
  for (auto& e : ev) cu("event", cudaEventCreate(&e));
  auto launch = [&]() {
    ck("time_kernel_ms", bs_render_forward(static_cast<int>(variant), mode_c(), s, d.pl, d.ranges,
                                           static_cast<uint32_t*>(c.order.p), width, height, patch_width,
                                           patch_height, bg, fo, rws, rwb, c.st));
  };
  launch();  // warm-up (first-launch costs)
  for (int i = 0; i < reps; ++i) {
    cu("flush", cudaMemsetAsync(fl, i & 0xff, kFlush, c.st));
    cu("event", cudaEventRecord(ev[2 * size_t(i)], c.st));
    launch();
    cu("event", cudaEventRecord(ev[2 * size_t(i) + 1], c.st));
  }
  c.sync();
  std::vector<float> ms(size_t(reps), 0.0f);
  for (int i = 0; i < reps; ++i) cu("event", cudaEventElapsedTime(&ms[size_t(i)], ev[2 * size_t(i)], ev[2 * size_t(i) + 1]));
  for (auto& e : ev) cudaEventDestroy(e);
  std::sort(ms.begin(), ms.end());
  return double(ms[size_t(reps) / 2]);  // median
}

// ---------------------------------------------------------------------------
// Work-trace model (src/kernels.cpp:27-38, 159-266): pure host bookkeeping.
std::int64_t warp_steps_pixelwise(const std::vector<std::optional<std::int64_t>>& term_indices, std::int64_t list_len) {
  std::int64_t m = 0;
  for (const auto& t : term_indices) m = std::max(m, t ? *t : list_len);
  return m;
}

std::int64_t warp_steps_gaussianwise(std::optional<std::int64_t> term_index, std::int64_t list_len) {
  return ((term_index ? *term_index : list_len) + kWarpLanes - 1) / kWarpLanes;
}

std::vector<TaskSpec> make_task_specs(KernelVariant variant, int width, int height, int patch_width,
                                      int patch_height) {
  const int cols = grid_cols(width, patch_width), rows = grid_cols(height, patch_height);
  const int slots = patch_width * patch_height;
  const bool fine = variant == KernelVariant::FineGrainedCombined;
  const int per_tile = fine ? (slots + kFinePixelsPerTask - 1) / kFinePixelsPerTask : 1;
  std::vector<TaskSpec> tasks(size_t(cols) * rows * per_tile);
  for (int tile = 0; tile < cols * rows; ++tile) {
    const int ox = (tile % cols) * patch_width, oy = (tile / cols) * patch_height;
    auto place = [&](TaskSpec& task, int warp, int slot) {
      const int px = ox + slot % patch_width, py = oy + slot / patch_width;
      if (px < width && py < height) task.warp_pixels[size_t(warp)].push_back({px, py});
    };
    for (int s = 0; s < per_tile; ++s) {
      TaskSpec& task = tasks[size_t(tile) * per_tile + s];
      task.task_id = tile * per_tile + s;
      task.tile_id = tile;
      if (fine) {
        for (int w = 0; w < kWarpsPerTask; ++w)
          if (s * kFinePixelsPerTask + w < slots) place(task, w, s * kFinePixelsPerTask + w);
      } else {
        for (int slot = 0; slot < slots; ++slot) place(task, (slot / kWarpLanes) % kWarpsPerTask, slot);
      }
    }
  }
  return tasks;
}

WorkTrace trace_from_work(KernelVariant variant, const std::vector<TileWork>& tiles) {
  WorkTrace trace;
  trace.variant = variant;
  const bool pixwise = variant == KernelVariant::Naive || variant == KernelVariant::DynamicBlocks ||
                       variant == KernelVariant::SharedMemOpt;
  const bool fine = variant == KernelVariant::FineGrainedCombined;
  auto groups = [](std::int32_t consumed) { return (std::int64_t(consumed) + kWarpLanes - 1) / kWarpLanes; };
  std::int32_t next_id = 0;
  for (size_t tile = 0; tile < tiles.size(); ++tile) {
    const TileWork& tw = tiles[tile];
    const int slots = int(tw.consumed.size());
    const std::int64_t chunks = (std::int64_t(tw.list_len) + kBlockThreads - 1) / kBlockThreads;
    if (fine) {
      for (int s = 0; s < (slots + kFinePixelsPerTask - 1) / kFinePixelsPerTask; ++s) {
        TaskTrace t;
        t.task_id = next_id++;
        t.tile_id = std::int32_t(tile);
        t.shared_chunks = chunks;
        for (int w = 0; w < kWarpsPerTask; ++w) {
          const int slot = s * kFinePixelsPerTask + w;
          if (slot >= slots || tw.consumed[size_t(slot)] < 0) continue;
          const std::int64_t gcount = groups(tw.consumed[size_t(slot)]);
          t.warps[size_t(w)] = WarpCounts{gcount, gcount, 1, 1};
        }
        trace.tasks.push_back(t);
      }
      continue;
    }
    TaskTrace t;
    t.task_id = next_id++;
    t.tile_id = std::int32_t(tile);
    t.shared_chunks = chunks;
    for (int slot = 0; slot < slots; ++slot) {
      const std::int32_t consumed = tw.consumed[size_t(slot)];
      if (consumed < 0) continue;
      WarpCounts& wc = t.warps[size_t((slot / kWarpLanes) % kWarpsPerTask)];
      if (pixwise) {
        wc.compute_steps = std::max<std::int64_t>(wc.compute_steps, consumed);
        wc.writeback_ops = 1;
      } else {
        const std::int64_t gcount = groups(consumed);
        wc.compute_steps += gcount;
        wc.prefix_groups += gcount;
        wc.reduce_ops += 1;
        wc.writeback_ops += 1;
      }
    }
    trace.tasks.push_back(t);
  }
  return trace;
}

std::string trace_csv(const WorkTrace& trace, const std::string& config_comment) {
  std::ostringstream out;
  out << "# " << config_comment << "\n"
      << "task_id,tile_id,warp_id,compute_steps,chunks,prefix_groups,reduce_ops,writeback_ops\n";
  for (const TaskTrace& t : trace.tasks)
    for (int w = 0; w < kWarpsPerTask; ++w) {
      const WarpCounts& c = t.warps[size_t(w)];
      out << t.task_id << ',' << t.tile_id << ',' << w << ',' << c.compute_steps << ',' << t.shared_chunks << ','
          << c.prefix_groups << ',' << c.reduce_ops << ',' << c.writeback_ops << "\n";
    }
  return out.str();
}

// ---------------------------------------------------------------------------
SelectionState checkpoint(SelectionState state, int iter, double t_balanced_ms, double t_baseline_ms) {
  if (state.switched) throw std::logic_error("checkpoint: selection already switched");
  if (state.check_interval <= 0 || iter % state.check_interval != 0)
    throw std::invalid_argument("checkpoint: iter is not a multiple of the interval");
  state.history.push_back({iter, t_balanced_ms, t_baseline_ms});
  if (t_balanced_ms > t_baseline_ms) {
    state.switched = true;
    state.current = KernelVariant::SharedMemOpt;
  }
  return state;
}

SelectionState checkpoint(SelectionState state, int iter, const TileBinning& binning,
                          const std::vector<Gaussian2D>& gaussians, int width, int height, int patch_width,
                          int patch_height) {
  if (state.switched) throw std::logic_error("checkpoint: selection already switched");
  const double tb = time_kernel_ms(KernelVariant::FineGrainedCombined, binning, gaussians, width, height,
                                   patch_width, patch_height);
  const double ts = time_kernel_ms(KernelVariant::SharedMemOpt, binning, gaussians, width, height, patch_width,
                                   patch_height);
  return checkpoint(std::move(state), iter, tb, ts);
}

KernelVariant select_variant(const TileHistogram& h, int width, int height, int patch_width, int patch_height) {
  bs_tile_histogram s{};
  s.min = h.min;
  s.max = h.max;
  s.p50 = h.p50;
  s.p99 = h.p99;
  s.mean = h.mean;
  s.total = std::accumulate(h.counts.begin(), h.counts.end(), std::uint64_t(0));
  s.tiles = int32_t(h.counts.size());
  int32_t sms = 0;
  if (bs_device_sm_count(&sms) != BS_OK) sms = 148;
  const int v = bs_select_variant(&s, width, height, patch_width, patch_height, sms);
  ck("select_variant", v < 0 ? v : BS_OK);
  return static_cast<KernelVariant>(v);
}

// ---------------------------------------------------------------------------
// Training run on measured times (src/adaptive.cpp:34-129 semantics).
TrainingRunReport run_training(const GeoTrajectoryParams& tp, int check_interval) {
  if (check_interval <= 0) throw std::invalid_argument("run_training: bad check interval");
  if (tp.total_iters <= 0 || tp.keyframes <= 0) throw std::invalid_argument("run_training: bad trajectory");
  TrainingRunReport report;
  report.iterations.reserve(size_t(tp.total_iters));
  SelectionState state;
  state.check_interval = check_interval;
  Camera cam;
  cam.view_transform = {1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1};
  cam.focal = {tp.focal, tp.focal};
  cam.width = tp.width;
  cam.height = tp.height;
  const int kf = std::min(tp.keyframes, tp.total_iters);
  int seg = -1;
  double t_bal = 0.0, t_base = 0.0;
  for (int iter = 0; iter < tp.total_iters; ++iter) {
    const int s = int(int64_t(iter) * kf / tp.total_iters);  // keyframe segment of this iteration
    if (s != seg) {
      seg = s;
      const double x = kf > 1 ? double(s) / double(kf - 1) : 0.0;
      ClusterSceneParams p;
      p.n_gaussians = tp.n_gaussians;
      p.seed = tp.seed;
      p.background_fraction = tp.background_fraction_start * (1 - x) + tp.background_fraction_end * x;
      p.cluster_sigma = tp.cluster_sigma_start * (1 - x) + tp.cluster_sigma_end * x;
      std::vector<Gaussian3D> g = gen_clustered_scene(p, cam);
      const float os = float(tp.opacity_scale_start * (1 - x) + tp.opacity_scale_end * x);
      for (Gaussian3D& q : g) q.opacity *= os;
      const std::vector<Gaussian2D> g2 = project_all(g, cam);
      const TileBinning b = bin_tiles(g2, tp.width, tp.height, tp.patch_width, tp.patch_height);
      t_bal = time_kernel_ms(KernelVariant::FineGrainedCombined, b, g2, tp.width, tp.height, tp.patch_width,
                             tp.patch_height, 5);
      t_base = time_kernel_ms(KernelVariant::SharedMemOpt, b, g2, tp.width, tp.height, tp.patch_width,
                              tp.patch_height, 5);
    }
    report.always_balanced_ms += t_bal;
    report.always_baseline_ms += t_base;
    IterationRecord rec;
    rec.iter = iter;
    if (!state.switched && iter % check_interval == 0) {
      rec.is_checkpoint = true;
      rec.t_balanced = t_bal;
      rec.t_baseline = t_base;
      report.benchmark_overhead_ms += t_bal + t_base;
      state = checkpoint(std::move(state), iter, t_bal, t_base);
      if (state.switched) report.inflection_iter = iter;
    }
    rec.variant = state.current;
    rec.ms = state.current == KernelVariant::FineGrainedCombined ? t_bal : t_base;
    report.adaptive_ms += rec.ms;
    report.iterations.push_back(rec);
  }
  report.adaptive_ms += report.benchmark_overhead_ms;
  return report;
}

SpeedupSummary speedup_summary(const TrainingRunReport& report) {
  SpeedupSummary s;
  double all_chosen = 0.0, post_chosen = 0.0;
  for (const IterationRecord& rec : report.iterations) {
    all_chosen += rec.ms;
    if (report.inflection_iter && rec.iter >= *report.inflection_iter) post_chosen += rec.ms;
  }
  const double all_base = report.always_baseline_ms;
  if (report.inflection_iter) {
    // after the switch the chosen kernel is the baseline
    const double post_base = post_chosen, pre_base = all_base - post_base, pre_chosen = all_chosen - post_chosen;
    if (pre_chosen > 0.0) s.pre_inflection = pre_base / pre_chosen;
    if (post_chosen > 0.0) s.post_inflection = post_base / post_chosen;
  } else if (all_chosen > 0.0) {
    s.pre_inflection = all_base / all_chosen;
  }
  s.overall = all_chosen > 0.0 ? all_base / all_chosen : 1.0;
  return s;
}

std::string report_csv(const TrainingRunReport& report, const std::string& config_comment) {
  std::ostringstream out;
  out.precision(17);
  out << "# " << config_comment << "\n";
  out << "iter,variant,ms,is_checkpoint,t_balanced,t_baseline\n";
  for (const IterationRecord& rec : report.iterations) {
    out << rec.iter << ',' << variant_name(rec.variant) << ',' << rec.ms << ',' << (rec.is_checkpoint ? 1 : 0) << ',';
    if (rec.is_checkpoint)
      out << rec.t_balanced << ',' << rec.t_baseline;
    else
      out << ',';
    out << "\n";
  }
  const SpeedupSummary s = speedup_summary(report);
  out << "# summary inflection_iter="
      << (report.inflection_iter ? std::to_string(*report.inflection_iter) : std::string("none"))
      << " adaptive_ms=" << report.adaptive_ms << " benchmark_overhead_ms=" << report.benchmark_overhead_ms
      << " always_balanced_ms=" << report.always_balanced_ms << " always_baseline_ms=" << report.always_baseline_ms
      << " speedup_pre=" << (s.pre_inflection ? std::to_string(*s.pre_inflection) : std::string("none"))
      << " speedup_post=" << (s.post_inflection ? std::to_string(*s.post_inflection) : std::string("none"))
      << " speedup_overall=" << s.overall << "\n";
  return out.str();
}

// ---------------------------------------------------------------------------
Deviation compare_outputs(const RenderOutput& reference, const RenderOutput& candidate) {
  if (reference.width != candidate.width || reference.height != candidate.height)
    throw std::invalid_argument("compare_outputs: dimension mismatch");
  Deviation d;
  auto scan = [&](const std::vector<float>& a, const std::vector<float>& b) {
    for (size_t i = 0; i < a.size(); ++i) {
      const double e = std::abs(double(a[i]) - double(b[i]));
      d.max_abs = std::max(d.max_abs, e);
      d.max_rel = std::max(d.max_rel, e / std::max(1.0, std::abs(double(a[i]))));
    }
  };
  scan(reference.color, candidate.color);
  scan(reference.alpha, candidate.alpha);
  scan(reference.depth, candidate.depth);
  d.contrib_equal = reference.contrib == candidate.contrib && reference.term == candidate.term;
  return d;
}

void write_ppm(const RenderOutput& r, const std::string& path) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("cannot open for writing: " + path);
  out << "P6\n" << r.width << ' ' << r.height << "\n255\n";
  std::vector<unsigned char> px(r.color.size());
  for (size_t i = 0; i < r.color.size(); ++i)
    px[i] = static_cast<unsigned char>(std::lround(std::clamp(r.color[i], 0.0f, 1.0f) * 255.0f));
  out.write(reinterpret_cast<const char*>(px.data()), std::streamsize(px.size()));
  if (!out) throw std::runtime_error("write failed: " + path);
}

void write_float_grid(const std::vector<float>& grid, int width, int height, const std::string& path) {
  if (grid.size() != size_t(width) * size_t(height)) throw std::invalid_argument("write_float_grid: size mismatch");
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("cannot open for writing: " + path);
  out.write(reinterpret_cast<const char*>(grid.data()), std::streamsize(grid.size() * 4));
  if (!out) throw std::runtime_error("write failed: " + path);
}

std::string render_digest_csv(const RenderOutput& r, const std::string& config_comment) {
  std::ostringstream csv;
  csv.precision(17);
  csv << "# " << config_comment << "\nplane,min,max,mean\n";
  const size_t P = r.pixels();
  auto row = [&](const char* name, size_t stride, size_t off, const std::vector<float>& v) {
    double lo = P ? 1e300 : 0.0, hi = P ? -1e300 : 0.0, sum = 0.0;
    for (size_t i = 0; i < P; ++i) {
      const double x = v[i * stride + off];
      lo = std::min(lo, x);
      hi = std::max(hi, x);
      sum += x;
    }
    csv << name << ',' << lo << ',' << hi << ',' << (P ? sum / double(P) : 0.0) << "\n";
  };
  row("r", 3, 0, r.color);
  row("g", 3, 1, r.color);
  row("b", 3, 2, r.color);
  row("alpha", 1, 0, r.alpha);
  row("depth", 1, 0, r.depth);
  return csv.str();
}

std::vector<Gaussian3D> gen_clustered_scene(const ClusterSceneParams& p, const Camera& cam) {
  if (p.n_gaussians < 0 || p.n_clusters < 1) throw std::invalid_argument("gen_clustered_scene: invalid params");
  std::vector<Gaussian3D> out(size_t(p.n_gaussians));
  const bs_camera cc = to_c(cam);
  ck("gen_clustered_scene",
     bs_host_gen_clustered_scene(p.n_gaussians, p.n_clusters, p.seed, p.cluster_sigma, p.background_fraction, &cc,
                                 reinterpret_cast<bs_gaussian3d*>(out.data())));
  return out;
}

std::uint64_t fnv1a64(const void* data, std::size_t size, std::uint64_t h) {
  const auto* b = static_cast<const unsigned char*>(data);
  for (std::size_t i = 0; i < size; ++i) h = (h ^ b[i]) * 0x100000001b3ull;
  return h;
}

}  // namespace splatsim

extern "C" int bs_host_run_training(const bs_training_params* p, int32_t check_interval, char* csv, size_t csv_cap,
                                    size_t* csv_len) {
  if (!p) return BS_ERR_INVALID_ARGUMENT;
  try {
    splatsim::GeoTrajectoryParams tp;
    tp.total_iters = p->total_iters;
    tp.keyframes = p->keyframes;
    tp.width = p->width;
    tp.height = p->height;
    tp.patch_width = p->patch_width;
    tp.patch_height = p->patch_height;
    tp.focal = p->focal;
    tp.n_gaussians = p->n_gaussians;
    tp.seed = p->seed;
    tp.background_fraction_start = p->background_fraction_start;
    tp.background_fraction_end = p->background_fraction_end;
    tp.cluster_sigma_start = p->cluster_sigma_start;
    tp.cluster_sigma_end = p->cluster_sigma_end;
    tp.opacity_scale_start = p->opacity_scale_start;
    tp.opacity_scale_end = p->opacity_scale_end;
    const std::string out = splatsim::report_csv(splatsim::run_training(tp, check_interval), "bs_host_run_training");
    if (csv_len) *csv_len = out.size();
    if (csv && csv_cap) {
      const size_t n = std::min(out.size(), csv_cap - 1);
      std::memcpy(csv, out.data(), n);
      csv[n] = 0;
    }
    return BS_OK;
  } catch (const std::invalid_argument&) {
    return BS_ERR_INVALID_ARGUMENT;
  } catch (const std::logic_error&) {
    return BS_ERR_LOGIC;
  } catch (...) {
    return BS_ERR_CUDA;
  }
}
