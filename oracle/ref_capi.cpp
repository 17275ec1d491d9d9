// oracle/ref_capi.cpp — extern "C" surface over the REFERENCE ITSELF.
//
// TEST INFRASTRUCTURE ONLY.  Built by `make -C oracle ref` into
// oracle/_ref/libsplatsim_ref.so from the reference's own, unmodified sources
// (/root/reference/proj/core/src/{scene,preprocess,blend,kernels,image_io,
// workload,machine,adaptive}.cpp) compiled against oracle/ref_shim (an
// Eigen-subset shim, see its header) and the nlohmann/json 3.11.3 header that
// ships with the image (the reference's vendor/ dir is not in the mount).
// Loaded only by tests/ (tests/ref_lib.py) and by bench.py's --impl reference
// arm.  Nothing here restates reference logic: every entry point converts the
// POD types the oracle uses to the reference's types and calls the reference
// function named in its comment.  Only the reference symbols' C wrappers are
// exported (-fvisibility=hidden), so this library can share a process with
// the product library's C++ API without symbol clashes.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "splatsim/adaptive.hpp"
#include "splatsim/blend.hpp"
#include "splatsim/image_io.hpp"
#include "splatsim/kernels.hpp"
#include "splatsim/preprocess.hpp"
#include "splatsim/rng.hpp"
#include "splatsim/scene.hpp"
#include "splatsim/workload.hpp"

#define REF_API extern "C" __attribute__((visibility("default")))

namespace {

using namespace splatsim;

// The oracle's POD layouts (oracle/oracle.hpp): rot w,x,y,z; view row-major.
struct PodG3 {
  float mean[3], scale[3], rot[4], opacity, color[3];
};
struct PodCam {
  float view[16];
  float focal[2];
  int32_t width, height;
};
struct PodG2 {
  float x, y, conic_a, conic_b, conic_c, opacity, color[3], depth, radius;
};
static_assert(sizeof(PodG3) == 56 && sizeof(PodG2) == 44 && sizeof(PodCam) == 80);

Camera cam_of(const PodCam& c) {
  Camera k;
  for (int r = 0; r < 4; ++r)
    for (int q = 0; q < 4; ++q) k.view_transform(r, q) = c.view[r * 4 + q];
  k.focal = {c.focal[0], c.focal[1]};
  k.width = c.width;
  k.height = c.height;
  return k;
}
Gaussian3D g3_of(const PodG3& p) {
  Gaussian3D g;
  g.mean = {p.mean[0], p.mean[1], p.mean[2]};
  g.scale = {p.scale[0], p.scale[1], p.scale[2]};
  g.rotation = Eigen::Quaternionf(p.rot[0], p.rot[1], p.rot[2], p.rot[3]);
  g.opacity = p.opacity;
  g.color = {p.color[0], p.color[1], p.color[2]};
  return g;
}
PodG3 pod_of(const Gaussian3D& g) {
  PodG3 p;
  for (int k = 0; k < 3; ++k) {
    p.mean[k] = g.mean[k];
    p.scale[k] = g.scale[k];
    p.color[k] = g.color[k];
  }
  p.rot[0] = g.rotation.w();
  p.rot[1] = g.rotation.x();
  p.rot[2] = g.rotation.y();
  p.rot[3] = g.rotation.z();
  p.opacity = g.opacity;
  return p;
}
Gaussian2D g2_of(const PodG2& p) {
  Gaussian2D g;
  g.xy = {p.x, p.y};
  g.conic_a = p.conic_a;
  g.conic_b = p.conic_b;
  g.conic_c = p.conic_c;
  g.opacity = p.opacity;
  g.color = {p.color[0], p.color[1], p.color[2]};
  g.depth = p.depth;
  g.radius = p.radius;
  return g;
}
PodG2 pod_of(const Gaussian2D& g) {
  return PodG2{g.xy.x(), g.xy.y(), g.conic_a, g.conic_b, g.conic_c, g.opacity,
               {g.color.x(), g.color.y(), g.color.z()}, g.depth, g.radius};
}
std::vector<Gaussian2D> g2_vec(const PodG2* g, int64_t n) {
  std::vector<Gaussian2D> v(size_t(std::max<int64_t>(n, 0)));
  for (int64_t i = 0; i < n; ++i) v[i] = g2_of(g[i]);
  return v;
}
TileBinning binning_of(const uint32_t* ranges, const uint32_t* pl, int64_t K, int W, int H, int pw, int ph) {
  TileBinning b;
  b.tile_cols = (W + pw - 1) / pw;
  b.tile_rows = (H + ph - 1) / ph;
  b.tile_ranges.resize(size_t(b.tile_count()));
  for (int t = 0; t < b.tile_count(); ++t) b.tile_ranges[t] = {ranges[2 * t], ranges[2 * t + 1]};
  if (K > 0) b.point_list.assign(pl, pl + K);
  return b;
}
int copy_str(const std::string& s, char* out, size_t cap) {
  if (out && cap > 0) {
    const size_t n = std::min(cap - 1, s.size());
    std::memcpy(out, s.data(), n);
    out[n] = 0;
  }
  return int(s.size());
}
struct Planes {
  float *color, *alpha, *depth, *final_t;
  int32_t *contrib, *term;
};
// copies the pixels of tile t of o into the output planes
void copy_tile(const RenderOutput& o, int t, int cols, int pw, int ph, const Planes& P) {
  const int tx = t % cols, ty = t / cols;
  const int x0 = tx * pw, y0 = ty * ph, x1 = std::min(o.width, x0 + pw), y1 = std::min(o.height, y0 + ph);
  for (int y = y0; y < y1; ++y)
    for (int x = x0; x < x1; ++x) {
      const size_t p = size_t(y) * size_t(o.width) + size_t(x);
      for (int c = 0; c < 3; ++c) P.color[3 * p + c] = o.color[3 * p + c];
      P.alpha[p] = o.alpha[p];
      P.depth[p] = o.depth[p];
      P.final_t[p] = o.final_t[p];
      P.contrib[p] = o.contrib[p];
      P.term[p] = o.term[p];
    }
}

}  // namespace

REF_API int ref_abi_version() { return 1; }

// src/workload.cpp:198-246 gen_clustered_scene
REF_API int ref_gen_clustered_scene(int n, int n_clusters, uint64_t seed, double sigma, double bgfrac,
                                    const PodCam* cam, PodG3* out) {
  ClusterSceneParams p;
  p.n_gaussians = n;
  p.n_clusters = n_clusters;
  p.seed = seed;
  p.cluster_sigma = sigma;
  p.background_fraction = bgfrac;
  try {
    const auto v = gen_clustered_scene(p, cam_of(*cam));
    for (size_t i = 0; i < v.size(); ++i) out[i] = pod_of(v[i]);
  } catch (...) {
    return -1;
  }
  return 0;
}

// src/scene.cpp:67-71 covariance_of (row-major 3x3 out)
REF_API void ref_covariance_of(const PodG3* g, float out[9]) {
  const Eigen::Matrix3f s = covariance_of(g3_of(*g));
  for (int i = 0; i < 9; ++i) out[i] = s(i / 3, i % 3);
}

// src/preprocess.cpp:10-15 project_covariance (row-major in/out)
REF_API void ref_project_covariance(const double jac[6], const double R[9], const double S[9], double out[4]) {
  Eigen::Matrix<double, 2, 3> j;
  Eigen::Matrix3d r, s;
  for (int i = 0; i < 6; ++i) j(i / 3, i % 3) = jac[i];
  for (int i = 0; i < 9; ++i) {
    r(i / 3, i % 3) = R[i];
    s(i / 3, i % 3) = S[i];
  }
  const Eigen::Matrix2d o = project_covariance(j, r, s);
  out[0] = o(0, 0);
  out[1] = o(0, 1);
  out[2] = o(1, 0);
  out[3] = o(1, 1);
}

// src/preprocess.cpp:17-55 project_gaussian: 1 if visible
REF_API int ref_project_gaussian(const PodG3* g, const PodCam* cam, PodG2* out) {
  const auto p = project_gaussian(g3_of(*g), cam_of(*cam));
  if (!p) return 0;
  *out = pod_of(*p);
  return 1;
}

// src/preprocess.cpp:57-64 project_all on `threads` contiguous chunks (the
// reference is a per-Gaussian map with order-preserving compaction, so the
// concatenation of the chunks' outputs is its output); returns the count
REF_API int64_t ref_project_all(const PodG3* g, int64_t n, const PodCam* cam, PodG2* out, int threads) {
  const Camera c = cam_of(*cam);
  const int nt = std::max(1, std::min<int>(threads, int(std::max<int64_t>(1, n / 4096))));
  std::vector<std::vector<Gaussian2D>> part(static_cast<size_t>(nt));
  std::vector<std::thread> pool;
  for (int t = 0; t < nt; ++t)
    pool.emplace_back([&, t] {
      const int64_t b = n * t / nt, e = n * (t + 1) / nt;
      std::vector<Gaussian3D> in(size_t(e - b));
      for (int64_t i = b; i < e; ++i) in[size_t(i - b)] = g3_of(g[i]);
      part[size_t(t)] = project_all(in, c);
    });
  for (auto& th : pool) th.join();
  int64_t m = 0;
  for (const auto& v : part)
    for (const Gaussian2D& x : v) out[m++] = pod_of(x);
  return m;
}

// src/preprocess.cpp:66-115 bin_tiles; returns K, writes point_list only if
// K <= cap, ranges (2T, [start, end) pairs) always
REF_API int64_t ref_bin_tiles(const PodG2* g, int64_t n, int W, int H, int pw, int ph, uint32_t* point_list,
                              int64_t cap, uint32_t* ranges) {
  const TileBinning b = bin_tiles(g2_vec(g, n), W, H, pw, ph);
  for (int t = 0; t < b.tile_count(); ++t) {
    ranges[2 * t] = b.tile_ranges[t].first;
    ranges[2 * t + 1] = b.tile_ranges[t].second;
  }
  const int64_t K = int64_t(b.point_list.size());
  if (K <= cap && K > 0) std::memcpy(point_list, b.point_list.data(), size_t(K) * 4);
  return K;
}

// src/preprocess.cpp:117-136 tile_load_histogram
REF_API void ref_tile_load_histogram(const uint32_t* ranges, int cols, int rows, uint32_t* counts, uint32_t* mn,
                                     uint32_t* mx, double* mean, uint32_t* p50, uint32_t* p99) {
  TileBinning b;
  b.tile_cols = cols;
  b.tile_rows = rows;
  b.tile_ranges.resize(size_t(cols) * size_t(rows));
  for (size_t t = 0; t < b.tile_ranges.size(); ++t) b.tile_ranges[t] = {ranges[2 * t], ranges[2 * t + 1]};
  const TileHistogram h = tile_load_histogram(b);
  if (!h.counts.empty()) std::memcpy(counts, h.counts.data(), h.counts.size() * 4);
  *mn = h.min;
  *mx = h.max;
  *mean = h.mean;
  *p50 = h.p50;
  *p99 = h.p99;
}

// src/preprocess.cpp:138-147 binning_csv
REF_API int ref_binning_csv(const uint32_t* ranges, int cols, int rows, const char* comment, char* out, size_t cap) {
  TileBinning b;
  b.tile_cols = cols;
  b.tile_rows = rows;
  b.tile_ranges.resize(size_t(cols) * size_t(rows));
  for (size_t t = 0; t < b.tile_ranges.size(); ++t) b.tile_ranges[t] = {ranges[2 * t], ranges[2 * t + 1]};
  return copy_str(binning_csv(b, comment), out, cap);
}

// src/blend.cpp:8-14 eval_alpha
REF_API void ref_eval_alpha(const PodG2* g, float px, float py, float* power, float* alpha) {
  const AlphaEval e = eval_alpha(g2_of(*g), px, py);
  *power = e.power;
  *alpha = e.alpha;
}

// src/blend.cpp:16-42 blend_pixel
REF_API void ref_blend_pixel(const float* alphas, const float* colors, const float* depths, int n, const float bg[3],
                             float* out_color3, float* out_alpha, float* out_depth, float* final_t, int32_t* contrib,
                             int32_t* term) {
  std::vector<BlendStep> s(size_t(std::max(0, n)));
  for (int i = 0; i < n; ++i) {
    s[i].alpha = alphas[i];
    for (int c = 0; c < 3; ++c) s[i].color[c] = colors ? colors[3 * i + c] : 0.0f;
    s[i].depth = depths ? depths[i] : 0.0f;
  }
  const PixelResult r = blend_pixel(s, Eigen::Vector3f(bg[0], bg[1], bg[2]));
  for (int c = 0; c < 3; ++c) out_color3[c] = r.color[c];
  *out_alpha = r.out_alpha;
  *out_depth = r.out_depth;
  *final_t = r.final_t;
  *contrib = r.contrib_count;
  *term = r.term_index.value_or(0);
}

// src/blend.cpp:44-53 termination_index (0 = none)
REF_API int ref_termination_index(const float* alphas, int n) {
  std::vector<BlendStep> s(size_t(std::max(0, n)));
  for (int i = 0; i < n; ++i) s[i].alpha = alphas[i];
  return termination_index(s).value_or(0);
}

// include/splatsim/blend.hpp:69-83 warp_prefix_product<float>
REF_API void ref_warp_prefix_product_f32(const float f[32], float t_in, float out[32], float* t_out) {
  std::array<float, 32> a;
  std::copy(f, f + 32, a.begin());
  const auto p = warp_prefix_product<float>(a, t_in);
  std::copy(p.per_lane.begin(), p.per_lane.end(), out);
  *t_out = p.t_out;
}

// src/kernels.cpp:268-301 run_kernel(variant, ...).  threads > 1: the tiles
// are dealt to threads (longest-processing-time first by pixels x list
// length), each thread calls run_kernel on a TileBinning holding only its
// tiles' lists (the others empty) and its tiles' pixels are copied out —
// tiles are independent in the reference (every pixel reads only its own
// tile's list), so the result equals one run_kernel call.  trace_csv_out
// (optional, threads == 1 only): trace_csv(run.trace, comment).
REF_API int ref_run_kernel(int variant, const uint32_t* ranges, const uint32_t* point_list, int64_t K,
                           const PodG2* g, int64_t n, int W, int H, int pw, int ph, const float bg[3], int threads,
                           float* color, float* alpha, float* depth, float* final_t, int32_t* contrib, int32_t* term,
                           char* trace_csv_out, size_t trace_cap) {
  if (variant < 0 || variant > 4) return -1;
  try {
    const auto gs = g2_vec(g, n);
    const Eigen::Vector3f bgv(bg[0], bg[1], bg[2]);
    const KernelVariant v = static_cast<KernelVariant>(variant);
    const Planes P{color, alpha, depth, final_t, contrib, term};
    const int cols = (W + pw - 1) / pw, rows = (H + ph - 1) / ph, T = cols * rows;
    if (threads <= 1) {
      const KernelRun run = run_kernel(v, binning_of(ranges, point_list, K, W, H, pw, ph), gs, W, H, pw, ph, bgv);
      for (int t = 0; t < T; ++t) copy_tile(run.output, t, cols, pw, ph, P);
      if (trace_csv_out) copy_str(trace_csv(run.trace, "ref"), trace_csv_out, trace_cap);
      return 0;
    }
    // LPT deal of tiles to threads by faithful work (pixels x list length)
    std::vector<int> order(static_cast<size_t>(T));
    std::iota(order.begin(), order.end(), 0);
    auto len = [&](int t) { return int64_t(ranges[2 * t + 1] - ranges[2 * t]); };
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return len(a) > len(b); });
    std::vector<int64_t> load(static_cast<size_t>(threads), 0);
    std::vector<std::vector<int>> mine(static_cast<size_t>(threads));
    for (int t : order) {
      const size_t k = size_t(std::min_element(load.begin(), load.end()) - load.begin());
      mine[k].push_back(t);
      load[k] += len(t) * int64_t(pw) * ph + 1;
    }
    std::vector<std::thread> pool;
    for (int k = 0; k < threads; ++k)
      pool.emplace_back([&, k] {
        TileBinning b;
        b.tile_cols = cols;
        b.tile_rows = rows;
        b.tile_ranges.assign(size_t(T), {0u, 0u});
        for (int t : mine[size_t(k)]) {
          const uint32_t s = uint32_t(b.point_list.size());
          b.point_list.insert(b.point_list.end(), point_list + ranges[2 * t], point_list + ranges[2 * t + 1]);
          b.tile_ranges[size_t(t)] = {s, uint32_t(b.point_list.size())};
        }
        const KernelRun run = run_kernel(v, b, gs, W, H, pw, ph, bgv);
        for (int t : mine[size_t(k)]) copy_tile(run.output, t, cols, pw, ph, P);
      });
    for (auto& th : pool) th.join();
  } catch (...) {
    return -2;
  }
  return 0;
}

// src/kernels.cpp:159-206 make_task_specs: returns the task count; when the
// buffers are given, per task (task_id, tile_id, pixels) and per pixel
// (warp, x, y), tasks in order
REF_API int64_t ref_make_task_specs(int variant, int W, int H, int pw, int ph, int32_t* task_tile,
                                    int32_t* task_npix, int32_t* pix_wxy, int64_t pix_cap) {
  const auto tasks = make_task_specs(static_cast<KernelVariant>(variant), W, H, pw, ph);
  int64_t q = 0;
  for (size_t i = 0; i < tasks.size(); ++i) {
    if (task_tile) task_tile[2 * i] = tasks[i].task_id, task_tile[2 * i + 1] = tasks[i].tile_id;
    if (task_npix) task_npix[i] = int32_t(tasks[i].pixel_count());
    for (int w = 0; w < kWarpsPerTask; ++w)
      for (const auto& p : tasks[i].warp_pixels[w]) {
        if (pix_wxy && q < pix_cap) pix_wxy[3 * q] = w, pix_wxy[3 * q + 1] = p.x(), pix_wxy[3 * q + 2] = p.y();
        ++q;
      }
  }
  return int64_t(tasks.size());
}

// src/kernels.cpp:208-266 trace_from_work + :303-313 trace_csv, on explicit
// TileWork (list_len per tile; consumed[T * cap], -1 = outside the image)
REF_API int ref_trace_csv(int variant, const int32_t* list_len, const int32_t* consumed, int T, int cap,
                          const char* comment, char* out, size_t out_cap) {
  std::vector<TileWork> tiles(static_cast<size_t>(std::max(0, T)));
  for (int t = 0; t < T; ++t) {
    tiles[t].list_len = list_len[t];
    tiles[t].consumed.assign(consumed + int64_t(t) * cap, consumed + int64_t(t + 1) * cap);
  }
  return copy_str(trace_csv(trace_from_work(static_cast<KernelVariant>(variant), tiles), comment), out, out_cap);
}

// src/kernels.cpp:27-38 warp_steps_*
REF_API int64_t ref_warp_steps_pixelwise(const int64_t* terms, int n, int64_t list_len) {
  std::vector<std::optional<int64_t>> t(size_t(std::max(0, n)));
  for (int i = 0; i < n; ++i)
    if (terms[i] > 0) t[i] = terms[i];
  return warp_steps_pixelwise(t, list_len);
}
REF_API int64_t ref_warp_steps_gaussianwise(int64_t term, int64_t list_len) {
  return warp_steps_gaussianwise(term > 0 ? std::optional<int64_t>(term) : std::nullopt, list_len);
}

// src/image_io.cpp: write_ppm (:21-36), write_float_grid (:38-48),
// render_digest_csv (:50-72), compare_outputs (:74-90) on a frame given as planes
namespace {
RenderOutput frame_of(int W, int H, const float* color, const float* alpha, const float* depth,
                      const float* final_t, const int32_t* contrib, const int32_t* term) {
  RenderOutput o;
  o.width = W;
  o.height = H;
  const size_t P = size_t(W) * size_t(H);
  o.color.assign(color, color + 3 * P);
  o.alpha.assign(alpha, alpha + P);
  o.depth.assign(depth, depth + P);
  o.final_t.assign(final_t, final_t + P);
  o.contrib.assign(contrib, contrib + P);
  o.term.assign(term, term + P);
  return o;
}
}  // namespace

REF_API int ref_write_ppm(int W, int H, const float* color, const char* path) {
  std::vector<float> z(size_t(W) * size_t(H), 0.0f);
  std::vector<int32_t> zi(z.size(), 0);
  try {
    write_ppm(frame_of(W, H, color, z.data(), z.data(), z.data(), zi.data(), zi.data()), path);
  } catch (...) {
    return -1;
  }
  return 0;
}
REF_API int ref_write_float_grid(const float* grid, int64_t n, int W, int H, const char* path) {
  try {
    write_float_grid(std::vector<float>(grid, grid + n), W, H, path);
  } catch (...) {
    return -1;
  }
  return 0;
}
REF_API int ref_render_digest_csv(int W, int H, const float* color, const float* alpha, const float* depth,
                                  const float* final_t, const int32_t* contrib, const int32_t* term,
                                  const char* comment, char* out, size_t cap) {
  return copy_str(render_digest_csv(frame_of(W, H, color, alpha, depth, final_t, contrib, term), comment), out, cap);
}
REF_API int ref_compare_outputs(int W, int H, const float* const* a, const int32_t* const* ai, int Wb, int Hb,
                                const float* const* b, const int32_t* const* bi, double* max_abs, double* max_rel,
                                int* contrib_equal) {
  try {
    const Deviation d = compare_outputs(frame_of(W, H, a[0], a[1], a[2], a[3], ai[0], ai[1]),
                                        frame_of(Wb, Hb, b[0], b[1], b[2], b[3], bi[0], bi[1]));
    *max_abs = d.max_abs;
    *max_rel = d.max_rel;
    *contrib_equal = d.contrib_equal ? 1 : 0;
  } catch (...) {
    return -1;  // std::invalid_argument on a dims mismatch
  }
  return 0;
}

// src/scene.cpp:73-166: parse a scene and serialize it again; validation
// errors come back as the SceneError text (return -1)
REF_API int ref_scene_roundtrip(const char* json_text, char* out, size_t cap) {
  try {
    return copy_str(serialize_scene(parse_scene(json_text)), out, cap);
  } catch (const SceneError& e) {
    copy_str(e.what(), out, cap);
    return -1;
  }
}
// serialize_scene of (camera, config, gaussians) given as PODs
REF_API int ref_serialize_scene(const PodCam* cam, int pw, int ph, const float bg[3], uint64_t seed, const PodG3* g,
                                int64_t n, char* out, size_t cap) {
  Scene s;
  s.camera = cam_of(*cam);
  s.config.patch_width = pw;
  s.config.patch_height = ph;
  s.config.background = {bg[0], bg[1], bg[2]};
  s.config.seed = seed;
  for (int64_t i = 0; i < n; ++i) s.gaussians.push_back(g3_of(g[i]));
  return copy_str(serialize_scene(s), out, cap);
}

// include/splatsim/rng.hpp fnv1a64
REF_API uint64_t ref_fnv1a64(const void* data, size_t size, uint64_t h) { return fnv1a64(data, size, h); }
