// oracle/oracle_capi.cpp — extern "C" surface of the CPU oracle for ctypes.
// TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py.  Never by the product.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <thread>
#include <vector>

#include "oracle.hpp"

using namespace oracle;

namespace {

TileBinning make_binning(const uint32_t* ranges, const uint32_t* point_list, int64_t K, int W, int H, int pw,
                         int ph) {
  TileBinning b;
  b.tile_cols = (W + pw - 1) / pw;
  b.tile_rows = (H + ph - 1) / ph;
  b.tile_ranges.assign(ranges, ranges + 2 * size_t(b.tile_count()));
  b.point_list.assign(point_list, point_list + K);
  return b;
}

void copy_out(const RenderOutput& o, float* color, float* alpha, float* depth, float* final_t, int32_t* contrib,
              int32_t* term) {
  const size_t P = size_t(o.width) * size_t(o.height);
  std::memcpy(color, o.color.data(), P * 3 * sizeof(float));
  std::memcpy(alpha, o.alpha.data(), P * sizeof(float));
  std::memcpy(depth, o.depth.data(), P * sizeof(float));
  std::memcpy(final_t, o.final_t.data(), P * sizeof(float));
  std::memcpy(contrib, o.contrib.data(), P * sizeof(int32_t));
  std::memcpy(term, o.term.data(), P * sizeof(int32_t));
}

// Restatement of glibc 2.39 expf (sysdeps/ieee754/flt-32/e_expf.c, the
// ARM optimized-routines algorithm; x86-64 dispatches the FMA build
// __expf_fma).  32-entry 2^(i/32) table + cubic in double.  Used only to pin
// the algorithm/constants that the GPU's exact-alpha path re-implements.
const uint64_t kExp2fTab[32] = {
    0x3ff0000000000000ull, 0x3fefd9b0d3158574ull, 0x3fefb5586cf9890full, 0x3fef9301d0125b51ull,
    0x3fef72b83c7d517bull, 0x3fef54873168b9aaull, 0x3fef387a6e756238ull, 0x3fef1e9df51fdee1ull,
    0x3fef06fe0a31b715ull, 0x3feef1a7373aa9cbull, 0x3feedea64c123422ull, 0x3feece086061892dull,
    0x3feebfdad5362a27ull, 0x3feeb42b569d4f82ull, 0x3feeab07dd485429ull, 0x3feea47eb03a5585ull,
    0x3feea09e667f3bcdull, 0x3fee9f75e8ec5f74ull, 0x3feea11473eb0187ull, 0x3feea589994cce13ull,
    0x3feeace5422aa0dbull, 0x3feeb737b0cdc5e5ull, 0x3feec49182a3f090ull, 0x3feed503b23e255dull,
    0x3feee89f995ad3adull, 0x3feeff76f2fb5e47ull, 0x3fef199bdd85529cull, 0x3fef3720dcef9069ull,
    0x3fef5818dcfba487ull, 0x3fef7c97337b9b5full, 0x3fefa4afa2a490daull, 0x3fefd0765b6e4540ull};

float restated_expf(float x) {
  const double InvLn2N = 0x1.71547652b82fep+0 * 32;
  const double C0 = 0x1.c6af84b912394p-5 / 32 / 32 / 32, C1 = 0x1.ebfce50fac4f3p-3 / 32 / 32,
               C2 = 0x1.62e42ff0c52d6p-1 / 32;
  const double SHIFT = 0x1.8p+52;
  const double xd = x;
  const double z = InvLn2N * xd;
  double kd = z + SHIFT;
  uint64_t ki;
  std::memcpy(&ki, &kd, 8);
  kd -= SHIFT;
  const double r = z - kd;
  uint64_t t = kExp2fTab[ki % 32] + (ki << 47);
  double s;
  std::memcpy(&s, &t, 8);
  const double zz = std::fma(C0, r, C1);
  const double r2 = r * r;
  double y = std::fma(C2, r, 1.0);
  y = std::fma(zz, r2, y);
  y = y * s;
  return float(y);
}

}  // namespace

extern "C" {

int orc_abi_version() { return 1; }

int orc_gen_clustered_scene(int n, int n_clusters, uint64_t seed, double sigma, double bgfrac, const Camera* cam,
                            Gaussian3D* out) {
  ClusterSceneParams p;
  p.n_gaussians = n;
  p.n_clusters = n_clusters;
  p.seed = seed;
  p.cluster_sigma = sigma;
  p.background_fraction = bgfrac;
  try {
    auto v = gen_clustered_scene(p, *cam);
    std::memcpy(out, v.data(), v.size() * sizeof(Gaussian3D));
  } catch (...) {
    return -1;
  }
  return 0;
}

void orc_covariance_of(const Gaussian3D* g, float out[9]) {
  Mat3f s = covariance_of(*g);
  for (int i = 0; i < 9; ++i) out[i] = s.m[i / 3][i % 3];
}

void orc_project_covariance(const double jac[6], const double R[9], const double S[9], double out[4]) {
  double j[2][3] = {{jac[0], jac[1], jac[2]}, {jac[3], jac[4], jac[5]}};
  Mat3d r, s;
  for (int i = 0; i < 9; ++i) {
    r.m[i / 3][i % 3] = R[i];
    s.m[i / 3][i % 3] = S[i];
  }
  double o[2][2];
  project_covariance(j, r, s, o);
  out[0] = o[0][0]; out[1] = o[0][1]; out[2] = o[1][0]; out[3] = o[1][1];
}

int orc_project_gaussian(const Gaussian3D* g, const Camera* cam, Gaussian2D* out) {
  auto p = project_gaussian(*g, *cam);
  if (!p) return 0;
  *out = *p;
  return 1;
}

int64_t orc_project_all(const Gaussian3D* g, int64_t n, const Camera* cam, Gaussian2D* out) {
  int64_t m = 0;
  for (int64_t i = 0; i < n; ++i)
    if (auto p = project_gaussian(g[i], *cam)) out[m++] = *p;
  return m;
}

// Returns K.  point_list is written only when K <= cap; ranges (2*T) always.
int64_t orc_bin_tiles(const Gaussian2D* g, int64_t n, int W, int H, int pw, int ph, uint32_t* point_list, int64_t cap,
                      uint32_t* ranges) {
  TileBinning b = bin_tiles(g, size_t(n), W, H, pw, ph);
  std::memcpy(ranges, b.tile_ranges.data(), b.tile_ranges.size() * sizeof(uint32_t));
  const int64_t K = int64_t(b.point_list.size());
  if (K <= cap && K > 0) std::memcpy(point_list, b.point_list.data(), size_t(K) * sizeof(uint32_t));
  return K;
}

void orc_tile_load_histogram(const uint32_t* ranges, int tile_cols, int tile_rows, uint32_t* counts, uint32_t* mn,
                             uint32_t* mx, double* mean, uint32_t* p50, uint32_t* p99) {
  TileBinning b;
  b.tile_cols = tile_cols;
  b.tile_rows = tile_rows;
  b.tile_ranges.assign(ranges, ranges + 2 * size_t(tile_cols) * size_t(tile_rows));
  TileHistogram h = tile_load_histogram(b);
  if (!h.counts.empty()) std::memcpy(counts, h.counts.data(), h.counts.size() * sizeof(uint32_t));
  *mn = h.min; *mx = h.max; *mean = h.mean; *p50 = h.p50; *p99 = h.p99;
}

void orc_eval_alpha(const Gaussian2D* g, float px, float py, float* power, float* alpha) {
  AlphaEval e = eval_alpha(*g, px, py);
  *power = e.power;
  *alpha = e.alpha;
}

static std::vector<BlendStep> steps_of(const float* alphas, const float* colors, const float* depths, int n) {
  std::vector<BlendStep> s(size_t(std::max(0, n)));
  for (int i = 0; i < n; ++i) {
    s[i].alpha = alphas[i];
    for (int c = 0; c < 3; ++c) s[i].color[c] = colors ? colors[3 * i + c] : 0.0f;
    s[i].depth = depths ? depths[i] : 0.0f;
  }
  return s;
}

void orc_blend_pixel(int gaussianwise, const float* alphas, const float* colors, const float* depths, int n,
                     const float bg[3], float* out_color3, float* out_alpha, float* out_depth, float* final_t,
                     int32_t* contrib, int32_t* term) {
  auto s = steps_of(alphas, colors, depths, n);
  PixelResult r = gaussianwise ? blend_pixel_gaussianwise(s, bg) : blend_pixel(s, bg);
  for (int c = 0; c < 3; ++c) out_color3[c] = r.color[c];
  *out_alpha = r.out_alpha;
  *out_depth = r.out_depth;
  *final_t = r.final_t;
  *contrib = r.contrib_count;
  *term = r.term_index;
}

int orc_termination_index(const float* alphas, int n) { return termination_index(steps_of(alphas, nullptr, nullptr, n)); }

void orc_warp_prefix_product_f32(const float f[32], float t_in, float out[32], float* t_out) {
  std::array<float, 32> a;
  for (int i = 0; i < 32; ++i) a[i] = f[i];
  auto p = warp_prefix_product<float>(a, t_in);
  for (int i = 0; i < 32; ++i) out[i] = p.per_lane[i];
  *t_out = p.t_out;
}

void orc_warp_prefix_product_f64(const double f[32], double t_in, double out[32], double* t_out) {
  std::array<double, 32> a;
  for (int i = 0; i < 32; ++i) a[i] = f[i];
  auto p = warp_prefix_product<double>(a, t_in);
  for (int i = 0; i < 32; ++i) out[i] = p.per_lane[i];
  *t_out = p.t_out;
}

int orc_render(int variant, const uint32_t* ranges, const uint32_t* point_list, int64_t K, const Gaussian2D* g,
               int64_t n, int W, int H, int pw, int ph, const float bg[3], int lazy, int threads, const int32_t* tiles,
               int n_tiles, float* color, float* alpha, float* depth, float* final_t, int32_t* contrib,
               int32_t* term) {
  if (variant < 0 || variant > 4) return -1;
  try {
    TileBinning b = make_binning(ranges, point_list, K, W, H, pw, ph);
    RenderOptions opt;
    opt.lazy = lazy != 0;
    opt.threads = threads <= 0 ? int(std::thread::hardware_concurrency()) : threads;
    opt.tiles = tiles;
    opt.n_tiles = n_tiles;
    RenderOutput o = render(Variant(variant), b, g, size_t(n), W, H, pw, ph, bg, opt);
    copy_out(o, color, alpha, depth, final_t, contrib, term);
  } catch (...) {
    return -2;
  }
  return 0;
}

int64_t orc_warp_steps_pixelwise(const int64_t* terms, int n, int64_t list_len) {
  return warp_steps_pixelwise(std::vector<int64_t>(terms, terms + n), list_len);
}
int64_t orc_warp_steps_gaussianwise(int64_t term, int64_t list_len) { return warp_steps_gaussianwise(term, list_len); }

uint64_t orc_fnv1a64(const void* data, size_t size, uint64_t h) { return fnv1a64(data, size, h); }

float orc_libm_expf(float x) { return std::exp(x); }

// Counts x in [lo, hi] (every float, stepping by bit pattern) where the
// restated algorithm differs from libm expf; reports the first few.
int64_t orc_expf_exhaustive_check(float lo, float hi, float* bad_x, int max_bad) {
  int64_t bad = 0;
  uint32_t ulo, uhi;
  std::memcpy(&ulo, &lo, 4);
  std::memcpy(&uhi, &hi, 4);
  auto check = [&](float x) {
    const float a = std::exp(x), b = restated_expf(x);
    if (std::memcmp(&a, &b, 4) != 0) {
      if (bad < max_bad) bad_x[bad] = x;
      ++bad;
    }
  };
  // walk the negative range [lo, hi] (lo <= hi <= 0); negative float bit
  // patterns grow as the value decreases.
  if (!(lo <= hi && hi <= 0.0f && lo < 0.0f)) return -1;
  const uint32_t ustart = (hi == 0.0f) ? 0x80000000u : uhi;
  // split the bit-pattern range over the host threads; collect per thread
  const unsigned nt = std::max(1u, std::thread::hardware_concurrency());
  const uint64_t span = uint64_t(ulo) - ustart + 1;
  std::vector<std::vector<float>> hits(nt);
  std::vector<int64_t> counts(nt, 0);
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < nt; ++t) {
    pool.emplace_back([&, t]() {
      const uint64_t b = ustart + span * t / nt, e = ustart + span * (t + 1) / nt;
      for (uint64_t u = b; u < e; ++u) {
        float x;
        const uint32_t u32 = uint32_t(u);
        std::memcpy(&x, &u32, 4);
        const float a = std::exp(x), r = restated_expf(x);
        if (std::memcmp(&a, &r, 4) != 0) {
          if (hits[t].size() < size_t(max_bad)) hits[t].push_back(x);
          ++counts[t];
        }
      }
    });
  }
  for (auto& th : pool) th.join();
  for (unsigned t = 0; t < nt; ++t) {
    for (float x : hits[t])
      if (bad < max_bad) bad_x[bad++] = x;
  }
  bad = 0;
  for (int64_t c : counts) bad += c;
  (void)check;
  return bad;
}

// Count of i in [0, n) with y[i] != libm expf(float with bits first_bits + i),
// over all host threads (exhaustive sweeps of the device exp).
int64_t orc_expf_compare_range(uint32_t first_bits, int64_t n, const float* y) {
  const unsigned nt = std::max(1u, std::thread::hardware_concurrency());
  std::vector<int64_t> bad(nt, 0);
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < nt; ++t)
    pool.emplace_back([&, t]() {
      const int64_t b = n * int64_t(t) / int64_t(nt), e = n * int64_t(t + 1) / int64_t(nt);
      for (int64_t i = b; i < e; ++i) {
        const uint32_t u = first_bits + uint32_t(i);
        float x;
        std::memcpy(&x, &u, 4);
        const float a = std::exp(x);
        if (std::memcmp(&a, &y[i], 4) != 0) ++bad[t];
      }
    });
  for (auto& th : pool) th.join();
  int64_t s = 0;
  for (int64_t b : bad) s += b;
  return s;
}

// Count of i with y[i] != libm expf(x[i]) bitwise.
int64_t orc_expf_compare_batch(const float* x, const float* y, int64_t n) {
  int64_t bad = 0;
  for (int64_t i = 0; i < n; ++i) {
    const float a = std::exp(x[i]);
    if (std::memcmp(&a, &y[i], 4) != 0) ++bad;
  }
  return bad;
}

// Backward render: grads = n x 10 doubles (x, y, conic a, b, c, opacity, r,
// g, b, depth), accumulated (caller zeroes).  0 = ok, -1 = grid mismatch.
int orc_render_backward(const uint32_t* ranges, const uint32_t* point_list, int64_t k, const Gaussian2D* g, int64_t n,
                        int W, int H, int pw, int ph, const float bg[3], const float* dl_dcolor, const float* dl_dalpha,
                        const float* dl_ddepth, double* grads) {
  TileBinning b;
  b.tile_cols = (W + pw - 1) / pw;
  b.tile_rows = (H + ph - 1) / ph;
  b.point_list.assign(point_list, point_list + k);
  b.tile_ranges.assign(ranges, ranges + 2 * size_t(b.tile_count()));
  std::vector<SplatGrad> out(static_cast<size_t>(n));
  try {
    render_backward(b, g, size_t(n), W, H, pw, ph, bg, dl_dcolor, dl_dalpha, dl_ddepth, out.data());
  } catch (...) {
    return -1;
  }
  for (int64_t i = 0; i < n; ++i) {
    const SplatGrad& o = out[size_t(i)];
    const double v[10] = {o.xy[0], o.xy[1], o.conic[0], o.conic[1], o.conic[2], o.opacity,
                          o.color[0], o.color[1], o.color[2], o.depth};
    for (int j = 0; j < 10; ++j) grads[10 * i + j] += v[j];
  }
  return 0;
}

}  // extern "C"
