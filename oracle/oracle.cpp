// oracle/oracle.cpp — CPU restatement of the reference forward path.
// TEST INFRASTRUCTURE ONLY (see oracle.hpp header).  Compiled -ffp-contract=off.
#include "oracle.hpp"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <numeric>
#include <stdexcept>
#include <thread>

namespace oracle {

// ---------------------------------------------------------------------------
// Variant names — include/splatsim/kernels.hpp:13-26, src/kernels.cpp:10-25
std::string_view variant_name(Variant v) {
  switch (v) {
    case Variant::Naive: return "Naive";
    case Variant::DynamicBlocks: return "DynamicBlocks";
    case Variant::GaussianWise: return "GaussianWise";
    case Variant::FineGrainedCombined: return "FineGrainedCombined";
    case Variant::SharedMemOpt: return "SharedMemOpt";
  }
  return "?";
}
std::optional<Variant> variant_from_name(std::string_view s) {
  for (int i = 0; i < 5; ++i)
    if (variant_name(Variant(i)) == s) return Variant(i);
  return std::nullopt;
}
// src/kernels.cpp:42-45
bool variant_is_pixelwise(Variant v) {
  return v == Variant::Naive || v == Variant::DynamicBlocks || v == Variant::SharedMemOpt;
}

void RenderOutput::init(int w, int h) {
  width = w;
  height = h;
  const size_t p = size_t(w) * size_t(h);
  color.assign(p * 3, 0.0f);
  alpha.assign(p, 0.0f);
  depth.assign(p, 0.0f);
  final_t.assign(p, 1.0f);
  contrib.assign(p, 0);
  term.assign(p, 0);
}

// ---------------------------------------------------------------------------
// P1 covariance_of — src/scene.cpp:67-71.
//   r = rotation.normalized().toRotationMatrix(); m = r * diag(scale); m * m^T
// normalized(): Eigen stores coeffs (x,y,z,w); squaredNorm of a Packet4f is
// predux((x2,y2,z2,w2)) = (x2+z2)+(y2+w2) (Eigen 3.4 SSE predux); then / sqrt.
// toRotationMatrix(): Eigen Quaternion.h formula.  3x3 float products are not
// vectorisable (3 % 4 != 0): coefficient = a0 + (a1 + a2).
Mat3f covariance_of(const Gaussian3D& g) {
  float qw = g.rot[0], qx = g.rot[1], qy = g.rot[2], qz = g.rot[3];
  const float n2 = (qx * qx + qz * qz) + (qy * qy + qw * qw);
  if (n2 > 0.0f) {
    const float n = std::sqrt(n2);
    qx = qx / n; qy = qy / n; qz = qz / n; qw = qw / n;
  }
  const float tx = 2.0f * qx, ty = 2.0f * qy, tz = 2.0f * qz;
  const float twx = tx * qw, twy = ty * qw, twz = tz * qw;
  const float txx = tx * qx, txy = ty * qx, txz = tz * qx;
  const float tyy = ty * qy, tyz = tz * qy, tzz = tz * qz;
  float r[3][3];
  r[0][0] = 1.0f - (tyy + tzz); r[0][1] = txy - twz;          r[0][2] = txz + twy;
  r[1][0] = txy + twz;          r[1][1] = 1.0f - (txx + tzz); r[1][2] = tyz - twx;
  r[2][0] = txz - twy;          r[2][1] = tyz + twx;          r[2][2] = 1.0f - (txx + tyy);
  float m[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) m[i][j] = r[i][j] * g.scale[j];
  Mat3f s;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) s.m[i][j] = m[i][0] * m[j][0] + (m[i][1] * m[j][1] + m[i][2] * m[j][2]);
  return s;
}

// P2 project_covariance — src/preprocess.cpp:10-15.  t = J*R (2x3 double,
// vectorised: left-to-right); (t*Sigma) evaluated into a temporary, then
// times t^T; every 2-row double product sums left-to-right.
void project_covariance(const double jac[2][3], const Mat3d& R, const Mat3d& S, double out[2][2]) {
  double t[2][3], u[2][3];
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 3; ++j) t[i][j] = (jac[i][0] * R.m[0][j] + jac[i][1] * R.m[1][j]) + jac[i][2] * R.m[2][j];
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 3; ++j) u[i][j] = (t[i][0] * S.m[0][j] + t[i][1] * S.m[1][j]) + t[i][2] * S.m[2][j];
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j) out[i][j] = (u[i][0] * t[j][0] + u[i][1] * t[j][1]) + u[i][2] * t[j][2];
}

// P3 project_gaussian — src/preprocess.cpp:17-55
std::optional<Gaussian2D> project_gaussian(const Gaussian3D& g, const Camera& cam) {
  // rot * mean (3x3 float, scalar redux a0+(a1+a2)) + trans
  const float* V = cam.view;
  float p[3];
  for (int i = 0; i < 3; ++i)
    p[i] = (V[i * 4 + 0] * g.mean[0] + (V[i * 4 + 1] * g.mean[1] + V[i * 4 + 2] * g.mean[2])) + V[i * 4 + 3];
  if (!(p[2] > kNearPlane)) return std::nullopt;

  const double x = p[0], y = p[1], z = p[2];
  const double fx = cam.focal[0], fy = cam.focal[1];
  double jac[2][3] = {{fx / z, 0.0, -fx * x / (z * z)}, {0.0, fy / z, -fy * y / (z * z)}};
  Mat3d R, S;
  const Mat3f sf = covariance_of(g);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      R.m[i][j] = double(V[i * 4 + j]);
      S.m[i][j] = double(sf.m[i][j]);
    }
  double c[2][2];
  project_covariance(jac, R, S, c);

  const double det = c[0][0] * c[1][1] - c[0][1] * c[1][0];
  if (!(det > 0.0) || !std::isfinite(det)) return std::nullopt;
  const double mid = 0.5 * (c[0][0] + c[1][1]);
  const double lambda_max = mid + std::sqrt(std::max(0.0, mid * mid - det));
  if (!(lambda_max > 0.0)) return std::nullopt;

  Gaussian2D out;
  out.x = static_cast<float>(fx * x / z) + 0.5f * float(cam.width);
  out.y = static_cast<float>(fy * y / z) + 0.5f * float(cam.height);
  out.conic_a = static_cast<float>(c[1][1] / det);
  out.conic_b = static_cast<float>(-c[0][1] / det);
  out.conic_c = static_cast<float>(c[0][0] / det);
  out.opacity = g.opacity;
  out.color[0] = g.color[0];
  out.color[1] = g.color[1];
  out.color[2] = g.color[2];
  out.depth = static_cast<float>(z);
  out.radius = static_cast<float>(3.0 * std::sqrt(lambda_max));
  if (!std::isfinite(out.conic_a) || !std::isfinite(out.conic_b) || !std::isfinite(out.conic_c) ||
      !std::isfinite(out.radius))
    return std::nullopt;
  return out;
}

// P4 project_all — src/preprocess.cpp:57-64 (order-preserving compaction)
std::vector<Gaussian2D> project_all(const std::vector<Gaussian3D>& gs, const Camera& cam) {
  std::vector<Gaussian2D> out;
  out.reserve(gs.size());
  for (const Gaussian3D& g : gs)
    if (auto p = project_gaussian(g, cam)) out.push_back(*p);
  return out;
}

// ---------------------------------------------------------------------------
// P5 bin_tiles — src/preprocess.cpp:66-115
TileBinning bin_tiles(const Gaussian2D* gs, size_t n, int width, int height, int pw, int ph) {
  TileBinning b;
  b.tile_cols = (width + pw - 1) / pw;
  b.tile_rows = (height + ph - 1) / ph;
  const int tiles = b.tile_count();
  b.tile_ranges.assign(size_t(tiles) * 2, 0u);
  struct Entry { uint32_t tile; float depth; uint32_t index; };
  std::vector<Entry> entries;
  for (uint32_t i = 0; i < n; ++i) {
    const Gaussian2D& g = gs[i];
    const float r = std::ceil(g.radius);
    const float x0 = g.x - r, x1 = g.x + r;
    const float y0 = g.y - r, y1 = g.y + r;
    if (x1 < 0.0f || y1 < 0.0f || x0 >= float(width) || y0 >= float(height)) continue;
    const int tx0 = std::max(0, int(std::floor(x0 / float(pw))));
    const int tx1 = std::min(b.tile_cols - 1, int(std::floor(x1 / float(pw))));
    const int ty0 = std::max(0, int(std::floor(y0 / float(ph))));
    const int ty1 = std::min(b.tile_rows - 1, int(std::floor(y1 / float(ph))));
    for (int ty = ty0; ty <= ty1; ++ty)
      for (int tx = tx0; tx <= tx1; ++tx) entries.push_back({uint32_t(ty * b.tile_cols + tx), g.depth, i});
  }
  std::sort(entries.begin(), entries.end(), [](const Entry& a, const Entry& c) {
    if (a.tile != c.tile) return a.tile < c.tile;
    if (a.depth != c.depth) return a.depth < c.depth;
    return a.index < c.index;
  });
  b.point_list.resize(entries.size());
  size_t pos = 0;
  for (int t = 0; t < tiles; ++t) {
    const size_t start = pos;
    while (pos < entries.size() && entries[pos].tile == uint32_t(t)) {
      b.point_list[pos] = entries[pos].index;
      ++pos;
    }
    b.tile_ranges[2 * size_t(t)] = uint32_t(start);
    b.tile_ranges[2 * size_t(t) + 1] = uint32_t(pos);
  }
  return b;
}

// P6 tile_load_histogram — src/preprocess.cpp:117-136
TileHistogram tile_load_histogram(const TileBinning& b) {
  TileHistogram h;
  const int T = b.tile_count();
  h.counts.resize(T);
  for (int t = 0; t < T; ++t) h.counts[t] = b.tile_ranges[2 * t + 1] - b.tile_ranges[2 * t];
  if (h.counts.empty()) return h;
  std::vector<uint32_t> s = h.counts;
  std::sort(s.begin(), s.end());
  h.min = s.front();
  h.max = s.back();
  h.mean = std::accumulate(s.begin(), s.end(), 0.0) / double(s.size());
  auto rank = [&](double q) {
    size_t k = size_t(std::ceil(q * double(s.size())));
    return s[std::min(s.size() - 1, k == 0 ? 0 : k - 1)];
  };
  h.p50 = rank(0.50);
  h.p99 = rank(0.99);
  return h;
}

// ---------------------------------------------------------------------------
// R1 eval_alpha — src/blend.cpp:8-14.  std::exp(float) -> libm expf.
AlphaEval eval_alpha(const Gaussian2D& g, float px, float py) {
  const float dx = px - g.x;
  const float dy = py - g.y;
  const float power = -0.5f * (g.conic_a * dx * dx + g.conic_c * dy * dy) - g.conic_b * dx * dy;
  const float alpha = std::min(kAlphaClamp, g.opacity * std::exp(power));
  return {power, alpha};
}

static void finalize(PixelResult& r, const double col[3], double depth, float t, const float bg[3]) {
  r.final_t = t;
  r.out_alpha = 1.0f - t;
  r.out_depth = static_cast<float>(depth);
  for (int c = 0; c < 3; ++c) r.color[c] = static_cast<float>(col[c] + static_cast<double>(bg[c]) * t);
}

// R2 blend_pixel — src/blend.cpp:16-42
PixelResult blend_pixel(std::span<const BlendStep> steps, const float bg[3]) {
  double col[3] = {0, 0, 0}, weight = 0.0, depth = 0.0;
  float t = 1.0f;
  PixelResult r;
  for (size_t i = 0; i < steps.size(); ++i) {
    const BlendStep& s = steps[i];
    if (s.alpha < kAlphaSkip) continue;
    const float tmp_t = t * (1.0f - s.alpha);
    if (tmp_t < kStopThreshold) {
      r.term_index = int(i) + 1;
      break;
    }
    const double w = static_cast<double>(s.alpha) * static_cast<double>(t);
    col[0] += s.color[0] * w;
    col[1] += s.color[1] * w;
    col[2] += s.color[2] * w;
    weight += w;
    depth += s.depth * w;
    t = tmp_t;
    ++r.contrib_count;
  }
  (void)weight;
  finalize(r, col, depth, t, bg);
  return r;
}

// R3 termination_index — src/blend.cpp:44-53
int termination_index(std::span<const BlendStep> steps) {
  float t = 1.0f;
  for (size_t i = 0; i < steps.size(); ++i) {
    if (steps[i].alpha < kAlphaSkip) continue;
    const float tmp_t = t * (1.0f - steps[i].alpha);
    if (tmp_t < kStopThreshold) return int(i) + 1;
    t = tmp_t;
  }
  return 0;
}

// R6 blend_pixel_gaussianwise — src/kernels.cpp:57-107
PixelResult blend_pixel_gaussianwise(std::span<const BlendStep> steps, const float bg[3]) {
  double col[3] = {0, 0, 0}, weight = 0.0, depth = 0.0;
  float t = 1.0f;
  PixelResult r;
  const size_t n = steps.size();
  for (size_t base = 0; base < n && !r.term_index; base += 32) {
    const size_t count = std::min<size_t>(32, n - base);
    std::array<float, 32> factors;
    std::array<bool, 32> skip;
    for (size_t lane = 0; lane < 32; ++lane) {
      const bool active = lane < count;
      skip[lane] = !active || steps[base + lane].alpha < kAlphaSkip;
      factors[lane] = skip[lane] ? 1.0f : 1.0f - steps[base + lane].alpha;
    }
    const WarpPrefix<float> prefix = warp_prefix_product<float>(factors, t);
    float serial_t = t;
    size_t commit_end = count;
    for (size_t lane = 0; lane < count; ++lane) {
      if (skip[lane]) continue;
      const float tmp_t = serial_t * factors[lane];
      if (tmp_t < kStopThreshold) {
        r.term_index = int(base + lane) + 1;
        commit_end = lane;
        break;
      }
      serial_t = tmp_t;
    }
    for (size_t lane = 0; lane < commit_end; ++lane) {
      if (skip[lane]) continue;
      const float t_before = lane == 0 ? t : prefix.per_lane[lane - 1];
      const BlendStep& s = steps[base + lane];
      const double w = static_cast<double>(s.alpha) * static_cast<double>(t_before);
      col[0] += s.color[0] * w;
      col[1] += s.color[1] * w;
      col[2] += s.color[2] * w;
      weight += w;
      depth += s.depth * w;
      ++r.contrib_count;
    }
    t = serial_t;
  }
  (void)weight;
  finalize(r, col, depth, t, bg);
  return r;
}

// R4/R7 render_reference (src/blend.cpp:55-107) / render_gaussianwise
// (src/kernels.cpp:109-155).  Faithful mode builds the BlendStep list for the
// whole tile list per pixel (src/blend.cpp:85-92); lazy mode stops building it
// once the serial stop rule fires — identical output, since no step after the
// termination index is ever read by either blend function.
static void render_tile(Variant v, const TileBinning& b, const Gaussian2D* gs, int width, int height, int pw,
                        int ph, const float bg[3], bool lazy, int t, std::vector<BlendStep>& steps,
                        RenderOutput& out) {
  const uint32_t start = b.tile_ranges[2 * size_t(t)], end = b.tile_ranges[2 * size_t(t) + 1];
  const int tx = t % b.tile_cols, ty = t / b.tile_cols;
  const int x0 = tx * pw, y0 = ty * ph;
  const int x1 = std::min(width, x0 + pw), y1 = std::min(height, y0 + ph);
  const bool pixwise = variant_is_pixelwise(v);
  for (int py = y0; py < y1; ++py) {
    for (int px = x0; px < x1; ++px) {
      const float sx = float(px) + 0.5f, sy = float(py) + 0.5f;
      steps.clear();
      steps.reserve(end - start);
      float lt = 1.0f;  // lazy-mode serial transmittance (decision only)
      for (uint32_t k = start; k < end; ++k) {
        const Gaussian2D& g = gs[b.point_list[k]];
        const AlphaEval e = eval_alpha(g, sx, sy);
        const float alpha = e.power > 0.0f ? 0.0f : e.alpha;
        steps.push_back({alpha, {g.color[0], g.color[1], g.color[2]}, g.depth});
        if (lazy && !(alpha < kAlphaSkip)) {
          const float tmp = lt * (1.0f - alpha);
          if (tmp < kStopThreshold) break;
          lt = tmp;
        }
      }
      const PixelResult r = pixwise ? blend_pixel(steps, bg) : blend_pixel_gaussianwise(steps, bg);
      const size_t p = size_t(py) * size_t(width) + size_t(px);
      out.color[p * 3 + 0] = r.color[0];
      out.color[p * 3 + 1] = r.color[1];
      out.color[p * 3 + 2] = r.color[2];
      out.alpha[p] = r.out_alpha;
      out.depth[p] = r.out_depth;
      out.final_t[p] = r.final_t;
      out.contrib[p] = r.contrib_count;
      out.term[p] = r.term_index;
    }
  }
}

RenderOutput render(Variant v, const TileBinning& b, const Gaussian2D* gs, size_t n, int width, int height,
                    int pw, int ph, const float bg[3], const RenderOptions& opt) {
  (void)n;
  const int cols = (width + pw - 1) / pw;
  const int rows = (height + ph - 1) / ph;
  if (cols != b.tile_cols || rows != b.tile_rows)
    throw std::invalid_argument("render_reference: binning grid does not match image dims");
  RenderOutput out;
  out.init(width, height);
  std::vector<int32_t> todo;
  if (opt.tiles) {
    todo.assign(opt.tiles, opt.tiles + opt.n_tiles);
  } else {
    todo.resize(b.tile_count());
    std::iota(todo.begin(), todo.end(), 0);
  }
  const int threads = std::max(1, opt.threads);
  std::atomic<size_t> next{0};
  auto worker = [&]() {
    std::vector<BlendStep> steps;
    for (;;) {
      const size_t i = next.fetch_add(1);
      if (i >= todo.size()) break;
      render_tile(v, b, gs, width, height, pw, ph, bg, opt.lazy, todo[i], steps, out);
    }
  };
  if (threads == 1) {
    worker();
  } else {
    std::vector<std::thread> pool;
    for (int i = 0; i < threads; ++i) pool.emplace_back(worker);
    for (auto& th : pool) th.join();
  }
  return out;
}

// ---------------------------------------------------------------------------
// Backward render.  Per pixel, the forward of blend_pixel
// (src/blend.cpp:16-42) is replayed to find the committed entries k with
// their alpha_k, transmittance T_k and weight w_k = alpha_k T_k; then, with
// colour = sum_k c_k w_k + bg t_final, depth = sum_k d_k w_k, out_alpha =
// 1 - t_final:
//   d colour / d alpha_k = c_k T_k - S_k / (1 - alpha_k),
//     S_k = sum_{j>k} c_j w_j + bg t_final          (same for depth, no bg)
//   d out_alpha / d alpha_k = t_final / (1 - alpha_k)
//   alpha = min(0.99, o G), G = exp(power): zero gradient when clamped;
//   power = -0.5 (a dx^2 + c dy^2) - b dx dy, dx = px + 0.5 - x.
void render_backward(const TileBinning& b, const Gaussian2D* gs, size_t n, int width, int height, int pw, int ph,
                     const float bg[3], const float* dl_dcolor, const float* dl_dalpha, const float* dl_ddepth,
                     SplatGrad* out) {
  (void)n;
  const int cols = (width + pw - 1) / pw, rows = (height + ph - 1) / ph;
  if (cols != b.tile_cols || rows != b.tile_rows)
    throw std::invalid_argument("render_backward: binning grid does not match image dims");
  struct Commit { uint32_t id; double alpha, T, G, a0, dx, dy; };
  std::vector<Commit> cm;
  for (int t = 0; t < b.tile_count(); ++t) {
    const uint32_t start = b.tile_ranges[2 * size_t(t)], end = b.tile_ranges[2 * size_t(t) + 1];
    const int tx = t % cols, ty = t / cols;
    const int x0 = tx * pw, y0 = ty * ph, x1 = std::min(width, x0 + pw), y1 = std::min(height, y0 + ph);
    for (int py = y0; py < y1; ++py)
      for (int px = x0; px < x1; ++px) {
        const size_t pp = size_t(py) * size_t(width) + size_t(px);
        if (dl_dcolor[3 * pp] == 0.0f && dl_dcolor[3 * pp + 1] == 0.0f && dl_dcolor[3 * pp + 2] == 0.0f &&
            dl_dalpha[pp] == 0.0f && dl_ddepth[pp] == 0.0f)
          continue;  // contributes nothing (lets tests sample tiles of large frames)
        const float sx = float(px) + 0.5f, sy = float(py) + 0.5f;
        cm.clear();
        float tt = 1.0f;
        double C[3] = {0, 0, 0}, D = 0;
        for (uint32_t k = start; k < end; ++k) {
          const Gaussian2D& g = gs[b.point_list[k]];
          const AlphaEval e = eval_alpha(g, sx, sy);
          const float alpha = e.power > 0.0f ? 0.0f : e.alpha;
          if (alpha < kAlphaSkip) continue;
          const float tmp = tt * (1.0f - alpha);
          if (tmp < kStopThreshold) break;
          const double w = double(alpha) * double(tt);
          for (int c = 0; c < 3; ++c) C[c] += g.color[c] * w;
          D += g.depth * w;
          const double G = std::exp(double(e.power));
          cm.push_back({b.point_list[k], double(alpha), double(tt), G, double(g.opacity) * G,
                        double(sx) - double(g.x), double(sy) - double(g.y)});
          tt = tmp;
        }
        const size_t p = size_t(py) * size_t(width) + size_t(px);
        const double tf = tt;
        double S[3], SD = D;
        for (int c = 0; c < 3; ++c) S[c] = C[c] + double(bg[c]) * tf;
        const double gC[3] = {dl_dcolor[3 * p], dl_dcolor[3 * p + 1], dl_dcolor[3 * p + 2]};
        const double gA = dl_dalpha[p], gD = dl_ddepth[p];
        for (const Commit& q : cm) {
          const Gaussian2D& g = gs[q.id];
          SplatGrad& o = out[q.id];
          const double w = q.alpha * q.T;
          for (int c = 0; c < 3; ++c) S[c] -= g.color[c] * w;
          SD -= g.depth * w;
          const double inv = 1.0 / (1.0 - q.alpha);
          double dla = gA * tf * inv + gD * (g.depth * q.T - SD * inv);
          for (int c = 0; c < 3; ++c) dla += gC[c] * (g.color[c] * q.T - S[c] * inv);
          for (int c = 0; c < 3; ++c) o.color[c] += gC[c] * w;
          o.depth += gD * w;
          if (q.a0 > double(kAlphaClamp)) continue;  // alpha clamped at 0.99
          o.opacity += dla * q.G;
          const double dlp = dla * double(g.opacity) * q.G;
          o.conic[0] += dlp * (-0.5 * q.dx * q.dx);
          o.conic[1] += dlp * (-q.dx * q.dy);
          o.conic[2] += dlp * (-0.5 * q.dy * q.dy);
          o.xy[0] += dlp * (double(g.conic_a) * q.dx + double(g.conic_b) * q.dy);
          o.xy[1] += dlp * (double(g.conic_c) * q.dy + double(g.conic_b) * q.dx);
        }
      }
  }
}

// ---------------------------------------------------------------------------
// R10 — src/kernels.cpp:27-38
int64_t warp_steps_pixelwise(const std::vector<int64_t>& term_or_zero, int64_t list_len) {
  int64_t steps = 0;
  for (int64_t t : term_or_zero) steps = std::max(steps, t > 0 ? t : list_len);
  return steps;
}
int64_t warp_steps_gaussianwise(int64_t term_or_zero, int64_t list_len) {
  const int64_t consumed = term_or_zero > 0 ? term_or_zero : list_len;
  return (consumed + 31) / 32;
}

// V-1 compare_outputs — src/image_io.cpp:74-90
Deviation compare_outputs(const RenderOutput& a, const RenderOutput& b) {
  if (a.width != b.width || a.height != b.height) throw std::invalid_argument("compare_outputs: dimension mismatch");
  Deviation d;
  auto scan = [&](const std::vector<float>& x, const std::vector<float>& y) {
    for (size_t i = 0; i < x.size(); ++i) {
      const double e = std::abs(static_cast<double>(x[i]) - y[i]);
      d.max_abs = std::max(d.max_abs, e);
      d.max_rel = std::max(d.max_rel, e / std::max(1.0, std::abs(static_cast<double>(x[i]))));
    }
  };
  scan(a.color, b.color);
  scan(a.alpha, b.alpha);
  scan(a.depth, b.depth);
  d.contrib_equal = a.contrib == b.contrib && a.term == b.term;
  return d;
}

// ---------------------------------------------------------------------------
// G-1 Rng — include/splatsim/rng.hpp:11-58
double Rng::uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
double Rng::normal() {
  double u1 = uniform();
  double u2 = uniform();
  if (u1 <= 0.0) u1 = 0x1.0p-53;
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586477 * u2);
}
uint64_t fnv1a64(const void* data, size_t size, uint64_t h) {
  const auto* p = static_cast<const unsigned char*>(data);
  for (size_t i = 0; i < size; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

// gen_clustered_scene — src/workload.cpp:198-246.  Braced initialiser lists
// evaluate left to right, so draws happen in x, y, z order.  Vector4d
// normalize(): Packet2d redux (q0^2+q2^2)+(q1^2+q3^2), then divide.
std::vector<Gaussian3D> gen_clustered_scene(const ClusterSceneParams& p, const Camera& cam) {
  if (p.n_gaussians < 0 || p.n_clusters < 1) throw std::invalid_argument("gen_clustered_scene: invalid params");
  constexpr uint64_t kSceneSalt = 0x7363656e65ull;
  std::vector<Gaussian3D> out;
  out.reserve(size_t(p.n_gaussians));
  Rng rng(p.seed ^ kSceneSalt, 0);
  const double fx = cam.focal[0], fy = cam.focal[1];
  struct Center { double x, y, z; };
  std::vector<Center> centers(size_t(p.n_clusters));
  for (Center& c : centers) {
    const double u = rng.uniform(0.12, 0.88) * cam.width;
    const double v = rng.uniform(0.12, 0.88) * cam.height;
    c.z = rng.uniform(3.0, 8.0);
    c.x = (u - 0.5 * cam.width) * c.z / fx;
    c.y = (v - 0.5 * cam.height) * c.z / fy;
  }
  for (int i = 0; i < p.n_gaussians; ++i) {
    Gaussian3D g{};
    const bool background = rng.uniform() < p.background_fraction;
    if (background) {
      const double z = rng.uniform(3.0, 9.0);
      const double mx = (rng.uniform(0.05, 0.95) * cam.width - 0.5 * cam.width) * z / fx;
      const double my = (rng.uniform(0.05, 0.95) * cam.height - 0.5 * cam.height) * z / fy;
      g.mean[0] = float(mx);
      g.mean[1] = float(my);
      g.mean[2] = float(z);
    } else {
      const Center& c = centers[rng.below(centers.size())];
      const double sigma = p.cluster_sigma * c.z;
      const double mx = c.x + sigma * rng.normal();
      const double my = c.y + sigma * rng.normal();
      const double mz = std::max(0.5, c.z + sigma * rng.normal());
      g.mean[0] = float(mx);
      g.mean[1] = float(my);
      g.mean[2] = float(mz);
    }
    const double base = 0.01 * static_cast<double>(g.mean[2]);
    for (int a = 0; a < 3; ++a) g.scale[a] = float(base * std::exp(0.4 * rng.normal()));
    double q[4];
    for (int k = 0; k < 4; ++k) q[k] = rng.normal();
    const double n2 = (q[0] * q[0] + q[2] * q[2]) + (q[1] * q[1] + q[3] * q[3]);
    if (n2 > 0.0) {
      const double n = std::sqrt(n2);
      for (double& v : q) v = v / n;
    }
    for (int k = 0; k < 4; ++k) g.rot[k] = float(q[k]);  // Quaternionf(w, x, y, z)
    g.opacity = float(rng.uniform(0.2, 0.95));
    for (int c = 0; c < 3; ++c) g.color[c] = float(rng.uniform());
    out.push_back(g);
  }
  return out;
}

}  // namespace oracle
