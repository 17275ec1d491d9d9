// oracle/oracle.hpp — CPU restatement of the reference forward-render path.
//
// TEST INFRASTRUCTURE ONLY.  This is the parity checker for the B200 product
// (paper_2412_17378_b200/).  Only tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py may load it.  The product
// never links, calls or falls back to it.
//
// What it restates (reference = /root/reference/proj/core, "splatsim"):
//   covariance_of            src/scene.cpp:67-71
//   project_covariance       src/preprocess.cpp:10-15
//   project_gaussian/_all    src/preprocess.cpp:17-64
//   bin_tiles                src/preprocess.cpp:66-115
//   tile_load_histogram      src/preprocess.cpp:117-136
//   eval_alpha/blend_pixel   src/blend.cpp:8-42, termination_index :44-53
//   warp_prefix_product      include/splatsim/blend.hpp:69-83
//   render_reference         src/blend.cpp:55-107
//   blend_pixel_gaussianwise src/kernels.cpp:57-107, render_gaussianwise :109-155
//   warp_steps_*/trace       src/kernels.cpp:27-38, 159-266, run_kernel :268-301
//   compare_outputs          src/image_io.cpp:74-90
//   Rng / fnv1a64            include/splatsim/rng.hpp:11-69
//   gen_clustered_scene      src/workload.cpp:198-246
//
// Pinning status:
//   * PINNED TO THE REFERENCE ITSELF: oracle/_ref (make -C oracle ref) builds
//     /root/reference/proj/core/src/*.cpp unmodified against an Eigen-subset
//     shim (oracle/ref_shim) and the image's nlohmann/json header;
//     tests/test_ref_oracle.py checks this restatement against it bit for
//     bit (scene generator, P1-P6, every render variant on C1, the golden
//     fixtures, the blend KATs) and tests/test_ref_host.py the product's host
//     bookkeeping.  The reference ships no golden vectors of its own.
//   * expf: the oracle calls libm expf exactly as the reference does
//     (std::exp(float), src/blend.cpp:12).  The third-party dependency is
//     glibc 2.39 libm (x86-64 ifunc __expf_fma).
//   * Eigen 3.x fixed-size products (unpinned version, absent here): the
//     evaluation order below — and the shim's — is the one Eigen 3.4 uses on
//     x86-64 with SSE2 (the reference's flags: no -march).  Products that are
//     vectorised (Lhs rows a multiple of the packet size: 2x3 double products)
//     sum left-to-right; scalar coefficient-based products (3x3 float) reduce
//     as a0 + (a1 + a2) (redux_novec_unroller).  P1-P3 bits therefore rest on
//     that documented order; everything else is pinned by executing the
//     reference's code.
//
// Compiled with -ffp-contract=off, as proj/CMakeLists.txt:11-12 does.
#pragma once

#include <array>
#include <cstdint>
#include <optional>
#include <span>
#include <string_view>
#include <vector>

namespace oracle {

struct Vec3f { float x = 0, y = 0, z = 0; };
struct Quatf { float w = 1, x = 0, y = 0, z = 0; };
struct Mat3f { float m[3][3]; };
struct Mat3d { double m[3][3]; };

// include/splatsim/scene.hpp:16-22 (fields, not Eigen memory layout)
struct Gaussian3D {
  float mean[3];
  float scale[3];
  float rot[4];  // w, x, y, z
  float opacity;
  float color[3];
};
static_assert(sizeof(Gaussian3D) == 56);

// include/splatsim/scene.hpp:24-29
struct Camera {
  float view[16];  // row-major world->camera
  float focal[2];
  int32_t width;
  int32_t height;
};

// include/splatsim/preprocess.hpp:16-25
struct Gaussian2D {
  float x, y;
  float conic_a, conic_b, conic_c;
  float opacity;
  float color[3];
  float depth;
  float radius;
};
static_assert(sizeof(Gaussian2D) == 44);

// include/splatsim/preprocess.hpp:28-36
struct TileBinning {
  int tile_cols = 0;
  int tile_rows = 0;
  std::vector<uint32_t> point_list;
  std::vector<uint32_t> tile_ranges;  // 2*T, [start, end) pairs
  int tile_count() const { return tile_cols * tile_rows; }
};

// include/splatsim/preprocess.hpp:38-45
struct TileHistogram {
  std::vector<uint32_t> counts;
  uint32_t min = 0, max = 0;
  double mean = 0.0;
  uint32_t p50 = 0, p99 = 0;
};

inline constexpr float kNearPlane = 0.01f;     // preprocess.hpp:47
inline constexpr float kAlphaClamp = 0.99f;    // blend.hpp:13
inline constexpr float kAlphaSkip = 1.0f / 255.0f;  // blend.hpp:14
inline constexpr float kStopThreshold = 1e-4f;  // blend.hpp:15

struct BlendStep {
  float alpha = 0.0f;
  float color[3] = {0, 0, 0};
  float depth = 0.0f;
};

struct PixelResult {
  float color[3] = {0, 0, 0};
  float out_alpha = 0.0f;
  float out_depth = 0.0f;
  float final_t = 1.0f;
  int contrib_count = 0;
  int term_index = 0;  // 0 = none (std::optional<int> in the reference)
};

struct AlphaEval { float power; float alpha; };

struct RenderOutput {
  int width = 0, height = 0;
  std::vector<float> color, alpha, depth, final_t;
  std::vector<int32_t> contrib, term;
  void init(int w, int h);
};

// ---- Backward render (not in the reference: the analytic
// gradient of render_reference's serial semantics, src/blend.cpp:8-42, with
// the forward's skip / stop decisions held fixed).  Per splat, accumulated
// over every pixel: d/d(x, y, conic_a, conic_b, conic_c, opacity, r, g, b,
// depth).  Double precision; pinned by finite differences of render().
struct SplatGrad {
  double xy[2] = {0, 0};
  double conic[3] = {0, 0, 0};
  double opacity = 0;
  double color[3] = {0, 0, 0};
  double depth = 0;
};
void render_backward(const TileBinning& b, const Gaussian2D* gs, size_t n, int width, int height, int pw, int ph,
                     const float bg[3], const float* dl_dcolor, const float* dl_dalpha, const float* dl_ddepth,
                     SplatGrad* out);

enum class Variant : int { Naive = 0, DynamicBlocks = 1, GaussianWise = 2, FineGrainedCombined = 3, SharedMemOpt = 4 };
std::string_view variant_name(Variant v);
std::optional<Variant> variant_from_name(std::string_view s);
bool variant_is_pixelwise(Variant v);

// ---- P1-P4 ----
Mat3f covariance_of(const Gaussian3D& g);
void project_covariance(const double jac[2][3], const Mat3d& view_rot, const Mat3d& cov3d, double out[2][2]);
std::optional<Gaussian2D> project_gaussian(const Gaussian3D& g, const Camera& cam);
std::vector<Gaussian2D> project_all(const std::vector<Gaussian3D>& gs, const Camera& cam);

// ---- P5-P6 ----
TileBinning bin_tiles(const Gaussian2D* gs, size_t n, int width, int height, int pw, int ph);
TileHistogram tile_load_histogram(const TileBinning& b);

// ---- R1-R7 ----
AlphaEval eval_alpha(const Gaussian2D& g, float px, float py);
PixelResult blend_pixel(std::span<const BlendStep> steps, const float bg[3]);
int termination_index(std::span<const BlendStep> steps);  // 0 = none

template <typename T>
struct WarpPrefix { std::array<T, 32> per_lane; T t_out; };
template <typename T>
WarpPrefix<T> warp_prefix_product(const std::array<T, 32>& factors, T t_in) {
  std::array<T, 32> acc = factors;
  for (int offset = 1; offset < 32; offset *= 2) {
    std::array<T, 32> shifted;
    for (int lane = 0; lane < 32; ++lane) shifted[lane] = lane >= offset ? acc[lane - offset] : T(1);
    for (int lane = 0; lane < 32; ++lane)
      if (lane >= offset) acc[lane] *= shifted[lane];
  }
  WarpPrefix<T> out;
  for (int lane = 0; lane < 32; ++lane) out.per_lane[lane] = t_in * acc[lane];
  out.t_out = out.per_lane[31];
  return out;
}

PixelResult blend_pixel_gaussianwise(std::span<const BlendStep> steps, const float bg[3]);

struct RenderOptions {
  bool lazy = false;            // stop evaluating a pixel's list after its term (same output)
  int threads = 1;              // tiles in parallel; output is identical for any value
  const int32_t* tiles = nullptr;  // optional subset of tiles to render (others keep init values)
  int n_tiles = 0;
};

// render_reference (pixel-wise semantics) / render_gaussianwise.
RenderOutput render(Variant v, const TileBinning& b, const Gaussian2D* gs, size_t n, int width, int height,
                    int pw, int ph, const float bg[3], const RenderOptions& opt = {});

// ---- R8-R10: work trace (src/kernels.cpp:27-38, 208-301) ----
int64_t warp_steps_pixelwise(const std::vector<int64_t>& term_or_zero, int64_t list_len);
int64_t warp_steps_gaussianwise(int64_t term_or_zero, int64_t list_len);

// ---- V-1 ----
struct Deviation { double max_abs = 0, max_rel = 0; bool contrib_equal = true; };
Deviation compare_outputs(const RenderOutput& ref, const RenderOutput& cand);

// ---- G-1 ----
class Rng {
 public:
  explicit Rng(uint64_t seed, uint64_t stream = 0) : state_(mix(seed ^ mix(stream + 0x9e3779b97f4a7c15ull))) {}
  uint64_t next_u64() { state_ += 0x9e3779b97f4a7c15ull; return mix(state_); }
  double uniform();
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  uint64_t below(uint64_t n) { return n ? next_u64() % n : 0; }
  double normal();
  static uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
 private:
  uint64_t state_;
};
uint64_t fnv1a64(const void* data, size_t size, uint64_t h = 0xcbf29ce484222325ull);

struct ClusterSceneParams {
  int n_gaussians = 2000;
  int n_clusters = 4;
  uint64_t seed = 42;
  double cluster_sigma = 0.035;
  double background_fraction = 0.12;
};
std::vector<Gaussian3D> gen_clustered_scene(const ClusterSceneParams& p, const Camera& cam);

}  // namespace oracle
