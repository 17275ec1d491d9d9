// splatsim_host.cpp — host-side pieces of the product library.
//
// Scene synthesis (the reference's workload module, src/workload.cpp:198-246
// with the counter RNG of include/splatsim/rng.hpp) used to build the
// measurement inputs.  Runs on the host: it draws from a serial splitmix64
// stream, exactly like the reference, so any parallel device version would
// have to replay that stream anyway.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "splatsim_b200.h"

namespace {

// include/splatsim/rng.hpp:11-58 (counter-based splitmix64).
class SplitMix {
 public:
  SplitMix(uint64_t seed, uint64_t stream) : s_(mix(seed ^ mix(stream + 0x9e3779b97f4a7c15ull))) {}
  static uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  uint64_t u64() {
    s_ += 0x9e3779b97f4a7c15ull;
    return mix(s_);
  }
  double uni() { return static_cast<double>(u64() >> 11) * 0x1.0p-53; }
  double uni(double lo, double hi) { return lo + (hi - lo) * uni(); }
  uint64_t below(uint64_t n) { return n ? u64() % n : 0; }
  double gauss() {  // Box-Muller, one draw per call (rng.hpp:43-48)
    double u1 = uni();
    const double u2 = uni();
    if (u1 <= 0.0) u1 = 0x1.0p-53;
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586477 * u2);
  }

 private:
  uint64_t s_;
};

}  // namespace

extern "C" int bs_host_gen_clustered_scene(int32_t n, int32_t n_clusters, uint64_t seed, double cluster_sigma,
                                           double background_fraction, const bs_camera* cam, bs_gaussian3d* out) {
  if (n < 0 || n_clusters < 1 || !cam || (n > 0 && !out)) return BS_ERR_INVALID_ARGUMENT;
  SplitMix rng(seed ^ 0x7363656e65ull /* "scene" */, 0);
  const double fx = cam->focal[0], fy = cam->focal[1];
  const double W = cam->width, H = cam->height;
  std::vector<double> cx(n_clusters), cy(n_clusters), cz(n_clusters);
  for (int c = 0; c < n_clusters; ++c) {
    const double u = rng.uni(0.12, 0.88) * W;
    const double v = rng.uni(0.12, 0.88) * H;
    cz[c] = rng.uni(3.0, 8.0);
    cx[c] = (u - 0.5 * W) * cz[c] / fx;
    cy[c] = (v - 0.5 * H) * cz[c] / fy;
  }
  for (int32_t i = 0; i < n; ++i) {
    bs_gaussian3d g;
    std::memset(&g, 0, sizeof(g));
    if (rng.uni() < background_fraction) {
      const double z = rng.uni(3.0, 9.0);
      const double mx = (rng.uni(0.05, 0.95) * W - 0.5 * W) * z / fx;
      const double my = (rng.uni(0.05, 0.95) * H - 0.5 * H) * z / fy;
      g.mean[0] = static_cast<float>(mx);
      g.mean[1] = static_cast<float>(my);
      g.mean[2] = static_cast<float>(z);
    } else {
      const uint64_t c = rng.below(static_cast<uint64_t>(n_clusters));
      const double sigma = cluster_sigma * cz[c];
      const double mx = cx[c] + sigma * rng.gauss();
      const double my = cy[c] + sigma * rng.gauss();
      const double mz = std::max(0.5, cz[c] + sigma * rng.gauss());
      g.mean[0] = static_cast<float>(mx);
      g.mean[1] = static_cast<float>(my);
      g.mean[2] = static_cast<float>(mz);
    }
    const double base = 0.01 * static_cast<double>(g.mean[2]);
    for (int a = 0; a < 3; ++a) g.scale[a] = static_cast<float>(base * std::exp(0.4 * rng.gauss()));
    double q[4];
    for (double& v : q) v = rng.gauss();
    // Eigen Vector4d::normalize(): SSE2 packet redux (q0^2+q2^2)+(q1^2+q3^2)
    const double n2 = (q[0] * q[0] + q[2] * q[2]) + (q[1] * q[1] + q[3] * q[3]);
    if (n2 > 0.0) {
      const double nn = std::sqrt(n2);
      for (double& v : q) v = v / nn;
    }
    for (int k = 0; k < 4; ++k) g.rot[k] = static_cast<float>(q[k]);
    g.opacity = static_cast<float>(rng.uni(0.2, 0.95));
    for (int k = 0; k < 3; ++k) g.color[k] = static_cast<float>(rng.uni());
    out[i] = g;
  }
  return BS_OK;
}
