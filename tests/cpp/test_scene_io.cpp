// Scene JSON I/O (src/scene.cpp:41-179 semantics), host only: bit-exact float
// round trips through serialize/parse and save/load, the reference's
// validation rules and SceneError messages, parsing of reference-layout files.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>

#include "splatsim_b200.hpp"

static int failures = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    if (!(cond)) {                                                         \
      std::printf("CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                          \
    }                                                                      \
  } while (0)

template <size_t N>
static bool same(const std::array<float, N>& a, const std::array<float, N>& b) {
  return std::memcmp(a.data(), b.data(), N * sizeof(float)) == 0;
}

static std::string error_of(const std::string& text) {
  try {
    splatsim::parse_scene(text);
  } catch (const splatsim::SceneError& e) {
    return e.what();
  }
  return "";
}

int main(int argc, char** argv) {
  const std::string tmp = argc > 1 ? argv[1] : "/tmp/scene_io_test.json";
  std::mt19937 rng(7);
  std::uniform_real_distribution<float> u(0.0f, 1.0f), w(-50.0f, 50.0f);
  splatsim::Scene s;
  s.camera.width = 1920;
  s.camera.height = 1080;
  s.camera.focal = {1000.0f, 999.5f};
  const float c = std::cos(0.3f), sn = std::sin(0.3f);
  s.camera.view_transform = {c, 0, sn, 0.25f, 0, 1, 0, -1.5f, -sn, 0, c, 3.0f, 0, 0, 0, 1};
  s.config.patch_width = 16;
  s.config.patch_height = 16;
  s.config.background = {0.1f, 0.2f, 0.3f};
  s.config.seed = 18446744073709551557ull;  // > 2^63: exact through the integer path
  for (int i = 0; i < 2000; ++i) {
    splatsim::Gaussian3D g;
    g.mean = {w(rng), w(rng), i == 0 ? -0.0f : w(rng)};
    g.scale = {u(rng) + 1e-7f, i == 1 ? 1.17549435e-38f : u(rng) + 1e-3f, 3.4e38f};
    float q[4] = {u(rng) - 0.5f, u(rng) - 0.5f, u(rng) - 0.5f, u(rng) - 0.5f};
    const float n = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    g.rotation = {q[0] / n, q[1] / n, q[2] / n, q[3] / n};
    g.opacity = i == 2 ? 1.0f : u(rng);
    g.color = {u(rng), 0.1f, i == 3 ? 1e-45f : u(rng)};  // a subnormal
    s.gaussians.push_back(g);
  }
  bool valid = true;
  try {
    splatsim::validate(s);
  } catch (const splatsim::SceneError& e) {
    std::printf("unexpected: %s\n", e.what());
    valid = false;
  }
  CHECK(valid);
  // serialize -> parse: every float bit-identical
  const std::string text = splatsim::serialize_scene(s);
  const splatsim::Scene r = splatsim::parse_scene(text);
  CHECK(r.gaussians.size() == s.gaussians.size());
  bool bits = same(r.camera.view_transform, s.camera.view_transform) && same(r.camera.focal, s.camera.focal) &&
              same(r.config.background, s.config.background) && r.camera.width == 1920 && r.camera.height == 1080 &&
              r.config.patch_width == 16 && r.config.patch_height == 16 && r.config.seed == s.config.seed;
  for (size_t i = 0; i < s.gaussians.size() && bits; ++i) {
    const auto &a = s.gaussians[i], &b = r.gaussians[i];
    bits = same(a.mean, b.mean) && same(a.scale, b.scale) && same(a.rotation, b.rotation) && same(a.color, b.color) &&
           std::memcmp(&a.opacity, &b.opacity, 4) == 0;
  }
  CHECK(bits);
  CHECK(splatsim::serialize_scene(r) == text);  // idempotent text
  // save / load through a file
  splatsim::save_scene(s, tmp);
  const splatsim::Scene f = splatsim::load_scene(tmp);
  CHECK(f.gaussians.size() == s.gaussians.size() && same(f.gaussians[5].mean, s.gaussians[5].mean));
  // a reference-layout file (keys in any order, integers where floats go)
  const std::string ref_json = R"({"gaussians": [{"rot": [1, 0, 0, 0], "opacity": 0.5, "mean": [0, 0, 10],
    "scale": [1, 2, 3], "color": [1, 0.5, 0]}], "camera": {"focal": [100, 100], "dims": [64, 48],
    "view": [1,0,0,0, 0,1,0,0, 0,0,1,0, 0,0,0,1]}})";
  const splatsim::Scene g = splatsim::parse_scene(ref_json);
  CHECK(g.gaussians.size() == 1 && g.gaussians[0].scale[1] == 2.0f && g.gaussians[0].rotation[0] == 1.0f);
  CHECK(g.camera.width == 64 && g.config.patch_width == 16 && g.config.patch_height == 8);  // defaults (scene.hpp:31-36)
  // validation and parse errors name the field, as the reference does
  CHECK(error_of("{}") == "camera: missing");
  CHECK(error_of("{\"camera\":{}}") == "view: missing");
  CHECK(error_of(R"({"camera": {"focal": [100, 100], "dims": [64, 48], "view": [1,0,0,0, 0,1,0,0, 0,0,1,0, 0,0,0,1]}})") ==
        "gaussians: missing array");
  std::string bad = ref_json;
  bad.replace(bad.find("\"rot\": [1, 0, 0, 0]"), 19, "\"rot\": [1, 1, 0, 0]");
  CHECK(error_of(bad) == "gaussians[0].rot: quaternion not unit length");
  bad = ref_json;
  bad.replace(bad.find("\"opacity\": 0.5"), 14, "\"opacity\": 1.5");
  CHECK(error_of(bad) == "gaussians[0].opacity: must be in [0,1]");
  bad = ref_json;
  bad.replace(bad.find("\"scale\": [1, 2, 3]"), 18, "\"scale\": [1, 0, 3]");
  CHECK(error_of(bad) == "gaussians[0].scale: components must be strictly positive");
  bad = ref_json;
  bad.replace(bad.find("\"mean\": [0, 0, 10]"), 18, "\"mean\": [0, \"x\", 1]");
  CHECK(error_of(bad) == "gaussians[0].mean[1]: not a number");
  bad = ref_json;
  bad.replace(bad.find("0,0,1,0, 0,0,0,1"), 16, "0,0,2,0, 0,0,0,1");
  CHECK(error_of(bad) == "camera.view: rotation block is not orthonormal");
  CHECK(error_of("{\"camera\": [1,2") .rfind("scene file:", 0) == 0);
  splatsim::Scene z = s;
  z.camera.width = 0;
  bool threw = false;
  try {
    splatsim::save_scene(z, tmp);
  } catch (const splatsim::SceneError& e) {
    threw = std::string(e.what()) == "camera.dims: must be positive";
  }
  CHECK(threw);
  std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
