// scene_io.cpp — scene JSON I/O and validation (src/scene.cpp:41-179).
//
// Host-only.  The reference reads/writes with nlohmann/json, which is not
// vendored in the mount; this is a small recursive-descent reader (objects,
// arrays, numbers via strtod — correctly rounded —, strings, literals) and a
// writer that emits keys in sorted order with two-space indentation like
// nlohmann's dump(2), numbers as the shortest text that parses back to the
// same double (std::to_chars), so float -> double -> text -> double -> float
// is the identity and save/load round-trips are bit-exact.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>

#include "splatsim_b200.hpp"

namespace splatsim {
namespace {

[[noreturn]] void fail(const std::string& what) { throw SceneError(what); }

struct Json {
  enum Kind { Null, Bool, Number, String, Array, Object } kind = Null;
  bool b = false;
  double num = 0.0;
  bool integral = false;  // written without '.', 'e' (ints / seeds)
  std::string text;       // number literal (for exact integers) or string
  std::vector<Json> arr;
  std::map<std::string, Json> obj;

  bool contains(const char* k) const { return kind == Object && obj.count(k); }
  const Json& at(const char* k) const { return obj.at(k); }
};

class Reader {
 public:
  explicit Reader(const std::string& s) : s_(s) {}
  Json parse() {
    Json v = value();
    ws();
    if (i_ != s_.size()) error("trailing characters");
    return v;
  }

 private:
  [[noreturn]] void error(const std::string& what) {
    fail("scene file: parse error at byte " + std::to_string(i_) + ": " + what);
  }
  void ws() {
    while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\n' || s_[i_] == '\r' || s_[i_] == '\t')) ++i_;
  }
  bool lit(const char* w) {
    const size_t n = std::strlen(w);
    if (s_.compare(i_, n, w) == 0) {
      i_ += n;
      return true;
    }
    return false;
  }
  Json value() {
    ws();
    if (i_ >= s_.size()) error("unexpected end of input");
    const char c = s_[i_];
    Json v;
    if (c == '{') {
      v.kind = Json::Object;
      ++i_;
      ws();
      if (i_ < s_.size() && s_[i_] == '}') {
        ++i_;
        return v;
      }
      for (;;) {
        ws();
        if (i_ >= s_.size() || s_[i_] != '"') error("expected object key");
        std::string k = str();
        ws();
        if (i_ >= s_.size() || s_[i_] != ':') error("expected ':'");
        ++i_;
        v.obj[k] = value();
        ws();
        if (i_ < s_.size() && s_[i_] == ',') {
          ++i_;
          continue;
        }
        if (i_ < s_.size() && s_[i_] == '}') {
          ++i_;
          return v;
        }
        error("expected ',' or '}'");
      }
    }
    if (c == '[') {
      v.kind = Json::Array;
      ++i_;
      ws();
      if (i_ < s_.size() && s_[i_] == ']') {
        ++i_;
        return v;
      }
      for (;;) {
        v.arr.push_back(value());
        ws();
        if (i_ < s_.size() && s_[i_] == ',') {
          ++i_;
          continue;
        }
        if (i_ < s_.size() && s_[i_] == ']') {
          ++i_;
          return v;
        }
        error("expected ',' or ']'");
      }
    }
    if (c == '"') {
      v.kind = Json::String;
      v.text = str();
      return v;
    }
    if (lit("true")) {
      v.kind = Json::Bool;
      v.b = true;
      return v;
    }
    if (lit("false")) {
      v.kind = Json::Bool;
      return v;
    }
    if (lit("null")) return v;
    return number();
  }
  std::string str() {
    ++i_;  // opening quote
    std::string out;
    while (i_ < s_.size() && s_[i_] != '"') {
      char c = s_[i_++];
      if (c == '\\') {
        if (i_ >= s_.size()) error("bad escape");
        const char e = s_[i_++];
        switch (e) {
          case '"': out += '"'; break;
          case '\\': out += '\\'; break;
          case '/': out += '/'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'n': out += '\n'; break;
          case 'r': out += '\r'; break;
          case 't': out += '\t'; break;
          case 'u': {
            if (i_ + 4 > s_.size()) error("bad \\u escape");
            const unsigned cp = unsigned(std::strtoul(s_.substr(i_, 4).c_str(), nullptr, 16));
            i_ += 4;
            if (cp < 0x80) {
              out += char(cp);
            } else if (cp < 0x800) {
              out += char(0xC0 | (cp >> 6));
              out += char(0x80 | (cp & 0x3F));
            } else {
              out += char(0xE0 | (cp >> 12));
              out += char(0x80 | ((cp >> 6) & 0x3F));
              out += char(0x80 | (cp & 0x3F));
            }
            break;
          }
          default: error("bad escape");
        }
      } else {
        out += c;
      }
    }
    if (i_ >= s_.size()) error("unterminated string");
    ++i_;
    return out;
  }
  Json number() {
    const size_t b = i_;
    if (i_ < s_.size() && (s_[i_] == '-' || s_[i_] == '+')) ++i_;
    bool integral = true;
    while (i_ < s_.size()) {
      const char c = s_[i_];
      if (c >= '0' && c <= '9') {
        ++i_;
      } else if (c == '.' || c == 'e' || c == 'E' || c == '+' || c == '-') {
        integral = false;
        ++i_;
      } else {
        break;
      }
    }
    if (i_ == b) error("unexpected character");
    Json v;
    v.kind = Json::Number;
    v.text = s_.substr(b, i_ - b);
    char* end = nullptr;
    v.num = std::strtod(v.text.c_str(), &end);  // correctly rounded
    if (!end || *end) error("bad number");
    v.integral = integral;
    return v;
  }
  const std::string& s_;
  size_t i_ = 0;
};

void read_floats(const Json& j, const char* field, float* out, int n) {
  if (!j.contains(field)) fail(std::string(field) + ": missing");
  const Json& a = j.at(field);
  if (a.kind != Json::Array || int(a.arr.size()) != n)
    fail(std::string(field) + ": expected array of " + std::to_string(n) + " numbers");
  for (int i = 0; i < n; ++i) {
    if (a.arr[size_t(i)].kind != Json::Number) fail(std::string(field) + "[" + std::to_string(i) + "]: not a number");
    out[i] = static_cast<float>(a.arr[size_t(i)].num);
  }
}

int get_int(const Json& j, const char* what) {
  if (j.kind != Json::Number) fail(std::string(what) + ": not a number");
  return int(j.num);
}

bool finite3(const std::array<float, 3>& v) {
  return std::isfinite(v[0]) && std::isfinite(v[1]) && std::isfinite(v[2]);
}

// -- writer ------------------------------------------------------------------
std::string num(double v) {
  char buf[64];
  const auto r = std::to_chars(buf, buf + sizeof(buf), v);  // shortest round-trip
  std::string s(buf, r.ptr);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";  // nlohmann writes floats with a point
  return s;
}

void write_array(std::ostringstream& o, const float* v, int n, int ind) {
  const std::string pad(size_t(ind + 2), ' ');
  o << "[\n";
  for (int i = 0; i < n; ++i) o << pad << num(double(v[i])) << (i + 1 < n ? ",\n" : "\n");
  o << std::string(size_t(ind), ' ') << "]";
}

void write_ints(std::ostringstream& o, long long a, long long b, int ind) {
  const std::string pad(size_t(ind + 2), ' ');
  o << "[\n" << pad << a << ",\n" << pad << b << "\n" << std::string(size_t(ind), ' ') << "]";
}

}  // namespace

void validate(const Scene& scene) {
  const Camera& cam = scene.camera;
  if (cam.width <= 0 || cam.height <= 0) fail("camera.dims: must be positive");
  if (!(cam.focal[0] > 0.0f) || !(cam.focal[1] > 0.0f)) fail("camera.focal: must be positive");
  float worst = 0.0f;  // max |R R^T - I| over the 3x3 rotation block
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      float d = 0.0f;
      for (int k = 0; k < 3; ++k) d += cam.view_transform[size_t(r * 4 + k)] * cam.view_transform[size_t(c * 4 + k)];
      worst = std::max(worst, std::abs(d - (r == c ? 1.0f : 0.0f)));
    }
  if (!(worst <= 1e-5f)) fail("camera.view: rotation block is not orthonormal");
  if (scene.config.patch_width <= 0 || scene.config.patch_height <= 0) fail("config.patch: must be positive");
  for (int c = 0; c < 3; ++c) {
    const float b = scene.config.background[size_t(c)];
    if (!(b >= 0.0f && b <= 1.0f)) fail("config.background: channels must be in [0,1]");
  }
  for (size_t i = 0; i < scene.gaussians.size(); ++i) {
    const Gaussian3D& g = scene.gaussians[i];
    const std::string at = "gaussians[" + std::to_string(i) + "].";
    if (!finite3(g.mean)) fail(at + "mean: not finite");
    if (!finite3(g.scale) || !(std::min({g.scale[0], g.scale[1], g.scale[2]}) > 0.0f))
      fail(at + "scale: components must be strictly positive");
    const auto& q = g.rotation;
    const float norm = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    if (!(std::abs(norm - 1.0f) <= 1e-6f)) fail(at + "rot: quaternion not unit length");
    if (!(g.opacity >= 0.0f && g.opacity <= 1.0f)) fail(at + "opacity: must be in [0,1]");
    for (int c = 0; c < 3; ++c)
      if (!(g.color[size_t(c)] >= 0.0f && g.color[size_t(c)] <= 1.0f)) fail(at + "color: channels must be in [0,1]");
  }
}

Scene parse_scene(const std::string& json_text) {
  const Json j = Reader(json_text).parse();
  if (j.kind != Json::Object) fail("scene file: top level is not an object");
  Scene scene;
  if (!j.contains("camera")) fail("camera: missing");
  const Json& jc = j.at("camera");
  read_floats(jc, "view", scene.camera.view_transform.data(), 16);
  read_floats(jc, "focal", scene.camera.focal.data(), 2);
  if (!jc.contains("dims") || jc.at("dims").kind != Json::Array || jc.at("dims").arr.size() != 2)
    fail("camera.dims: expected [width, height]");
  scene.camera.width = get_int(jc.at("dims").arr[0], "camera.dims");
  scene.camera.height = get_int(jc.at("dims").arr[1], "camera.dims");
  if (j.contains("config")) {
    const Json& jf = j.at("config");
    if (jf.contains("patch")) {
      if (jf.at("patch").kind != Json::Array || jf.at("patch").arr.size() != 2) fail("config.patch: expected [w, h]");
      scene.config.patch_width = get_int(jf.at("patch").arr[0], "config.patch");
      scene.config.patch_height = get_int(jf.at("patch").arr[1], "config.patch");
    }
    if (jf.contains("background")) read_floats(jf, "background", scene.config.background.data(), 3);
    if (jf.contains("seed")) {
      const Json& sd = jf.at("seed");
      if (sd.kind != Json::Number) fail("config.seed: not a number");
      scene.config.seed = sd.integral ? std::strtoull(sd.text.c_str(), nullptr, 10) : std::uint64_t(sd.num);
    }
  }
  if (!j.contains("gaussians") || j.at("gaussians").kind != Json::Array) fail("gaussians: missing array");
  const auto& ga = j.at("gaussians").arr;
  scene.gaussians.reserve(ga.size());
  for (size_t idx = 0; idx < ga.size(); ++idx) {
    const Json& jg = ga[idx];
    Gaussian3D g;
    try {
      read_floats(jg, "mean", g.mean.data(), 3);
      read_floats(jg, "scale", g.scale.data(), 3);
      read_floats(jg, "rot", g.rotation.data(), 4);  // [w, x, y, z] (src/scene.cpp:124)
      if (!jg.contains("opacity") || jg.at("opacity").kind != Json::Number) fail("opacity: missing or not a number");
      g.opacity = static_cast<float>(jg.at("opacity").num);
      read_floats(jg, "color", g.color.data(), 3);
    } catch (const SceneError& e) {
      fail("gaussians[" + std::to_string(idx) + "]." + e.what());
    }
    scene.gaussians.push_back(g);
  }
  validate(scene);
  return scene;
}

std::string serialize_scene(const Scene& scene) {
  std::ostringstream o;
  o << "{\n  \"camera\": {\n    \"dims\": ";
  write_ints(o, scene.camera.width, scene.camera.height, 4);
  o << ",\n    \"focal\": ";
  write_array(o, scene.camera.focal.data(), 2, 4);
  o << ",\n    \"view\": ";
  write_array(o, scene.camera.view_transform.data(), 16, 4);
  o << "\n  },\n  \"config\": {\n    \"background\": ";
  write_array(o, scene.config.background.data(), 3, 4);
  o << ",\n    \"patch\": ";
  write_ints(o, scene.config.patch_width, scene.config.patch_height, 4);
  o << ",\n    \"seed\": " << scene.config.seed << "\n  },\n  \"gaussians\": [";
  for (size_t i = 0; i < scene.gaussians.size(); ++i) {
    const Gaussian3D& g = scene.gaussians[i];
    o << (i ? ",\n" : "\n") << "    {\n      \"color\": ";
    write_array(o, g.color.data(), 3, 6);
    o << ",\n      \"mean\": ";
    write_array(o, g.mean.data(), 3, 6);
    o << ",\n      \"opacity\": " << num(double(g.opacity)) << ",\n      \"rot\": ";
    write_array(o, g.rotation.data(), 4, 6);
    o << ",\n      \"scale\": ";
    write_array(o, g.scale.data(), 3, 6);
    o << "\n    }";
  }
  o << (scene.gaussians.empty() ? "]" : "\n  ]") << "\n}";
  return o.str();
}

Scene load_scene(const std::string& path) {
  std::ifstream in(path);
  if (!in) fail("cannot open scene file: " + path);
  std::ostringstream ss;
  ss << in.rdbuf();
  return parse_scene(ss.str());
}

void save_scene(const Scene& scene, const std::string& path) {
  validate(scene);
  std::ofstream out(path);
  if (!out) fail("cannot open for writing: " + path);
  out << serialize_scene(scene) << '\n';
  if (!out) fail("write failed: " + path);
}

}  // namespace splatsim
