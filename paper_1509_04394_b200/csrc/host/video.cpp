// FPVD codec and synthetic marker scenes (see video.hpp).
#include "video.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <iterator>
#include <random>

#include "json.hpp"

namespace fuseplan {

namespace {

constexpr char kFpvdMagic[4] = {'F', 'P', 'V', 'D'};
constexpr std::uint32_t kFpvdVersion = 1;

void append_u32(std::string& s, std::uint32_t v) {
  char b[4];
  std::memcpy(b, &v, 4);  // little-endian hosts, like the reference
  s.append(b, 4);
}

std::uint32_t take_u32(const std::string& s, std::size_t& at) {
  require(at + 4 <= s.size(), ErrorKind::Input, "video file truncated");
  std::uint32_t v;
  std::memcpy(&v, s.data() + at, 4);
  at += 4;
  return v;
}

}  // namespace

// video.cpp:46-62: header {magic, version, W, H, F, C, elem_type} + payload.
std::string encode_fpvd(const HostVideo& v) {
  std::string s(kFpvdMagic, 4);
  append_u32(s, kFpvdVersion);
  for (int x : {v.dims.width, v.dims.height, v.dims.frames, v.dims.channels})
    append_u32(s, std::uint32_t(x));
  append_u32(s, std::uint32_t(v.elem));
  if (v.elem == ElemType::U8)
    s.append(reinterpret_cast<const char*>(v.u8.data()), v.u8.size());
  else
    s.append(reinterpret_cast<const char*>(v.f32.data()), v.f32.size() * 4);
  return s;
}

// video.cpp:64-93.
HostVideo decode_fpvd(const std::string& bytes) {
  require(bytes.size() >= 4 && std::memcmp(bytes.data(), kFpvdMagic, 4) == 0,
          ErrorKind::Input, "not an FPVD video file");
  std::size_t at = 4;
  require(take_u32(bytes, at) == kFpvdVersion, ErrorKind::Input,
          "unsupported FPVD version");
  HostVideo v;
  v.dims.width = int(take_u32(bytes, at));
  v.dims.height = int(take_u32(bytes, at));
  v.dims.frames = int(take_u32(bytes, at));
  v.dims.channels = int(take_u32(bytes, at));
  v.dims.fps = 1;
  std::uint32_t et = take_u32(bytes, at);
  require(et <= 1, ErrorKind::Input, "unknown FPVD element type");
  v.elem = ElemType(et);
  v.dims.validate();
  std::size_t n = std::size_t(v.dims.element_count());
  std::size_t esz = v.elem == ElemType::U8 ? 1 : 4;
  require(bytes.size() == at + n * esz, ErrorKind::Input, "video payload size mismatch");
  if (v.elem == ElemType::U8)
    v.u8.assign(bytes.begin() + std::ptrdiff_t(at), bytes.end());
  else {
    v.f32.resize(n);
    std::memcpy(v.f32.data(), bytes.data() + at, n * 4);
  }
  return v;
}

HostVideo read_fpvd_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  require(in.good(), ErrorKind::Input, "cannot open video file: " + path);
  std::string bytes((std::istreambuf_iterator<char>(in)),
                    std::istreambuf_iterator<char>());
  return decode_fpvd(bytes);
}

void write_fpvd_file(const std::string& path, const HostVideo& v) {
  std::ofstream out(path, std::ios::binary);
  require(out.good(), ErrorKind::Input, "cannot write video file: " + path);
  std::string s = encode_fpvd(v);
  out.write(s.data(), std::streamsize(s.size()));
}

// The C++ API's float volume through the same codec: u8 payloads store
// uint8_t(clamp(v, 0, 255)) (video.cpp:57, truncation), f32 payloads the floats.
std::string encode_video(const VideoData& video) {
  HostVideo h;
  h.dims = video.dims;
  h.elem = video.elem_type;
  if (h.elem == ElemType::U8) {
    h.u8.resize(video.data.size());
    std::transform(video.data.begin(), video.data.end(), h.u8.begin(), [](float f) {
      return std::uint8_t(std::clamp(f, 0.0f, 255.0f));
    });
  } else {
    h.f32 = video.data;
  }
  return encode_fpvd(h);
}

VideoData decode_video(const std::string& bytes) {
  HostVideo h = decode_fpvd(bytes);
  VideoData v;
  v.dims = h.dims;
  v.elem_type = h.elem;
  if (h.elem == ElemType::U8)
    v.data.assign(h.u8.begin(), h.u8.end());  // float(u8), video.cpp:87
  else
    v.data = std::move(h.f32);
  return v;
}

void write_video_file(const std::string& path, const VideoData& video) {
  std::ofstream out(path, std::ios::binary);
  require(out.good(), ErrorKind::Input, "cannot write video file: " + path);
  const std::string s = encode_video(video);
  out.write(s.data(), std::streamsize(s.size()));
}

VideoData read_video_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  require(in.good(), ErrorKind::Input, "cannot read video file: " + path);
  std::string bytes((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  return decode_video(bytes);
}

SyntheticSceneSpec parse_synth_spec(const std::string& text) {
  nlohmann::ordered_json j;
  try {
    j = nlohmann::ordered_json::parse(text);
  } catch (const nlohmann::ordered_json::exception& e) {
    throw Error(ErrorKind::Input, std::string("synth: bad JSON: ") + e.what());
  }
  SyntheticSceneSpec s;
  s.dims.width = j.value("width", 64);
  s.dims.height = j.value("height", 64);
  s.dims.frames = j.value("frames", 32);
  s.dims.channels = j.value("channels", 4);
  s.dims.fps = j.value("fps", 1);
  s.noise_sigma = j.value("noise_sigma", 0.0);
  s.background = j.value("background", 0.0);
  s.seed = j.value("seed", std::uint64_t(0));
  if (j.contains("markers"))
    for (const auto& jm : j["markers"]) {
      MarkerSpec m;
      m.start_x = jm.value("x", 0.0);
      m.start_y = jm.value("y", 0.0);
      m.vx = jm.value("vx", 0.0);
      m.vy = jm.value("vy", 0.0);
      m.radius = jm.value("radius", 3.0);
      m.intensity = jm.value("intensity", 255.0);
      s.markers.push_back(m);
    }
  return s;
}

namespace {

// Triangle-wave position in [0, limit] (synth.cpp:12-18).
double bounce(double u, double limit) {
  if (limit <= 0.0) return 0.0;
  const double period = 2.0 * limit;
  double m = std::fmod(u, period);
  if (m < 0.0) m += period;
  return m <= limit ? m : period - m;
}

// Fraction of a 4x4 grid of sub-samples of pixel (px, py) inside the disc
// (synth.cpp:21-31).
double coverage(int px, int py, double cx, double cy, double r) {
  int inside = 0;
  for (int sy = 0; sy < 4; ++sy)
    for (int sx = 0; sx < 4; ++sx) {
      double dx = px + (sx + 0.5) / 4.0 - 0.5 - cx;
      double dy = py + (sy + 0.5) / 4.0 - 0.5 - cy;
      inside += dx * dx + dy * dy <= r * r;
    }
  return inside / 16.0;
}

}  // namespace

HostVideo synth_scene(const SyntheticSceneSpec& spec,
                      std::vector<std::vector<std::pair<double, double>>>* truth) {
  spec.dims.validate();
  for (const MarkerSpec& m : spec.markers) {
    require(m.start_x >= 0 && m.start_x <= spec.dims.width - 1 && m.start_y >= 0 &&
                m.start_y <= spec.dims.height - 1,
            ErrorKind::Input, "marker start position outside the frame");
    require(m.radius > 0, ErrorKind::Input, "marker radius must be > 0");
  }
  const VideoDims& d = spec.dims;
  HostVideo v;
  v.dims = d;
  v.elem = ElemType::F32;
  v.f32.assign(std::size_t(d.element_count()), 0.0f);
  if (truth) truth->assign(spec.markers.size(), {});
  std::mt19937_64 rng(spec.seed);
  std::normal_distribution<double> noise(0.0, spec.noise_sigma);
  const std::size_t plane = std::size_t(d.width) * d.height;
  std::vector<std::pair<double, double>> centre(spec.markers.size());
  for (int t = 0; t < d.frames; ++t) {
    for (std::size_t i = 0; i < spec.markers.size(); ++i) {
      const MarkerSpec& m = spec.markers[i];
      centre[i] = {bounce(m.start_x + m.vx * t, d.width - 1.0),
                   bounce(m.start_y + m.vy * t, d.height - 1.0)};
      if (truth) (*truth)[i].push_back(centre[i]);
    }
    for (int y = 0; y < d.height; ++y)
      for (int x = 0; x < d.width; ++x) {
        double level = spec.background;
        for (std::size_t i = 0; i < spec.markers.size(); ++i) {
          const MarkerSpec& m = spec.markers[i];
          double c = coverage(x, y, centre[i].first, centre[i].second, m.radius);
          level = std::max(level, spec.background + c * (m.intensity - spec.background));
        }
        // one normal draw per (t, y, x, c), in that order (synth.cpp:70-74)
        for (int c = 0; c < d.channels; ++c) {
          double val = level;
          if (spec.noise_sigma > 0.0) val += noise(rng);
          v.f32[(std::size_t(t) * d.channels + c) * plane + std::size_t(y) * d.width +
                x] = float(std::clamp(val, 0.0, 255.0));
        }
      }
  }
  return v;
}

}  // namespace fuseplan
