// Host-side video formats either side of the hot path: the FPVD raw planar
// file (/root/reference/proj/src/video.cpp:46-109) and the synthetic marker
// scene generator (/root/reference/proj/src/synth.cpp:35-78).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../../include/fuseplan/fuseplan.hpp"
#include "../../../include/fuseplan/video.hpp"

namespace fuseplan {

// A planar [t][c][y][x] volume.  u8 files keep their bytes; f32 files keep
// floats.  (The reference holds everything as float; the device path reads
// bytes directly, which is what makes the u8 ingest 4x cheaper.)
struct HostVideo {
  VideoDims dims;
  ElemType elem = ElemType::U8;
  std::vector<std::uint8_t> u8;
  std::vector<float> f32;
  const void* data() const {
    return elem == ElemType::U8 ? static_cast<const void*>(u8.data())
                                : static_cast<const void*>(f32.data());
  }
};

std::string encode_fpvd(const HostVideo& v);
HostVideo decode_fpvd(const std::string& bytes);
HostVideo read_fpvd_file(const std::string& path);
void write_fpvd_file(const std::string& path, const HostVideo& v);

struct MarkerSpec {
  double start_x = 0.0, start_y = 0.0;
  double vx = 0.0, vy = 0.0;
  double radius = 3.0;
  double intensity = 255.0;
};

struct SyntheticSceneSpec {
  VideoDims dims;
  std::vector<MarkerSpec> markers;
  double noise_sigma = 0.0;
  double background = 0.0;
  std::uint64_t seed = 0;
};

// Parses the fp_simulate synth JSON (capi.cpp:116-144 field names/defaults).
SyntheticSceneSpec parse_synth_spec(const std::string& json_text);

// Float-valued scene (unrounded, as the reference's synth_video returns) plus
// the exact marker centres per frame.
HostVideo synth_scene(const SyntheticSceneSpec& spec,
                      std::vector<std::vector<std::pair<double, double>>>* truth);

}  // namespace fuseplan
