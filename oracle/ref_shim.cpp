// TEST INFRASTRUCTURE ONLY.  A thin extern "C" shim over the UNMODIFIED
// reference sources (compiled where they lie under /root/reference by
// oracle/Makefile into oracle/_ref/libfuseplan_ref.so).  Nothing here
// re-implements reference logic: every entry point calls the reference's own
// functions -- parse_pipeline / parse_device (config.cpp:98-190), plan /
// render_plan (planner.cpp:342-442), run_sequential / run_tiled
// (simulator.cpp:158-333), synth_video (synth.cpp:35-78) and the FPVD codec
// (video.cpp:46-94).
//
// ref_run_sequential_strips() runs the reference's run_sequential on
// horizontal row strips in parallel threads (each strip extended by the
// pipeline's cumulative y-halo so the kept rows are exact); it is how the
// bench's reference arm uses every host core without touching the
// reference's code.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "fuseplan/config.hpp"
#include "fuseplan/planner.hpp"
#include "fuseplan/codegen.hpp"
#include "fuseplan/simulator.hpp"
#include "fuseplan/tracking.hpp"
#include "fuseplan/video.hpp"
#include "json.hpp"

using namespace fuseplan;

namespace {

int fail(const std::exception& e, char* err, int errcap, int code) {
  if (err && errcap > 0) {
    std::strncpy(err, e.what(), std::size_t(errcap) - 1);
    err[errcap - 1] = '\0';
  }
  return code;
}

int kind_code(const Error& e) {
  switch (e.kind()) {
    case ErrorKind::Infeasible: return 1;
    case ErrorKind::Input: return 2;
    default: return 3;
  }
}

VideoData make_video(const Pipeline& p, const void* video, int is_u8,
                     int y0 = 0, int rows = -1) {
  VideoDims d = p.video;
  int full_h = d.height;
  if (rows < 0) rows = full_h;
  d.height = rows;
  VideoData v = VideoData::zeros(d, is_u8 ? ElemType::U8 : ElemType::F32);
  std::size_t wh_full = std::size_t(d.width) * full_h;
  for (int t = 0; t < d.frames; ++t)
    for (int c = 0; c < d.channels; ++c)
      for (int y = 0; y < rows; ++y) {
        std::size_t src = (std::size_t(t) * d.channels + c) * wh_full +
                          std::size_t(y0 + y) * d.width;
        for (int x = 0; x < d.width; ++x)
          v.at(x, y, t, c) =
              is_u8 ? float(static_cast<const std::uint8_t*>(video)[src + x])
                    : static_cast<const float*>(video)[src + x];
      }
  return v;
}

}  // namespace

// Plan options in the C ABI's JSON (the reference's parse_plan_options,
// capi.cpp:88-110, restated: that function lives in capi.cpp, which is not
// built here): halo_mode, transfer_variant, force_partition as the
// reference's "1-2,3-5,6" string (or, for older fixtures, [[a, b], ...]),
// tile {x, y, t}.
static PlanOptions shim_options(const char* options_json) {
  PlanOptions opts;
  if (!options_json || !*options_json) return opts;
  auto j = nlohmann::json::parse(options_json);
  if (j.contains("halo_mode"))
    opts.halo_mode = halo_mode_from_string(j["halo_mode"].get<std::string>());
  if (j.contains("transfer_variant"))
    opts.transfer_variant =
        transfer_variant_from_string(j["transfer_variant"].get<std::string>());
  if (j.contains("force_partition")) {
    std::vector<std::pair<int, int>> iv;
    const auto& fpj = j["force_partition"];
    if (fpj.is_string()) {
      std::string str = fpj.get<std::string>(), tok;
      std::size_t pos = 0;
      while (pos <= str.size()) {
        std::size_t c = str.find(',', pos);
        if (c == std::string::npos) c = str.size();
        tok = str.substr(pos, c - pos);
        std::size_t dash = tok.find('-');
        int a = std::stoi(tok.substr(0, dash));
        int b = dash == std::string::npos ? a : std::stoi(tok.substr(dash + 1));
        iv.emplace_back(a, b);
        pos = c + 1;
      }
    } else {
      for (auto& e : fpj) iv.emplace_back(e[0].get<int>(), e[1].get<int>());
    }
    opts.forced_partition = iv;
  }
  if (j.contains("tile"))
    opts.forced_tile = TileShape{j["tile"].value("x", 1), j["tile"].value("y", 1),
                                 j["tile"].value("t", 1)};
  return opts;
}

extern "C" {

// Plan JSON through the reference planner.  Returns 0 / fp_status-like code.
int ref_plan_json(const char* pipeline_json, const char* device_json,
                  const char* options_json, char* out, int cap, char* err,
                  int errcap) {
  try {
    Pipeline p = parse_pipeline(pipeline_json);
    Device d = parse_device(device_json);
    PlanOptions opts = shim_options(options_json);
    std::string s = render_plan(plan(p, d, opts));
    if (int(s.size()) + 1 > cap) return -int(s.size()) - 1;
    std::memcpy(out, s.c_str(), s.size() + 1);
    return 0;
  } catch (const Error& e) {
    return fail(e, err, errcap, kind_code(e));
  } catch (const std::exception& e) {
    return fail(e, err, errcap, 3);
  }
}

// run_sequential on a planar [t][c][y][x] video (u8 or f32).  final_out gets
// the last executed stage ([t][y][x] float); stage_outs (nullable) gets every
// executed stage back to back.  Returns 0 or an error code.
int ref_run_sequential(const char* pipeline_json, const void* video, int is_u8,
                       float* final_out, float* stage_outs, char* err,
                       int errcap) {
  try {
    Pipeline p = parse_pipeline(pipeline_json);
    VideoData v = make_video(p, video, is_u8);
    SequentialResult r = run_sequential(p, v);
    std::memcpy(final_out, r.final_output.data.data(),
                r.final_output.data.size() * sizeof(float));
    if (stage_outs) {
      std::size_t off = 0;
      for (const auto& s : r.stage_outputs) {
        std::memcpy(stage_outs + off, s.data.data(),
                    s.data.size() * sizeof(float));
        off += s.data.size();
      }
    }
    return 0;
  } catch (const Error& e) {
    return fail(e, err, errcap, kind_code(e));
  } catch (const std::exception& e) {
    return fail(e, err, errcap, 3);
  }
}

// The reference's run_sequential over row strips in `nthreads` threads.  The
// pipeline must be frame-local in y except for stencil halos; each strip is
// extended by the cumulative y halo (sum of y_lo / y_hi over the kernels) so
// the kept rows never see a strip edge.  Output: final stage, [t][y][x].
int ref_run_sequential_strips(const char* pipeline_json, const void* video,
                              int is_u8, float* final_out, int nthreads,
                              char* err, int errcap) {
  try {
    Pipeline p = parse_pipeline(pipeline_json);
    int H = p.video.height, W = p.video.width, F = p.video.frames;
    int hlo = 0, hhi = 0;
    for (const auto& k : p.kernels) {
      hlo += k.halo.y_lo;
      hhi += k.halo.y_hi;
    }
    nthreads = std::max(1, std::min(nthreads, H));
    std::vector<std::thread> pool;
    std::vector<std::string> errors(static_cast<std::size_t>(nthreads));
    for (int i = 0; i < nthreads; ++i) {
      int y0 = int(std::int64_t(H) * i / nthreads);
      int y1 = int(std::int64_t(H) * (i + 1) / nthreads);
      pool.emplace_back([&, i, y0, y1] {
        try {
          int e0 = std::max(0, y0 - hlo), e1 = std::min(H, y1 + hhi);
          Pipeline sp = p;
          sp.video.height = e1 - e0;
          VideoData v = make_video(p, video, is_u8, e0, e1 - e0);
          v.dims.height = e1 - e0;
          SequentialResult r = run_sequential(sp, v);
          for (int t = 0; t < F; ++t)
            for (int y = y0; y < y1; ++y)
              std::memcpy(final_out + (std::size_t(t) * H + y) * W,
                          &r.final_output.data[(std::size_t(t) * (e1 - e0) +
                                                (y - e0)) *
                                               W],
                          sizeof(float) * W);
        } catch (const std::exception& e) {
          errors[std::size_t(i)] = e.what();
        }
      });
    }
    for (auto& t : pool) t.join();
    for (auto& e : errors)
      if (!e.empty()) throw Error(ErrorKind::Internal, e);
    return 0;
  } catch (const Error& e) {
    return fail(e, err, errcap, kind_code(e));
  } catch (const std::exception& e) {
    return fail(e, err, errcap, 3);
  }
}

// run_tiled for the plan the reference planner makes; traffic4 gets
// {gmem_reads, gmem_writes, smem_reads, smem_writes}.
// generate_plan_sources (codegen.cpp:425-465): the manifest JSON of the plan
// the options select (the pseudo-CUDA files themselves are not returned).
int ref_codegen_manifest(const char* pipeline_json, const char* device_json,
                         const char* options_json, const char* name, char* out, int cap,
                         char* err, int errcap) {
  try {
    Pipeline p = parse_pipeline(pipeline_json);
    Device d = parse_device(device_json);
    FusionPlan fp = plan(p, d, shim_options(options_json));
    std::string s = generate_plan_sources(fp, p, d, name).manifest_json;
    if (int(s.size()) + 1 > cap) return -int(s.size()) - 1;
    std::memcpy(out, s.c_str(), s.size() + 1);
    return 0;
  } catch (const Error& e) {
    return fail(e, err, errcap, kind_code(e));
  } catch (const std::exception& e) {
    return fail(e, err, errcap, 3);
  }
}

int ref_run_tiled(const char* pipeline_json, const char* device_json,
                  const char* options_json, const void* video, int is_u8,
                  float* final_out, long long* traffic4, char* err,
                  int errcap) {
  try {
    Pipeline p = parse_pipeline(pipeline_json);
    Device d = parse_device(device_json);
    PlanOptions opts = shim_options(options_json);
    FusionPlan fp = plan(p, d, opts);
    VideoData v = make_video(p, video, is_u8);
    TiledResult r = run_tiled(fp, p, v);
    std::memcpy(final_out, r.final_output.data.data(),
                r.final_output.data.size() * sizeof(float));
    if (traffic4) {
      traffic4[0] = r.traffic.gmem_reads;
      traffic4[1] = r.traffic.gmem_writes;
      traffic4[2] = r.traffic.smem_reads;
      traffic4[3] = r.traffic.smem_writes;
    }
    return 0;
  } catch (const Error& e) {
    return fail(e, err, errcap, kind_code(e));
  } catch (const std::exception& e) {
    return fail(e, err, errcap, 3);
  }
}

// synth_video (synth.cpp:35-78) followed by the FPVD u8 round trip
// (video.cpp:46-94, truncating encode), written as planar u8.
int ref_synth_u8(const char* synth_json, std::uint8_t* out, char* err,
                 int errcap) {
  try {
    auto j = nlohmann::json::parse(synth_json);
    SyntheticSceneSpec spec;
    spec.dims.width = j.value("width", 64);
    spec.dims.height = j.value("height", 64);
    spec.dims.frames = j.value("frames", 32);
    spec.dims.channels = j.value("channels", 4);
    spec.noise_sigma = j.value("noise_sigma", 0.0);
    spec.background = j.value("background", 0.0);
    spec.seed = j.value("seed", std::uint64_t(0));
    if (j.contains("markers"))
      for (const auto& jm : j["markers"]) {
        MarkerSpec m;
        m.start_x = jm.value("x", 0.0);
        m.start_y = jm.value("y", 0.0);
        m.vx = jm.value("vx", 0.0);
        m.vy = jm.value("vy", 0.0);
        m.radius = jm.value("radius", 3.0);
        m.intensity = jm.value("intensity", 255.0);
        spec.markers.push_back(m);
      }
    SyntheticScene scene = synth_video(spec);
    VideoData q = decode_video(encode_video(scene.video));
    for (std::size_t i = 0; i < q.data.size(); ++i)
      out[i] = std::uint8_t(q.data[i]);
    return 0;
  } catch (const Error& e) {
    return fail(e, err, errcap, kind_code(e));
  } catch (const std::exception& e) {
    return fail(e, err, errcap, 3);
  }
}

}  // extern "C"
