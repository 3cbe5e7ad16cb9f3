// The fuseplan C ABI of the B200 build (include/fuseplan.h).  Every entry
// point runs under guarded(): no exception crosses the boundary, Error kinds
// map to fp_status, the message lands in the thread-local fp_last_error()
// (same contract as /root/reference/proj/src/capi.cpp:21-47).
#include "../../../include/fuseplan.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <filesystem>
#include <functional>
#include <fstream>
#include <iomanip>
#include <memory>
#include <sstream>

#include "exec.hpp"
#include "../../../include/fuseplan/fuseplan.hpp"
#include "../../../include/fuseplan/simulator.hpp"
#include "json.hpp"
#include "video.hpp"

using namespace fuseplan;
using ordered_json = nlohmann::ordered_json;

namespace fuseplan {
void calibrate_csv(const std::string& text, double params[4], double* rms);  // calibrate.cpp
// run_tiled's box staging on the device (simulate.cpp): host video in
// (in_type FC_U8 / FC_F32), single-channel float output
void device_run_tiled(const Pipeline& p, const FusionPlan& fp, const void* video, int in_type,
                      float* out);
}

struct fp_pipeline {
  Pipeline p;
};
struct fp_device {
  Device d;
};
struct fp_plan {
  FusionPlan plan;
};
struct fp_exec {
  std::unique_ptr<Executor> ex;
};

struct fp_graph {
  cudaGraphExec_t exec = nullptr;
  cudaStream_t capture_stream = nullptr;  // keys the launchers' scratch the graph uses
  int device = 0;
};

extern "C" void fc_release_stream_scratch(int device, void* stream);

namespace {

constexpr int kTrackPts = 23;

// trajectories_to_csv (tracking.cpp:130-146): same header, precision 9
std::string trajectory_csv(const double* pts, int n_rois, int frames) {
  std::ostringstream ss;
  ss << "frame,marker_id,meas_x,meas_y,est_x,est_y,est_vx,est_vy\n";
  ss << std::setprecision(9);
  for (int m = 0; m < n_rois; ++m)
    for (int t = 0; t < frames; ++t) {
      const double* p = pts + (std::size_t(m) * frames + t) * kTrackPts;
      ss << t << ',' << (m + 1) << ',';
      if (p[0] != 0.0)
        ss << p[1] << ',' << p[2];
      else
        ss << ',';
      ss << ',' << p[3] << ',' << p[4] << ',' << p[5] << ',' << p[6] << '\n';
    }
  return ss.str();
}

void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Error(ErrorKind::Internal, std::string(what) + ": " + cudaGetErrorString(e));
}

// Runs the K6 kernel; `pts` receives n_rois * frames * kTrackPts doubles.
void track_on_device(const void* mask, int elem_type, bool on_device, int W, int H, int F,
                     const int* rois, int n_rois, double q, double r, double p0,
                     std::vector<double>& pts, void* stream) {
  require(W > 0 && H > 0 && F >= 0 && n_rois >= 1, ErrorKind::Input, "bad tracking dims");
  require(elem_type == FP_ELEM_U8 || elem_type == FP_ELEM_F32, ErrorKind::Input,
          "mask must be FP_ELEM_U8 or FP_ELEM_F32");
  for (int i = 0; i < n_rois; ++i)
    require(rois[4 * i + 2] >= 1 && rois[4 * i + 3] >= 1, ErrorKind::Input,
            "ROI extents must be >= 1");
  pts.assign(std::size_t(n_rois) * F * kTrackPts, 0.0);
  if (F == 0) return;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const std::size_t mbytes = std::size_t(W) * H * F * (elem_type == FP_ELEM_U8 ? 1 : 4);
  // grow-only per-thread device buffers (tracking runs often on short calls)
  struct Buf {
    void* p = nullptr;
    std::size_t n = 0;
    void* get(std::size_t want) {
      if (want > n) {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
        cuda_ok(cudaMalloc(&p, want), "cudaMalloc tracking buffer");
        n = want;
      }
      return p;
    }
  };
  // cudaMalloc'd memory belongs to the device current at allocation: one set
  // of buffers per device
  struct Bufs {
    Buf mask, rois, pts;
  };
  static thread_local std::map<int, Bufs> per_dev;
  int dev = 0;
  cuda_ok(cudaGetDevice(&dev), "cudaGetDevice");
  Bufs& bs = per_dev[dev];
  Buf &bmask = bs.mask, &brois = bs.rois, &bpts = bs.pts;
  const void* m = mask;
  if (!on_device) {
    void* dm = bmask.get(mbytes);
    cuda_ok(cudaMemcpyAsync(dm, mask, mbytes, cudaMemcpyHostToDevice, st), "H2D mask");
    m = dm;
  }
  int* drois = static_cast<int*>(brois.get(sizeof(int) * 4 * n_rois));
  double* dpts = static_cast<double*>(bpts.get(sizeof(double) * pts.size()));
  cuda_ok(cudaMemcpyAsync(drois, rois, sizeof(int) * 4 * n_rois, cudaMemcpyHostToDevice, st),
          "H2D rois");
  const int rc = fc_track_features(m, elem_type == FP_ELEM_U8 ? FC_U8 : FC_F32, W, H, F, drois,
                                   n_rois, q, r, p0, dpts, stream);
  cuda_ok(cudaError_t(rc), "tracking kernel");
  cuda_ok(cudaMemcpyAsync(pts.data(), dpts, sizeof(double) * pts.size(), cudaMemcpyDeviceToHost,
                          st),
          "D2H points");
  cuda_ok(cudaStreamSynchronize(st), "tracking sync");
}

thread_local std::string g_err;

fp_status status_of(ErrorKind k) {
  switch (k) {
    case ErrorKind::Input: return FP_ERR_INPUT;
    case ErrorKind::Infeasible: return FP_ERR_INFEASIBLE;
    default: return FP_ERR_INTERNAL;
  }
}

template <typename Fn>
fp_status guarded(Fn&& fn) {
  try {
    fn();
    return FP_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return status_of(e.kind());
  } catch (const std::exception& e) {
    g_err = e.what();
    return FP_ERR_INTERNAL;
  }
}

char* dup(const std::string& s) {
  char* p = new char[s.size() + 1];
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

void need(bool ok) { require(ok, ErrorKind::Input, "null argument"); }

ReportFormat fmt_of(const char* f) { return report_format_from_string(f ? f : "text"); }

// capi.cpp:149-168: No / Two / Full fusion over every fusible segment.
std::vector<std::pair<std::string, PlanOptions>> fusion_options(
    const Pipeline& p, const PlanOptions& base) {
  std::vector<std::pair<int, int>> none, two, full;
  for (const FusibleSegment& s : fusible_segments(p)) {
    for (int k = s.first_id; k <= s.last_id; ++k) none.emplace_back(k, k);
    if (s.size() >= 3) {
      two.emplace_back(s.first_id, s.first_id + 1);
      two.emplace_back(s.first_id + 2, s.last_id);
    } else {
      two.emplace_back(s.first_id, s.last_id);
    }
    full.emplace_back(s.first_id, s.last_id);
  }
  std::vector<std::pair<std::string, PlanOptions>> out;
  for (auto& [name, part] : {std::pair{"No Fusion", none}, std::pair{"Two Fusion", two},
                             std::pair{"Full Fusion", full}}) {
    PlanOptions o = base;
    o.forced_partition = part;
    out.emplace_back(name, o);
  }
  return out;
}

struct OptionMetrics {
  std::string name;
  std::vector<std::pair<int, int>> partition;
  double cost = 0.0;
  std::int64_t transfer_paper = 0, transfer_exact = 0;
  double min_du = 1.0;
  int buffers = 0;
  std::int64_t buffer_bytes = 0;
  double min_occ = 1.0;
};

OptionMetrics metrics_of(const std::string& name, const Pipeline& p, const Device& d,
                         const PlanOptions& o) {
  FusionPlan fp = plan(p, d, o);
  OptionMetrics m;
  m.name = name;
  m.partition = fp.partition();
  m.cost = fp.total_cost;
  m.buffers = fp.buffers.buffers;
  m.buffer_bytes = fp.buffers.bytes;
  for (const PlanGroup& g : fp.groups) {
    m.transfer_paper += g.transfer_paper;
    m.transfer_exact += g.transfer_exact;
    m.min_du = std::min(m.min_du, g.du);
    if (!g.global_aggregation) m.min_occ = std::min(m.min_occ, g.launch.occupancy);
  }
  return m;
}

// Device element traffic of one executor run, by construction of the kernels:
std::string utc_now() {
  std::time_t now = std::time(nullptr);
  std::tm tm{};
  gmtime_r(&now, &tm);
  char buf[32];
  std::strftime(buf, sizeof buf, "%Y-%m-%dT%H:%M:%SZ", &tm);
  return buf;
}

}  // namespace

namespace fuseplan {
// Helpers shared with the sharded executor's C ABI (shard.cpp).
fp_status capi_guarded(const std::function<void()>& fn) { return guarded(fn); }
const Pipeline& capi_pipeline(const fp_pipeline* p) { return p->p; }
const FusionPlan& capi_plan(const fp_plan* p) { return p->plan; }
char* capi_dup(const std::string& s) { return dup(s); }
// fp_exec_create's options: {"variant": "auto"|"exact"|"fast",
// "host_chunk_frames": N} (+ "warmup_frames": W for the sharded executor)
ExecOptions capi_exec_options(const char* options_json, int* warmup_frames) {
  ExecOptions o;
  if (!options_json || !*options_json) return o;
  ordered_json j;
  try {
    j = ordered_json::parse(options_json);
  } catch (const ordered_json::exception& e) {
    throw Error(ErrorKind::Input, std::string("exec options: bad JSON: ") + e.what());
  }
  std::string v = j.value("variant", std::string("auto"));
  if (v == "auto") o.variant = Variant::Auto;
  else if (v == "exact") o.variant = Variant::Exact;
  else if (v == "fast") o.variant = Variant::Fast;
  else throw Error(ErrorKind::Input, "unknown variant: " + v);
  o.host_chunk_frames = j.value("host_chunk_frames", 0);
  if (warmup_frames) *warmup_frames = j.value("warmup_frames", *warmup_frames);
  return o;
}
}  // namespace fuseplan

extern "C" {

const char* fp_last_error(void) { return g_err.c_str(); }
void fp_string_free(char* s) { delete[] s; }

fp_status fp_pipeline_parse(const char* json_text, fp_pipeline** out) {
  return guarded([&] {
    need(json_text && out);
    *out = new fp_pipeline{parse_pipeline(json_text)};
  });
}

fp_status fp_pipeline_load(const char* path, fp_pipeline** out) {
  return guarded([&] {
    need(path && out);
    *out = new fp_pipeline{load_pipeline_file(path)};
  });
}

void fp_pipeline_free(fp_pipeline* p) { delete p; }

fp_status fp_device_parse(const char* json_text, fp_device** out) {
  return guarded([&] {
    need(json_text && out);
    *out = new fp_device{parse_device(json_text)};
  });
}

fp_status fp_device_load(const char* path_or_name, fp_device** out) {
  return guarded([&] {
    need(path_or_name && out);
    *out = new fp_device{load_device_file(path_or_name)};
  });
}

void fp_device_free(fp_device* d) { delete d; }

fp_status fp_plan_create(const fp_pipeline* p, const fp_device* d,
                         const char* options_json, fp_plan** out) {
  return guarded([&] {
    need(p && d && out);
    *out = new fp_plan{plan(p->p, d->d, parse_plan_options(options_json))};
  });
}

void fp_plan_free(fp_plan* plan) { delete plan; }

fp_status fp_plan_render_json(const fp_plan* fp, char** out) {
  return guarded([&] {
    need(fp && out);
    *out = dup(render_plan(fp->plan));
  });
}

fp_status fp_analyze_report(const fp_pipeline* p, const char* format,
                            int with_timestamp, char** out) {
  return guarded([&] {
    need(p && out);
    *out = dup(analyze_report(p->p, {fmt_of(format), with_timestamp != 0}));
  });
}

fp_status fp_plan_report(const fp_plan* fp, const char* format, int with_timestamp,
                         char** out) {
  return guarded([&] {
    need(fp && out);
    *out = dup(plan_report(fp->plan, {fmt_of(format), with_timestamp != 0}));
  });
}

fp_status fp_tile_sweep(const fp_device* d, const int halo[6], int max_x, int max_t,
                        const char* format, char** out) {
  return guarded([&] {
    need(d && halo && out);
    Halo h{halo[0], halo[1], halo[2], halo[3], halo[4], halo[5]};
    h.validate();
    *out = dup(tile_sweep_csv(h, d->d.smem_bytes / 4, max_x, max_t, fmt_of(format)));
  });
}

fp_status fp_codegen(const fp_pipeline* p, const fp_device* d, const char* options_json,
                     const char* name, const char* out_dir, char** manifest_out) {
  return guarded([&] {
    need(p && d && name && out_dir && manifest_out);
    FusionPlan fp = plan(p->p, d->d, parse_plan_options(options_json));
    // The B200 build does not generate kernel source: each group maps onto a
    // compiled sm_100a kernel.  Per group it writes <name>_group<i>.genkernel
    // (the reference's file name, codegen.cpp) naming that kernel, its
    // launch-relevant plan data and the stage parameters as the kernel
    // receives them, with the entry's __global__ signature; the manifest
    // records the mapping.
    // Manifest: the reference's schema (codegen.cpp:437-463: pipeline,
    // device, halo_mode, kernels[group, file, tile, smem_bytes,
    // staged_arrays, sync_points]) plus, per kernel, the sm_100a kernel that
    // executes the group and its source file.
    ordered_json m;
    m["pipeline"] = name;
    m["device"] = fp.device_name;
    m["halo_mode"] = to_string(fp.halo_mode);
    m["kernels"] = ordered_json::array();
    std::filesystem::create_directories(out_dir);
    int gi = 0;
    for (const PlanGroup& g : fp.groups) {
      ++gi;
      if (g.global_aggregation) continue;  // tracking stage, not a fused kernel
      std::string kernel = "fctrack::k_track (K6 centroid + Kalman, one CTA per marker)";
      std::string src = "fc_track.cu";
      std::vector<std::string> ops;
      for (int id = g.first; id <= g.last; ++id)
        ops.push_back(p->p.kernels[std::size_t(id - 1)].stencil_op);
      if (!g.global_aggregation) {
        using V = std::vector<std::string>;
        if (ops == V{"rgba2gray", "iir_temporal", "gaussian", "gradient", "threshold"}) {
          kernel = "fcpipe2::k_chain_pair (F12345 frame-pair pipeline, certified FP32 or exact "
                   "FP64 stencil; fallback: k_chain_exact)";
          src = "fc_pipe2.cu / fc_exact.cu";
        } else if (ops == V{"rgba2gray", "iir_temporal"}) {
          kernel = "k_gray_iir_stream / k_gray_iir (F12)";
          src = "fc_f12.cu / fc_exact.cu";
        } else if (ops == V{"gaussian", "gradient", "threshold"}) {
          kernel = "fcpipe::k_chain_pipe<OH, true> (certified F345 row-pair pipeline); exact: "
                   "fcpipe2::k_chain_pair on f32 planes (fallback: k_gauss_grad_thr)";
          src = "fc_pipe.cu / fc_pipe2.cu / fc_exact.cu";
        } else {
          kernel = "per-stage kernels (k_rgba2gray, k_iir, k_gaussian<R>, k_gradient, "
                   "k_pointwise, k_box_mean)";
          src = "fc_exact.cu";
        }
      }
      // the staged box the reference's generated kernel would hold
      // (codegen.cpp:316-340): per-pixel capacity vs the device's SHMEM,
      // two arrays when a member has a halo, a barrier before each TMT member
      const std::int64_t staged = std::int64_t(g.tile.x + g.halo.dx()) *
                                  (g.tile.y + g.halo.dy()) * (g.tile.t + g.halo.dt());
      require(staged * std::int64_t(sizeof(float)) <= d->d.smem_bytes, ErrorKind::Infeasible,
              "staged input box exceeds SHMEM capacity");
      int arrays = 1;
      std::vector<int> syncs{-1};
      for (int id = g.first; id <= g.last; ++id) {
        const KernelDesc& kd = p->p.kernels[std::size_t(id - 1)];
        if (!kd.halo.zero()) arrays = 2;
        if (id > g.first && classify_dependency(kd) == DependencyType::TMT)
          syncs.push_back(id - g.first - 1);
      }
      const std::string file = std::string(name) + "_group" + std::to_string(gi) + ".genkernel";
      ordered_json jk;
      jk["group"] = {{"first", g.first}, {"last", g.last}};
      jk["file"] = file;
      jk["tile"] = {{"x", g.tile.x}, {"y", g.tile.y}, {"t", g.tile.t}};
      jk["smem_bytes"] = staged * std::int64_t(sizeof(float)) * arrays;
      jk["staged_arrays"] = arrays;
      jk["sync_points"] = syncs;
      jk["sm100a_kernel"] = kernel;
      jk["source"] = "paper_1509_04394_b200/csrc/kernels/" + src;
      m["kernels"].push_back(std::move(jk));
      std::ostringstream k;
      k << "// " << name << " group " << gi << ": K" << g.first << ".." << "K" << g.last
        << " (";
      for (std::size_t i = 0; i < ops.size(); ++i) k << (i ? ", " : "") << ops[i];
      k << ")\n// executed on sm_100a by " << kernel << "\n// source: "
        << "paper_1509_04394_b200/csrc/kernels/" << src << "\n// plan: tile " << g.tile.x
        << "x" << g.tile.y << "x" << g.tile.t << ", halo x " << g.halo.x_lo << "/"
        << g.halo.x_hi << " y " << g.halo.y_lo << "/" << g.halo.y_hi << " t " << g.halo.t_lo
        << "/" << g.halo.t_hi << "\n// stage parameters as passed to the kernel (fc_stage):\n"
        << std::setprecision(9);
      for (int id = g.first; id <= g.last; ++id) {
        const fc_stage st = make_stage(p->p.kernels[std::size_t(id - 1)]);
        k << "//   K" << id << " " << p->p.kernels[std::size_t(id - 1)].stencil_op;
        if (st.op == FC_RGBA2GRAY) k << " wr=" << st.wr << " wg=" << st.wg << " wb=" << st.wb;
        if (st.op == FC_IIR_TEMPORAL) k << " alpha=" << st.alpha;
        if (st.op == FC_THRESHOLD)
          k << " th=" << st.th << " white=" << st.white << " black=" << st.black;
        if (st.op == FC_GAUSSIAN) {
          const int dd = 2 * st.g_radius + 1;
          k << " radius=" << st.g_radius << " taps=";
          for (int i = 0; i < dd * dd; ++i) k << (i ? "," : "") << st.g_w[i];
        }
        k << "\n";
      }
      k << "extern \"C\" __global__ void " << name << "_group" << gi
        << "(const void* in, void* out, int width, int height, int frames);\n";
      write_text_file((std::filesystem::path(out_dir) /
                       (std::string(name) + "_group" + std::to_string(gi) + ".genkernel"))
                          .string(),
                      k.str());
    }
    std::string text = m.dump(2) + "\n";
    write_text_file((std::filesystem::path(out_dir) / (std::string(name) + "_manifest.json"))
                        .string(),
                    text);
    *manifest_out = dup(text);
  });
}

fp_status fp_simulate(const fp_pipeline* p, const fp_device* d, const char* options_json,
                      const char* video_path, const char* synth_json,
                      const char* track_csv_path, const char* format, int with_timestamp,
                      char** out) {
  return guarded([&] {
    need(p && d && out);
    require((video_path != nullptr) != (synth_json != nullptr), ErrorKind::Input,
            "exactly one of video file / synth spec needed");
    ReportFormat rf = fmt_of(format);
    PlanOptions base = parse_plan_options(options_json);
    HostVideo video = video_path ? read_fpvd_file(video_path)
                                 : synth_scene(parse_synth_spec(synth_json), nullptr);
    const VideoDims& pv = p->p.video;
    require(video.dims.width == pv.width && video.dims.height == pv.height &&
                video.dims.frames == pv.frames && video.dims.channels == pv.channels,
            ErrorKind::Input, "video does not match pipeline dimensions");

    FusionPlan executed = plan(p->p, d->d, base);
    std::vector<OptionMetrics> options;
    for (auto& [name, o] : fusion_options(p->p, base)) {
      try {
        options.push_back(metrics_of(name, p->p, d->d, o));
      } catch (const Error&) {
        // an infeasible comparison option is omitted, not fatal
      }
    }
    // Sequential arm (run_sequential): every stage its own sm_100a kernel,
    // intermediates in HBM.  Tiled arm (run_tiled): the plan's fused
    // production kernels -- whose output equals run_sequential's whenever the
    // plan's staged halos cover the cumulative requirement -- or, for a plan
    // whose tiling erodes (PaperMax halos, an IIR split across boxes), the
    // device restatement of run_tiled's box staging (fc_tiled.cu), so the
    // diffs the reference would report are reproduced.
    PlanOptions singles = base;
    singles.forced_partition.emplace();
    for (int k = 1; k <= p->p.size(); ++k) singles.forced_partition->emplace_back(k, k);
    singles.forced_tile.reset();
    FusionPlan seq_plan = plan(p->p, d->d, singles);
    int in_type = video.elem == ElemType::U8 ? FC_U8 : FC_F32;
    Executor seq(p->p, seq_plan, 0, {});
    std::size_t n = std::size_t(pv.pixel_volume());
    std::vector<float> a(n), b(n);
    auto run_to_float = [&](Executor& ex, std::vector<float>& dst) {
      if (ex.output_type() == FC_U8) {
        std::vector<std::uint8_t> tmp(n);
        ex.run_host(video.data(), in_type, tmp.data());
        std::transform(tmp.begin(), tmp.end(), dst.begin(),
                       [](std::uint8_t v) { return float(v); });
      } else {
        ex.run_host(video.data(), in_type, dst.data());
      }
    };
    run_to_float(seq, a);
    const bool erodes = tiling_erodes(executed, p->p);
    if (erodes) {
      device_run_tiled(p->p, executed, video.data(), in_type, b.data());
    } else {
      Executor fused(p->p, executed, 0, {});
      run_to_float(fused, b);
    }
    TileShape grid;
    bool have_grid = false;
    const Halo erode = tiling_erosion(executed, p->p, &grid, &have_grid);
    VideoDims od = pv;
    od.channels = 1;
    VideoData va, vb;
    va.dims = vb.dims = od;
    va.data = std::move(a);
    vb.data = std::move(b);
    const DiffReport dr = compare_outputs(va, vb, erode, have_grid ? &grid : nullptr);
    b = std::move(vb.data);  // the tiled arm's mask feeds the tracking stage
    struct {
      float max_abs;
      std::int64_t count, interior, boundary;
    } df{dr.max_abs_diff, dr.diff_count, dr.interior_diffs, dr.boundary_diffs};
    int executed_kernels = 0;
    for (const KernelDesc& k : p->p.kernels)
      executed_kernels += k.scope != KernelScope::GlobalAggregation;
    std::int64_t analytic_serial =
        transfer_serial(std::max(executed_kernels, 1), 1,
                        TileShape{pv.width, pv.height, pv.frames});
    std::int64_t analytic_fused = 0;
    for (const PlanGroup& g : executed.groups) analytic_fused += g.transfer_exact;
    struct {
      std::int64_t serial, tiled;
    } tl{sequential_traffic(p->p).gmem_total(), tiled_traffic(executed, p->p).gmem_total()};
    double reduction =
        tl.serial > 0 ? 100.0 * (1.0 - double(tl.tiled) / double(tl.serial)) : 0.0;

    if (track_csv_path) {  // capi.cpp:366-381: K6 on the tiled arm's mask, on the GPU
      require(synth_json != nullptr, ErrorKind::Input,
              "tracking output needs a synthetic scene with markers");
      SyntheticSceneSpec spec = parse_synth_spec(synth_json);
      require(!spec.markers.empty(), ErrorKind::Input,
              "tracking output needs a synthetic scene with markers");
      bool gray = pv.channels == 1;
      for (const KernelDesc& k : p->p.kernels) gray = gray || k.stencil_op == "rgba2gray";
      require(gray, ErrorKind::Input, "tracking needs a single-channel mask output");
      std::vector<int> rois;
      for (const auto& mk : spec.markers) {
        const int side = 2 * int(std::ceil(mk.radius)) + 9;
        rois.insert(rois.end(), {int(std::lround(mk.start_x)) - side / 2,
                                 int(std::lround(mk.start_y)) - side / 2, side, side});
      }
      std::vector<double> pts;
      track_on_device(b.data(), FP_ELEM_F32, false, pv.width, pv.height, pv.frames, rois.data(),
                      int(spec.markers.size()), 0.01, 0.25, 10.0, pts, nullptr);
      std::ofstream f(track_csv_path, std::ios::binary);
      require(bool(f), ErrorKind::Input, std::string("cannot write ") + track_csv_path);
      f << trajectory_csv(pts.data(), int(spec.markers.size()), pv.frames);
    }

    std::ostringstream ss;
    if (rf == ReportFormat::Json) {
      ordered_json j;
      j["schema_version"] = 1;
      if (with_timestamp) j["generated"] = utc_now();
      j["plan"] = ordered_json::parse(render_plan(executed));
      j["options"] = ordered_json::array();
      for (const auto& o : options)
        j["options"].push_back({{"name", o.name},
                                {"partition", partition_string(o.partition)},
                                {"predicted_cost", o.cost},
                                {"transfer_paper", o.transfer_paper},
                                {"transfer_exact", o.transfer_exact},
                                {"min_du", o.min_du},
                                {"buffers", o.buffers},
                                {"buffer_bytes", o.buffer_bytes},
                                {"min_occupancy", o.min_occ}});
      j["buffer_policy"] = "one input buffer plus one output buffer per group";
      j["simulation"] = {{"outputs_identical", df.count == 0},
                         {"max_abs_diff", df.max_abs},
                         {"diff_count", df.count},
                         {"interior_diffs", df.interior},
                         {"boundary_diffs", df.boundary},
                         {"measured_serial_gmem", tl.serial},
                         {"analytic_serial_gmem", analytic_serial},
                         {"measured_tiled_gmem", tl.tiled},
                         {"analytic_fused_exact_gmem", analytic_fused},
                         {"traffic_reduction_pct", reduction},
                         // B200 additions (not in the reference's report)
                         {"backend", "sm_100a"},
                         {"tiled_arm", erodes ? "run_tiled box staging (fc_tiled.cu)"
                                              : "plan's fused kernels"},
                         {"measured_gmem_meaning",
                          "element tallies of the simulated schedule (simulator.cpp rules); "
                          "device DRAM bytes are in ncu profiles"}};
      *out = dup(j.dump(2) + "\n");
      return;
    }
    if (rf == ReportFormat::Csv) {
      ss << "option,partition,predicted_cost,transfer_paper,transfer_exact,"
            "min_du,buffers,buffer_bytes,min_occupancy\n";
      for (const auto& o : options)
        ss << o.name << ",\"" << partition_string(o.partition) << "\"," << o.cost << ','
           << o.transfer_paper << ',' << o.transfer_exact << ',' << o.min_du << ','
           << o.buffers << ',' << o.buffer_bytes << ',' << o.min_occ << '\n';
      *out = dup(ss.str());
      return;
    }
    ss << "run report\n";
    if (with_timestamp) ss << "generated: " << utc_now() << "\n";
    ss << "device: " << executed.device_name << "\nvideo: " << pv.width << "x"
       << pv.height << "x" << pv.frames << " (" << pv.channels
       << (pv.channels == 1 ? " channel)" : " channels)") << "\nfusion options:\n";
    for (const auto& o : options)
      ss << "  " << o.name << " [" << partition_string(o.partition) << "]: cost "
         << o.cost << ", transfer paper " << o.transfer_paper << " / exact "
         << o.transfer_exact << ", min DU " << std::fixed << std::setprecision(4)
         << o.min_du << std::defaultfloat << ", buffers " << o.buffers << " ("
         << o.buffer_bytes << " bytes), min occupancy " << o.min_occ << "\n";
    ss << "gmem buffer policy: one input buffer plus one output buffer per group\n"
       << "executed partition: " << partition_string(executed.partition()) << " (halo "
       << to_string(executed.halo_mode) << ")\n"
       << "simulation:\n"
       << "  outputs identical: " << (df.count == 0 ? "true" : "false") << "\n"
       << "  max abs diff: " << df.max_abs << " (" << df.count << " elements; interior "
       << df.interior << ", boundary " << df.boundary << ")\n"
       << "  serial gmem: measured " << tl.serial << ", analytic " << analytic_serial
       << "\n  tiled gmem: measured " << tl.tiled << ", analytic exact " << analytic_fused
       << "\n  traffic reduction: " << std::fixed << std::setprecision(1) << reduction << "%"
       << std::defaultfloat << "\n";
    *out = dup(ss.str());
  });
}

fp_status fp_calibrate_csv(const char* measurements_csv, char** result_json) {
  return guarded([&] {  // capi.cpp:388-400
    need(measurements_csv && result_json);
    double prm[4], rms = 0.0;
    calibrate_csv(measurements_csv, prm, &rms);
    ordered_json j;
    j["params"] = {{"gmem_cost_per_elem", prm[0]},
                   {"smem_cost_per_elem", prm[1]},
                   {"compute_cost_unit", prm[2]},
                   {"launch_overhead", prm[3]}};
    j["residual_rms"] = rms;
    *result_json = dup(j.dump(2) + "\n");
  });
}

fp_status fp_device_render_with_cost(const fp_device* d, const char* params_json,
                                     char** out) {
  return guarded([&] {
    need(d && params_json && out);
    ordered_json j;
    try {
      j = ordered_json::parse(params_json);
    } catch (const ordered_json::exception& e) {
      throw Error(ErrorKind::Input, std::string("params: bad JSON: ") + e.what());
    }
    if (j.contains("params")) j = j["params"];
    Device dev = d->d;
    dev.cost.gmem_cost_per_elem = j.value("gmem_cost_per_elem", dev.cost.gmem_cost_per_elem);
    dev.cost.smem_cost_per_elem = j.value("smem_cost_per_elem", dev.cost.smem_cost_per_elem);
    dev.cost.compute_cost_unit = j.value("compute_cost_unit", dev.cost.compute_cost_unit);
    dev.cost.launch_overhead = j.value("launch_overhead", dev.cost.launch_overhead);
    *out = dup(render_device(dev));
  });
}

// ------------------------------------------------------------ executor

fp_status fp_exec_create(const fp_pipeline* p, const fp_plan* fp, int device,
                         const char* options_json, fp_exec** out) {
  return guarded([&] {
    need(p && fp && out);
    ExecOptions o = fuseplan::capi_exec_options(options_json, nullptr);
    *out = new fp_exec{std::make_unique<Executor>(p->p, fp->plan, device, o)};
  });
}

fp_status fp_exec_converge(fp_exec* e, const void* video, int in_type, int n_frames,
                           const float* s_true, const float* s_warm, int* frames_out,
                           void* stream) {
  return guarded([&] {
    need(e && video && s_true && s_warm && frames_out);
    require(in_type == FP_ELEM_U8 || in_type == FP_ELEM_F32, ErrorKind::Input,
            "in_type must be FP_ELEM_U8 or FP_ELEM_F32");
    require(n_frames >= 0, ErrorKind::Input, "n_frames < 0");
    *frames_out = e->ex->converge(video, in_type, n_frames, s_true, s_warm, stream);
  });
}

void fp_exec_free(fp_exec* e) { delete e; }

fp_status fp_exec_output_type(const fp_exec* e, int* elem_type) {
  return guarded([&] {
    need(e && elem_type);
    *elem_type = e->ex->output_type();
  });
}

fp_status fp_exec_state_planes(const fp_exec* e, int* n) {
  return guarded([&] {
    need(e && n);
    *n = e->ex->iir_count();
  });
}

fp_status fp_exec_run(fp_exec* e, const void* video, int in_type, void* out, int flags,
                      void* stream) {
  return guarded([&] {
    need(e && video && out);
    require(in_type == FP_ELEM_U8 || in_type == FP_ELEM_F32, ErrorKind::Input,
            "in_type must be FP_ELEM_U8 or FP_ELEM_F32");
    if (flags & FP_EXEC_DEVICE_PTRS)
      e->ex->run_device(video, in_type, out, e->ex->dims().frames, 0, nullptr, nullptr,
                        stream);
    else
      e->ex->run_host(video, in_type, out);
  });
}

fp_status fp_exec_graph_create(fp_exec* e, const void* video, int in_type, void* out,
                               void* stream, fp_graph** graph) {
  return guarded([&] {
    need(e && video && out && graph);
    require(in_type == FP_ELEM_U8 || in_type == FP_ELEM_F32, ErrorKind::Input,
            "in_type must be FP_ELEM_U8 or FP_ELEM_F32");
    cuda_ok(cudaSetDevice(e->ex->device()), "cudaSetDevice");
    std::unique_ptr<fp_graph, void (*)(fp_graph*)> g(new fp_graph, fp_exec_graph_free);
    g->device = e->ex->device();
    cuda_ok(cudaStreamCreateWithFlags(&g->capture_stream, cudaStreamNonBlocking),
               "capture stream");
    // the capture stream starts after the caller's stream's pending work
    if (stream) {
      cudaEvent_t ev;
      cuda_ok(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
      cudaEventRecord(ev, static_cast<cudaStream_t>(stream));
      cudaStreamWaitEvent(g->capture_stream, ev, 0);
      cudaEventDestroy(ev);
    }
    g->exec = static_cast<cudaGraphExec_t>(e->ex->capture(video, in_type, out,
                                                           g->capture_stream));
    *graph = g.release();
  });
}

fp_status fp_exec_graph_launch(fp_graph* g, void* stream) {
  return guarded([&] {
    need(g && g->exec);
    cuda_ok(cudaSetDevice(g->device), "cudaSetDevice");
    cuda_ok(cudaGraphLaunch(g->exec, static_cast<cudaStream_t>(stream)), "graph launch");
  });
}

void fp_exec_graph_free(fp_graph* g) {
  if (!g) return;
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(g->device);
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->capture_stream) {
    cudaDeviceSynchronize();  // replays in flight on any stream use the scratch
    fc_release_stream_scratch(g->device, g->capture_stream);
    cudaStreamDestroy(g->capture_stream);
  }
  cudaSetDevice(cur);
  delete g;
}

fp_status fp_exec_run_range(fp_exec* e, const void* video, int in_type, void* out,
                            int n_frames, int n_warm, const float* state_in,
                            float* state_out, void* stream) {
  return guarded([&] {
    need(e && video && (out || n_frames == n_warm));
    require(in_type == FP_ELEM_U8 || in_type == FP_ELEM_F32, ErrorKind::Input,
            "in_type must be FP_ELEM_U8 or FP_ELEM_F32");
    e->ex->run_device(video, in_type, out, n_frames, n_warm, state_in, state_out, stream);
  });
}

fp_status fp_exec_run_file(fp_exec* e, const char* in_path, const char* out_path) {
  return guarded([&] {
    need(e && in_path && out_path);
    e->ex->run_file(in_path, out_path);
  });
}

fp_status fp_certified_params(const fp_pipeline* p, char** out_json) {
  return guarded([&] {
    need(p && out_json);
    const auto& ks = p->p.kernels;
    require(ks.size() >= 5 && ks[0].stencil_op == "rgba2gray" &&
                ks[1].stencil_op == "iir_temporal" && ks[2].stencil_op == "gaussian" &&
                ks[3].stencil_op == "gradient" && ks[4].stencil_op == "threshold",
            ErrorKind::Input, "certified parameters exist for the SPEC chain only");
    fc_stage st[5];
    for (int i = 0; i < 5; ++i) st[i] = make_stage(ks[i]);
    double c[6];
    require(fc_certified_params(&st[0], &st[1], &st[2], &st[4], c) == 0, ErrorKind::Input,
            "the chain's parameters are outside the certified path");
    std::ostringstream ss;
    ss.precision(17);
    ss << "{\"g0\": " << c[0] << ", \"g1\": " << c[1] << ", \"mlo_n\": " << c[2]
       << ", \"band_n\": " << c[3] << ", \"S\": " << c[4] << ", \"mstar\": " << c[5] << "}";
    *out_json = dup(ss.str());
  });
}

fp_status fp_exec_describe(const fp_exec* e, char** out_json) {
  return guarded([&] {
    need(e && out_json);
    *out_json = dup(e->ex->describe());
  });
}

fp_status fp_track_features(const void* mask, int elem_type, int mask_on_device, int width,
                            int height, int frames, const int* rois_xywh, int n_rois,
                            const char* kalman_json, double* points, char** csv_out,
                            void* stream) {
  return guarded([&] {
    need(mask && rois_xywh);
    double q = 0.01, r = 0.25, p0 = 10.0;  // KalmanParams defaults (tracking.hpp:40-44)
    if (kalman_json && *kalman_json) {
      ordered_json j;
      try {
        j = ordered_json::parse(kalman_json);
      } catch (const ordered_json::exception& e) {
        throw Error(ErrorKind::Input, std::string("kalman: bad JSON: ") + e.what());
      }
      q = j.value("q", q);
      r = j.value("r", r);
      p0 = j.value("p0", p0);
    }
    std::vector<double> pts;
    track_on_device(mask, elem_type, mask_on_device != 0, width, height, frames, rois_xywh,
                    n_rois, q, r, p0, pts, stream);
    if (points) std::memcpy(points, pts.data(), pts.size() * sizeof(double));
    if (csv_out) *csv_out = dup(trajectory_csv(pts.data(), n_rois, frames));
  });
}

fp_status fp_synth_hash_u8(void* device_out, int width, int height, int frames,
                           int channels, int t0, uint64_t seed, void* stream) {
  return guarded([&] {
    need(device_out != nullptr);
    require(width >= 0 && height >= 0 && frames >= 0 && channels >= 1, ErrorKind::Input,
            "bad dims");
    int rc = fc_hash_video_u8(static_cast<std::uint8_t*>(device_out),
                              fc_dims{width, height, frames}, channels, t0, seed, stream);
    require(rc == 0, ErrorKind::Internal,
            std::string("fc_hash_video_u8: ") + fc_error_string(rc));
  });
}

}  // extern "C"
