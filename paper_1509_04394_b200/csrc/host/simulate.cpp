// The C++ API's executors (include/fuseplan/simulator.hpp), GPU-backed:
// run_sequential / run_tiled / compare_outputs of the reference
// (/root/reference/proj/src/simulator.cpp:158-368), plus the plan-derived
// traffic tallies and erosion fp_simulate reports.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <span>

#include "../../../include/fuseplan/fuseplan.hpp"
#include "../../../include/fuseplan/simulator.hpp"
#include "exec.hpp"

namespace fuseplan {

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Error(ErrorKind::Internal, std::string(what) + ": " + cudaGetErrorString(e));
}

void ck(int rc, const char* what) {
  if (rc != 0) throw Error(ErrorKind::Internal, std::string(what) + ": " + fc_error_string(rc));
}

struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  void alloc(std::size_t bytes, const char* what) {
    if (p) cudaFree(p);
    p = nullptr;
    ck(cudaMalloc(&p, bytes), what);
  }
};

// sum over the boxes along one axis of (box extent + halo): the staged
// extents of run_group_box's boxes (edge boxes clipped to the video)
std::int64_t axis_sum(int extent, int tile, int halo) {
  std::int64_t s = 0;
  for (int b = 0; b < extent; b += tile) s += std::min(tile, extent - b) + halo;
  return s;
}

std::int64_t window_volume(const KernelDesc& k) {
  return std::int64_t(k.halo.dx() + 1) * (k.halo.dy() + 1) * (k.halo.dt() + 1);
}

void require_device() {
  int n = 0;
  const cudaError_t e = cudaGetDeviceCount(&n);
  require(e == cudaSuccess && n > 0, ErrorKind::Internal,
          std::string("no CUDA device available: ") + cudaGetErrorString(e));
}

}  // namespace

// ---------------------------------------------------------------- tallies

TrafficCounters sequential_traffic(const Pipeline& p) {  // simulator.cpp:158-177
  TrafficCounters t;
  const std::int64_t px = p.video.pixel_volume();
  for (const KernelDesc& k : p.kernels)
    if (k.scope != KernelScope::GlobalAggregation) {
      t.gmem_reads += px;
      t.gmem_writes += px;
    }
  return t;
}

TrafficCounters tiled_traffic(const FusionPlan& fp, const Pipeline& p) {  // :238-333
  TrafficCounters t;
  const VideoDims& v = p.video;
  const std::int64_t px = v.pixel_volume();
  for (const PlanGroup& g : fp.groups) {
    if (g.global_aggregation) continue;
    std::span<const KernelDesc> members(p.kernels.data() + (g.first - 1),
                                        std::size_t(g.last - g.first + 1));
    if (!g.tiled) {
      for (std::size_t i = 0; i < members.size(); ++i) {
        t.gmem_reads += px;
        t.gmem_writes += px;
      }
      continue;
    }
    const std::int64_t staged = axis_sum(v.width, g.tile.x, g.halo.dx()) *
                                axis_sum(v.height, g.tile.y, g.halo.dy()) *
                                axis_sum(v.frames, g.tile.t, g.halo.dt());
    t.gmem_reads += staged;  // staging the haloed input boxes
    t.smem_writes += staged;
    for (const KernelDesc& k : members) {
      t.smem_reads += staged * window_volume(k);
      t.smem_writes += staged;
    }
    t.gmem_writes += px;  // write-back of the output boxes
    t.smem_reads += px;
  }
  return t;
}

Halo tiling_erosion(const FusionPlan& fp, const Pipeline& p, TileShape* grid,
                    bool* have_grid) {
  Halo e;
  if (have_grid) *have_grid = false;
  for (const PlanGroup& g : fp.groups) {
    if (!g.tiled) continue;
    std::span<const KernelDesc> members(p.kernels.data() + (g.first - 1),
                                        std::size_t(g.last - g.first + 1));
    const Halo cum = fused_halo(members, HaloMode::Cumulative);
    e.x_lo = std::max(e.x_lo, cum.x_lo - g.halo.x_lo);
    e.x_hi = std::max(e.x_hi, cum.x_hi - g.halo.x_hi);
    e.y_lo = std::max(e.y_lo, cum.y_lo - g.halo.y_lo);
    e.y_hi = std::max(e.y_hi, cum.y_hi - g.halo.y_hi);
    e.t_lo = std::max(e.t_lo, cum.t_lo - g.halo.t_lo);
    e.t_hi = std::max(e.t_hi, cum.t_hi - g.halo.t_hi);
    if (have_grid && !*have_grid) {
      *grid = g.tile;
      *have_grid = true;
    }
  }
  return e;
}

bool tiling_erodes(const FusionPlan& fp, const Pipeline& p) {
  const Halo e = tiling_erosion(fp, p, nullptr, nullptr);
  if (e.x_lo > 0 || e.x_hi > 0 || e.y_lo > 0 || e.y_hi > 0 || e.t_lo > 0 || e.t_hi > 0)
    return true;
  for (const PlanGroup& g : fp.groups) {
    if (!g.tiled) continue;
    for (int id = g.first; id <= g.last; ++id)
      if (p.kernels[std::size_t(id - 1)].stencil_op == "iir_temporal" &&
          (g.tile.t < p.video.frames || g.halo.t_lo > 0))
        return true;  // the IIR restarts per box
  }
  return false;
}

// ---------------------------------------------------------------- compare

DiffReport compare_outputs(const VideoData& a, const VideoData& b, const Halo& erode,
                           const TileShape* tile_grid) {
  require(a.dims.width == b.dims.width && a.dims.height == b.dims.height &&
              a.dims.frames == b.dims.frames && a.dims.channels == b.dims.channels,
          ErrorKind::Input, "compare_outputs: dimension mismatch");
  const TileShape grid = tile_grid ? *tile_grid
                                   : TileShape{a.dims.width, a.dims.height, a.dims.frames};
  auto interior_1d = [](int c, int extent, int step, int lo, int hi) {
    const int start = (c / step) * step;
    const int end = std::min(start + step, extent);
    return (c - start) >= lo && (end - 1 - c) >= hi;
  };
  DiffReport r;
  for (int t = 0; t < a.dims.frames; ++t)
    for (int c = 0; c < a.dims.channels; ++c)
      for (int y = 0; y < a.dims.height; ++y)
        for (int x = 0; x < a.dims.width; ++x) {
          const float d = std::abs(a.at(x, y, t, c) - b.at(x, y, t, c));
          if (d == 0.0f) continue;
          r.max_abs_diff = std::max(r.max_abs_diff, d);
          ++r.diff_count;
          const bool in = interior_1d(x, a.dims.width, grid.x, erode.x_lo, erode.x_hi) &&
                          interior_1d(y, a.dims.height, grid.y, erode.y_lo, erode.y_hi) &&
                          interior_1d(t, a.dims.frames, grid.t, erode.t_lo, erode.t_hi);
          ++(in ? r.interior_diffs : r.boundary_diffs);
        }
  return r;
}

// ---------------------------------------------------------------- device runs

// run_tiled (simulator.cpp:298-333) on the device: whole-frame groups as
// per-stage kernels, tiled groups through fc_tiled_group's box staging.
void device_run_tiled(const Pipeline& p, const FusionPlan& fp, const void* video, int in_type,
                      float* host_out) {
  require_device();
  const VideoDims& v = p.video;
  const std::int64_t hw = std::int64_t(v.width) * v.height, px = hw * v.frames;
  const std::size_t vbytes = std::size_t(px) * v.channels * (in_type == FC_U8 ? 1 : 4);
  ck(cudaSetDevice(0), "cudaSetDevice");
  DevBuf dvid, da, db, dscr, dst;
  dvid.alloc(vbytes, "cudaMalloc video");
  ck(cudaMemcpy(dvid.p, video, vbytes, cudaMemcpyHostToDevice), "H2D video");
  da.alloc(std::size_t(px) * 4, "cudaMalloc plane");
  db.alloc(std::size_t(px) * 4, "cudaMalloc plane");
  const void* cur = dvid.p;
  int cur_type = in_type, cur_ch = v.channels;
  float* bufs[2] = {static_cast<float*>(da.p), static_cast<float*>(db.p)};
  int which = 0;
  const fc_dims d{v.width, v.height, v.frames};
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  for (const PlanGroup& g : fp.groups) {
    if (g.global_aggregation) continue;
    std::vector<fc_stage> st;
    for (int id = g.first; id <= g.last; ++id)
      st.push_back(make_stage(p.kernels[std::size_t(id - 1)]));
    if (!g.tiled) {
      for (const fc_stage& s : st) {
        float* out = bufs[which];
        if (cur_type == FC_U8 && s.op != FC_RGBA2GRAY) {  // widen a 1-channel u8 input
          fc_stage conv{};
          conv.op = FC_IDENTITY;
          ck(fc_stage_spatial(&conv, cur, FC_U8, out, FC_F32, d, nullptr), "u8 widen");
          cur = out;
          cur_type = FC_F32;
          which ^= 1;
          out = bufs[which];
        }
        if (s.op == FC_IIR_TEMPORAL)
          ck(fc_stage_iir(&s, static_cast<const float*>(cur), out, d, 0, nullptr, nullptr,
                          nullptr),
             "iir");
        else
          ck(fc_stage_spatial(&s, cur, cur_type, out, FC_F32, d, nullptr), "stage");
        cur = out;
        cur_type = FC_F32;
        cur_ch = 1;
        which ^= 1;
      }
      continue;
    }
    const int halo[6] = {g.halo.x_lo, g.halo.x_hi, g.halo.y_lo,
                         g.halo.y_hi, g.halo.t_lo, g.halo.t_hi};
    const int ctas = sms * 4;
    dscr.alloc(std::size_t(fc_tiled_scratch_bytes(g.tile.x, g.tile.y, g.tile.t, halo, cur_ch,
                                                  ctas)),
               "cudaMalloc box scratch");
    dst.alloc(st.size() * sizeof(fc_stage), "cudaMalloc stages");
    ck(cudaMemcpy(dst.p, st.data(), st.size() * sizeof(fc_stage), cudaMemcpyHostToDevice),
       "H2D stages");
    float* out = bufs[which];
    ck(fc_tiled_group(static_cast<const fc_stage*>(dst.p), int(st.size()), cur, cur_type, cur_ch,
                      out, d, g.tile.x, g.tile.y, g.tile.t, halo, static_cast<float*>(dscr.p),
                      ctas, nullptr),
       "tiled group");
    cur = out;
    cur_type = FC_F32;
    cur_ch = 1;
    which ^= 1;
  }
  if (cur_type == FC_U8) {  // no executable stage consumed the video
    std::vector<std::uint8_t> tmp(static_cast<std::size_t>(px));
    ck(cudaMemcpy(tmp.data(), cur, tmp.size(), cudaMemcpyDeviceToHost), "D2H");
    std::transform(tmp.begin(), tmp.end(), host_out, [](std::uint8_t x) { return float(x); });
  } else {
    ck(cudaMemcpy(host_out, cur, std::size_t(px) * 4, cudaMemcpyDeviceToHost), "D2H");
  }
}

SequentialResult run_sequential(const Pipeline& pipeline, const VideoData& video) {
  require(video.dims.width == pipeline.video.width &&
              video.dims.height == pipeline.video.height &&
              video.dims.channels == pipeline.video.channels,
          ErrorKind::Input, "video does not match pipeline dimensions");
  require_device();
  VideoDims vd = video.dims;
  const std::int64_t hw = std::int64_t(vd.width) * vd.height, px = hw * vd.frames;
  SequentialResult r;
  ck(cudaSetDevice(0), "cudaSetDevice");
  DevBuf din, da, db;
  din.alloc(video.data.size() * 4 + 4, "cudaMalloc video");
  ck(cudaMemcpy(din.p, video.data.data(), video.data.size() * 4, cudaMemcpyHostToDevice),
     "H2D video");
  da.alloc(std::size_t(px) * 4 + 4, "cudaMalloc plane");
  db.alloc(std::size_t(px) * 4 + 4, "cudaMalloc plane");
  const float* cur = static_cast<const float*>(din.p);
  float* bufs[2] = {static_cast<float*>(da.p), static_cast<float*>(db.p)};
  int which = 0;
  const fc_dims d{vd.width, vd.height, vd.frames};
  VideoDims od = vd;
  od.channels = 1;
  for (const KernelDesc& k : pipeline.kernels) {
    if (k.scope == KernelScope::GlobalAggregation) continue;  // tracking stage (:168)
    const fc_stage s = make_stage(k);
    float* out = bufs[which];
    if (s.op == FC_IIR_TEMPORAL)
      ck(fc_stage_iir(&s, cur, out, d, 0, nullptr, nullptr, nullptr), "iir");
    else
      ck(fc_stage_spatial(&s, cur, FC_F32, out, FC_F32, d, nullptr), "stage");
    ck(cudaDeviceSynchronize(), "stage");
    VideoData o = VideoData::zeros(od);
    ck(cudaMemcpy(o.data.data(), out, std::size_t(px) * 4, cudaMemcpyDeviceToHost), "D2H stage");
    r.stage_outputs.push_back(std::move(o));
    r.traffic.gmem_reads += px;
    r.traffic.gmem_writes += px;
    ++r.executed_kernels;
    cur = out;
    which ^= 1;
  }
  r.final_output = r.stage_outputs.empty() ? video : r.stage_outputs.back();
  return r;
}

TiledResult run_tiled(const FusionPlan& plan, const Pipeline& pipeline, const VideoData& video) {
  require(video.dims.width == pipeline.video.width &&
              video.dims.height == pipeline.video.height &&
              video.dims.frames == pipeline.video.frames &&
              video.dims.channels == pipeline.video.channels,
          ErrorKind::Input, "video does not match pipeline dimensions");
  require_device();
  TiledResult r;
  VideoDims od = video.dims;
  od.channels = 1;
  r.final_output = VideoData::zeros(od);
  if (tiling_erodes(plan, pipeline)) {
    device_run_tiled(pipeline, plan, video.data.data(), FC_F32, r.final_output.data.data());
  } else {
    Executor ex(pipeline, plan, 0, {});
    const std::size_t n = r.final_output.data.size();
    if (ex.output_type() == FC_U8) {
      std::vector<std::uint8_t> tmp(n);
      ex.run_host(video.data.data(), FC_F32, tmp.data());
      std::transform(tmp.begin(), tmp.end(), r.final_output.data.begin(),
                     [](std::uint8_t x) { return float(x); });
    } else {
      ex.run_host(video.data.data(), FC_F32, r.final_output.data.data());
    }
  }
  r.traffic = tiled_traffic(plan, pipeline);
  return r;
}

}  // namespace fuseplan
