// Public C++ API: the reference's two executors and the output comparison
// (/root/reference/proj/include/fuseplan/simulator.hpp:10-60), GPU-backed.
//
//   run_sequential  every executable kernel as its own sm_100a kernel over
//                   the whole volume (the paper's "No Fusion" regime), every
//                   stage output kept (stage_outputs[k], bit-identical to the
//                   reference's);
//   run_tiled       the plan's fused partitions: the production kernels when
//                   the plan's staged halos cover the cumulative requirement
//                   (their output is then run_sequential's), the device
//                   restatement of the reference's box staging when they do
//                   not (PaperMax halos, an IIR cut into boxes shorter than
//                   the video), so tile-edge erosion is reproduced;
//   compare_outputs the reference's diff report (simulator.cpp:335-368).
//
// TrafficCounters are the reference's element tallies of the simulated
// schedule (simulator.cpp:158-333 counting rules), computed from the plan's
// geometry.  Both executors need a CUDA device (Error(Internal) otherwise);
// there is no CPU execution path.
#pragma once

#include <cstdint>
#include <vector>

#include "fuseplan/fuseplan.hpp"
#include "fuseplan/video.hpp"

namespace fuseplan {

struct TrafficCounters {
  std::int64_t gmem_reads = 0;
  std::int64_t gmem_writes = 0;
  std::int64_t smem_reads = 0;
  std::int64_t smem_writes = 0;

  std::int64_t gmem_total() const { return gmem_reads + gmem_writes; }
  TrafficCounters& operator+=(const TrafficCounters& o) {
    gmem_reads += o.gmem_reads;
    gmem_writes += o.gmem_writes;
    smem_reads += o.smem_reads;
    smem_writes += o.smem_writes;
    return *this;
  }
};

struct SequentialResult {
  std::vector<VideoData> stage_outputs;  // one per executed kernel
  VideoData final_output;
  TrafficCounters traffic;
  int executed_kernels = 0;  // tile-local kernels only
};

SequentialResult run_sequential(const Pipeline& pipeline, const VideoData& video);

struct TiledResult {
  VideoData final_output;
  TrafficCounters traffic;
};

TiledResult run_tiled(const FusionPlan& plan, const Pipeline& pipeline, const VideoData& video);

struct DiffReport {
  float max_abs_diff = 0.0f;
  std::int64_t diff_count = 0;
  std::int64_t interior_diffs = 0;
  std::int64_t boundary_diffs = 0;
};

// Diffs inside each tile's interior (eroded by `erode` per side) vs near a
// tile boundary; tile_grid null = one tile (the whole video).
DiffReport compare_outputs(const VideoData& a, const VideoData& b, const Halo& erode,
                           const TileShape* tile_grid);

// The plan-derived pieces fp_simulate reports (B200 build helpers).
TrafficCounters sequential_traffic(const Pipeline& pipeline);
TrafficCounters tiled_traffic(const FusionPlan& plan, const Pipeline& pipeline);
// Erosion of the tiled groups' halos vs the cumulative requirement and the
// first tiled group's tile (nullptr when no group is tiled).
Halo tiling_erosion(const FusionPlan& plan, const Pipeline& pipeline, TileShape* grid,
                    bool* have_grid);
// True when run_tiled differs from run_sequential for this plan.
bool tiling_erodes(const FusionPlan& plan, const Pipeline& pipeline);

}  // namespace fuseplan
