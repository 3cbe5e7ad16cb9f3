// fuseplan C++ API of the B200 build.
//
// The names, fields and semantics mirror the reference's public C++ surface
// so callers of the reference compile against this header unchanged:
//   descriptors   /root/reference/proj/include/fuseplan/types.hpp:13-128
//   catalog       .../stencil_catalog.hpp:10-33
//   config I/O    .../config.hpp:10-24
//   dependency    .../dependency.hpp:11-40
//   tiling        .../tiling.hpp:15-97
//   planner       .../planner.hpp:12-106
// The implementation is this build's own (model.cpp, planner.cpp); the
// reference's CPU simulator is NOT part of the product -- execution goes to
// the sm_100a kernels through exec.hpp.
#pragma once

#include <cstdint>
#include <map>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace fuseplan {

// ---------------------------------------------------------------- errors
// Input -> FP_ERR_INPUT (2), Infeasible -> FP_ERR_INFEASIBLE (1),
// Internal -> FP_ERR_INTERNAL (3)  (types.hpp:13-27, capi.cpp:23-34).
enum class ErrorKind { Input, Infeasible, Internal };

class Error : public std::runtime_error {
 public:
  Error(ErrorKind kind, const std::string& msg)
      : std::runtime_error(msg), kind_(kind) {}
  ErrorKind kind() const { return kind_; }

 private:
  ErrorKind kind_;
};

inline void require(bool ok, ErrorKind kind, const std::string& msg) {
  if (!ok) throw Error(kind, msg);
}

// ---------------------------------------------------------------- descriptors
struct VideoDims {
  int width = 0;
  int height = 0;
  int frames = 0;
  int fps = 1;
  int channels = 1;
  std::int64_t pixel_volume() const {
    return std::int64_t(width) * height * frames;
  }
  std::int64_t element_count() const { return pixel_volume() * channels; }
  void validate() const;
};

std::int64_t frame_count(std::int64_t duration_seconds, std::int64_t fps);

// Per-side stencil footprint (the data-access-pattern descriptor).
struct Halo {
  int x_lo = 0, x_hi = 0;
  int y_lo = 0, y_hi = 0;
  int t_lo = 0, t_hi = 0;
  int dx() const { return x_lo + x_hi; }
  int dy() const { return y_lo + y_hi; }
  int dt() const { return t_lo + t_hi; }
  bool zero() const { return dx() == 0 && dy() == 0 && dt() == 0; }
  static Halo symmetric(int rx, int ry, int rt = 0) {
    return Halo{rx, rx, ry, ry, rt, rt};
  }
  void validate() const;
  bool operator==(const Halo&) const = default;
};

enum class OperationType {
  SinglePoint,
  Rectangular,
  SingleFrame,
  MultiFrame,
  SpatioTemporal
};
enum class DependencyType { TT, TMT, KK };
enum class KernelScope { TileLocal, GlobalAggregation };

using StencilParams = std::map<std::string, double>;

struct KernelDesc {
  int id = 0;
  std::string name;
  OperationType op_type = OperationType::SinglePoint;
  bool multi_frame = false;
  Halo halo;
  KernelScope scope = KernelScope::TileLocal;
  std::string stencil_op;
  StencilParams params;
  int in_channels = 1;
  int out_channels = 1;
  int in_bytes_per_elem = 4;
  int out_bytes_per_elem = 4;
  double compute_weight = 1.0;
};

struct Pipeline {
  VideoDims video;
  std::vector<KernelDesc> kernels;
  int size() const { return int(kernels.size()); }
  void validate() const;
};

struct CostParams {
  double gmem_cost_per_elem = 100.0;
  double smem_cost_per_elem = 1.0;
  double compute_cost_unit = 1.0;
  double launch_overhead = 10000.0;
  void validate() const;
};

// B200 extension of the device profile (not in the reference): the cost of a
// plan group as THIS build's executor runs it.  The reference's Eq-2 model
// (predict_cost) prices tiles, halos and SHMEM windows; the B200 executor
// streams every group (frame pipeline / time scan / per-stage kernels), so a
// group's time is the launches it takes plus pixels x the measured ns/pixel
// of the kernel class that runs it (calibrated on a B200:
// scripts/calibrate_streaming.py).  Classes: "chain" / "chain_exact" (the
// whole SPEC chain, certified / FP64), "gray_iir", "gauss_grad_thr" /
// "gauss_grad_thr_exact", and one per catalog op for unfused stages.
struct StreamingCost {
  double launch_ns = 0.0;
  std::map<std::string, double> ns_per_px;
  double rate(const std::string& cls) const;
};

struct Device {
  std::string name;
  std::int64_t smem_bytes = 0;
  int sm_count = 0;
  int warp_size = 32;
  int max_threads_per_block = 1024;
  int max_blocks_per_sm = 16;
  int max_warps_per_sm = 64;
  CostParams cost;
  std::optional<StreamingCost> streaming;  // "streaming_cost" (B200 extension)
  void validate() const;
};

const char* to_string(OperationType t);
const char* to_string(DependencyType t);
const char* to_string(KernelScope s);
OperationType operation_type_from_string(const std::string& s);
KernelScope scope_from_string(const std::string& s);

// ---------------------------------------------------------------- catalog
struct StencilOpInfo {
  std::string name;
  int in_channels = 1;
  int out_channels = 1;
  bool causal_recurrence = false;
  bool global_aggregation = false;
};
const StencilOpInfo& stencil_op_info(const std::string& name);
bool stencil_op_known(const std::string& name);
Halo stencil_op_halo(const std::string& name, const StencilParams& params);
double stencil_op_default_weight(const std::string& name,
                                 const StencilParams& params);

// ---------------------------------------------------------------- config I/O
Pipeline parse_pipeline(const std::string& json_text);
Device parse_device(const std::string& json_text);
std::string render_pipeline(const Pipeline& p);
std::string render_device(const Device& d);
Pipeline load_pipeline_file(const std::string& path);
Device load_device_file(const std::string& path_or_name);
std::string read_text_file(const std::string& path);
void write_text_file(const std::string& path, const std::string& text);

// ---------------------------------------------------------------- dependency
struct OperationClass {
  OperationType primary = OperationType::SinglePoint;
  bool single_frame = true;
};
OperationClass classify_operation(const Halo& halo, bool multi_frame);
DependencyType classify_dependency(const KernelDesc& consumer);

struct BoundaryClassification {
  int consumer_id = 0;
  DependencyType dep_type = DependencyType::TT;
  std::string reason;
};
std::vector<BoundaryClassification> classify_boundaries(const Pipeline& p);

struct FusibleSegment {
  int first_id = 0;
  int last_id = 0;
  std::vector<KernelDesc> kernels;
  int size() const { return last_id - first_id + 1; }
};
std::vector<FusibleSegment> fusible_segments(const Pipeline& p);

// ---------------------------------------------------------------- tiling
enum class HaloMode { PaperMax, Cumulative };
enum class TransferVariant { PaperFormula, ExactVolume };
const char* to_string(HaloMode m);
const char* to_string(TransferVariant v);
HaloMode halo_mode_from_string(const std::string& s);
TransferVariant transfer_variant_from_string(const std::string& s);

struct TileShape {
  int x = 1, y = 1, t = 1;
  std::int64_t volume() const { return std::int64_t(x) * y * t; }
  bool operator==(const TileShape&) const = default;
};

Halo fused_halo(std::span<const KernelDesc> kernels, HaloMode mode);
Halo fused_halo(const std::vector<KernelDesc>& kernels, HaloMode mode);
TileShape input_box(const TileShape& tile, const Halo& halo);
std::int64_t block_count(const VideoDims& video, const TileShape& tile);
double data_utilization(const TileShape& tile, const Halo& halo);
double objective_v(const TileShape& tile, const Halo& halo);

struct TileSearchResult {
  TileShape tile;
  double du = 0.0;
  double objective_v = 0.0;
  bool feasible = false;
  std::int64_t smem_bytes_used = 0;
};

struct LaunchLimits {
  int max_x = 1 << 20;
  int max_t = 1 << 20;
  int min_t = 1;
  bool constrain_input_box = false;
};

TileSearchResult optimal_tile(const Halo& halo, std::int64_t budget_elems,
                              const LaunchLimits& limits = {},
                              int elem_bytes = 4);
double continuous_seed_x(const Halo& halo, std::int64_t budget_elems);
std::int64_t transfer_serial(int n_kernels, std::int64_t blocks,
                             const TileShape& tile);
std::int64_t transfer_fused(std::int64_t blocks, const TileShape& tile,
                            const Halo& halo, TransferVariant variant);

struct OccupancyResult {
  int blocks_per_sm = 0;
  double occupancy = 0.0;
};
OccupancyResult occupancy(const Device& device, int threads_per_block,
                          std::int64_t smem_per_block);

struct BufferReport {
  int buffers = 0;
  std::int64_t bytes = 0;
};
BufferReport gmem_buffers(const Pipeline& pipeline,
                          const std::vector<std::pair<int, int>>& partition);

// ---------------------------------------------------------------- planner
struct CostBreakdown {
  double t_access = 0.0;
  double t_compute = 0.0;
  double t_write = 0.0;
  double launch = 0.0;
  double total() const { return t_access + t_compute + t_write + launch; }
};

struct CandidateFusedKernel {
  int first = 0, last = 0;
  std::vector<int> selector;
  Halo halo;
  TileSearchResult tile;
  CostBreakdown breakdown;
  double cost = 0.0;
  bool feasible = false;
};

struct PlanOptions {
  HaloMode halo_mode = HaloMode::Cumulative;
  TransferVariant transfer_variant = TransferVariant::ExactVolume;
  std::optional<std::vector<std::pair<int, int>>> forced_partition;
  std::optional<TileShape> forced_tile;
  // B200 extension (not in the reference; default = reference semantics):
  // the GPU executor streams recurrence groups frame by frame with the IIR
  // state in registers / a carry plane, so a group containing the IIR need not
  // hold the whole time extent in shared memory (planner.cpp select_group_tile
  // otherwise pins t = F, planner.cpp:73 of the reference).
  bool iir_streaming = false;
  // B200 extension: which cost model prices the groups.  Auto = the
  // device's "streaming_cost" when its profile has one (which also lifts the
  // IIR t-pin, as iir_streaming does), else the reference's Eq-2 model;
  // "reference" forces Eq 2 (plans byte-identical to the reference's).
  enum class CostModel { Auto, Reference, Streaming } cost_model = CostModel::Auto;
};

bool uses_streaming_cost(const Device& dev, const PlanOptions& opt);
// Executor kernel class of a contiguous group whose first kernel is `first_id`
// (1 = reads the video), and its cost under the streaming model.
std::string streaming_class_of(std::span<const KernelDesc> ks, int first_id,
                               const VideoDims& video);

struct LaunchConfig {
  int th_x = 1, th_y = 1, th_t = 1;
  std::int64_t blocks = 0;
  int blocks_per_sm = 0;
  double occupancy = 0.0;
};

struct PlanGroup {
  int first = 0, last = 0;
  std::vector<std::string> kernel_names;
  Halo halo;
  TileShape tile;
  bool tiled = false;
  bool global_aggregation = false;
  std::int64_t smem_bytes_used = 0;
  double du = 1.0;
  LaunchConfig launch;
  CostBreakdown cost;
  std::int64_t blocks = 0;
  std::int64_t transfer_paper = 0;
  std::int64_t transfer_exact = 0;
};

struct FusionPlan {
  HaloMode halo_mode = HaloMode::Cumulative;
  TransferVariant transfer_variant = TransferVariant::ExactVolume;
  VideoDims video;
  std::string device_name;
  std::vector<FusibleSegment> segments;
  std::vector<PlanGroup> groups;
  double total_cost = 0.0;
  bool streaming_cost = false;  // B200 extension: groups priced by StreamingCost
  BufferReport buffers;
  std::vector<std::pair<int, int>> partition() const;
};

int group_elem_bytes(std::span<const KernelDesc> kernels);
std::vector<CandidateFusedKernel> enumerate_candidates(
    const FusibleSegment& segment, const Device& device,
    const VideoDims& video, const PlanOptions& options = {});
CostBreakdown predict_cost(std::span<const KernelDesc> kernels,
                           const TileShape& tile, const Halo& halo,
                           const Device& device, const VideoDims& video);
std::vector<std::pair<int, int>> optimal_partition(
    const FusibleSegment& segment, const Device& device,
    const VideoDims& video, const PlanOptions& options = {});
double partition_dp(int n, const std::vector<std::vector<double>>& cost,
                    std::vector<std::pair<int, int>>* out_intervals);
double partition_branch_and_bound(
    int n, const std::vector<std::vector<double>>& cost,
    std::vector<std::pair<int, int>>* out_intervals);
FusionPlan plan(const Pipeline& pipeline, const Device& device,
                const PlanOptions& options = {});
std::string render_plan(const FusionPlan& plan);

// Plan options in the C-ABI JSON form (fuseplan.h:39-45):
// {"halo_mode", "transfer_variant", "force_partition": "1-2,3-5", "tile",
//  "iir_streaming"}.
PlanOptions parse_plan_options(const char* options_json);
std::vector<std::pair<int, int>> parse_partition_string(const std::string& s);
std::string partition_string(const std::vector<std::pair<int, int>>& p);

// ---------------------------------------------------------------- reports
enum class ReportFormat { Text, Json, Csv };
ReportFormat report_format_from_string(const std::string& s);
struct ReportOptions {
  ReportFormat format = ReportFormat::Text;
  bool timestamp = true;
};
std::string analyze_report(const Pipeline& pipeline, const ReportOptions& o);
std::string plan_report(const FusionPlan& plan, const ReportOptions& o);
std::string tile_sweep_csv(const Halo& halo, std::int64_t budget_elems,
                           int max_x, int max_t, ReportFormat fmt);

}  // namespace fuseplan
