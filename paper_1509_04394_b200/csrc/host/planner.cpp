// Tiling geometry, the cost model and the partition optimizer.
//
// Contract (what must match the reference bit for bit, because the chosen
// partition decides which fused sm_100a kernels run):
//   * fused_halo / input_box / block_count / DU / transfers  (tiling.cpp:28-212)
//   * optimal_tile: exact-rational DU maximisation, ties -> larger t, then
//     larger x                                                (tiling.cpp:98-145)
//   * predict_cost: Eq 2 with the same double accumulation order
//                                                              (planner.cpp:96-116)
//   * exact min-cost contiguous cover; equal costs resolved by the cut-set
//     bitstring order; DP and branch-and-bound must agree (planner.cpp:158-268)
//   * plan(): forced intervals + optimal runs between them   (planner.cpp:342-393)
// tests/test_planner.py checks render_plan() byte-for-byte against the
// reference planner on 146 cases (tests/golden/plans.json).
#include <algorithm>
#include <cmath>
#include <ctime>
#include <iomanip>
#include <limits>
#include <sstream>

#include "../../../include/fuseplan/fuseplan.hpp"
#include "json.hpp"

namespace fuseplan {

using ordered_json = nlohmann::ordered_json;

namespace {
constexpr double kInf = std::numeric_limits<double>::infinity();
}

// ---------------------------------------------------------------- enums

const char* to_string(HaloMode m) {
  return m == HaloMode::PaperMax ? "paper-max" : "cumulative";
}
const char* to_string(TransferVariant v) {
  return v == TransferVariant::PaperFormula ? "paper" : "exact";
}
HaloMode halo_mode_from_string(const std::string& s) {
  if (s == "paper-max") return HaloMode::PaperMax;
  if (s == "cumulative") return HaloMode::Cumulative;
  throw Error(ErrorKind::Input, "unknown halo mode: " + s);
}
TransferVariant transfer_variant_from_string(const std::string& s) {
  if (s == "paper") return TransferVariant::PaperFormula;
  if (s == "exact") return TransferVariant::ExactVolume;
  throw Error(ErrorKind::Input, "unknown transfer variant: " + s);
}

// ---------------------------------------------------------------- geometry

Halo fused_halo(std::span<const KernelDesc> kernels, HaloMode mode) {
  require(!kernels.empty(), ErrorKind::Input, "fused_halo: empty kernel list");
  Halo acc = kernels[0].halo;
  auto combine = [mode](int& a, int b) {
    a = mode == HaloMode::PaperMax ? std::max(a, b) : a + b;
  };
  for (const KernelDesc& k : kernels.subspan(1)) {
    combine(acc.x_lo, k.halo.x_lo);
    combine(acc.x_hi, k.halo.x_hi);
    combine(acc.y_lo, k.halo.y_lo);
    combine(acc.y_hi, k.halo.y_hi);
    combine(acc.t_lo, k.halo.t_lo);
    combine(acc.t_hi, k.halo.t_hi);
  }
  return acc;
}

Halo fused_halo(const std::vector<KernelDesc>& kernels, HaloMode mode) {
  return fused_halo(std::span<const KernelDesc>(kernels), mode);
}

TileShape input_box(const TileShape& tile, const Halo& halo) {
  return {tile.x + halo.dx(), tile.y + halo.dy(), tile.t + halo.dt()};
}

std::int64_t block_count(const VideoDims& video, const TileShape& tile) {
  require(tile.x >= 1 && tile.y >= 1 && tile.t >= 1, ErrorKind::Input,
          "tile dimensions must be >= 1");
  auto cdiv = [](std::int64_t a, std::int64_t b) { return (a + b - 1) / b; };
  return cdiv(video.width, tile.x) * cdiv(video.height, tile.y) *
         cdiv(video.frames, tile.t);
}

double data_utilization(const TileShape& tile, const Halo& halo) {
  return double(tile.volume()) / double(input_box(tile, halo).volume());
}

double objective_v(const TileShape& tile, const Halo& halo) {
  double side = double(tile.x + halo.dx());
  return side * side * (tile.t + halo.dt());
}

double continuous_seed_x(const Halo& halo, std::int64_t budget) {
  if (halo.dt() == 0) return std::sqrt(double(budget));
  if (halo.dx() == 0) return 1.0;
  return std::cbrt(double(budget) * halo.dx() / halo.dt());
}

TileSearchResult optimal_tile(const Halo& halo, std::int64_t budget,
                              const LaunchLimits& lim, int elem_bytes) {
  require(budget >= 1, ErrorKind::Infeasible, "SHMEM budget below one element");
  // Candidate (x, x, t): t is the largest temporal extent the budget allows
  // for this x.  DU = out / in compared exactly by cross multiplication.
  struct Best {
    bool any = false;
    TileShape tile;
    std::int64_t out = 0, in = 1;
  } best;
  std::int64_t x_cap = std::int64_t(std::sqrt(double(budget))) + 2;
  x_cap = std::min<std::int64_t>(lim.max_x, x_cap);
  for (std::int64_t x = 1; x <= x_cap; ++x) {
    std::int64_t t = lim.constrain_input_box
                         ? budget / ((x + halo.dx()) * (x + halo.dy())) - halo.dt()
                         : budget / (x * x);
    t = std::min<std::int64_t>(t, lim.max_t);
    if (t < lim.min_t) continue;
    TileShape cand{int(x), int(x), int(t)};
    std::int64_t in = input_box(cand, halo).volume();
    std::int64_t used = lim.constrain_input_box ? in : cand.volume();
    if (used > budget) continue;
    std::int64_t out = cand.volume();
    __int128 lhs = (__int128)out * best.in, rhs = (__int128)best.out * in;
    bool take = !best.any || lhs > rhs ||
                (lhs == rhs && std::make_pair(cand.t, cand.x) >
                                   std::make_pair(best.tile.t, best.tile.x));
    if (take) best = {true, cand, out, in};
  }
  require(best.any, ErrorKind::Infeasible, "no feasible tile under SHMEM budget");
  TileSearchResult r;
  r.tile = best.tile;
  r.feasible = true;
  r.du = data_utilization(r.tile, halo);
  r.objective_v = objective_v(r.tile, halo);
  r.smem_bytes_used = input_box(r.tile, halo).volume() * std::int64_t(elem_bytes);
  return r;
}

std::int64_t transfer_serial(int n_kernels, std::int64_t blocks,
                             const TileShape& tile) {
  require(n_kernels >= 1 && blocks >= 1, ErrorKind::Input,
          "transfer_serial: counts must be >= 1");
  return 2 * std::int64_t(n_kernels) * blocks * tile.volume();
}

std::int64_t transfer_fused(std::int64_t blocks, const TileShape& tile,
                            const Halo& halo, TransferVariant variant) {
  require(blocks >= 1, ErrorKind::Input, "transfer_fused: blocks must be >= 1");
  if (variant == TransferVariant::ExactVolume)
    return blocks * (input_box(tile, halo).volume() + tile.volume());
  // The paper's printed formula (SPEC §VI.D), deliberately verbatim: the halo
  // term has no per-block factor and no temporal face.
  std::int64_t face = std::int64_t(tile.x) * halo.dy() +
                      std::int64_t(tile.y) * halo.dx() +
                      std::int64_t(halo.dx()) * halo.dy();
  return 2 * blocks * tile.volume() + face * (tile.t + halo.dt());
}

OccupancyResult occupancy(const Device& d, int threads, std::int64_t smem) {
  require(threads >= 1 && threads <= d.max_threads_per_block, ErrorKind::Input,
          "threads_per_block out of range");
  require(smem <= d.smem_bytes, ErrorKind::Infeasible,
          "block SHMEM request exceeds device capacity");
  std::int64_t lim_smem = smem > 0 ? d.smem_bytes / smem : d.max_blocks_per_sm;
  std::int64_t lim_thr = std::int64_t(d.max_warps_per_sm) * d.warp_size / threads;
  OccupancyResult r;
  r.blocks_per_sm =
      int(std::min({lim_smem, std::int64_t(d.max_blocks_per_sm), lim_thr}));
  std::int64_t warps = (threads + d.warp_size - 1) / d.warp_size;
  r.occupancy = std::clamp(double(r.blocks_per_sm * warps) / d.max_warps_per_sm,
                           0.0, 1.0);
  return r;
}

BufferReport gmem_buffers(const Pipeline& p,
                          const std::vector<std::pair<int, int>>& part) {
  require(!part.empty(), ErrorKind::Input, "empty partition");
  int next = 1;
  for (auto [a, b] : part) {
    require(a == next && b >= a && b <= p.size(), ErrorKind::Input,
            "partition does not cover 1..n");
    next = b + 1;
  }
  require(next == p.size() + 1, ErrorKind::Input, "partition does not cover 1..n");
  BufferReport r;
  std::int64_t px = p.video.pixel_volume();
  r.buffers = int(part.size()) + 1;
  r.bytes = px * p.kernels.front().in_bytes_per_elem;
  for (auto [a, b] : part) r.bytes += px * p.kernels[b - 1].out_bytes_per_elem;
  return r;
}

// ---------------------------------------------------------------- cost model

int group_elem_bytes(std::span<const KernelDesc> kernels) {
  int w = 1;
  for (const KernelDesc& k : kernels)
    w = std::max({w, k.in_bytes_per_elem, k.out_bytes_per_elem});
  return w;
}

CostBreakdown predict_cost(std::span<const KernelDesc> kernels,
                           const TileShape& tile, const Halo& halo,
                           const Device& device, const VideoDims& video) {
  const CostParams& cp = device.cost;
  std::int64_t blocks = block_count(video, tile);
  double out = double(blocks * tile.volume());
  double in = double(blocks * input_box(tile, halo).volume());
  CostBreakdown c;
  c.t_access = cp.gmem_cost_per_elem * in;
  c.t_write = cp.gmem_cost_per_elem * out;
  for (const KernelDesc& k : kernels) {
    double window =
        double(k.halo.dx() + 1) * (k.halo.dy() + 1) * (k.halo.dt() + 1);
    c.t_compute += cp.compute_cost_unit * k.compute_weight * out;
    c.t_compute += cp.smem_cost_per_elem * out * (window + 1.0);
  }
  c.launch = cp.launch_overhead;
  return c;
}

// ---------------------------------------------------------------- B200 streaming cost
// (extension; see StreamingCost in fuseplan.hpp)

bool uses_streaming_cost(const Device& dev, const PlanOptions& opt) {
  using CM = PlanOptions::CostModel;
  if (opt.cost_model == CM::Reference) return false;
  if (opt.cost_model == CM::Streaming)
    require(dev.streaming.has_value(), ErrorKind::Input,
            "cost_model 'streaming' needs a device profile with streaming_cost");
  return dev.streaming.has_value();
}

namespace {
double kparam(const KernelDesc& k, const char* key, double dflt) {
  auto it = k.params.find(key);
  return it == k.params.end() ? dflt : it->second;
}
}  // namespace

// The launch group the executor (exec.cpp) builds for this interval, and for
// the fused classes whether the certified FP32 kernel applies (fc_common.cuh
// fast_params / stencil_params: IIR alpha in [0, 1], gaussian r = 2, a
// {0, 255} byte mask, th > 0).
std::string streaming_class_of(std::span<const KernelDesc> ks, int first_id,
                               const VideoDims& video) {
  std::vector<std::string> ops;
  for (const KernelDesc& k : ks) ops.push_back(k.stencil_op);
  using V = std::vector<std::string>;
  auto certified_tail = [&](const KernelDesc& g, const KernelDesc& t) {
    return int(kparam(g, "radius", 2)) == 2 && kparam(t, "th", 128.0) > 0.0 &&
           kparam(t, "white", 255.0) == 255.0 && kparam(t, "black", 0.0) == 0.0;
  };
  const bool reads_video = first_id == 1;
  if (reads_video && video.channels == 4 &&
      ops == V{"rgba2gray", "iir_temporal", "gaussian", "gradient", "threshold"}) {
    const int r = int(kparam(ks[2], "radius", 2));
    if (r >= 1 && r <= 3)
    {
      // the frame pipeline takes any alpha in [0, 1] and any width (a pitched
      // copy of the video when the width is not a multiple of 16)
      const float a = float(kparam(ks[1], "alpha", 0.5));
      return a >= 0.0f && a <= 1.0f && certified_tail(ks[2], ks[4]) ? "chain" : "chain_exact";
    }
  }
  if (reads_video && ops == V{"rgba2gray", "iir_temporal"}) return "gray_iir";
  if (ops == V{"gaussian", "gradient", "threshold"})
    return certified_tail(ks[0], ks[2]) && video.width % 4 == 0 ? "gauss_grad_thr"
                                                                 : "gauss_grad_thr_exact";
  return "stages";
}

namespace {

CostBreakdown streaming_cost(std::span<const KernelDesc> ks, int first_id, const Device& dev,
                             const VideoDims& video) {
  const StreamingCost& sc = *dev.streaming;
  const double px = double(video.pixel_volume());
  CostBreakdown c;
  if (std::any_of(ks.begin(), ks.end(), [](const KernelDesc& k) {
        return k.scope == KernelScope::GlobalAggregation;
      })) {
    c.launch = sc.launch_ns;  // the host-side tracking stage: one pass
    return c;
  }
  const std::string cls = streaming_class_of(ks, first_id, video);
  if (cls == "stages") {
    for (const KernelDesc& k : ks) {
      c.t_compute += px * sc.rate(k.stencil_op);
      c.launch += sc.launch_ns;
    }
  } else {
    c.t_compute = px * sc.rate(cls);
    c.launch = sc.launch_ns;
  }
  return c;
}

bool any_recurrence(std::span<const KernelDesc> ks) {
  return std::any_of(ks.begin(), ks.end(), [](const KernelDesc& k) {
    return stencil_op_info(k.stencil_op).causal_recurrence;
  });
}

bool any_aggregation(std::span<const KernelDesc> ks) {
  return std::any_of(ks.begin(), ks.end(), [](const KernelDesc& k) {
    return k.scope == KernelScope::GlobalAggregation;
  });
}

struct GroupTile {
  Halo halo;
  TileShape tile;
  std::int64_t smem = 0;
  bool feasible = false;
};

// Staging-box sizing for one candidate group (planner.cpp:56-85): the input
// box must fit SHMEM; a causal recurrence pins t to the whole video.
GroupTile size_group(std::span<const KernelDesc> ks, const Device& dev,
                     const VideoDims& video, const PlanOptions& opt) {
  GroupTile g;
  g.halo = fused_halo(ks, opt.halo_mode);
  int eb = group_elem_bytes(ks);
  if (opt.forced_tile) {
    g.tile = *opt.forced_tile;
    g.smem = input_box(g.tile, g.halo).volume() * eb;
    g.feasible = g.smem <= dev.smem_bytes;
    return g;
  }
  LaunchLimits lim;
  lim.constrain_input_box = true;
  lim.max_x = std::max(video.width, video.height);
  lim.max_t = video.frames;
  if (any_recurrence(ks) && !opt.iir_streaming && !uses_streaming_cost(dev, opt))
    lim.min_t = video.frames;
  try {
    TileSearchResult r = optimal_tile(g.halo, dev.smem_bytes / eb, lim, eb);
    g.tile = r.tile;
    g.smem = r.smem_bytes_used;
    g.feasible = r.feasible;
  } catch (const Error&) {
    g.tile = TileShape{1, 1, 1};
    g.smem = input_box(g.tile, g.halo).volume() * eb;
    g.feasible = false;
  }
  return g;
}

// Cut-set order: bit for boundary i weighs 2^(62-i); a smaller mask is the
// preferred partition at equal cost (fewer / later cuts win).
std::uint64_t cut_bit(int i) { return 1ULL << (62 - i); }

std::vector<std::pair<int, int>> cuts_to_intervals(std::uint64_t mask, int n) {
  std::vector<std::pair<int, int>> iv;
  int lo = 1;
  for (int i = 1; i < n; ++i)
    if (mask & cut_bit(i)) {
      iv.emplace_back(lo, i);
      lo = i + 1;
    }
  iv.emplace_back(lo, n);
  return iv;
}

void check_solver_input(int n) {
  require(n >= 1 && n < 62, ErrorKind::Input, "segment too long");
}

// One occupancy-limited thread block per tile: split the larger side until
// the block fits max_threads_per_block (planner.cpp:40-54).
std::pair<int, int> fold_block(const TileShape& tile, const Device& dev) {
  int tx = tile.x, ty = tile.y;
  while (std::int64_t(tx) * ty > dev.max_threads_per_block) {
    if (tx >= ty)
      tx = (tx + 1) / 2;
    else
      ty = (ty + 1) / 2;
  }
  return {tx, ty};
}

PlanGroup make_group(std::span<const KernelDesc> ks, int first, int last,
                     const Device& dev, const VideoDims& video,
                     const PlanOptions& opt) {
  PlanGroup g;
  g.first = first;
  g.last = last;
  for (const KernelDesc& k : ks) g.kernel_names.push_back(k.name);
  g.global_aggregation = any_aggregation(ks);
  g.tiled = ks.size() > 1 && !g.global_aggregation;
  GroupTile gt = size_group(ks, dev, video, opt);
  require(gt.feasible, ErrorKind::Infeasible,
          "group " + std::to_string(first) + "-" + std::to_string(last) +
              " does not fit SHMEM at any tile");
  g.halo = gt.halo;
  g.tile = gt.tile;
  g.smem_bytes_used = gt.smem;
  g.du = data_utilization(g.tile, g.halo);
  g.cost = uses_streaming_cost(dev, opt) ? streaming_cost(ks, first, dev, video)
                                          : predict_cost(ks, g.tile, g.halo, dev, video);
  g.blocks = block_count(video, g.tile);
  std::tie(g.launch.th_x, g.launch.th_y) = fold_block(g.tile, dev);
  g.launch.th_t = 1;
  g.launch.blocks = g.blocks;
  OccupancyResult occ = occupancy(dev, g.launch.th_x * g.launch.th_y,
                                  g.tiled ? g.smem_bytes_used : 0);
  g.launch.blocks_per_sm = occ.blocks_per_sm;
  g.launch.occupancy = occ.occupancy;
  if (g.tiled) {
    g.transfer_paper =
        transfer_fused(g.blocks, g.tile, g.halo, TransferVariant::PaperFormula);
    g.transfer_exact =
        transfer_fused(g.blocks, g.tile, g.halo, TransferVariant::ExactVolume);
  } else if (!g.global_aggregation) {
    g.transfer_paper = g.transfer_exact =
        transfer_serial(int(ks.size()), g.blocks, g.tile);
  }
  return g;
}

}  // namespace

std::vector<CandidateFusedKernel> enumerate_candidates(
    const FusibleSegment& seg, const Device& dev, const VideoDims& video,
    const PlanOptions& opt) {
  const int n = seg.size();
  std::vector<CandidateFusedKernel> cands;
  cands.reserve(std::size_t(n) * (n + 1) / 2);
  for (int a = 1; a <= n; ++a)
    for (int b = a; b <= n; ++b) {
      std::span<const KernelDesc> ks(seg.kernels.data() + (a - 1),
                                     std::size_t(b - a + 1));
      CandidateFusedKernel c;
      c.first = seg.first_id + a - 1;
      c.last = seg.first_id + b - 1;
      c.selector.assign(std::size_t(n), 0);
      std::fill(c.selector.begin() + (a - 1), c.selector.begin() + b, 1);
      GroupTile g = size_group(ks, dev, video, opt);
      c.halo = g.halo;
      c.tile.tile = g.tile;
      c.tile.smem_bytes_used = g.smem;
      // an aggregation kernel never fuses with a neighbour
      c.tile.feasible = g.feasible && !(ks.size() > 1 && any_aggregation(ks));
      c.feasible = c.tile.feasible;
      if (c.feasible) {
        c.tile.du = data_utilization(g.tile, g.halo);
        c.tile.objective_v = objective_v(g.tile, g.halo);
        c.breakdown = uses_streaming_cost(dev, opt)
                          ? streaming_cost(ks, c.first, dev, video)
                          : predict_cost(ks, g.tile, g.halo, dev, video);
        c.cost = c.breakdown.total();
      } else {
        c.cost = kInf;
      }
      cands.push_back(std::move(c));
    }
  return cands;
}

double partition_dp(int n, const std::vector<std::vector<double>>& cost,
                    std::vector<std::pair<int, int>>* out) {
  check_solver_input(n);
  // best[j]: cheapest cover of kernels 1..j; mask[j]: its cut set.
  std::vector<double> best(std::size_t(n) + 1, kInf);
  std::vector<std::uint64_t> mask(std::size_t(n) + 1, 0);
  best[0] = 0.0;
  for (int j = 1; j <= n; ++j)
    for (int i = 0; i < j; ++i) {
      if (std::isinf(best[i])) continue;
      double c = best[i] + cost[i][j - 1];
      if (std::isinf(c)) continue;
      std::uint64_t m = mask[i] | (i > 0 ? cut_bit(i) : 0);
      if (c < best[j] || (c == best[j] && m < mask[j])) {
        best[j] = c;
        mask[j] = m;
      }
    }
  if (out)
    *out = std::isinf(best[n]) ? std::vector<std::pair<int, int>>{}
                               : cuts_to_intervals(mask[n], n);
  return best[n];
}

double partition_branch_and_bound(int n,
                                  const std::vector<std::vector<double>>& cost,
                                  std::vector<std::pair<int, int>>* out) {
  check_solver_input(n);
  // Depth-first over exact covers of the chain: at position p choose the
  // interval [p+1, b].  Prune prefixes strictly worse than the incumbent;
  // equal-cost leaves are ordered by their cut mask.
  struct Search {
    int n;
    const std::vector<std::vector<double>>& cost;
    bool found = false;
    double best = kInf;
    std::uint64_t best_mask = ~0ULL;
    void go(int p, double acc, std::uint64_t m) {
      if (acc > best) return;
      if (p == n) {
        if (!found || acc < best || (acc == best && m < best_mask)) {
          found = true;
          best = acc;
          best_mask = m;
        }
        return;
      }
      for (int b = p + 1; b <= n; ++b) {
        double c = cost[p][b - 1];
        if (!std::isinf(c)) go(b, acc + c, b < n ? (m | cut_bit(b)) : m);
      }
    }
  } s{n, cost};
  s.go(0, 0.0, 0);
  if (out)
    *out = s.found ? cuts_to_intervals(s.best_mask, n)
                   : std::vector<std::pair<int, int>>{};
  return s.found ? s.best : kInf;
}

std::vector<std::pair<int, int>> optimal_partition(const FusibleSegment& seg,
                                                   const Device& dev,
                                                   const VideoDims& video,
                                                   const PlanOptions& opt) {
  const int n = seg.size();
  std::vector<CandidateFusedKernel> cands = enumerate_candidates(seg, dev, video, opt);
  std::vector<std::vector<double>> cost(std::size_t(n),
                                        std::vector<double>(std::size_t(n), kInf));
  auto it = cands.begin();
  for (int a = 0; a < n; ++a)
    for (int b = a; b < n; ++b) cost[a][b] = (it++)->cost;
  std::vector<std::pair<int, int>> dp_iv, bb_iv;
  double dp = partition_dp(n, cost, &dp_iv);
  double bb = partition_branch_and_bound(n, cost, &bb_iv);
  require(!std::isinf(dp), ErrorKind::Infeasible, "no feasible partition for segment");
  require(dp == bb && dp_iv == bb_iv, ErrorKind::Internal,
          "partition solvers disagree");
  for (auto& [a, b] : dp_iv) {
    a += seg.first_id - 1;
    b += seg.first_id - 1;
  }
  return dp_iv;
}

std::vector<std::pair<int, int>> FusionPlan::partition() const {
  std::vector<std::pair<int, int>> p;
  for (const PlanGroup& g : groups) p.emplace_back(g.first, g.last);
  return p;
}

FusionPlan plan(const Pipeline& pipeline, const Device& dev,
                const PlanOptions& opt) {
  pipeline.validate();
  dev.validate();
  FusionPlan fp;
  fp.halo_mode = opt.halo_mode;
  fp.transfer_variant = opt.transfer_variant;
  fp.video = pipeline.video;
  fp.device_name = dev.name;
  fp.streaming_cost = uses_streaming_cost(dev, opt);
  fp.segments = fusible_segments(pipeline);

  const auto& forced = opt.forced_partition;
  if (forced) {  // planner.cpp:315-337
    int prev = 0;
    for (auto [a, b] : *forced) {
      require(a >= 1 && b >= a && b <= pipeline.size(), ErrorKind::Input,
              "invalid interval " + std::to_string(a) + "-" + std::to_string(b));
      require(a > prev, ErrorKind::Input,
              "forced intervals overlap or are out of order");
      prev = b;
      bool inside = std::any_of(
          fp.segments.begin(), fp.segments.end(),
          [&](const FusibleSegment& s) { return a >= s.first_id && b <= s.last_id; });
      require(inside, ErrorKind::Infeasible,
              "forced interval " + std::to_string(a) + "-" + std::to_string(b) +
                  " crosses a KK boundary");
    }
  }

  std::vector<std::pair<int, int>> intervals;
  auto optimise_run = [&](int lo, int hi) {
    if (lo > hi) return;
    FusibleSegment run;
    run.first_id = lo;
    run.last_id = hi;
    run.kernels.assign(pipeline.kernels.begin() + (lo - 1),
                       pipeline.kernels.begin() + hi);
    auto part = optimal_partition(run, dev, pipeline.video, opt);
    intervals.insert(intervals.end(), part.begin(), part.end());
  };
  for (const FusibleSegment& seg : fp.segments) {
    int cursor = seg.first_id;
    if (forced)
      for (auto [a, b] : *forced) {
        if (a < seg.first_id || b > seg.last_id) continue;
        optimise_run(cursor, a - 1);
        intervals.emplace_back(a, b);
        cursor = b + 1;
      }
    optimise_run(cursor, seg.last_id);
  }
  for (auto [a, b] : intervals) {
    std::span<const KernelDesc> ks(pipeline.kernels.data() + (a - 1),
                                   std::size_t(b - a + 1));
    fp.groups.push_back(make_group(ks, a, b, dev, pipeline.video, opt));
  }
  fp.total_cost = 0.0;
  for (const PlanGroup& g : fp.groups) fp.total_cost += g.cost.total();
  fp.buffers = gmem_buffers(pipeline, fp.partition());
  return fp;
}

// Schema-versioned plan document; key order is part of the format
// (planner.cpp:395-442).
std::string render_plan(const FusionPlan& fp) {
  auto halo_json = [](const Halo& h) {
    return ordered_json{{"x_lo", h.x_lo}, {"x_hi", h.x_hi}, {"y_lo", h.y_lo},
                        {"y_hi", h.y_hi}, {"t_lo", h.t_lo}, {"t_hi", h.t_hi}};
  };
  ordered_json doc;
  doc["schema_version"] = 1;
  doc["halo_mode"] = to_string(fp.halo_mode);
  doc["transfer_variant"] = to_string(fp.transfer_variant);
  doc["device"] = fp.device_name;
  if (fp.streaming_cost) doc["cost_model"] = "streaming (B200 executor, ns)";
  doc["video"] = {{"width", fp.video.width},
                  {"height", fp.video.height},
                  {"frames", fp.video.frames},
                  {"channels", fp.video.channels}};
  doc["segments"] = ordered_json::array();
  for (const FusibleSegment& s : fp.segments)
    doc["segments"].push_back({{"first", s.first_id}, {"last", s.last_id}});
  doc["groups"] = ordered_json::array();
  for (const PlanGroup& g : fp.groups) {
    ordered_json jg;
    jg["interval"] = {{"first", g.first}, {"last", g.last}};
    jg["kernels"] = g.kernel_names;
    jg["tiled"] = g.tiled;
    jg["global_aggregation"] = g.global_aggregation;
    jg["halo"] = halo_json(g.halo);
    jg["tile"] = {{"x", g.tile.x}, {"y", g.tile.y}, {"t", g.tile.t}};
    jg["smem_bytes"] = g.smem_bytes_used;
    jg["data_utilization"] = g.du;
    jg["blocks"] = g.blocks;
    jg["launch"] = {{"th_x", g.launch.th_x},
                    {"th_y", g.launch.th_y},
                    {"th_t", g.launch.th_t},
                    {"blocks_per_sm", g.launch.blocks_per_sm},
                    {"occupancy", g.launch.occupancy}};
    jg["cost"] = {{"t_access", g.cost.t_access},
                  {"t_compute", g.cost.t_compute},
                  {"t_write", g.cost.t_write},
                  {"launch", g.cost.launch},
                  {"total", g.cost.total()}};
    jg["transfer_paper"] = g.transfer_paper;
    jg["transfer_exact"] = g.transfer_exact;
    doc["groups"].push_back(std::move(jg));
  }
  doc["total_cost"] = fp.total_cost;
  doc["gmem_buffers"] = {{"count", fp.buffers.buffers},
                         {"bytes", fp.buffers.bytes},
                         {"policy", "one input buffer plus one output buffer per group"}};
  return doc.dump(2) + "\n";
}

// ---------------------------------------------------------------- options
// capi.cpp:54-111: "a" or "a-b" items separated by commas, parsed with stoi.

std::vector<std::pair<int, int>> parse_partition_string(const std::string& s) {
  std::vector<std::pair<int, int>> out;
  std::size_t pos = 0;
  for (;;) {
    std::size_t comma = s.find(',', pos);
    std::string item = s.substr(pos, comma == std::string::npos ? std::string::npos
                                                                 : comma - pos);
    require(!item.empty(), ErrorKind::Input,
            "invalid interval '' in partition '" + s + "'");
    int a = 0, b = 0;
    try {
      std::size_t dash = item.find('-');
      a = std::stoi(item.substr(0, dash));
      b = dash == std::string::npos ? a : std::stoi(item.substr(dash + 1));
    } catch (const std::exception&) {
      throw Error(ErrorKind::Input, "invalid interval " + item);
    }
    require(a >= 1 && b >= a, ErrorKind::Input, "invalid interval " + item);
    out.emplace_back(a, b);
    if (comma == std::string::npos) break;
    pos = comma + 1;
  }
  return out;
}

std::string partition_string(const std::vector<std::pair<int, int>>& p) {
  std::string s;
  for (auto [a, b] : p) {
    if (!s.empty()) s += ',';
    s += std::to_string(a);
    if (b != a) s += "-" + std::to_string(b);
  }
  return s;
}

PlanOptions parse_plan_options(const char* text) {
  PlanOptions o;
  if (text == nullptr || *text == '\0') return o;
  ordered_json j;
  try {
    j = ordered_json::parse(text);
  } catch (const ordered_json::exception& e) {
    throw Error(ErrorKind::Input, std::string("options: bad JSON: ") + e.what());
  }
  // JSON type errors escape as std::exception -> FP_ERR_INTERNAL, as in
  // the reference's guarded() (capi.cpp:36-47).
  if (j.contains("halo_mode"))
    o.halo_mode = halo_mode_from_string(j["halo_mode"].get<std::string>());
  if (j.contains("transfer_variant"))
    o.transfer_variant =
        transfer_variant_from_string(j["transfer_variant"].get<std::string>());
  if (j.contains("force_partition"))
    o.forced_partition =
        parse_partition_string(j["force_partition"].get<std::string>());
  if (j.contains("tile")) {
    const auto& t = j["tile"];
    o.forced_tile = TileShape{t.value("x", 1), t.value("y", 1), t.value("t", 1)};
  }
  if (j.contains("iir_streaming")) o.iir_streaming = j["iir_streaming"].get<bool>();
  if (j.contains("cost_model")) {
    const std::string m = j["cost_model"].get<std::string>();
    if (m == "auto") o.cost_model = PlanOptions::CostModel::Auto;
    else if (m == "reference") o.cost_model = PlanOptions::CostModel::Reference;
    else if (m == "streaming") o.cost_model = PlanOptions::CostModel::Streaming;
    else throw Error(ErrorKind::Input, "unknown cost_model: " + m);
  }
  return o;
}

// ---------------------------------------------------------------- reports
// Text/JSON/CSV renderings for the C ABI's report entry points
// (report.cpp:56-201).  Presentation only.

ReportFormat report_format_from_string(const std::string& s) {
  if (s == "text") return ReportFormat::Text;
  if (s == "json") return ReportFormat::Json;
  if (s == "csv") return ReportFormat::Csv;
  throw Error(ErrorKind::Input, "unknown format: " + s);
}

namespace {

std::string utc_now() {
  std::time_t now = std::time(nullptr);
  std::tm tm{};
  gmtime_r(&now, &tm);
  char buf[32];
  std::strftime(buf, sizeof buf, "%Y-%m-%dT%H:%M:%SZ", &tm);
  return buf;
}

std::string dims_text(const VideoDims& v) {
  std::ostringstream ss;
  ss << v.width << "x" << v.height << "x" << v.frames << " (" << v.channels
     << (v.channels == 1 ? " channel)" : " channels)");
  return ss.str();
}

}  // namespace

std::string analyze_report(const Pipeline& p, const ReportOptions& o) {
  auto bounds = classify_boundaries(p);
  auto segs = fusible_segments(p);
  std::vector<std::pair<int, int>> seg_iv;
  for (const auto& s : segs) seg_iv.emplace_back(s.first_id, s.last_id);
  if (o.format == ReportFormat::Json) {
    ordered_json j;
    j["schema_version"] = 1;
    if (o.timestamp) j["generated"] = utc_now();
    j["video"] = {{"width", p.video.width}, {"height", p.video.height},
                  {"frames", p.video.frames}, {"channels", p.video.channels}};
    j["kernels"] = ordered_json::array();
    for (const auto& k : p.kernels)
      j["kernels"].push_back({{"id", k.id}, {"name", k.name},
                              {"op_type", to_string(k.op_type)},
                              {"scope", to_string(k.scope)}});
    j["boundaries"] = ordered_json::array();
    for (const auto& b : bounds)
      j["boundaries"].push_back({{"consumer", b.consumer_id},
                                 {"dependency", to_string(b.dep_type)},
                                 {"reason", b.reason}});
    j["segments"] = ordered_json::array();
    for (auto [a, b] : seg_iv) j["segments"].push_back({{"first", a}, {"last", b}});
    return j.dump(2) + "\n";
  }
  std::ostringstream ss;
  if (o.format == ReportFormat::Csv) {
    ss << "boundary,producer,consumer,dependency,reason\n";
    for (std::size_t i = 0; i < bounds.size(); ++i)
      ss << i + 1 << ',' << bounds[i].consumer_id - 1 << ',' << bounds[i].consumer_id
         << ',' << to_string(bounds[i].dep_type) << ",\"" << bounds[i].reason << "\"\n";
    return ss.str();
  }
  ss << "dependency analysis\n";
  if (o.timestamp) ss << "generated: " << utc_now() << "\n";
  ss << "video: " << dims_text(p.video) << "\nkernels:\n";
  for (const auto& k : p.kernels)
    ss << "  K" << k.id << "  " << k.name << "  [" << to_string(k.op_type) << ", "
       << to_string(k.scope) << "]\n";
  ss << "boundaries:\n";
  for (const auto& b : bounds)
    ss << "  K" << b.consumer_id - 1 << " -> K" << b.consumer_id << ": "
       << to_string(b.dep_type) << "  (" << b.reason << ")\n";
  ss << "fusible segments: " << partition_string(seg_iv) << "\n";
  return ss.str();
}

std::string plan_report(const FusionPlan& fp, const ReportOptions& o) {
  if (o.format == ReportFormat::Json) return render_plan(fp);
  std::ostringstream ss;
  if (o.format == ReportFormat::Csv) {
    ss << "group,first,last,tiled,tile_x,tile_y,tile_t,smem_bytes,"
          "data_utilization,blocks,occupancy,cost,transfer_paper,transfer_exact\n";
    int i = 0;
    for (const auto& g : fp.groups)
      ss << ++i << ',' << g.first << ',' << g.last << ',' << int(g.tiled) << ','
         << g.tile.x << ',' << g.tile.y << ',' << g.tile.t << ','
         << g.smem_bytes_used << ',' << g.du << ',' << g.blocks << ','
         << g.launch.occupancy << ',' << g.cost.total() << ',' << g.transfer_paper
         << ',' << g.transfer_exact << '\n';
    return ss.str();
  }
  ss << "fusion plan\n";
  if (o.timestamp) ss << "generated: " << utc_now() << "\n";
  ss << "device: " << fp.device_name << "\nvideo: " << dims_text(fp.video)
     << "\nhalo mode: " << to_string(fp.halo_mode)
     << ", transfer variant: " << to_string(fp.transfer_variant)
     << "\npartition: " << partition_string(fp.partition()) << "\n";
  for (const auto& g : fp.groups) {
    ss << "  group K" << g.first << "-K" << g.last << ": ";
    if (g.global_aggregation) {
      ss << "global aggregation stage (runs whole-video)\n";
    } else if (!g.tiled) {
      ss << "whole-frame launch, transfer " << g.transfer_exact << " elems, cost "
         << g.cost.total() << "\n";
    } else {
      ss << "tile " << g.tile.x << "x" << g.tile.y << "x" << g.tile.t << ", halo +"
         << g.halo.dx() << "/+" << g.halo.dy() << "/+" << g.halo.dt() << ", smem "
         << g.smem_bytes_used << " B, DU " << std::fixed << std::setprecision(4)
         << g.du << std::defaultfloat << ", occupancy " << g.launch.occupancy
         << ", cost " << g.cost.total() << "\n    transfers: paper "
         << g.transfer_paper << ", exact " << g.transfer_exact << " elems; blocks "
         << g.blocks << "\n";
    }
  }
  ss << "total predicted cost: " << fp.total_cost << "\ngmem buffers: "
     << fp.buffers.buffers << " (" << fp.buffers.bytes
     << " bytes; policy: one input buffer plus one output buffer per group)\n";
  return ss.str();
}

std::string tile_sweep_csv(const Halo& halo, std::int64_t budget, int max_x,
                           int max_t, ReportFormat fmt) {
  require(max_x >= 1 && max_t >= 1, ErrorKind::Input, "sweep bounds must be >= 1");
  ordered_json rows = ordered_json::array();
  std::ostringstream ss;
  ss << "x,y,t,du,v,feasible\n";
  for (int x = 1; x <= max_x; ++x)
    for (int t = 1; t <= max_t; ++t) {
      TileShape tile{x, x, t};
      bool ok = input_box(tile, halo).volume() <= budget;
      double du = ok ? data_utilization(tile, halo) : 0.0;
      double v = objective_v(tile, halo);
      rows.push_back({{"x", x}, {"y", x}, {"t", t}, {"du", du}, {"v", v},
                      {"feasible", ok}});
      ss << x << ',' << x << ',' << t << ',' << du << ',' << v << ',' << int(ok)
         << '\n';
    }
  return fmt == ReportFormat::Json ? rows.dump(2) + "\n" : ss.str();
}

}  // namespace fuseplan
