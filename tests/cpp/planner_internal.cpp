// C++-level checks of the optimizer internals, modelled on the reference's
// acceptance criteria 1-3 (acceptance.cpp:35-167): DP == branch-and-bound ==
// brute force on random cost tables; n(n+1)/2 candidates; optimal_tile ==
// exhaustive grid search; the continuous seed is stationary.
// Built and run by tests/test_planner_internal.py.
#include <cmath>
#include <cstdio>
#include <limits>
#include <random>

#include "fuseplan/fuseplan.hpp"

using namespace fuseplan;

static int failures = 0;
#define CHECK(c, ...)                      \
  do {                                     \
    if (!(c)) {                            \
      std::printf("FAIL %s: ", #c);        \
      std::printf(__VA_ARGS__);            \
      std::printf("\n");                   \
      ++failures;                          \
    }                                      \
  } while (0)

static double brute(int n, const std::vector<std::vector<double>>& cost,
                    std::vector<std::pair<int, int>>* out) {
  const double inf = std::numeric_limits<double>::infinity();
  double best = inf;
  std::uint64_t best_mask = ~0ULL;
  for (std::uint64_t m = 0; m < (1ULL << (n - 1)); ++m) {
    double total = 0.0;
    std::uint64_t mask = 0;
    int lo = 1;
    bool ok = true;
    for (int i = 1; i <= n && ok; ++i) {
      bool cut = i < n && ((m >> (i - 1)) & 1);
      if (cut || i == n) {
        double c = cost[lo - 1][i - 1];
        if (std::isinf(c)) ok = false;
        total += c;
        if (cut) mask |= 1ULL << (62 - i);
        lo = i + 1;
      }
    }
    if (ok && (total < best || (total == best && mask < best_mask))) {
      best = total;
      best_mask = mask;
    }
  }
  out->clear();
  if (!std::isinf(best)) {
    int lo = 1;
    for (int i = 1; i < n; ++i)
      if (best_mask & (1ULL << (62 - i))) {
        out->emplace_back(lo, i);
        lo = i + 1;
      }
    out->emplace_back(lo, n);
  }
  return best;
}

int main() {
  const double inf = std::numeric_limits<double>::infinity();
  std::mt19937_64 rng(101);
  // 1. solver agreement
  for (int trial = 0; trial < 300; ++trial) {
    int n = 1 + int(rng() % 12);
    std::vector<std::vector<double>> cost(n, std::vector<double>(n, inf));
    for (int a = 0; a < n; ++a)
      for (int b = a; b < n; ++b)
        cost[a][b] = (a != b && rng() % 8 == 0)
                         ? inf
                         : (trial % 3 == 0 ? double(1 + rng() % 4)  // many ties
                                           : 1.0 + double(rng() % 100000) / 1000.0);
    std::vector<std::pair<int, int>> dp_iv, bb_iv, br_iv;
    double dp = partition_dp(n, cost, &dp_iv);
    double bb = partition_branch_and_bound(n, cost, &bb_iv);
    double br = brute(n, cost, &br_iv);
    CHECK(dp == br && bb == br && dp_iv == br_iv && bb_iv == br_iv, "trial %d n=%d",
          trial, n);
  }
  // 2. candidate count
  VideoDims v{64, 64, 8, 1, 1};
  Device d;
  d.name = "t";
  d.smem_bytes = 1 << 24;
  d.sm_count = 13;
  for (int n = 1; n <= 50; ++n) {
    FusibleSegment seg;
    seg.first_id = 1;
    seg.last_id = n;
    for (int i = 1; i <= n; ++i) {
      KernelDesc k;
      k.id = i;
      k.name = "id";
      k.stencil_op = "identity";
      seg.kernels.push_back(k);
    }
    auto c = enumerate_candidates(seg, d, v);
    CHECK(int(c.size()) == n * (n + 1) / 2, "n=%d got %zu", n, c.size());
  }
  // 3. optimal_tile vs exhaustive grid search, continuous seed stationarity
  for (int trial = 0; trial < 60; ++trial) {
    int dx = int(rng() % 9), dt = int(rng() % 5);
    std::int64_t budget = std::int64_t(1) << (8 + rng() % 9);
    Halo h{dx / 2, dx - dx / 2, dx / 2, dx - dx / 2, 0, dt};
    TileSearchResult r = optimal_tile(h, budget);
    double best = 0.0;
    for (std::int64_t x = 1; x * x <= budget; ++x)
      for (std::int64_t t = 1; x * x * t <= budget; ++t)
        best = std::max(best, data_utilization(TileShape{int(x), int(x), int(t)}, h));
    CHECK(r.du == best, "trial %d du %.17g vs %.17g", trial, r.du, best);
    if (dx > 0 && dt > 0) {
      double xs = continuous_seed_x(h, budget);
      double lhs = xs * xs * xs * dt, rhs = double(budget) * dx;
      CHECK(std::abs(lhs - rhs) <= 1e-9 * std::abs(rhs), "seed trial %d", trial);
    }
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
