// Regenerates tests/golden/random_chains_*.npz inputs: the reference's own
// randomized bit-exactness suites, restated call for call so libstdc++'s
// std::mt19937_64 / uniform_*_distribution produce the same chains and videos
// (proj/tests/helpers.hpp:67-120 random_chain / random_video;
// test_simulator.cpp:228-243 seed 2024 x 25 trials, videos 1000 + trial;
// acceptance.cpp:276-293 seed 606 x 30 trials, videos 7000 + trial).
// Output: one line per trial "suite trial W H F op[,op...]" on stdout and the
// video floats (planar [t][y][x], C = 1) appended to the file named by argv[1].
//
//   g++ -O2 -std=c++17 gen_random_chains.cpp -o /tmp/gen && /tmp/gen videos.f32
#include <cstdio>
#include <random>
#include <string>
#include <vector>

static const char* kOps[7] = {"identity", "scale_offset", "gaussian", "gradient",
                              "threshold", "box_mean", "iir_temporal"};

struct Chain {
  int w, h, f;
  std::vector<int> ops;
};

static Chain random_chain(std::mt19937_64& rng, int max_len = 5) {
  std::uniform_int_distribution<int> dim_pick(0, 3);
  const int sizes[4] = {8, 16, 24, 32};
  Chain c;
  c.w = sizes[dim_pick(rng)];
  c.h = sizes[dim_pick(rng)];
  c.f = sizes[dim_pick(rng)] / 2;
  std::uniform_int_distribution<int> len_pick(2, max_len);
  std::uniform_int_distribution<int> op_pick(0, 6);
  const int len = len_pick(rng);
  for (int i = 0; i < len; ++i) c.ops.push_back(op_pick(rng));  // 6: recurrence allowed
  return c;
}

int main(int argc, char** argv) {
  if (argc < 2) return 1;
  std::FILE* fv = std::fopen(argv[1], "wb");
  const struct { const char* name; unsigned long long seed; int trials, video0; } suites[2] = {
      {"simulator2024", 2024, 25, 1000}, {"acceptance606", 606, 30, 7000}};
  for (const auto& s : suites) {
    std::mt19937_64 rng(s.seed);
    for (int t = 0; t < s.trials; ++t) {
      Chain c = random_chain(rng);
      std::printf("%s %d %d %d %d ", s.name, t, c.w, c.h, c.f);
      for (std::size_t i = 0; i < c.ops.size(); ++i)
        std::printf("%s%s", i ? "," : "", kOps[c.ops[i]]);
      std::printf("\n");
      std::mt19937_64 vr(s.video0 + t);
      std::uniform_real_distribution<float> dist(0.0f, 255.0f);
      std::vector<float> v(std::size_t(c.w) * c.h * c.f);
      for (float& x : v) x = dist(vr);
      std::fwrite(v.data(), sizeof(float), v.size(), fv);
    }
  }
  std::fclose(fv);
  return 0;
}
