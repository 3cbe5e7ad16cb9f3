// C++ caller of the GPU-backed executors of include/fuseplan/simulator.hpp:
// reads a pipeline, a device profile, plan options and an FPVD video, runs
// run_sequential and run_tiled, writes every stage output and the tiled
// output as raw float32 files into an output directory, and prints the
// compare_outputs report and traffic tallies as one JSON line.
#include <cstdio>
#include <fstream>
#include <sstream>
#include <string>

#include "fuseplan/config.hpp"
#include "fuseplan/planner.hpp"
#include "fuseplan/simulator.hpp"
#include "fuseplan/video.hpp"

using namespace fuseplan;

static std::string slurp(const char* path) {
  std::ifstream in(path);
  std::stringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

static void dump(const std::string& path, const VideoData& v) {
  std::ofstream out(path, std::ios::binary);
  out.write(reinterpret_cast<const char*>(v.data.data()), std::streamsize(v.data.size() * 4));
}

int main(int argc, char** argv) {
  if (argc < 6) return 2;
  try {
    Pipeline p = parse_pipeline(slurp(argv[1]));
    Device d = parse_device(slurp(argv[2]));
    PlanOptions o;
    if (std::string(argv[3]) == "paper-max") o.halo_mode = HaloMode::PaperMax;
    VideoData v = read_video_file(argv[4]);
    const std::string dir = argv[5];
    SequentialResult s = run_sequential(p, v);
    FusionPlan fp = plan(p, d, o);
    TiledResult t = run_tiled(fp, p, v);
    for (std::size_t k = 0; k < s.stage_outputs.size(); ++k)
      dump(dir + "/stage" + std::to_string(k) + ".f32", s.stage_outputs[k]);
    dump(dir + "/tiled.f32", t.final_output);
    TileShape grid;
    bool have = false;
    const Halo er = tiling_erosion(fp, p, &grid, &have);
    DiffReport r = compare_outputs(s.final_output, t.final_output, er, have ? &grid : nullptr);
    std::printf("{\"stages\": %zu, \"diff_count\": %lld, \"interior\": %lld, \"boundary\": %lld, "
                "\"seq_gmem\": %lld, \"tiled_gmem\": %lld, \"executed\": %d}\n",
                s.stage_outputs.size(), (long long)r.diff_count, (long long)r.interior_diffs,
                (long long)r.boundary_diffs, (long long)s.traffic.gmem_total(),
                (long long)t.traffic.gmem_total(), s.executed_kernels);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 0;
}
