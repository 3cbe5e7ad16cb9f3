// GPU executor: maps the groups of a FusionPlan onto sm_100a kernel
// variants and runs them over a device- or host-resident video.
//
// This is the B200 replacement for the reference's executors
// run_sequential / run_tiled (/root/reference/proj/src/simulator.cpp:158-333):
// a plan group of the SPEC chain becomes ONE fused kernel (F12, F345 or the
// streaming F12345); any other contiguous interval runs as its member stages
// back to back (the paper's "No Fusion" regime), so every partition the
// optimizer can return maps to device code.  There is no CPU fallback: a
// missing device or a launch failure is an Error(Internal).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../kernels/fc_kernels.h"
#include "../../../include/fuseplan/fuseplan.hpp"

namespace fuseplan {

enum class Variant { Auto = 0, Exact = 1, Fast = 2 };

struct ExecOptions {
  Variant variant = Variant::Auto;
  int host_chunk_frames = 0;  // 0 = auto; frames per H2D/compute/D2H chunk
};

// One launch unit of the executor.
struct LaunchGroup {
  int first = 0, last = 0;           // kernel ids (1-based, inclusive)
  enum Kind { Stages, GrayIir, GaussGradThr, Chain } kind = Stages;
  std::vector<fc_stage> stages;      // executed member stages
  bool reads_video = false;          // input is the video (else f32 planes)
  bool has_iir = false;
  int out_type = FC_F32;
  const char* kernel_name() const;
};

class Executor {
 public:
  Executor(const Pipeline& p, const FusionPlan& plan, int device,
           const ExecOptions& opt);
  ~Executor();
  Executor(const Executor&) = delete;
  Executor& operator=(const Executor&) = delete;

  int output_type() const { return out_type_; }
  const VideoDims& dims() const { return dims_; }
  int iir_count() const { return n_iir_; }

  // Device pointers.  video holds n_frames frames starting at the first
  // processed frame; the first n_warm are warm-up frames (IIR state only);
  // out receives n_frames - n_warm frames.  state_in / state_out: n_iir W*H
  // planes (nullable).  Asynchronous on `stream`.
  void run_device(const void* video, int in_type, void* out, int n_frames,
                  int n_warm, const float* state_in, float* state_out,
                  void* stream);

  // Host pointers (pinned or pageable): the video is streamed through the
  // device in frame chunks, the IIR state carried exactly from chunk to
  // chunk, H2D / compute / D2H of neighbouring chunks overlapped on two
  // streams.  Synchronous.
  void run_host(const void* video, int in_type, void* out);

  // FPVD file -> FPVD file (video.cpp:46-109 layout), streamed: chunks of
  // frames are read from disk into pinned buffers while the previous chunk
  // is on the GPU, the IIR carried exactly between chunks, the output
  // (1 channel, u8 mask or f32 planes) written as chunks complete.  The
  // video never has to fit in host memory.  Synchronous.
  void run_file(const std::string& in_path, const std::string& out_path);

  // T-shard carry check: video holds the shard's n_frames frames (device);
  // s_true / s_warm: the true carry and the warm state the shard started
  // from.  Returns how many leading frames of the shard differ (0 = none,
  // n_frames = the end state differs too); synchronous.  Needs a chain whose
  // IIR is its first stage or follows a single rgba2gray (else Input error).
  int converge(const void* video, int in_type, int n_frames, const float* s_true,
               const float* s_warm, void* stream);

  // CUDA graph of one whole run on fixed device buffers (run_device over all
  // frames): one uncaptured run first (every lazy allocation, plan and
  // kernel attribute is settled outside the capture), then the run captured
  // on `stream` and instantiated.  Returns the cudaGraphExec_t; replays
  // reuse the buffers, including the launchers' per-stream scratch of
  // `stream` -- so the caller owns `stream` for the graph's lifetime.
  void* capture(const void* video, int in_type, void* out, void* stream);
  int device() const { return device_; }

  std::string describe() const;  // JSON: launch groups and kernels
  std::int64_t launches_per_run() const;

 private:
  void ensure_scratch(std::size_t bytes);
  int device_ = 0;
  fc_knobs knobs_{};  // FUSEPLAN_* launcher knobs, read once at creation
  VideoDims dims_;
  ExecOptions opt_;
  std::vector<LaunchGroup> groups_;
  int out_type_ = FC_F32;
  int n_iir_ = 0;
  void* scratch_ = nullptr;
  std::size_t scratch_bytes_ = 0;
  void* own_stream_ = nullptr;
  // host-pointer streaming (run_host): device staging and copy streams kept
  // across calls (a per-call cudaMalloc / cudaFree of the staging buffers
  // cost tens to hundreds of ms and made end-to-end times erratic)
  void* stage_ = nullptr;
  std::size_t stage_bytes_ = 0;
  void* s_in_ = nullptr;
  void* s_out_ = nullptr;
  int* k_dev_ = nullptr;  // converge() result slot
  // pitched copy of planes 0-2 for the frame pipeline when the width is not a
  // multiple of 16 or the video base is not 16-byte aligned (TMA strides)
  void* pitched_ = nullptr;
  std::size_t pitched_bytes_ = 0;
  std::string last_chain_ = "none";
};

// fc_stage for one kernel descriptor, parameters converted as the
// reference converts them (simulator.cpp:21-106); gaussian taps from
// gaussian_taps().
fc_stage make_stage(const KernelDesc& k);

// simulator.cpp:27-44: taps in double, normalised by the dy-outer/dx-inner
// running sum, rounded to float.
std::vector<float> gaussian_taps(int radius, double sigma);

}  // namespace fuseplan
