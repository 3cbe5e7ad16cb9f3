// Variant dispatch for the streaming all-fused chain (F12345) and the F345
// group, plus the launcher knobs (fc_knobs, read from the environment once
// per executor).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "fc_kernels.h"
#include "fc_common.cuh"

#define FC_CHAIN_ARGS                                                          \
  const fc_stage *sgray, const fc_stage *si, const fc_stage *sg,               \
      const fc_stage *sthr, const void *video, int in_type, int gray_in,       \
      void *out, int out_type, fc_dims d, int n_warm, const float *state_in,   \
      float *state_out, void *stream

extern "C" int fc_chain_exact(FC_CHAIN_ARGS);  // fc_exact.cu: FP64 everywhere
extern "C" int fc_chain_pipe(const fc_stage* sgray, const fc_stage* si, const fc_stage* sg,
                             const fc_stage* sthr, const void* video, int in_type, int gray_in,
                             void* out, int out_type, fc_dims d, int n_warm,
                             const float* state_in, float* state_out, int pitch, int opitch,
                             void* stream);  // fc_pipe.cu: certified, headline
extern "C" int fc_chain_pipe2(const fc_stage* sgray, const fc_stage* si, const fc_stage* sg,
                              const fc_stage* sthr, const void* video, int in_type, int gray_in,
                              void* out, int out_type, fc_dims d, int n_warm,
                              const float* state_in, float* state_out, int pitch, int opitch,
                              void* stream);  // fc_pipe2.cu: certified, frame pairs
extern "C" long long fc_pipe2_recheck_count(void);
extern "C" int fc_chain_pipe2_exact(const fc_stage* sgray, const fc_stage* si,
                                    const fc_stage* sg, const fc_stage* sthr, const void* video,
                                    int in_type, int gray_in, void* out, int out_type, fc_dims d,
                                    int n_warm, const float* state_in, float* state_out,
                                    int pitch, int opitch, void* stream);  // fc_pipe2.cu: exact
extern "C" int fc_f345_pair_exact(const fc_stage* sg, const fc_stage* sthr, const float* in,
                                  void* out, int out_type, fc_dims d, void* stream);
extern "C" int fc_f345_pipe(const fc_stage* sg, const fc_stage* sthr, const float* in,
                            void* out, int out_type, fc_dims d, double in_max, void* stream);
extern "C" long long fc_pipe_recheck_count(void);

namespace {
thread_local fc_knobs g_knobs = {};

int env_int(const char* name) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : 0;
}
}  // namespace

extern "C" void fc_knobs_from_env(fc_knobs* k) {
  std::memset(k, 0, sizeof *k);
  k->pipe_oh = env_int("FUSEPLAN_PIPE_OH");
  k->pipe_segs = env_int("FUSEPLAN_PIPE_SEGS");
  k->pipe_seg_warm = env_int("FUSEPLAN_PIPE_SEG_WARM");
  k->pipe_skip = env_int("FUSEPLAN_PIPE_SKIP");
  if (const char* e = std::getenv("FUSEPLAN_PIPE_BAND_SCALE")) k->band_scale = float(std::atof(e));
  if (const char* e = std::getenv("FUSEPLAN_PIPE_PROFILE")) k->profile = e[0] == '2' ? 2 : 1;
  k->debug = std::getenv("FUSEPLAN_DEBUG") != nullptr;
  if (const char* e = std::getenv("FUSEPLAN_PIPE_DEBUG_PX"))
    k->dbg_px_on = std::sscanf(e, "%d,%d,%d", &k->dbg_px[0], &k->dbg_px[1], &k->dbg_px[2]) == 3;
  k->f12_stream = std::getenv("FUSEPLAN_F12_STREAM") != nullptr;
  k->f12_legacy = std::getenv("FUSEPLAN_F12_LEGACY") != nullptr;
  k->pipe_impl = env_int("FUSEPLAN_PIPE_IMPL");
  k->pipe_out = env_int("FUSEPLAN_PIPE_OUT");
}

extern "C" void fc_set_knobs(const fc_knobs* k) {
  if (k)
    g_knobs = *k;
  else
    std::memset(&g_knobs, 0, sizeof g_knobs);
}

extern "C" const fc_knobs* fc_get_knobs(void) { return &g_knobs; }

namespace {
thread_local const char* g_last_chain = "none";
}

// variant: 0 auto (certified frame pipeline when covered, else exact),
//          1 exact, 2 fast (certified frame pipeline or -1: fail loudly).
// video_pitch: row pitch of a pitched copy of the video for the frame
// pipeline (0: the video itself, pitch = width); `video` is always the
// contiguous video (the exact kernel's input).
extern "C" int fc_fused_chain_pitched(const fc_stage* sgray, const fc_stage* si,
                                      const fc_stage* sg, const fc_stage* sgrad,
                                      const fc_stage* sthr, const void* video,
                                      const void* pitched, int video_pitch, void* pitched_out,
                                      int out_pitch, int in_type, int gray_in, void* out,
                                      int out_type, fc_dims d, int n_warm,
                                      const float* state_in, float* state_out, int variant,
                                      void* stream) {
  (void)sgrad;
  if (variant == 2 || variant == 0) {
    // frame-pair pipeline (fc_pipe2.cu) unless the row-pair one is forced
    const bool pair = fc_get_knobs()->pipe_impl != 1;
    const auto fn = pair ? fc_chain_pipe2 : fc_chain_pipe;
    const int rc = fn(sgray, si, sg, sthr, pitched ? pitched : video, in_type, gray_in,
                      pitched_out ? pitched_out : out, out_type, d, n_warm, state_in, state_out,
                      pitched ? video_pitch : 0, pitched_out ? out_pitch : 0, stream);
    if (rc == 0 && pitched_out)  // the mask rows back to their contiguous layout
      return int(cudaMemcpy2DAsync(out, size_t(d.width), pitched_out, size_t(out_pitch),
                                   size_t(d.width), size_t(d.height) * (d.frames - n_warm),
                                   cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream)));
    if (rc != -1)
      g_last_chain = pair ? "certified FP32 frame-pair pipeline (fc_pipe2.cu)"
                          : "certified FP32 row-pair pipeline (fc_pipe.cu)";
    if (rc != -1 || variant == 2) return rc;  // -1: parameters not covered
  }
  // reference-exact: the frame-pair pipeline with the FP64 stencil role where
  // it applies (u8 RGBA in, 5x5 gaussian, {0, 255} byte mask), else the FP64
  // tile march (FUSEPLAN_PIPE_IMPL=3 forces the tiles)
  if (fc_get_knobs()->pipe_impl != 3) {
    const int rc = fc_chain_pipe2_exact(sgray, si, sg, sthr, pitched ? pitched : video, in_type,
                                        gray_in, pitched_out ? pitched_out : out, out_type, d,
                                        n_warm, state_in, state_out, pitched ? video_pitch : 0,
                                        pitched_out ? out_pitch : 0, stream);
    if (rc == 0 && pitched_out)
      return int(cudaMemcpy2DAsync(out, size_t(d.width), pitched_out, size_t(out_pitch),
                                   size_t(d.width), size_t(d.height) * (d.frames - n_warm),
                                   cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream)));
    if (rc != -1) {
      g_last_chain = "exact FP64 frame-pair pipeline (fc_pipe2.cu)";
      return rc;
    }
  }
  g_last_chain = "exact FP64 tiles (fc_exact.cu k_chain_exact)";
  return fc_chain_exact(sgray, si, sg, sthr, video, in_type, gray_in, out,
                        out_type, d, n_warm, state_in, state_out, stream);
}

extern "C" int fc_fused_chain(const fc_stage* sgray, const fc_stage* si,
                              const fc_stage* sg, const fc_stage* sgrad,
                              const fc_stage* sthr, const void* video,
                              int in_type, int gray_in, void* out, int out_type,
                              fc_dims d, int n_warm, const float* state_in,
                              float* state_out, int variant, void* stream) {
  return fc_fused_chain_pitched(sgray, si, sg, sgrad, sthr, video, nullptr, 0, nullptr, 0,
                                in_type, gray_in, out, out_type, d, n_warm, state_in, state_out,
                                variant, stream);
}

extern "C" const char* fc_last_chain_kernel(void) { return g_last_chain; }

extern "C" void fc_pipe_release_scratch(int device, void* stream);
extern "C" void fc_pipe2_release_scratch(int device, void* stream);
// the time-segment scratch both pipelines keep per (device, stream)
extern "C" void fc_release_stream_scratch(int device, void* stream) {
  fc_pipe_release_scratch(device, stream);
  fc_pipe2_release_scratch(device, stream);
}

// Would the certified frame pipeline take this chain with a video of row
// pitch `pitch` (values only: the pointer alignment is the caller's)?
extern "C" int fc_chain_pipe_applies(const fc_stage* sgray, const fc_stage* si,
                                     const fc_stage* sg, const fc_stage* sthr, int in_type,
                                     int gray_in, int out_type, fc_dims d, int pitch);

// Certification parameters of the fused chain (host only; for reports and
// the error-bound tests): out = {g0, g1, mlo_n, band_n, S, mstar}, where g0,
// g1 are the centre-normalised separable taps, S = 1 / h2^2 the scale of the
// normalised domain, mlo_n ~ S^2 M* and band_n the certified band on
// nd = mlo_n - gx^2 - gy^2 (fc_common.cuh certify_band_scaled).  Returns 0,
// or -1 when the chain is outside the certified path.
extern "C" int fc_certified_params(const fc_stage* sgray, const fc_stage* si, const fc_stage* sg,
                                   const fc_stage* sthr, double* out) {
  fccommon::FastParams p;
  static const unsigned char dummy[16] __attribute__((aligned(16))) = {};
  fc_dims d{16, 8, 1};
  if (!fccommon::fast_params(sgray, si, sg, sthr, dummy, FC_U8, 0, FC_U8, d, 16, &p)) return -1;
  const double e2 = double(p.h2);
  out[0] = p.g0;
  out[1] = p.g1;
  out[2] = p.mlo_n;
  out[3] = p.band_n;
  out[4] = 1.0 / (e2 * e2);
  out[5] = p.mstar;
  return 0;
}

extern "C" long long fc_last_recheck_count(void) {
  return fc_pipe_recheck_count() + fc_pipe2_recheck_count();
}

extern "C" int fc_fused_gauss_grad_thr_v(const fc_stage* sg, const fc_stage* sgrad,
                                         const fc_stage* sthr, const float* in, void* out,
                                         int out_type, fc_dims d, int variant, double in_max,
                                         void* stream) {
  if (variant != 1 && in_max > 0.0) {
    const int rc = fc_f345_pipe(sg, sthr, in, out, out_type, d, in_max, stream);
    if (rc != -1) {  // -1: parameters not covered -> exact
      g_last_chain = "certified FP32 row-pair pipeline on f32 planes (fc_pipe.cu, F345)";
      return rc;
    }
  }
  // reference-exact: the exact frame-pair pipeline with the plane loader,
  // else the FP64 tiles
  if (fc_get_knobs()->pipe_impl != 3) {
    const int rc = fc_f345_pair_exact(sg, sthr, in, out, out_type, d, stream);
    if (rc != -1) {
      g_last_chain = "exact FP64 frame-pair pipeline on f32 planes (fc_pipe2.cu, F345)";
      return rc;
    }
  }
  g_last_chain = "exact FP64 tiles on f32 planes (fc_exact.cu, F345)";
  return fc_fused_gauss_grad_thr(sg, sgrad, sthr, in, out, out_type, d, stream);
}
