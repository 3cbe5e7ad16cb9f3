/* Thin C ABI between the C++ host (executor.cpp) and the sm_100a kernels.
 * Raw device pointers, plain sizes, a cudaStream_t passed as void*, int
 * status (0 = ok, else a cudaError_t value; -1 = unsupported arguments).
 *
 * Layouts (HBM):
 *   video  : planar u8 or f32, [t][c][y][x]   (the FPVD payload order,
 *            /root/reference/proj/include/fuseplan/video.hpp:24-28)
 *   planes : f32 [t][y][x] for every intermediate stage
 *   mask   : u8  [t][y][x] (threshold output when white/black are bytes)
 */
#ifndef FC_KERNELS_H
#define FC_KERNELS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum fc_op {
  FC_RGBA2GRAY = 0,
  FC_IIR_TEMPORAL = 1,
  FC_GAUSSIAN = 2,
  FC_GRADIENT = 3,
  FC_THRESHOLD = 4,
  FC_IDENTITY = 5,
  FC_SCALE_OFFSET = 6,
  FC_BOX_MEAN = 7
};

#define FC_MAX_GAUSS_RADIUS 4

/* Parameters of one stencil stage, already converted the way the reference
 * converts them (float(param) for float ops, simulator.cpp:51-106; gaussian
 * taps from simulator.cpp:27-44 computed on the host with std::exp). */
typedef struct {
  int op;
  float wr, wg, wb;          /* rgba2gray */
  float alpha;               /* iir_temporal */
  int g_radius;              /* gaussian */
  float g_w[(2 * FC_MAX_GAUSS_RADIUS + 1) * (2 * FC_MAX_GAUSS_RADIUS + 1)];
  float th, white, black;    /* threshold */
  float scale, offset;       /* scale_offset */
  int rx, ry, rt;            /* box_mean */
} fc_stage;

typedef struct {
  int width, height, frames;
} fc_dims;

/* Element type codes. */
enum { FC_U8 = 0, FC_F32 = 1 };

/* ---- unfused stages (the paper's sequential baseline) -------------------
 * One launch per stage over the whole volume; input/output f32 planes except
 * rgba2gray (video in, 4 channels, u8 or f32) and threshold (u8 or f32 out).
 * IIR stages take the streaming-range arguments described below. */
int fc_stage_spatial(const fc_stage* st, const void* in, int in_type,
                     void* out, int out_type, fc_dims d, void* stream);

/* Streaming range for anything containing the causal IIR:
 *   in/out point at the first processed frame; n_frames are processed; the
 *   first n_warm are warm-up frames (state only, no output written; out
 *   then points at the first OUTPUT frame).  state_in (nullable): IIR plane
 *   to resume from; NULL restarts the recurrence at the first processed
 *   frame (y = x, simulator.cpp:57-62).  state_out (nullable): IIR plane after
 *   the last processed frame. */
int fc_stage_iir(const fc_stage* st, const float* in, float* out, fc_dims d,
                 int n_warm, const float* state_in, float* state_out,
                 void* stream);

/* ---- fused partitions ----------------------------------------------------
 * F12   : rgba2gray + iir                 video -> f32 planes  (time scan)
 * F345  : gaussian + gradient + threshold f32 planes -> mask   (per frame)
 * F12345: the whole SPEC chain            video -> mask        (streaming)
 * `gray_in` for F12345 = 1 when the video is already single-channel (the
 * chain then starts at the IIR; s_gray is ignored). */
int fc_fused_gray_iir(const fc_stage* s_gray, const fc_stage* s_iir,
                      const void* video, int in_type, float* out, fc_dims d,
                      int n_warm, const float* state_in, float* state_out,
                      void* stream);

int fc_fused_gauss_grad_thr(const fc_stage* s_gauss, const fc_stage* s_grad,
                            const fc_stage* s_thr, const float* in, void* out,
                            int out_type, fc_dims d, void* stream);

/* F345 with a variant: 1 = exact (FP64 kernel); 0 / 2 = the certified
 * frame-pipeline kernel when the inputs are known to lie in [0, in_max]
 * (in_max > 0; the executor's range analysis), else exact. */
int fc_fused_gauss_grad_thr_v(const fc_stage* s_gauss, const fc_stage* s_grad,
                              const fc_stage* s_thr, const float* in, void* out,
                              int out_type, fc_dims d, int variant, double in_max,
                              void* stream);

/* variant: 0 = auto, 1 = exact (FP64 gaussian everywhere),
 *          2 = certified FP32 fast path with exact recheck */
int fc_fused_chain(const fc_stage* s_gray, const fc_stage* s_iir,
                   const fc_stage* s_gauss, const fc_stage* s_grad,
                   const fc_stage* s_thr, const void* video, int in_type,
                   int gray_in, void* out, int out_type, fc_dims d, int n_warm,
                   const float* state_in, float* state_out, int variant,
                   void* stream);

/* F12345 with optional pitched buffers for the certified frame pipeline (its
 * TMA map needs a 16-byte row pitch and base; its mask stores 4-byte aligned
 * rows): `pitched` holds planes 0-2 of every frame at [t][4][H][video_pitch]
 * (NULL: use `video`); `pitched_out` (NULL: write `out`) receives the mask at
 * row pitch out_pitch and is copied into `out` afterwards.  `video` / `out`
 * are the contiguous arrays (the FP64 kernel's). */
int fc_fused_chain_pitched(const fc_stage* s_gray, const fc_stage* s_iir,
                           const fc_stage* s_gauss, const fc_stage* s_grad,
                           const fc_stage* s_thr, const void* video, const void* pitched,
                           int video_pitch, void* pitched_out, int out_pitch, int in_type,
                           int gray_in, void* out, int out_type, fc_dims d, int n_warm,
                           const float* state_in, float* state_out, int variant, void* stream);
/* Would the certified frame pipeline take this chain with row pitch `pitch`? */
int fc_chain_pipe_applies(const fc_stage* s_gray, const fc_stage* s_iir,
                          const fc_stage* s_gauss, const fc_stage* s_thr, int in_type,
                          int gray_in, int out_type, fc_dims d, int pitch);
/* Would the exact frame-pair pipeline (fc_pipe2.cu, FP64 stencil role) take
 * this chain with a video of row pitch `pitch`? */
int fc_chain_pipe2_exact_applies(const fc_stage* s_gray, const fc_stage* s_iir,
                                 const fc_stage* s_gauss, const fc_stage* s_thr, int in_type,
                                 int gray_in, int out_type, fc_dims d, int pitch);
/* The kernel the last fc_fused_chain* call on this thread ran. */
const char* fc_last_chain_kernel(void);

/* run_tiled's box staging (simulator.cpp:229-333) for one tiled plan group,
 * for fp_simulate's tiled arm when a plan's halo erodes (fc_tiled.cu): one
 * CTA per output box (boxes looped over `ctas` CTAs); dev_stages: the
 * group's members on the device; halo = {x_lo, x_hi, y_lo, y_hi, t_lo, t_hi};
 * in: [t][c][y][x] with in_ch channels (FC_U8 / FC_F32); out: f32 [t][y][x];
 * scratch: fc_tiled_scratch_bytes() of device memory. */
long long fc_tiled_scratch_bytes(int tile_x, int tile_y, int tile_t, const int* halo,
                                 int in_ch, int ctas);
int fc_tiled_group(const fc_stage* dev_stages, int n_stages, const void* in, int in_type,
                   int in_ch, float* out, fc_dims d, int tile_x, int tile_y, int tile_t,
                   const int* halo, float* scratch, int ctas, void* stream);

/* T-shard carry check (fc_shard.cu): for the pixels whose true and warm
 * start states differ, runs gray (unless gray_in) + IIR from both over the
 * shard's d.frames frames and stores in *k_dev (device int) the number of
 * leading frames in which some pixel's IIR still differs (0: states equal;
 * d.frames: some pixel never converged).  Asynchronous. */
int fc_iir_converge(const fc_stage* sgray, const fc_stage* si, const void* video, int in_type,
                    int gray_in, fc_dims d, const float* s_true, const float* s_warm,
                    int* k_dev, void* stream);

/* Deterministic counter-hash u8 video (splitmix64 finaliser of
 * index + seed * 0x9E3779B97F4A7C15, top byte), [t][c][y][x]; frames
 * [t0, t0 + d.frames).  Mirrors tests/golden/make_golden.py:hash_video. */
int fc_hash_video_u8(uint8_t* out, fc_dims d, int channels, int t0,
                     uint64_t seed, void* stream);

/* Count of pixels that took the exact recheck path in the last certified
 * launch on this stream's device (diagnostic; 0 if unavailable). */
long long fc_last_recheck_count(void);
/* Certification parameters of the fused chain, {g0, g1, mlo_n, band_n, S,
 * mstar} (fc_dispatch.cu); -1 when the chain is outside the certified path. */
int fc_certified_params(const fc_stage* sgray, const fc_stage* si, const fc_stage* sg,
                        const fc_stage* sthr, double* out);

/* K6 tracking: one CTA per marker (fc_track.cu).  rois_dev: n x (x, y, w, h)
 * int32 on the device; points_dev: n x frames x 23 doubles on the device. */
int fc_track_features(const void* mask, int elem_type, int W, int H, int F,
                      const int* rois_dev, int n_rois, double q, double r, double p0,
                      double* points_dev, void* stream);

const char* fc_error_string(int code);

/* Diagnostic / tuning knobs of the kernel launchers.  The executor reads the
 * FUSEPLAN_* environment ONCE, when it is created (fc_knobs_from_env), and
 * installs its copy on the calling thread before each run (fc_set_knobs); the
 * launchers never call getenv.  All-zero = the shipped defaults. */
typedef struct {
  int pipe_oh;        /* FUSEPLAN_PIPE_OH: force the frame-pipeline window height */
  int pipe_segs;      /* FUSEPLAN_PIPE_SEGS: force the number of time segments */
  int pipe_seg_warm;  /* FUSEPLAN_PIPE_SEG_WARM: IIR warm-up of a segment (0 = default) */
  int pipe_skip;      /* FUSEPLAN_PIPE_SKIP: timing experiments (1 IIR, 2 stencil math) */
  float band_scale;   /* FUSEPLAN_PIPE_BAND_SCALE: widen the certification band (tests) */
  int profile;        /* FUSEPLAN_PIPE_PROFILE: per-CTA spans (1 summary, 2 every CTA) */
  int debug;          /* FUSEPLAN_DEBUG: launcher decisions on stderr */
  int dbg_px_on, dbg_px[3]; /* FUSEPLAN_PIPE_DEBUG_PX=x,y,t */
  int f12_stream;     /* FUSEPLAN_F12_STREAM: force the streaming F12 kernel */
  int f12_legacy;     /* FUSEPLAN_F12_LEGACY: the per-pixel F12 kernel */
  int pipe_impl;      /* FUSEPLAN_PIPE_IMPL: 0 auto, 1 row-pair pipe, 2 frame-pair pipe,
                         3 no exact pipeline (FP64 tiles / k_chain_exact) */
  int pipe_out;       /* FUSEPLAN_PIPE_OUT: force the frame-pair window's output rows */
} fc_knobs;

void fc_knobs_from_env(fc_knobs* k);
void fc_set_knobs(const fc_knobs* k); /* NULL = defaults */
const fc_knobs* fc_get_knobs(void);

#ifdef __cplusplus
}
#endif

#endif
