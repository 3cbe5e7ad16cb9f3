/* fuseplan C ABI -- B200 build (libfuseplan_b200.so).
 *
 * Drop-in for the reference's C interface
 * (/root/reference/proj/include/fuseplan.h:14-93, implemented by
 * /root/reference/proj/src/capi.cpp:186-425): same opaque handles, same
 * status codes, same ownership rules (returned char* are freed with
 * fp_string_free), same thread-local fp_last_error().  Planning entry points
 * keep their exact semantics; fp_simulate executes on the GPU instead of the
 * CPU simulator.  The fp_exec_* block is new: the device executor that runs a
 * plan's fused partitions as sm_100a kernels.  No torch types cross this
 * boundary -- plain pointers, sizes and a cudaStream_t passed as void*.
 */
#ifndef FUSEPLAN_H
#define FUSEPLAN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* fuseplan.h:14-19 */
typedef enum {
  FP_OK = 0,
  FP_ERR_INFEASIBLE = 1,
  FP_ERR_INPUT = 2,
  FP_ERR_INTERNAL = 3
} fp_status;

/* fuseplan.h:21-23 */
typedef struct fp_pipeline fp_pipeline;
typedef struct fp_device fp_device;
typedef struct fp_plan fp_plan;

/* fuseplan.h:25-26 / capi.cpp:183-186: thread-local diagnostic of the most
 * recent failure on this thread; strings returned via char** are new[]'d. */
const char* fp_last_error(void);
void fp_string_free(char* s);

/* ---- inputs: fuseplan.h:30-37 / capi.cpp:188-217 ------------------------ */
fp_status fp_pipeline_parse(const char* json_text, fp_pipeline** out);
fp_status fp_pipeline_load(const char* path, fp_pipeline** out);
void fp_pipeline_free(fp_pipeline* p);
fp_status fp_device_parse(const char* json_text, fp_device** out);
fp_status fp_device_load(const char* path_or_name, fp_device** out);
void fp_device_free(fp_device* d);

/* ---- planning: fuseplan.h:39-50 / capi.cpp:219-234 ----------------------
 * options_json (may be NULL): {"halo_mode": "cumulative"|"paper-max",
 *   "transfer_variant": "exact"|"paper", "force_partition": "1-2,3-5",
 *   "tile": {"x": 32, "y": 32, "t": 4},
 *   "iir_streaming": false}
 * iir_streaming (B200 extension, default false = the reference's planner):
 * the device executor streams a group containing the causal IIR frame by
 * frame, so the planner need not pin that group's tile to t = F (the
 * reference's rule, planner.cpp:73); long videos (e.g. 800x600x16000, which
 * the reference reports infeasible) then plan normally. */
fp_status fp_plan_create(const fp_pipeline* p, const fp_device* d,
                         const char* options_json, fp_plan** out);
void fp_plan_free(fp_plan* plan);
fp_status fp_plan_render_json(const fp_plan* plan, char** out);

/* ---- reports: fuseplan.h:52-65 / capi.cpp:236-265 ----------------------- */
fp_status fp_analyze_report(const fp_pipeline* p, const char* format,
                            int with_timestamp, char** out);
fp_status fp_plan_report(const fp_plan* plan, const char* format,
                         int with_timestamp, char** out);
fp_status fp_tile_sweep(const fp_device* d, const int halo[6], int max_x,
                        int max_t, const char* format, char** out);

/* ---- fuseplan.h:67-71 / capi.cpp:267-284.  The reference emits uncompiled
 * pseudo-CUDA text; this build replaces it with real kernels, so fp_codegen
 * writes a manifest naming the sm_100a kernel each plan group runs. */
fp_status fp_codegen(const fp_pipeline* p, const fp_device* d,
                     const char* options_json, const char* name,
                     const char* out_dir, char** manifest_out);

/* ---- fuseplan.h:73-83 / capi.cpp:286-385.  Same arguments and report
 * format.  The "sequential" arm runs one sm_100a kernel per stage with
 * intermediates in HBM (the paper's No Fusion regime); the "tiled" arm runs
 * the plan's fused partitions; outputs are compared element for element.
 * Needs a CUDA device (FP_ERR_INTERNAL otherwise). */
fp_status fp_simulate(const fp_pipeline* p, const fp_device* d,
                      const char* options_json, const char* video_path,
                      const char* synth_json, const char* track_csv_path,
                      const char* format, int with_timestamp, char** out);

/* ---- fuseplan.h:85-93 / calibrate.cpp:10-54: least-squares fit of the
 * cost-model parameters from a measurements CSV (same columns, messages and
 * JSON result as the reference; Householder QR with column pivoting in place
 * of Eigen's ColPivHouseholderQR), and a device JSON re-rendered with fitted
 * parameters. */
fp_status fp_calibrate_csv(const char* measurements_csv, char** result_json);
fp_status fp_device_render_with_cost(const fp_device* d,
                                     const char* params_json, char** out);

/* ======================================================================
 * NEW: device executor (replaces run_sequential / run_tiled,
 * /root/reference/proj/include/fuseplan/simulator.hpp:44-53, as the way a
 * plan is executed).
 * ==================================================================== */
typedef struct fp_exec fp_exec;

enum { FP_ELEM_U8 = 0, FP_ELEM_F32 = 1 };
/* fp_exec_run flags */
enum { FP_EXEC_HOST_PTRS = 0, FP_EXEC_DEVICE_PTRS = 1 };

/* Builds an executor for `plan` over `p` on CUDA device `device`.
 * options_json (may be NULL): {"variant": "auto"|"exact"|"fast",
 *   "host_chunk_frames": N}.  "auto": the certified FP32 frame-pipeline
 *   kernel (exact FP64 recheck inside its error band) where it applies, else
 *   the FP64 kernels; "exact": FP64 kernels only; "fast": the frame pipeline
 *   or FP_ERR_INTERNAL when the chain is outside its coverage.  The FUSEPLAN_*
 *   diagnostic environment knobs are read once, here.  FP_ERR_INPUT if a
 *   stage has no device kernel, FP_ERR_INTERNAL if no CUDA device is present. */
fp_status fp_exec_create(const fp_pipeline* p, const fp_plan* plan, int device,
                         const char* options_json, fp_exec** out);
void fp_exec_free(fp_exec* e);

/* Element type of the final output (FP_ELEM_U8 for a byte-valued threshold
 * mask, else FP_ELEM_F32) and the number of IIR state planes. */
fp_status fp_exec_output_type(const fp_exec* e, int* elem_type);
fp_status fp_exec_state_planes(const fp_exec* e, int* n_planes);

/* Runs the whole pipeline.  video: planar [t][c][y][x] of the pipeline's
 * dims, element type in_type; out: [t][y][x] of fp_exec_output_type().
 * FP_EXEC_HOST_PTRS: host buffers, streamed through the device in frame
 * chunks (H2D / compute / D2H overlapped, IIR state carried exactly);
 * synchronous.  FP_EXEC_DEVICE_PTRS: device buffers, asynchronous on
 * `stream` (a cudaStream_t; NULL = the executor's own stream). */
fp_status fp_exec_run(fp_exec* e, const void* video, int in_type, void* out,
                      int flags, void* stream);

/* CUDA graph of a whole device-buffer run (fp_exec_run with
 * FP_EXEC_DEVICE_PTRS) on fixed buffers: the launches of one run (for small
 * frames several per run: time segments, seam check, fix-up) replay with one
 * cudaGraphLaunch.  fp_exec_graph_create runs the pipeline once uncaptured
 * (out is written), then captures a second run on `stream` (NULL: a
 * temporary non-blocking stream; the legacy default stream cannot capture)
 * and instantiates it.  Refill `video` in place between launches; the graph
 * always reads `video` and writes `out`.  fp_exec_graph_launch is
 * asynchronous on `stream` (NULL = the legacy default stream).  The
 * executor must outlive its graphs (they use its scratch buffers), and one
 * executor's graph launches must not overlap each other or its runs.
 * fp_exec_graph_free synchronises the graph's device. */
typedef struct fp_graph fp_graph;
fp_status fp_exec_graph_create(fp_exec* e, const void* video, int in_type, void* out,
                               void* stream, fp_graph** graph);
fp_status fp_exec_graph_launch(fp_graph* g, void* stream);
void fp_exec_graph_free(fp_graph* g);

/* Frame-range run on device buffers, for T-sharding: video holds n_frames
 * frames; the first n_warm only advance the IIR state (no output); out gets
 * n_frames - n_warm frames.  state_in (may be NULL = restart the recurrence
 * at the first frame) / state_out (may be NULL): n_planes * W * H floats. */
fp_status fp_exec_run_range(fp_exec* e, const void* video, int in_type,
                            void* out, int n_frames, int n_warm,
                            const float* state_in, float* state_out,
                            void* stream);

/* T-shard carry check: video holds a shard's n_frames frames
 * on the executor's device, which ran from the warm state s_warm (its IIR
 * restarted some frames before the shard); s_true is the true carry from the
 * previous shard (W*H floats each, device).  *frames_out = how many leading
 * frames of the shard's output differ from an exact run (0: none; n_frames:
 * the end state differs too), from a gray+IIR re-run of only the pixels
 * whose two states differ.  Re-running those frames from s_true makes the
 * shard exact.  Synchronous.  FP_ERR_INPUT unless the chain opens with
 * [rgba2gray,] iir_temporal. */
fp_status fp_exec_converge(fp_exec* e, const void* video, int in_type, int n_frames,
                           const float* s_true, const float* s_warm, int* frames_out,
                           void* stream);

/* ---- multi-GPU: one process, one host thread, N devices ------------------
 * The video is split along T into n_devices shards (devices[] may repeat a
 * device).  Each shard restarts its IIR "warmup_frames" (default 48) frames
 * early, runs on its device, and the shards' carries move device to device
 * (cudaMemcpyPeerAsync); a carry that differs from the shard's warm state
 * triggers a re-run of only the frames it affects (fp_exec_converge), in
 * rank order.  Output identical to a single-device run for any warm-up.
 * options_json: fp_exec_create's keys plus {"warmup_frames": W}. */
typedef struct fp_shard_exec fp_shard_exec;
fp_status fp_shard_exec_create(const fp_pipeline* p, const fp_plan* plan, const int* devices,
                               int n_devices, const char* options_json, fp_shard_exec** out);
void fp_shard_exec_free(fp_shard_exec* e);
/* Host buffers: planar [t][c][y][x] video of the pipeline's dims, element
 * type in_type; out [t][y][x] of the executor's output type.  Synchronous. */
fp_status fp_shard_exec_run(fp_shard_exec* e, const void* video, int in_type, void* out);
/* JSON: shards (device, frames, warm-up) and the last run's fix-ups. */
fp_status fp_shard_exec_stats(const fp_shard_exec* e, char** out_json);

/* FPVD file -> FPVD file (video.cpp:46-109), streamed through the GPU:
 * chunks of host_chunk_frames frames are read into pinned buffers while the
 * previous chunk runs, the IIR carried exactly between chunks, the output
 * (1 channel: u8 mask or f32 planes) written as chunks complete -- the video
 * never has to fit in host memory.  Synchronous. */
fp_status fp_exec_run_file(fp_exec* e, const char* in_path, const char* out_path);

/* ---- K6 tracking (tracking.cpp:84-128, capi.cpp:366-381), on the GPU -----
 * mask [frames][height][width], FP_ELEM_U8 or FP_ELEM_F32, "set" where
 * > 127; mask_on_device != 0: a device pointer (async on `stream`, the call
 * still returns after the points are on the host), else a host pointer.
 * rois_xywh: n_rois x (x, y, w, h) initial ROIs, one per marker.
 * kalman_json (nullable): {"q": 0.01, "r": 0.25, "p0": 10.0} (the reference's
 * KalmanParams defaults).
 * points (nullable, caller-owned, n_rois * frames * 23 doubles): per marker
 * and frame: measured (0/1), meas_x, meas_y, est_x, est_y, est_vx, est_vy,
 * covariance[16] row-major.
 * csv_out (nullable): the reference's trajectory CSV text
 * (trajectories_to_csv, tracking.cpp:130-146); free with fp_string_free. */
fp_status fp_track_features(const void* mask, int elem_type, int mask_on_device,
                            int width, int height, int frames, const int* rois_xywh,
                            int n_rois, const char* kalman_json, double* points,
                            char** csv_out, void* stream);

/* JSON: the launch groups and the kernel each runs. */
fp_status fp_exec_describe(const fp_exec* e, char** out_json);

/* Certification parameters of the all-fused SPEC chain (host only, no
 * device): JSON {g0, g1, mlo_n, band_n, S, mstar} -- the centre-normalised
 * separable taps, the normalised-domain threshold and certified band on
 * nd = mlo_n - gx^2 - gy^2, the scale S and the float threshold M* on m.
 * FP_ERR_INPUT when the chain is not the SPEC chain or its parameters are
 * outside the certified path.  Free with fp_string_free. */
fp_status fp_certified_params(const fp_pipeline* p, char** out_json);

/* Fills a device buffer with the deterministic counter-hash u8 test video
 * (frames [t0, t0 + frames) of a W x H x C volume). */
fp_status fp_synth_hash_u8(void* device_out, int width, int height,
                           int frames, int channels, int t0, uint64_t seed,
                           void* stream);

#ifdef __cplusplus
}
#endif

#endif /* FUSEPLAN_H */
