/* TEST INFRASTRUCTURE ONLY -- never linked into, loaded by, or called from the
 * product path.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may use this.
 *
 * CPU restatement of the reference hot path: the per-element stencil
 * semantics of /root/reference/proj/src/simulator.cpp (apply_stencil_at,
 * :48-108), the whole-volume stage driver (apply_stencil, :129-156) and the
 * sequential oracle (run_sequential, :158-177).  Written in plain C, built
 * with -O2 -ffp-contract=off (no FMA contraction, no fast-math) so every float
 * operation rounds exactly where the reference's does.
 *
 * Parity is pinned against the reference itself, compiled unmodified into
 * oracle/_ref/libfuseplan_ref.so by oracle/Makefile (see tests/test_oracle.py)
 * and against the golden vectors in tests/golden/.
 */
#ifndef FUSECHAIN_ORACLE_H
#define FUSECHAIN_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Stencil ops of the reference catalog (stencil_catalog.cpp:10-23). */
enum {
  ORC_RGBA2GRAY = 0,
  ORC_IIR_TEMPORAL = 1,
  ORC_GAUSSIAN = 2,
  ORC_GRADIENT = 3,
  ORC_THRESHOLD = 4,
  ORC_IDENTITY = 5,
  ORC_SCALE_OFFSET = 6,
  ORC_BOX_MEAN = 7,
  ORC_KALMAN_TRACK = 8 /* global aggregation: skipped by run_sequential */
};

/* One pipeline stage.  p[] holds the op's parameters with the reference's
 * defaults already applied (simulator.cpp:51-106):
 *   rgba2gray   p = {wr, wg, wb}
 *   iir         p = {alpha}
 *   gaussian    p = {radius, sigma}
 *   threshold   p = {th, white, black}
 *   scale_offset p = {scale, offset}
 *   box_mean    p = {radius_x, radius_y, radius_t}                      */
typedef struct {
  int op;
  double p[4];
} orc_stage;

/* Fills `out` ((2r+1)^2 floats, dy-major) with the reference's normalised
 * gaussian taps (simulator.cpp:27-44). */
void orc_gaussian_weights(int radius, double sigma, float* out);

/* apply_stencil (simulator.cpp:129-156) over a whole planar [t][c][y][x]
 * float volume.  in_ch is the input channel count (4 for rgba2gray, else 1);
 * the output has 1 channel.  Returns 0, or -1 for an unknown op. */
int orc_apply_stage(const orc_stage* st, const float* in, int width,
                    int height, int frames, int in_ch, float* out,
                    int nthreads);

/* Streaming restatement of run_sequential for chains whose only temporal
 * dependence is the causal IIR (no box_mean with radius_t > 0): frames are
 * processed in order, the IIR plane is carried, and each stage of frame t
 * reads the previous stage's frame-t plane with clamp-to-edge.
 *
 * video   : planar [t][c][y][x] u8 volume (c = in_ch) holding frames
 *           [0, frames) of the full video.
 * t_begin : first frame of the recurrence.  Frame t_begin is treated as the
 *           recurrence start (y = x), exactly like a warm-up restart; pass 0
 *           for the reference semantics.  Frames before t_begin are ignored.
 * t_out   : first frame whose final output is written (t_out >= t_begin).
 * out     : final-stage output, frames [t_out, frames), [t][y][x] float.
 * iir_state_out : optional W*H float plane, the IIR state after the last
 *           frame (NULL to skip).  iir_state_in: optional state to resume
 *           from (frame t_begin is then a normal recurrence step).
 * Returns 0, or -1 for an unsupported chain. */
int orc_chain_stream_u8(const uint8_t* video, int width, int height,
                        int frames, int in_ch, const orc_stage* stages,
                        int n_stages, int t_begin, int t_out, float* out,
                        const float* iir_state_in, float* iir_state_out,
                        int nthreads);

/* Same, for float input volumes. */
int orc_chain_stream_f32(const float* video, int width, int height,
                         int frames, int in_ch, const orc_stage* stages,
                         int n_stages, int t_begin, int t_out, float* out,
                         const float* iir_state_in, float* iir_state_out,
                         int nthreads);

#ifdef __cplusplus
}
#endif

#endif
