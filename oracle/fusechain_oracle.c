/* TEST INFRASTRUCTURE ONLY (see fusechain_oracle.h).  CPU restatement of the
 * reference hot path; every function cites the reference lines it follows.
 * Build: gcc -O2 -ffp-contract=off -fopenmp (oracle/Makefile).  FMA
 * contraction or -ffast-math would change the float results. */
#include "fusechain_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static inline int clampi(int v, int lo, int hi) {
  return v < lo ? lo : (v > hi ? hi : v);
}

/* simulator.cpp:27-44: weights in double, normalised by the sum accumulated
 * in dy-outer / dx-inner order, each rounded to float. */
void orc_gaussian_weights(int radius, double sigma, float* out) {
  int d = 2 * radius + 1;
  double* w = (double*)malloc(sizeof(double) * (size_t)d * d);
  double sum = 0.0;
  for (int dy = -radius; dy <= radius; ++dy)
    for (int dx = -radius; dx <= radius; ++dx) {
      double v = exp(-(dx * dx + dy * dy) / (2.0 * sigma * sigma));
      w[(dy + radius) * d + (dx + radius)] = v;
      sum += v;
    }
  for (int i = 0; i < d * d; ++i) out[i] = (float)(w[i] / sum);
  free(w);
}

/* A sampler over one float plane with clamp-to-edge (video.cpp:39-44). */
typedef struct {
  const float* p;
  int w, h;
} plane;

static inline float smp(const plane* s, int x, int y) {
  x = clampi(x, 0, s->w - 1);
  y = clampi(y, 0, s->h - 1);
  return s->p[(size_t)y * s->w + x];
}

/* Spatial part of apply_stencil_at (simulator.cpp:48-108) for the
 * frame-local ops.  `chan` are the input channel planes of one frame. */
static float eval_spatial(const orc_stage* st, const plane* chan, int x, int y,
                          const float* gw) {
  switch (st->op) {
    case ORC_RGBA2GRAY: { /* :51-56 */
      float wr = (float)st->p[0], wg = (float)st->p[1], wb = (float)st->p[2];
      return wr * smp(&chan[0], x, y) + wg * smp(&chan[1], x, y) +
             wb * smp(&chan[2], x, y);
    }
    case ORC_GAUSSIAN: { /* :63-74, FP64 accumulation, dy outer, dx inner */
      int r = (int)st->p[0];
      int d = 2 * r + 1;
      double acc = 0.0;
      for (int dy = -r; dy <= r; ++dy)
        for (int dx = -r; dx <= r; ++dx)
          acc += (double)gw[(dy + r) * d + (dx + r)] *
                 (double)smp(&chan[0], x + dx, y + dy);
      return (float)acc;
    }
    case ORC_GRADIENT: { /* :75-83 */
#define S(dx, dy) smp(&chan[0], x + (dx), y + (dy))
      float gx = (S(1, -1) + 2.0f * S(1, 0) + S(1, 1)) -
                 (S(-1, -1) + 2.0f * S(-1, 0) + S(-1, 1));
      float gy = (S(-1, 1) + 2.0f * S(0, 1) + S(1, 1)) -
                 (S(-1, -1) + 2.0f * S(0, -1) + S(1, -1));
#undef S
      return sqrtf(gx * gx + gy * gy);
    }
    case ORC_THRESHOLD: { /* :84-89 */
      float th = (float)st->p[0], white = (float)st->p[1],
            black = (float)st->p[2];
      return smp(&chan[0], x, y) >= th ? white : black;
    }
    case ORC_IDENTITY:
    case ORC_KALMAN_TRACK: /* :90 */
      return smp(&chan[0], x, y);
    case ORC_SCALE_OFFSET: { /* :91-95 */
      float scale = (float)st->p[0], offset = (float)st->p[1];
      return scale * smp(&chan[0], x, y) + offset;
    }
    default:
      return 0.0f;
  }
}

static int in_channels_of(int op) { return op == ORC_RGBA2GRAY ? 4 : 1; }

/* One output row of a frame-local stage.  Interior pixels of the gaussian and
 * the gradient (no clamp can trigger) take a loop without the sampler; the
 * arithmetic and its order are exactly eval_spatial's (same expressions, same
 * double accumulation order), so the result is bit-identical -- this only
 * makes the checker fast enough for full-volume parity runs. */
static void eval_row(const orc_stage* st, const plane* chan, int y, const float* gw,
                     float* dst) {
  const int W = chan[0].w, H = chan[0].h;
  int r = 0;
  if (st->op == ORC_GAUSSIAN) r = (int)st->p[0];
  else if (st->op == ORC_GRADIENT) r = 1;
  if (r == 0 || y < r || y >= H - r || W <= 2 * r) {
    for (int x = 0; x < W; ++x) dst[x] = eval_spatial(st, chan, x, y, gw);
    return;
  }
  for (int x = 0; x < r; ++x) dst[x] = eval_spatial(st, chan, x, y, gw);
  for (int x = W - r; x < W; ++x) dst[x] = eval_spatial(st, chan, x, y, gw);
  const float* p = chan[0].p;
  if (st->op == ORC_GAUSSIAN) { /* :63-74 */
    const int d = 2 * r + 1;
    double w[15 * 15];
    for (int i = 0; i < d * d && i < 15 * 15; ++i) w[i] = (double)gw[i];
    if (d > 15) {
      for (int x = r; x < W - r; ++x) dst[x] = eval_spatial(st, chan, x, y, gw);
      return;
    }
    for (int x = r; x < W - r; ++x) {
      double acc = 0.0;
      for (int dy = -r; dy <= r; ++dy) {
        const float* row = p + (size_t)(y + dy) * W + x;
        const double* wr = w + (dy + r) * d + r;
        for (int dx = -r; dx <= r; ++dx) acc += wr[dx] * (double)row[dx];
      }
      dst[x] = (float)acc;
    }
  } else { /* ORC_GRADIENT :75-83 */
    const float* up = p + (size_t)(y - 1) * W;
    const float* mid = p + (size_t)y * W;
    const float* dn = p + (size_t)(y + 1) * W;
    for (int x = 1; x < W - 1; ++x) {
      float gx = (up[x + 1] + 2.0f * mid[x + 1] + dn[x + 1]) -
                 (up[x - 1] + 2.0f * mid[x - 1] + dn[x - 1]);
      float gy = (dn[x - 1] + 2.0f * dn[x] + dn[x + 1]) -
                 (up[x - 1] + 2.0f * up[x] + up[x + 1]);
      dst[x] = sqrtf(gx * gx + gy * gy);
    }
  }
}

/* apply_stencil (simulator.cpp:129-156) over a whole volume. */
int orc_apply_stage(const orc_stage* st, const float* in, int width,
                    int height, int frames, int in_ch, float* out,
                    int nthreads) {
  size_t plane_sz = (size_t)width * height;
  if (nthreads < 1) nthreads = 1;
  if (st->op == ORC_IIR_TEMPORAL) {
    /* :136-147: per (c, y, x) scan over t; t = 0 passes the input through. */
    float alpha = (float)st->p[0];
#pragma omp parallel for num_threads(nthreads) schedule(static)
    for (long i = 0; i < (long)plane_sz; ++i) {
      float prev = 0.0f;
      for (int t = 0; t < frames; ++t) {
        float v = in[(size_t)t * plane_sz + i];
        prev = (t == 0) ? v : alpha * v + (1.0f - alpha) * prev; /* :57-62 */
        out[(size_t)t * plane_sz + i] = prev;
      }
    }
    return 0;
  }
  if (st->op == ORC_BOX_MEAN) {
    /* :96-106: double accumulation, dt outer, dy, dx inner, clamp in t. */
    int rx = (int)st->p[0], ry = (int)st->p[1], rt = (int)st->p[2];
    int vol = (2 * rx + 1) * (2 * ry + 1) * (2 * rt + 1);
#pragma omp parallel for num_threads(nthreads) schedule(static) collapse(2)
    for (int t = 0; t < frames; ++t)
      for (int y = 0; y < height; ++y)
        for (int x = 0; x < width; ++x) {
          double acc = 0.0;
          for (int dt = -rt; dt <= rt; ++dt) {
            int tt = clampi(t + dt, 0, frames - 1);
            plane pl = {in + (size_t)tt * plane_sz, width, height};
            for (int dy = -ry; dy <= ry; ++dy)
              for (int dx = -rx; dx <= rx; ++dx)
                acc += smp(&pl, x + dx, y + dy);
          }
          out[(size_t)t * plane_sz + (size_t)y * width + x] =
              (float)(acc / vol);
        }
    return 0;
  }
  if (in_ch != in_channels_of(st->op)) return -1;
  float* gw = NULL;
  if (st->op == ORC_GAUSSIAN) {
    int r = (int)st->p[0];
    gw = (float*)malloc(sizeof(float) * (size_t)(2 * r + 1) * (2 * r + 1));
    orc_gaussian_weights(r, st->p[1], gw);
  }
  if (st->op < 0 || st->op > ORC_KALMAN_TRACK) return -1;
#pragma omp parallel for num_threads(nthreads) schedule(static) collapse(2)
  for (int t = 0; t < frames; ++t)
    for (int y = 0; y < height; ++y) {
      plane chan[4];
      for (int c = 0; c < in_ch; ++c) {
        chan[c].p = in + ((size_t)t * in_ch + c) * plane_sz;
        chan[c].w = width;
        chan[c].h = height;
      }
      for (int x = 0; x < width; ++x)
        out[(size_t)t * plane_sz + (size_t)y * width + x] =
            eval_spatial(st, chan, x, y, gw);
    }
  free(gw);
  return 0;
}

/* Streaming run_sequential (simulator.cpp:158-177): frame t of stage k only
 * depends on frame t of stage k-1 (clamped spatially) and, for the IIR, on the
 * stage's own frame t-1 output -- the carried state plane. */
static int chain_stream(const void* video, int is_u8, int width, int height,
                        int frames, int in_ch, const orc_stage* stages,
                        int n_stages, int t_begin, int t_out, float* out,
                        const float* iir_state_in, float* iir_state_out,
                        int nthreads) {
  size_t plane_sz = (size_t)width * height;
  if (nthreads < 1) nthreads = 1;
  if (t_begin < 0 || t_out < t_begin || t_out > frames) return -1;
  int n_iir = 0;
  float* gw[64];
  if (n_stages > 64) return -1;
  int ch = in_ch;
  for (int k = 0; k < n_stages; ++k) {
    gw[k] = NULL;
    const orc_stage* st = &stages[k];
    if (st->op == ORC_KALMAN_TRACK) continue; /* :168 */
    if (st->op == ORC_BOX_MEAN && (int)st->p[2] != 0) return -1;
    if (st->op < 0 || st->op > ORC_KALMAN_TRACK) return -1;
    if (ch != in_channels_of(st->op)) return -1;
    ch = 1;
    if (st->op == ORC_IIR_TEMPORAL) ++n_iir;
    if (st->op == ORC_GAUSSIAN) {
      int r = (int)st->p[0];
      gw[k] = (float*)malloc(sizeof(float) * (size_t)(2 * r + 1) * (2 * r + 1));
      orc_gaussian_weights(r, st->p[1], gw[k]);
    }
  }
  float* state = (float*)calloc((size_t)(n_iir ? n_iir : 1) * plane_sz,
                                sizeof(float));
  if (iir_state_in)
    memcpy(state, iir_state_in, sizeof(float) * (size_t)n_iir * plane_sz);
  float* in_f = (float*)malloc(sizeof(float) * plane_sz * in_ch);
  float* bufA = (float*)malloc(sizeof(float) * plane_sz);
  float* bufB = (float*)malloc(sizeof(float) * plane_sz);

  for (int t = t_begin; t < frames; ++t) {
    int first = (t == t_begin) && (iir_state_in == NULL);
    /* frame t input planes as float (video.cpp:87: float(u8)) */
    size_t base = (size_t)t * in_ch * plane_sz;
#pragma omp parallel for num_threads(nthreads) schedule(static)
    for (long i = 0; i < (long)(plane_sz * in_ch); ++i)
      in_f[i] = is_u8 ? (float)((const uint8_t*)video)[base + i]
                      : ((const float*)video)[base + i];
    const float* cur = in_f;
    int cur_ch = in_ch;
    int iir_idx = 0;
    float* dst = bufA;
    for (int k = 0; k < n_stages; ++k) {
      const orc_stage* st = &stages[k];
      if (st->op == ORC_KALMAN_TRACK) continue;
      if (st->op == ORC_IIR_TEMPORAL) {
        float alpha = (float)st->p[0];
        float* s = state + (size_t)iir_idx * plane_sz;
#pragma omp parallel for num_threads(nthreads) schedule(static)
        for (long i = 0; i < (long)plane_sz; ++i) {
          float v = cur[i];
          float y = first ? v : alpha * v + (1.0f - alpha) * s[i];
          s[i] = y;
          dst[i] = y;
        }
        ++iir_idx;
      } else {
        plane chan[4];
        for (int c = 0; c < cur_ch; ++c) {
          chan[c].p = cur + (size_t)c * plane_sz;
          chan[c].w = width;
          chan[c].h = height;
        }
#pragma omp parallel for num_threads(nthreads) schedule(static)
        for (int y = 0; y < height; ++y)
          eval_row(st, chan, y, gw[k], dst + (size_t)y * width);
      }
      cur = dst;
      cur_ch = 1;
      dst = (dst == bufA) ? bufB : bufA;
    }
    if (t >= t_out)
      memcpy(out + (size_t)(t - t_out) * plane_sz, cur,
             sizeof(float) * plane_sz);
  }
  if (iir_state_out)
    memcpy(iir_state_out, state, sizeof(float) * (size_t)n_iir * plane_sz);
  for (int k = 0; k < n_stages; ++k) free(gw[k]);
  free(state);
  free(in_f);
  free(bufA);
  free(bufB);
  return 0;
}

int orc_chain_stream_u8(const uint8_t* video, int width, int height,
                        int frames, int in_ch, const orc_stage* stages,
                        int n_stages, int t_begin, int t_out, float* out,
                        const float* iir_state_in, float* iir_state_out,
                        int nthreads) {
  return chain_stream(video, 1, width, height, frames, in_ch, stages, n_stages,
                      t_begin, t_out, out, iir_state_in, iir_state_out,
                      nthreads);
}

int orc_chain_stream_f32(const float* video, int width, int height,
                         int frames, int in_ch, const orc_stage* stages,
                         int n_stages, int t_begin, int t_out, float* out,
                         const float* iir_state_in, float* iir_state_out,
                         int nthreads) {
  return chain_stream(video, 0, width, height, frames, in_ch, stages, n_stages,
                      t_begin, t_out, out, iir_state_in, iir_state_out,
                      nthreads);
}
