/* Test model of the certified frame-pair kernel's FP32 arithmetic
 * (paper_1509_04394_b200/csrc/kernels/fc_pipe2.cu stencil_role): the
 * centre-normalised separable gaussian (tap4n), the Sobel in the kernel's
 * order and nd = mlo_n - gy^2 - gx^2, op for op with explicit fmaf, on an
 * exact IIR plane.  Used by tests/test_certified_band.py to measure the
 * kernel's actual error against the certified band (CPU only, test code).
 *
 * Per-stage clamps as in the kernel: the gaussian reads the IIR plane at
 * clamped columns / rows (edge replication of the window cells), the Sobel
 * reads the gaussian plane at clamped columns (xlo / xhi selects) and rows
 * (the fixed-step y clamps). */
#include <math.h>
#include <stdlib.h>

static inline int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* tap4n(a, b, c, d, e) = FFMA2(g1, FADD2(b, d), FFMA2(g0, FADD2(a, e), c)) */
static inline float tap4n(float a, float b, float c, float d, float e, float g0, float g1) {
  return fmaf(g1, b + d, fmaf(g0, a + e, c));
}

/* iir: [F][H][W] exact IIR planes; nd: [F][H][W] out */
void fast_nd(const float* iir, int W, int H, int F, float g0, float g1, float mlo_n, float* nd) {
  float* hp = (float*)malloc(sizeof(float) * (size_t)W * H);
  float* gp = (float*)malloc(sizeof(float) * (size_t)W * H);
  for (int t = 0; t < F; ++t) {
    const float* I = iir + (size_t)t * W * H;
    for (int y = 0; y < H; ++y)
      for (int x = 0; x < W; ++x) {
        const float* r = I + (size_t)y * W;
        hp[(size_t)y * W + x] = tap4n(r[clampi(x - 2, 0, W - 1)], r[clampi(x - 1, 0, W - 1)], r[x],
                                      r[clampi(x + 1, 0, W - 1)], r[clampi(x + 2, 0, W - 1)], g0,
                                      g1);
      }
    for (int y = 0; y < H; ++y)
      for (int x = 0; x < W; ++x) {
#define HV(dy) hp[(size_t)clampi(y + (dy), 0, H - 1) * W + x]
        gp[(size_t)y * W + x] = tap4n(HV(-2), HV(-1), HV(0), HV(1), HV(2), g0, g1);
#undef HV
      }
    for (int y = 0; y < H; ++y)
      for (int x = 0; x < W; ++x) {
        float S[3], D[3];
        for (int k = 0; k < 3; ++k) {
          const int xx = clampi(x + k - 1, 0, W - 1);
          const float gm = gp[(size_t)clampi(y - 1, 0, H - 1) * W + xx];
          const float gc = gp[(size_t)y * W + xx];
          const float gq = gp[(size_t)clampi(y + 1, 0, H - 1) * W + xx];
          S[k] = fmaf(2.0f, gc, gm) + gq;
          D[k] = fmaf(-1.0f, gm, gq);
        }
        const float gx = fmaf(-1.0f, S[0], S[2]);
        const float gy = fmaf(2.0f, D[1], D[0]) + D[2];
        nd[(size_t)t * W * H + (size_t)y * W + x] = fmaf(-gx, gx, fmaf(-gy, gy, mlo_n));
      }
  }
  free(hp);
  free(gp);
}
