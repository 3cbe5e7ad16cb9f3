// Shared pieces of the certified fast kernels (fc_fast.cu tile march,
// fc_strip.cu strip march): mbarrier / TMA wrappers, the exact S1+S2
// arithmetic helpers, the FP32 stencil taps and the host-side certification
// of the FP32 path (weights, separable taps, M*, error band).
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>

#include "fc_kernels.h"

namespace fccommon {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// x (innermost, bytes) must be a multiple of 16 (measured on B200: other
// offsets raise an illegal-instruction fault; scripts/tma_probe.cu).
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

// float(byte k of w) + 2^23 in one PRMT: bytes {w.k, 0, 0, 0x4B}
template <int K>
__device__ __forceinline__ float magic(uint32_t w) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(w), "r"(0x4B000000u), "n"(0x7440 + K));
  return __uint_as_float(r);
}

// Same with the 0x4B000000 word in a register the compiler cannot see
// through (kernel parameter): the selector then stays an immediate instead
// of being re-materialised into a register for every PRMT.
template <int K>
__device__ __forceinline__ float magic_r(uint32_t w, uint32_t k4b) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(w), "r"(k4b), "n"(0x7440 + K));
  return __uint_as_float(r);
}

// magic_r with a per-lane selector (0x7440 + byte index) in a register
__device__ __forceinline__ float magic_rs(uint32_t w, uint32_t k4b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(w), "r"(k4b), "r"(sel));
  return __uint_as_float(r);
}

// 0xFF where nd < 0, else 0, for four values -> one word: PRMT's
// sign-replicate mode (selector nibble 8 + byte) on byte 3 of each float.
__device__ __forceinline__ uint32_t pack_neg(float a, float b, float c, float d) {
  uint32_t ab, cd, r;
  asm("prmt.b32 %0, %1, %2, 0x00FB;" : "=r"(ab) : "r"(__float_as_uint(a)), "r"(__float_as_uint(b)));
  asm("prmt.b32 %0, %1, %2, 0x00FB;" : "=r"(cd) : "r"(__float_as_uint(c)), "r"(__float_as_uint(d)));
  asm("prmt.b32 %0, %1, %2, 0x5410;" : "=r"(r) : "r"(ab), "r"(cd));
  return r;
}

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 splat(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 lo2(float4 v) { return make_float2(v.x, v.y); }
__device__ __forceinline__ float2 hi2(float4 v) { return make_float2(v.z, v.w); }

// fl(w * c), c in [0,255] held as c + 2^23: FMA(w, c + 2^23, -w 2^23)
// rounds the exact product w*c once (w 2^23 is exact).
__device__ __forceinline__ float2 wprod(float2 m, float w, float wm) {
  return __ffma2_rn(splat(w), m, splat(wm));
}

// Centre-normalised separable 5-tap pass (centre tap 1; g0 at |d| = 2, g1 at
// |d| = 1): 4 packed ops, at most 3 roundings per term -- the order
// certify_band_scaled and tests/cpp/fast_model.c assume.  No packed multiply
// feeds a packed add (ptxas would contract the pair, fc_sobel.cuh).
__device__ __forceinline__ float2 tap4n(float2 a, float2 b, float2 c, float2 d, float2 e,
                                        float g0, float g1) {
  return __ffma2_rn(splat(g1), __fadd2_rn(b, d), __ffma2_rn(splat(g0), __fadd2_rn(a, e), c));
}

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return min(max(v, lo), hi); }

// 0xFF where dm >= 0 (white), else 0, for four values -> one word.  dm is
// never -0 for m < M* (Sterbenz: the difference of nearby floats is exact),
// so the sign bit is the decision.
__device__ __forceinline__ uint32_t pack_white(float a, float b, float c, float d) {
  uint32_t sa = uint32_t(__float_as_int(a) >> 31), sb = uint32_t(__float_as_int(b) >> 31);
  uint32_t sc = uint32_t(__float_as_int(c) >> 31), sd = uint32_t(__float_as_int(d) >> 31);
  return ~__byte_perm(__byte_perm(sa, sb, 0x0040), __byte_perm(sc, sd, 0x0040), 0x5410);
}

// ------------------------------------------------------------------ host

// Parameters of the certified FP32 path, shared by both fast kernels.
struct FastParams {
  float wr, wg, wb, wrm, wgm, wbm;  // gray weights (x 0.5 when alpha = 0.5), -w*2^23
  float ia, ib;                     // IIR alpha and float(1 - alpha) (general alpha)
  int alpha_half;                   // alpha == 0.5: folded into the weights, one FMA
  float h0, h1, h2;                 // separable fast taps: |d|=2, |d|=1, centre
  float taps[25];                   // reference taps for the exact recheck
  float mstar, band, th_val;
  float mlo;        // largest float below M*: white <=> m > mlo <=> mlo - m < 0
  uint32_t k4b;     // 0x4B000000 (see magic_r)
  // Centre-normalised taps (fc_pipe.cu): g0 = h0 / h2, g1 = h1 / h2, centre 1,
  // so a 5-tap pass is 4 packed ops; G, gx, gy come out scaled by S = 1 / h2^2
  // and m by S^2.  mlo_n ~ S^2 M*, band_n: the certified band in that domain.
  float g0, g1, mlo_n, band_n;
};

// M* = the smallest float m with sqrtf(m) >= th (white <=> m >= M*)
inline float threshold_mstar(float th) {
  float m = th * th;
  while (m > 0.0f && std::sqrt(std::nextafter(m, 0.0f)) >= th) m = std::nextafter(m, 0.0f);
  while (std::sqrt(m) < th) m = std::nextafter(m, INFINITY);
  return m;
}

// Certified error band on m = gx^2 + gy^2 (u = 2^-24, all stencil inputs >= 0):
//   kappa : relative error of the FP32 separable gaussian vs the reference's
//           FP64-accumulated, float-rounded value: <= 8.1u (two passes of at
//           most 4 roundings per term) + dw (separable vs reference taps) + u
//           (the reference's final rounding) + 25 * 2^-53 (its double sums);
//   E     : |gx_f - gx_ref| <= (kappa + 6.1u) * S, S = sum of the six taps'
//           |values| <= 8 gmax (3 roundings on each side);
//   Em(m) <= 4 E sqrt(m) + 2 E^2 + 4.1 u m   (|g.| <= sqrt(m), 2 roundings
//           in each of m_f and m_ref) + 2u (M* + m) (the strip kernel forms
//           mlo - gy^2 - gx^2 with two FMAs instead of m - M*);
//   B solves B >= Em(M* + B); m_f >= M* + B certifies white, m_f < M* - B
//   black.  The returned band is 2B (margin).
inline float certify_band(float mstar, double gmax, double dw) {
  const double u = std::ldexp(1.0, -24);
  double kappa = 8.1 * u + dw + u + 25.0 * std::ldexp(1.0, -53);
  double E = (kappa + 6.1 * u) * 8.0 * gmax;
  double B = 1.0;
  for (int it = 0; it < 60; ++it)
    B = 4.0 * E * std::sqrt(double(mstar) + B) + 2.0 * E * E + 4.1 * u * (double(mstar) + B) +
        2.0 * u * (2.0 * double(mstar) + B);
  return float(2.0 * B + 1e-3);
}

// The same certification in the scaled domain of the centre-normalised taps:
// gx, gy scaled by S, m by S^2, threshold T = S^2 M* represented by the float
// mlo_n (|mlo_n - T| enters the band).  dw is measured against S x the
// reference taps; a normalised pass has at most 3 roundings per term (< the 4
// the 8.1u term allows).
inline float certify_band_scaled(double T, float mlo_n, double gmax_s, double dw) {
  const double u = std::ldexp(1.0, -24);
  double kappa = 8.1 * u + dw + u + 25.0 * std::ldexp(1.0, -53);
  double E = (kappa + 6.1 * u) * 8.0 * gmax_s;
  const double dT = std::fabs(double(mlo_n) - T);
  double B = 1.0;
  for (int it = 0; it < 60; ++it)
    B = 4.0 * E * std::sqrt(T + B) + 2.0 * E * E + 4.1 * u * (T + B) + 2.0 * u * (2.0 * T + B) +
        dT;
  return float(2.0 * B * (1.0 + 1e-6) + 1e-3 * T / 16384.0);
}

// Coverage of the certified path + its parameters.  Returns false when the
// chain is outside it (u8 RGBA video, {0,255} u8 mask, IIR alpha = 0.5,
// gaussian r = 2 with separable taps, threshold > 0, width a multiple of 16
// (TMA strides), 16-byte aligned base); the caller then runs the exact kernel.
// Stencil half of the certified path (S3-S5): separable / centre-normalised
// taps, M*, and the certified bands for inputs in [0, in_max].
inline bool stencil_params(const fc_stage* sg, const fc_stage* sthr, int out_type,
                           double in_max, FastParams* p) {
  if (out_type != FC_U8) return false;
  if (sg->g_radius != 2 || !(sthr->th > 0.0f)) return false;
  if (sthr->white != 255.0f || sthr->black != 0.0f) return false;
  if (!(in_max > 0.0) || !std::isfinite(in_max)) return false;
  // Separable fast taps from the centre row of the reference taps: in exact
  // arithmetic w[2][k] / sum_k w[2][k] is the normalised 1-D gaussian.
  double e[5], row = 0.0, es = 0.0;
  for (int k = 0; k < 5; ++k) row += double(sg->g_w[10 + k]);
  for (int k = 0; k < 5; ++k) es += (e[k] = double(sg->g_w[10 + k]) / row);
  p->h0 = float(e[0] / es);
  p->h1 = float(e[1] / es);
  p->h2 = float(e[2] / es);
  const float hh[5] = {p->h0, p->h1, p->h2, p->h1, p->h0};
  double dw = 0.0;  // worst relative mismatch of h_i h_j vs the reference taps
  for (int j = 0; j < 5; ++j)
    for (int i = 0; i < 5; ++i) {
      double ref = sg->g_w[j * 5 + i];
      dw = std::max(dw, std::fabs(double(hh[j]) * hh[i] - ref) / ref);
    }
  if (!(dw < 1e-5)) return false;  // not separable enough to certify
  std::memcpy(p->taps, sg->g_w, sizeof p->taps);
  p->th_val = sthr->th;
  p->mstar = threshold_mstar(sthr->th);
  p->mlo = std::nextafter(p->mstar, 0.0f);
  double tap_sum = 0.0;
  for (int k = 0; k < 25; ++k) tap_sum += sg->g_w[k];
  p->band = certify_band(p->mstar, in_max * tap_sum * 1.001, dw);
  // centre-normalised taps and their certification (scaled domain)
  const double S = 1.0 / (e[2] / es * (e[2] / es));
  p->g0 = float((e[0] / es) / (e[2] / es));
  p->g1 = float((e[1] / es) / (e[2] / es));
  const double gg[5] = {p->g0, p->g1, 1.0, p->g1, p->g0};
  double dwn = 0.0;
  for (int j = 0; j < 5; ++j)
    for (int i = 0; i < 5; ++i) {
      const double ref = S * double(sg->g_w[j * 5 + i]);
      dwn = std::max(dwn, std::fabs(gg[j] * gg[i] - ref) / ref);
    }
  if (!(dwn < 1e-5)) return false;
  const double T = S * S * double(p->mstar);
  p->mlo_n = float(T);
  p->band_n = certify_band_scaled(T, p->mlo_n, S * in_max * tap_sum * 1.001, dwn);
  return true;
}

// Gray + IIR half of both frame pipelines (exact S1+S2): the u8 RGBA video's
// layout requirements and the folded weights.  pitch: bytes between the
// video's rows (>= width; the TMA map needs it and the base address 16-byte
// aligned).  Returns the upper bound of the IIR values (0: not covered).
inline double iir_params(const fc_stage* sgray, const fc_stage* si, const void* video,
                         int in_type, int gray_in, fc_dims d, int pitch, FastParams* p) {
  if (in_type != FC_U8 || gray_in || sgray == nullptr) return 0.0;
  // any alpha in [0, 1] keeps the IIR a convex combination (the value bound
  // the certification needs); 0.5 takes the folded one-FMA update
  if (!(si->alpha >= 0.0f && si->alpha <= 1.0f)) return 0.0;
  if (sgray->wr < 0.0f || sgray->wg < 0.0f || sgray->wb < 0.0f) return 0.0;
  // width % 4: every stencil lane owns 4 whole columns (its mask store, the
  // edge replication of the IIR cells and the Sobel x clamp assume it)
  if (pitch < d.width || pitch % 16 != 0 || d.width % 4 != 0 || d.height < 1) return 0.0;
  if (reinterpret_cast<uintptr_t>(video) % 16 != 0) return 0.0;
  std::memset(p, 0, sizeof *p);
  p->alpha_half = si->alpha == 0.5f;
  p->ia = si->alpha;
  p->ib = 1.0f - si->alpha;  // host float arithmetic == the reference's
  // alpha = 0.5 folded into the gray weights (exact power-of-two scale)
  const float fold = p->alpha_half ? 0.5f : 1.0f;
  p->wr = sgray->wr * fold;
  p->wg = sgray->wg * fold;
  p->wb = sgray->wb * fold;
  p->wrm = -p->wr * 8388608.0f;
  p->wgm = -p->wg * 8388608.0f;
  p->wbm = -p->wb * 8388608.0f;
  p->k4b = 0x4B000000u;
  // IIR values are convex combinations of gray values in [0, gray_max]
  return 255.0 * (double(sgray->wr) + double(sgray->wg) + double(sgray->wb));
}

inline bool fast_params(const fc_stage* sgray, const fc_stage* si, const fc_stage* sg,
                        const fc_stage* sthr, const void* video, int in_type, int gray_in,
                        int out_type, fc_dims d, int pitch, FastParams* p) {
  const double gray_max = iir_params(sgray, si, video, in_type, gray_in, d, pitch, p);
  return gray_max > 0.0 && stencil_params(sg, sthr, out_type, gray_max, p);
}

// The exact frame pipeline (FP64 gaussian in the reference's order, float
// Sobel, m >= M*): any 5x5 gaussian, a {0, 255} byte mask, th > 0.
inline bool exact_params(const fc_stage* sgray, const fc_stage* si, const fc_stage* sg,
                         const fc_stage* sthr, const void* video, int in_type, int gray_in,
                         int out_type, fc_dims d, int pitch, FastParams* p) {
  if (iir_params(sgray, si, video, in_type, gray_in, d, pitch, p) <= 0.0) return false;
  if (out_type != FC_U8 || sg->g_radius != 2 || !(sthr->th > 0.0f)) return false;
  if (sthr->white != 255.0f || sthr->black != 0.0f) return false;
  std::memcpy(p->taps, sg->g_w, sizeof p->taps);
  p->th_val = sthr->th;
  p->mstar = threshold_mstar(sthr->th);
  p->mlo = std::nextafter(p->mstar, 0.0f);
  return true;
}

inline PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* ptr = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

// 3-D map over f32 planes [T][H][W] with a box of (bw, rows, 1): one copy
// brings a haloed window of one frame (the F345 input of the pipe kernel).
inline bool plane_tensor_map(CUtensorMap* map, const void* planes, fc_dims d, int bw, int rows) {
  auto enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[3] = {cuuint64_t(d.width), cuuint64_t(d.height), cuuint64_t(d.frames)};
  cuuint64_t strides[2] = {cuuint64_t(d.width) * 4, cuuint64_t(d.width) * d.height * 4};
  cuuint32_t box[3] = {cuuint32_t(bw), cuuint32_t(rows), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(planes), dims, strides,
             box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

// 3-D map over the planar video [4T][H][pitch] u8 (width W used) with a box
// of (bw, rows, 3): one copy brings the R, G, B planes of a haloed window of
// one frame.
inline bool rgb_tensor_map(CUtensorMap* map, const void* video, fc_dims d, int bw, int rows,
                           int pitch) {
  auto enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[3] = {cuuint64_t(d.width), cuuint64_t(d.height), cuuint64_t(4) * d.frames};
  cuuint64_t strides[2] = {cuuint64_t(pitch), cuuint64_t(pitch) * d.height};
  cuuint32_t box[3] = {cuuint32_t(bw), cuuint32_t(rows), 3};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(video), dims, strides,
             box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace fccommon
