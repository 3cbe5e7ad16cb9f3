// Reference-exact sm_100a kernels for every stage of the SPEC chain and the
// rest of the stencil catalog, plus the exact fused partitions.
//
// Arithmetic contract (simulator.cpp:48-108): every
// float op is an explicit round-to-nearest intrinsic (__fmul_rn/__fadd_rn/
// __fsub_rn/__fsqrt_rn) so nothing is contracted; the gaussian accumulates
// in FP64 in dy-outer/dx-inner order (a DFMA equals the reference's
// "acc += double(w) * src" because a float*float product is exact in double);
// no flush-to-zero (the IIR decays into subnormals on dark pixels).
// Borders: every stage reads ITS OWN input clamped to the video
// (simulator.cpp:202-210): inside fused tiles a stage's out-of-video halo cell
// holds that stage's value at the clamped position.
#include <cuda_runtime.h>

#include <utility>

#include <algorithm>
#include <cstdint>

#include "fc_kernels.h"

namespace fc {

__device__ __forceinline__ int clampi(int v, int lo, int hi) {
  return min(max(v, lo), hi);
}

template <typename T>
__device__ __forceinline__ float to_f(T v);
template <>
__device__ __forceinline__ float to_f<uint8_t>(uint8_t v) {
  return float(v);
}
template <>
__device__ __forceinline__ float to_f<float>(float v) {
  return v;
}

template <typename T>
__device__ __forceinline__ T from_level(float v);
template <>
__device__ __forceinline__ uint8_t from_level<uint8_t>(float v) {
  return uint8_t(v);  // only used for white/black values that are bytes
}
template <>
__device__ __forceinline__ float from_level<float>(float v) {
  return v;
}

// simulator.cpp:51-56
__device__ __forceinline__ float gray_op(const fc_stage& s, float r, float g,
                                         float b) {
  return __fadd_rn(__fadd_rn(__fmul_rn(s.wr, r), __fmul_rn(s.wg, g)),
                   __fmul_rn(s.wb, b));
}

// simulator.cpp:57-62 with beta = float(1 - alpha) computed in float
__device__ __forceinline__ float iir_op(float alpha, float beta, float x,
                                        float prev) {
  return __fadd_rn(__fmul_rn(alpha, x), __fmul_rn(beta, prev));
}

// simulator.cpp:75-83; s(dx,dy) supplied by the caller
template <typename S>
__device__ __forceinline__ float sobel_op(S s) {
  float gx = __fsub_rn(
      __fadd_rn(__fadd_rn(s(1, -1), __fmul_rn(2.0f, s(1, 0))), s(1, 1)),
      __fadd_rn(__fadd_rn(s(-1, -1), __fmul_rn(2.0f, s(-1, 0))), s(-1, 1)));
  float gy = __fsub_rn(
      __fadd_rn(__fadd_rn(s(-1, 1), __fmul_rn(2.0f, s(0, 1))), s(1, 1)),
      __fadd_rn(__fadd_rn(s(-1, -1), __fmul_rn(2.0f, s(0, -1))), s(1, -1)));
  return __fsqrt_rn(__fadd_rn(__fmul_rn(gx, gx), __fmul_rn(gy, gy)));
}

// ------------------------------------------------------------ unfused stages
// The paper's sequential baseline: one launch per stage, every intermediate
// plane in HBM.  Each kernel is a vectorised stream over its own bytes
// (uint4 / float4 accesses, several frames or pixels per thread) so that the
// fused-versus-sequential comparison is made against efficient unfused
// kernels; frames are looped inside the grid (no gridDim.z limit).

// fl(w * c) for a byte c held as the float c + 2^23 (one PRMT): the FMA
// w * (c + 2^23) - w 2^23 rounds the exact product w c once (w 2^23 exact).
template <int K>
__device__ __forceinline__ float byte_magic(uint32_t w) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(w), "r"(0x4B000000u), "n"(0x7440 + K));
  return __uint_as_float(r);
}

// simulator.cpp:51-56 on four pixels packed as bytes of r, g, b words
__device__ __forceinline__ float4 gray4(const fc_stage& s, float wrm, float wgm, float wbm,
                                        uint32_t r, uint32_t g, uint32_t b) {
#define FC_G(K)                                                                   \
  __fadd_rn(__fadd_rn(__fmaf_rn(s.wr, byte_magic<K>(r), wrm),                     \
                      __fmaf_rn(s.wg, byte_magic<K>(g), wgm)),                    \
            __fmaf_rn(s.wb, byte_magic<K>(b), wbm))
  return make_float4(FC_G(0), FC_G(1), FC_G(2), FC_G(3));
#undef FC_G
}

// u8 RGBA -> gray, 16 pixels per work item (hw % 16 == 0, 16-byte aligned)
__global__ void k_rgba2gray_u8x16(const uint8_t* __restrict__ in, float* __restrict__ out,
                                  fc_stage s, long long hw, long long n16) {
  const float wrm = -s.wr * 8388608.0f, wgm = -s.wg * 8388608.0f, wbm = -s.wb * 8388608.0f;
  const long long q = hw / 16;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n16;
       i += (long long)gridDim.x * blockDim.x) {
    const long long t = i / q, p = (i - t * q) * 16;
    const uint8_t* f = in + t * 4 * hw + p;
    const uint4 r = __ldcs(reinterpret_cast<const uint4*>(f));
    const uint4 g = __ldcs(reinterpret_cast<const uint4*>(f + hw));
    const uint4 b = __ldcs(reinterpret_cast<const uint4*>(f + 2 * hw));
    float4* o = reinterpret_cast<float4*>(out + t * hw + p);
    __stcs(o + 0, gray4(s, wrm, wgm, wbm, r.x, g.x, b.x));
    __stcs(o + 1, gray4(s, wrm, wgm, wbm, r.y, g.y, b.y));
    __stcs(o + 2, gray4(s, wrm, wgm, wbm, r.z, g.z, b.z));
    __stcs(o + 3, gray4(s, wrm, wgm, wbm, r.w, g.w, b.w));
  }
}

template <typename InT>
__global__ void k_rgba2gray(const InT* __restrict__ in, float* __restrict__ out,
                            fc_stage s, long long hw, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    long long t = i / hw, p = i - t * hw;
    const InT* f = in + t * 4 * hw + p;
    out[i] = gray_op(s, to_f(f[0]), to_f(f[hw]), to_f(f[2 * hw]));
  }
}

// One thread per pixel scans t (simulator.cpp:136-147).  Loads of later
// frames do not depend on the carried state, so the unrolled loop keeps
// several frames in flight.
__global__ void k_iir(const float* __restrict__ in, float* __restrict__ out,
                      float alpha, float beta, long long hw, int n_frames,
                      int n_warm, const float* __restrict__ state_in,
                      float* __restrict__ state_out) {
  long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (p >= hw) return;
  float prev = state_in ? state_in[p] : 0.0f;
  bool fresh = state_in == nullptr;
#pragma unroll 8
  for (int t = 0; t < n_frames; ++t) {
    float x = in[t * hw + p];
    prev = (fresh && t == 0) ? x : iir_op(alpha, beta, x, prev);
    if (t >= n_warm) out[(t - n_warm) * hw + p] = prev;
  }
  if (state_out) state_out[p] = prev;
}

// Same scan on four pixels per thread (float4), eight frames of loads issued
// ahead of the recurrence (hw % 4 == 0, 16-byte aligned planes).
__global__ void k_iir_x4(const float* __restrict__ in, float* __restrict__ out, float alpha,
                         float beta, long long hw, int n_frames, int n_warm,
                         const float* __restrict__ state_in, float* __restrict__ state_out) {
  const long long p = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * 4;
  if (p >= hw) return;
  const float4* src = reinterpret_cast<const float4*>(in + p);
  float4* dst = reinterpret_cast<float4*>(out + p);
  const long long step = hw / 4;
  float4 y = state_in ? *reinterpret_cast<const float4*>(state_in + p)
                      : make_float4(0.f, 0.f, 0.f, 0.f);
  const bool fresh = state_in == nullptr;
  constexpr int U = 8;
  int t = 0;
  for (; t < n_frames; t += U) {
    float4 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (t + u < n_frames) x[u] = __ldcs(src + (long long)(t + u) * step);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (t + u >= n_frames) break;
      if (fresh && t + u == 0) {
        y = x[u];
      } else {
        y.x = iir_op(alpha, beta, x[u].x, y.x);
        y.y = iir_op(alpha, beta, x[u].y, y.y);
        y.z = iir_op(alpha, beta, x[u].z, y.z);
        y.w = iir_op(alpha, beta, x[u].w, y.w);
      }
      if (t + u >= n_warm) __stcs(dst + (long long)(t + u - n_warm) * step, y);
    }
  }
  if (state_out) *reinterpret_cast<float4*>(state_out + p) = y;
}

// Gaussian weights widened to double once on the host (kernel parameter:
// the DFMA reads them from the constant bank, no register or LDS cost).
struct GaussW {
  double w[(2 * FC_MAX_GAUSS_RADIUS + 1) * (2 * FC_MAX_GAUSS_RADIUS + 1)];
};

// fn(integral_constant<int, I>) for I = I0 .. N - 1, unrolled at compile time
template <int I, int N, typename Fn>
__device__ __forceinline__ void unroll_steps(Fn&& fn) {
  if constexpr (I < N) {
    fn(std::integral_constant<int, I>{});
    unroll_steps<I + 1, N>(fn);
  }
}

// Row-marching unfused stencils (no shared memory, no CTA barrier): a thread
// owns 4 consecutive columns of a band of RB rows and marches the band's rows
// plus the halo, loading each input row once (L1-cached, clamped to the
// frame: the stage's own per-stage clamp) and keeping the rows it still
// needs in registers.
constexpr int RB = 32;     // output rows per band
constexpr int RTHR = 128;  // threads per CTA (512 columns)

// 4 + 2P consecutive input columns x - P .. x + 3 + P of row y (clamped)
template <int P>
__device__ __forceinline__ void load_cols(const float* __restrict__ row, int x, int W,
                                          bool interior, float (&v)[4 + 2 * P]) {
  if (interior) {  // x - 4 .. x + 7 in three aligned float4 (W % 4 == 0)
    const float4 a = __ldg(reinterpret_cast<const float4*>(row + x - 4));
    const float4 b = __ldg(reinterpret_cast<const float4*>(row + x));
    const float4 c = __ldg(reinterpret_cast<const float4*>(row + x + 4));
    const float w12[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x, c.y, c.z, c.w};
#pragma unroll
    for (int j = 0; j < 4 + 2 * P; ++j) v[j] = w12[4 - P + j];
  } else {
#pragma unroll
    for (int j = 0; j < 4 + 2 * P; ++j) v[j] = __ldg(row + clampi(x - P + j, 0, W - 1));
  }
}

__device__ __forceinline__ void store4(float* __restrict__ o, int x, int W, bool vec,
                                       float a, float b, float c, float d) {
  if (vec) {
    __stcs(reinterpret_cast<float4*>(o), make_float4(a, b, c, d));
  } else {
    const float m[4] = {a, b, c, d};
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (x + j < W) o[j] = m[j];
  }
}

// Exact FP64 gaussian (simulator.cpp:63-74).  Each loaded row r feeds the K
// output rows g = r - R .. r + R that read it, as their tap row dy = r - g + R:
// every output's 25 (K^2) products accumulate in the reference's dy-outer /
// dx-inner order, and a step carries K x 4 independent DFMA chains.
template <int R>
__global__ void __launch_bounds__(RTHR) k_gaussian_rows(const float* __restrict__ in,
                                                        float* __restrict__ out, GaussW gw,
                                                        int W, int H, int F) {
  constexpr int K = 2 * R + 1, NV = 4 + 2 * R;
  const int x = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
  if (x >= W) return;
  const int y0 = blockIdx.y * RB, y1 = min(y0 + RB, H);
  // vector loads / stores need 16-byte aligned planes (W % 4 == 0 keeps the
  // rows aligned)
  const bool al_in = (reinterpret_cast<uintptr_t>(in) & 15) == 0;
  const bool al_out = (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  const bool interior = al_in && (W & 3) == 0 && x >= 4 && x + 8 <= W && R <= 4;
  const bool vec = al_out && (W & 3) == 0 && x + 3 < W;
  const long long hw = (long long)W * H;
  for (int t = blockIdx.z; t < F; t += gridDim.z) {
    const float* f = in + t * hw;
    float* o = out + t * hw;
    double acc[K][4];  // output row g at ring index g % K
    // steps r = y0 - R .. y1 - 1 + R in bodies of K (ring indices
    // compile-time: step r uses ring slot (r + R - dy) % K for tap row dy,
    // counted from the band start so the slots are fixed per body position)
    auto step = [&](int r, auto pos_t) {
      constexpr int POS = decltype(pos_t)::value;  // (r - (y0 - R)) % K
      float vf[NV];
      load_cols<R>(f + (long long)clampi(r, 0, H - 1) * W, x, W, interior, vf);
      double v[NV];
#pragma unroll
      for (int j = 0; j < NV; ++j) v[j] = double(vf[j]);
#pragma unroll
      for (int dy = 0; dy < K; ++dy) {
        // output row g = r + R - dy, ring slot (g - (y0 - 2R)) % K = (POS + 2R - dy) % K
        constexpr int dummy = 0;
        (void)dummy;
        const int gs = (POS + 2 * R - dy + K) % K;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          double tt = dy == 0 ? 0.0 : acc[gs][j];
#pragma unroll
          for (int dx = 0; dx < K; ++dx) tt = __fma_rn(gw.w[dy * K + dx], v[j + dx], tt);
          acc[gs][j] = tt;
        }
      }
      // the row completing this step: g = r - R (its last tap row dy = 2R)
      const int g = r - R;
      if (g >= y0 && g < y1) {
        const int gs = (POS + 2 * R - (K - 1) + K) % K;
        store4(o + (long long)g * W + x, x, W, vec, __double2float_rn(acc[gs][0]),
               __double2float_rn(acc[gs][1]), __double2float_rn(acc[gs][2]),
               __double2float_rn(acc[gs][3]));
      }
    };
    int r = y0 - R;
    const int rend = y1 + R;  // exclusive
#pragma unroll 1
    for (; r + K <= rend; r += K)
      unroll_steps<0, K>([&](auto i_t) { step(r + decltype(i_t)::value, i_t); });
    unroll_steps<0, K>([&](auto i_t) {
      if (r + decltype(i_t)::value < rend) step(r + decltype(i_t)::value, i_t);
    });
  }
}

// Sobel magnitude (simulator.cpp:75-83) on 4 columns per thread, a 3-row
// window in registers.
__global__ void __launch_bounds__(RTHR) k_gradient_rows(const float* __restrict__ in,
                                                        float* __restrict__ out, int W, int H,
                                                        int F) {
  const int x = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
  if (x >= W) return;
  const int y0 = blockIdx.y * RB, y1 = min(y0 + RB, H);
  const bool al_in = (reinterpret_cast<uintptr_t>(in) & 15) == 0;
  const bool al_out = (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  const bool interior = al_in && (W & 3) == 0 && x >= 4 && x + 8 <= W;
  const bool vec = al_out && (W & 3) == 0 && x + 3 < W;
  const long long hw = (long long)W * H;
  for (int t = blockIdx.z; t < F; t += gridDim.z) {
    const float* f = in + t * hw;
    float* o = out + t * hw;
    float w[3][6];  // rows at ring index r % 3, columns x - 1 .. x + 4
    auto load = [&](int r, auto slot_t) {
      constexpr int SL = decltype(slot_t)::value;
      load_cols<1>(f + (long long)clampi(r, 0, H - 1) * W, x, W, interior, w[SL]);
    };
    auto emit = [&](int y, auto m_t) {  // rows y-1, y, y+1 at slots (M+2)%3, M, (M+1)%3
      constexpr int M = decltype(m_t)::value;
      float m[4];
#pragma unroll
      for (int j = 0; j < 4; ++j)
        m[j] = sobel_op([&](int dx, int dy) {
          return w[(M + 3 + dy) % 3][1 + j + dx];
        });
      store4(o + (long long)y * W + x, x, W, vec, m[0], m[1], m[2], m[3]);
    };
    // slot of row r: (r - (y0 - 1)) % 3; output row y uses rows y-1 .. y+1
    load(y0 - 1, std::integral_constant<int, 0>{});
    load(y0, std::integral_constant<int, 1>{});
    int y = y0;
#pragma unroll 1
    for (; y + 3 <= y1; y += 3) {
      load(y + 1, std::integral_constant<int, 2>{});
      emit(y, std::integral_constant<int, 1>{});
      load(y + 2, std::integral_constant<int, 0>{});
      emit(y + 1, std::integral_constant<int, 2>{});
      load(y + 3, std::integral_constant<int, 1>{});
      emit(y + 2, std::integral_constant<int, 0>{});
    }
    if (y < y1) {
      load(y + 1, std::integral_constant<int, 2>{});
      emit(y, std::integral_constant<int, 1>{});
    }
    if (y + 1 < y1) {
      load(y + 2, std::integral_constant<int, 0>{});
      emit(y + 1, std::integral_constant<int, 2>{});
    }
  }
}

__device__ __forceinline__ float point_op(const fc_stage& s, float v) {
  if (s.op == FC_THRESHOLD) return v >= s.th ? s.white : s.black;  // simulator.cpp:84-89
  if (s.op == FC_SCALE_OFFSET) return __fadd_rn(__fmul_rn(s.scale, v), s.offset);  // :91-95
  return v;  // identity :90
}

template <typename OutT>
__global__ void k_pointwise(const float* __restrict__ in, OutT* __restrict__ out,
                            fc_stage s, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = from_level<OutT>(point_op(s, in[i]));
}

// Four elements per thread (n % 4 == 0, 16-byte aligned).
__global__ void k_pointwise_x4_u8(const float* __restrict__ in, uint8_t* __restrict__ out,
                                  fc_stage s, long long n4) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    const float4 v = __ldcs(reinterpret_cast<const float4*>(in) + i);
    const uint32_t r = uint32_t(from_level<uint8_t>(point_op(s, v.x))) |
                       uint32_t(from_level<uint8_t>(point_op(s, v.y))) << 8 |
                       uint32_t(from_level<uint8_t>(point_op(s, v.z))) << 16 |
                       uint32_t(from_level<uint8_t>(point_op(s, v.w))) << 24;
    reinterpret_cast<uint32_t*>(out)[i] = r;
  }
}

__global__ void k_pointwise_x4_f32(const float* __restrict__ in, float* __restrict__ out,
                                   fc_stage s, long long n4) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    const float4 v = __ldcs(reinterpret_cast<const float4*>(in) + i);
    __stcs(reinterpret_cast<float4*>(out) + i,
           make_float4(point_op(s, v.x), point_op(s, v.y), point_op(s, v.z), point_op(s, v.w)));
  }
}

// float(u8) (video.cpp:87) for a single-channel u8 video entering a stage
// that reads f32 planes.
__global__ void k_u8_to_f32(const uint8_t* __restrict__ in, float* __restrict__ out,
                            long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = float(in[i]);
}

// box_mean (simulator.cpp:96-106): double accumulation dt, dy, dx, clamp in
// x, y and t; result float(acc / volume).
__global__ void k_box_mean(const float* __restrict__ in, float* __restrict__ out,
                           int rx, int ry, int rt, int W, int H, int F) {
  long long hw = (long long)W * H, n = hw * F;
  double vol = double((2 * rx + 1) * (2 * ry + 1) * (2 * rt + 1));
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    int t = int(i / hw);
    int p = int(i - t * hw);
    int y = p / W, x = p - y * W;
    double acc = 0.0;
    for (int dt = -rt; dt <= rt; ++dt) {
      const float* f = in + clampi(t + dt, 0, F - 1) * hw;
      for (int dy = -ry; dy <= ry; ++dy) {
        const float* row = f + (long long)clampi(y + dy, 0, H - 1) * W;
        for (int dx = -rx; dx <= rx; ++dx)
          acc = __dadd_rn(acc, double(row[clampi(x + dx, 0, W - 1)]));
      }
    }
    out[i] = __double2float_rn(__ddiv_rn(acc, vol));
  }
}

// ------------------------------------------------------------ F12

template <typename InT>
__global__ void k_gray_iir(const InT* __restrict__ video, float* __restrict__ out,
                           fc_stage sg, float alpha, float beta, long long hw,
                           int n_frames, int n_warm,
                           const float* __restrict__ state_in,
                           float* __restrict__ state_out) {
  long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (p >= hw) return;
  float prev = state_in ? state_in[p] : 0.0f;
  bool fresh = state_in == nullptr;
#pragma unroll 4
  for (int t = 0; t < n_frames; ++t) {
    const InT* f = video + (long long)t * 4 * hw + p;
    float x = gray_op(sg, to_f(f[0]), to_f(f[hw]), to_f(f[2 * hw]));
    prev = (fresh && t == 0) ? x : iir_op(alpha, beta, x, prev);
    if (t >= n_warm) out[(t - n_warm) * hw + p] = prev;
  }
  if (state_out) state_out[p] = prev;
}

// ------------------------------------------------------------ F345
// One CTA per (32x16 tile, frame).  Stage the IIR plane with a halo of R+1
// as double (converted once per element), compute the gaussian on the
// tile+1 ring (centres clamped to the video, so the ring's out-of-video cells
// carry the edge value the gradient must see), then Sobel + threshold.
constexpr int FW = 32, FH = 16, FT = 256;

// The staged double plane of the fused exact kernels: rows of DP doubles
// (even, so every row is 16-byte aligned), ring column c of the gaussian at
// staged column c + R (staged column 0 = video column x0 - 1 - R).
template <int R>
struct RingGeom {
  static constexpr int K = 2 * R + 1;
  static constexpr int GW = FW + 2, GH = FH + 2;       // ring: the tile + 1
  static constexpr int RG = (GW + 3) / 4;              // 4-wide ring groups per row
  static constexpr int DW = 4 * RG + 2 * R;            // staged columns read
  static constexpr int DP = DW + (DW & 1);             // row pitch (even)
  static constexpr int DH = GH + 2 * R;
};

// Exact FP64 gaussian of the ring (simulator.cpp:63-74, dy-outer / dx-inner
// accumulation): a thread computes four neighbouring ring cells from one
// pass over 4 + 2R staged doubles per row (LDS.128 pairs); cells whose
// centre is clamped to the video (border tiles) take the per-cell form.
template <int R>
__device__ __forceinline__ void ring_gaussian(const double* __restrict__ d, float* __restrict__ g,
                                              const GaussW& gw, int x0, int y0, int W, int H) {
  using G = RingGeom<R>;
  constexpr int K = G::K;
  for (int item = threadIdx.x; item < G::RG * G::GH; item += FT) {
    const int ry = item / G::RG, rc = 4 * (item - ry * G::RG);
    const int cy = clampi(y0 + ry - 1, 0, H - 1) - (y0 - 1 - R);  // staged row of the centre
    bool plain = true;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int xv = x0 - 1 + rc + j;
      plain = plain && (rc + j >= G::GW || (xv >= 0 && xv <= W - 1));
    }
    if (plain) {
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int dy = 0; dy < K; ++dy) {
        const double* row = d + (cy - R + dy) * G::DP + rc;
        double v[4 + 2 * R + 1];
#pragma unroll
        for (int q = 0; q < (4 + 2 * R + 1) / 2; ++q) {
          const double2 t = *reinterpret_cast<const double2*>(row + 2 * q);
          v[2 * q] = t.x;
          v[2 * q + 1] = t.y;
        }
#pragma unroll
        for (int dx = 0; dx < K; ++dx)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[j] = __fma_rn(gw.w[dy * K + dx], v[j + dx], acc[j]);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (rc + j < G::GW) g[ry * G::GW + rc + j] = __double2float_rn(acc[j]);
    } else {
      for (int j = 0; j < 4 && rc + j < G::GW; ++j) {
        const int cx = clampi(x0 - 1 + rc + j, 0, W - 1) - (x0 - 1 - R);
        double acc = 0.0;
        for (int dy = 0; dy < K; ++dy)
          for (int dx = 0; dx < K; ++dx)
            acc = __fma_rn(gw.w[dy * K + dx], d[(cy - R + dy) * G::DP + cx - R + dx], acc);
        g[ry * G::GW + rc + j] = __double2float_rn(acc);
      }
    }
  }
}

template <int R, typename OutT>
__device__ __forceinline__ void ring_sobel_threshold(const float* __restrict__ g,
                                                     OutT* __restrict__ o, float th, float white,
                                                     float black, int x0, int y0, int W, int H) {
  using G = RingGeom<R>;
  for (int i = threadIdx.x; i < FW * FH; i += FT) {
    const int ty = i / FW, tx = i - ty * FW;
    const int x = x0 + tx, y = y0 + ty;
    if (x >= W || y >= H) continue;
    const float m =
        sobel_op([&](int dx, int dy) { return g[(ty + 1 + dy) * G::GW + tx + 1 + dx]; });
    o[(long long)y * W + x] = from_level<OutT>(m >= th ? white : black);
  }
}

template <int R, typename OutT>
__global__ void __launch_bounds__(FT) k_gauss_grad_thr(
    const float* __restrict__ in, OutT* __restrict__ out, GaussW gw,
    float th, float white, float black, int W, int H) {
  using G = RingGeom<R>;
  __shared__ __align__(16) double d[G::DH * G::DP];
  __shared__ float g[G::GH * G::GW];
  const int x0 = blockIdx.x * FW, y0 = blockIdx.y * FH;
  const long long hw = (long long)W * H;
  const float* f = in + blockIdx.z * hw;
  for (int i = threadIdx.x; i < G::DP * G::DH; i += FT) {
    const int sy = i / G::DP, sx = i - sy * G::DP;
    const int gx = clampi(x0 - 1 - R + sx, 0, W - 1);
    const int gy = clampi(y0 - 1 - R + sy, 0, H - 1);
    d[i] = double(__ldg(f + (long long)gy * W + gx));
  }
  __syncthreads();
  ring_gaussian<R>(d, g, gw, x0, y0, W, H);
  __syncthreads();
  ring_sobel_threshold<R>(g, out + blockIdx.z * hw, th, white, black, x0, y0, W, H);
}

// ------------------------------------------------------------ F12345 exact
// Streaming all-fused chain: one CTA per spatial tile marches over t, the IIR
// state of its staged cells lives in registers, the frame's inputs for t+1
// are loaded while t is computed.  Reference-exact everywhere (FP64
// gaussian); the certified kernel is fc_pipe.cu's frame pipeline.
template <int R>
struct ChainGeom {
  static constexpr int NS = (RingGeom<R>::DP * RingGeom<R>::DH + FT - 1) / FT;  // cells / thread
};

template <int R, typename InT, typename OutT, bool GRAY_IN>
__global__ void __launch_bounds__(FT) k_chain_exact(
    const InT* __restrict__ video, OutT* __restrict__ out, fc_stage sgray,
    float alpha, float beta, GaussW gw, float th, float white, float black,
    int W, int H, int n_frames, int n_warm, const float* __restrict__ state_in,
    float* __restrict__ state_out) {
  using G = RingGeom<R>;
  constexpr int NS = ChainGeom<R>::NS, NCELL = G::DP * G::DH;
  constexpr int C = GRAY_IN ? 1 : 4;
  __shared__ __align__(16) double d[NCELL];
  __shared__ float g[G::GH * G::GW];
  const int x0 = blockIdx.x * FW, y0 = blockIdx.y * FH;
  const long long hw = (long long)W * H;
  const int tid = threadIdx.x;

  // loop-invariant clamped source offsets of the owned IIR cells
  int src[NS];
  float st[NS];
  const bool fresh = state_in == nullptr;
#pragma unroll
  for (int k = 0; k < NS; ++k) {
    const int i = tid + k * FT;
    const int sy = i / G::DP, sx = i - sy * G::DP;
    const int gx = clampi(x0 - 1 - R + sx, 0, W - 1);
    const int gy = clampi(y0 - 1 - R + sy, 0, H - 1);
    src[k] = gy * W + gx;
    st[k] = (i < NCELL && state_in) ? state_in[src[k]] : 0.0f;
  }
  float cur[NS][3], nxt[NS][3];
  auto load = [&](int t, float (&v)[NS][3]) {
    const InT* f = video + (long long)t * C * hw;
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      if (tid + k * FT < NCELL) {
#pragma unroll
        for (int c = 0; c < (GRAY_IN ? 1 : 3); ++c) v[k][c] = to_f(__ldg(f + c * hw + src[k]));
      }
    }
  };
  load(0, cur);
  for (int t = 0; t < n_frames; ++t) {
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      const int i = tid + k * FT;
      if (i < NCELL) {
        const float x = GRAY_IN ? cur[k][0] : gray_op(sgray, cur[k][0], cur[k][1], cur[k][2]);
        st[k] = (fresh && t == 0) ? x : iir_op(alpha, beta, x, st[k]);
        d[i] = double(st[k]);
      }
    }
    if (t + 1 < n_frames) load(t + 1, nxt);
    __syncthreads();
    if (t >= n_warm) ring_gaussian<R>(d, g, gw, x0, y0, W, H);
    __syncthreads();
    if (t >= n_warm)
      ring_sobel_threshold<R>(g, out + (long long)(t - n_warm) * hw, th, white, black, x0, y0,
                              W, H);
#pragma unroll
    for (int k = 0; k < NS; ++k)
#pragma unroll
      for (int c = 0; c < 3; ++c) cur[k][c] = nxt[k][c];
  }
  if (state_out) {
    // write back the state of the cells that are the tile's own pixels
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      const int i = tid + k * FT;
      const int sy = i / G::DP, sx = i - sy * G::DP;
      const int x = x0 - 1 - R + sx, y = y0 - 1 - R + sy;
      if (i < NCELL && sx >= R + 1 && sx < R + 1 + FW && sy >= R + 1 && sy < R + 1 + FH &&
          x < W && y < H)
        state_out[(long long)y * W + x] = st[k];
    }
  }
}

// ------------------------------------------------------------ synthetic input

__global__ void k_hash_video(uint8_t* __restrict__ out, long long n, int C, int H,
                             int W, long long t0, unsigned long long seed_term) {
  long long per_frame = (long long)C * H * W;
  long long base = t0 * per_frame;
  for (long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * 16; i < n;
       i += (long long)gridDim.x * blockDim.x * 16) {
    if (i + 16 <= n) {
      uint32_t words[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t wv = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          unsigned long long z = (unsigned long long)(base + i + q * 4 + b) + seed_term;
          z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
          z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
          z ^= z >> 31;
          wv |= uint32_t(z >> 56) << (8 * b);
        }
        words[q] = wv;
      }
      *reinterpret_cast<uint4*>(out + i) = make_uint4(words[0], words[1], words[2], words[3]);
    } else {
      for (long long j = i; j < n; ++j) {
        unsigned long long z = (unsigned long long)(base + j) + seed_term;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        out[j] = uint8_t(z >> 56);
      }
    }
  }
}

inline int grid_for(long long n, int block) {
  long long g = (n + block - 1) / block;
  return int(g > 148LL * 64 ? 148LL * 64 : (g < 1 ? 1 : g));
}

inline int status() { return int(cudaGetLastError()); }

}  // namespace fc

using namespace fc;

extern "C" {

const char* fc_error_string(int code) {
  if (code == -1) return "unsupported kernel arguments";
  return cudaGetErrorString(cudaError_t(code));
}

int fc_stage_spatial(const fc_stage* s, const void* in, int in_type, void* out,
                     int out_type, fc_dims d, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  long long hw = (long long)d.width * d.height, n = hw * d.frames;
  if (n == 0) return 0;
  auto aligned = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  // row-marching stencils: column groups x bands of RB rows x ~4 frames per
  // CTA (frames looped inside, z <= 65535): many short CTAs keep the hardware
  // scheduler's dynamic balance
  auto rows_frame_groups = [&]() { return std::max(1, std::min(65535, (d.frames + 3) / 4)); };
  const int quads = (d.width + 3) / 4;  // 4-column groups of a row
  const int rthr = std::min(RTHR, (quads + 31) / 32 * 32);
  switch (s->op) {
    case FC_RGBA2GRAY:
      if (out_type != FC_F32) return -1;
      if (in_type == FC_U8 && hw % 16 == 0 && aligned(in) && aligned(out))
        k_rgba2gray_u8x16<<<grid_for(n / 16, 256), 256, 0, st>>>(
            static_cast<const uint8_t*>(in), static_cast<float*>(out), *s, hw, n / 16);
      else if (in_type == FC_U8)
        k_rgba2gray<uint8_t><<<grid_for(n, 256), 256, 0, st>>>(
            static_cast<const uint8_t*>(in), static_cast<float*>(out), *s, hw, n);
      else
        k_rgba2gray<float><<<grid_for(n, 256), 256, 0, st>>>(
            static_cast<const float*>(in), static_cast<float*>(out), *s, hw, n);
      return status();
    case FC_GAUSSIAN: {
      if (in_type != FC_F32 || out_type != FC_F32) return -1;
      auto f = static_cast<const float*>(in);
      auto o = static_cast<float*>(out);
      GaussW w;
      const int K = 2 * s->g_radius + 1;
      for (int i = 0; i < K * K; ++i) w.w[i] = double(s->g_w[i]);
#define FC_GK(R)                                                                     \
  k_gaussian_rows<R><<<dim3((quads + rthr - 1) / rthr, (d.height + RB - 1) / RB,         \
                           rows_frame_groups()),                                         \
                       rthr, 0, st>>>(f, o, w, d.width, d.height, d.frames)
      switch (s->g_radius) {
        case 0: FC_GK(0); break;
        case 1: FC_GK(1); break;
        case 2: FC_GK(2); break;
        case 3: FC_GK(3); break;
        case 4: FC_GK(4); break;
        default: return -1;
      }
#undef FC_GK
      return status();
    }
    case FC_GRADIENT:
      if (in_type != FC_F32 || out_type != FC_F32) return -1;
      k_gradient_rows<<<dim3((quads + rthr - 1) / rthr, (d.height + RB - 1) / RB,
                             rows_frame_groups()),
                        rthr, 0, st>>>(static_cast<const float*>(in), static_cast<float*>(out),
                                       d.width, d.height, d.frames);
      return status();
    case FC_THRESHOLD:
    case FC_IDENTITY:
    case FC_SCALE_OFFSET:
      if (s->op == FC_IDENTITY && in_type == FC_U8 && out_type == FC_F32) {
        k_u8_to_f32<<<grid_for(n, 256), 256, 0, st>>>(
            static_cast<const uint8_t*>(in), static_cast<float*>(out), n);
        return status();
      }
      if (in_type != FC_F32) return -1;
      if (n % 4 == 0 && aligned(in) && aligned(out)) {
        if (out_type == FC_U8)
          k_pointwise_x4_u8<<<grid_for(n / 4, 256), 256, 0, st>>>(
              static_cast<const float*>(in), static_cast<uint8_t*>(out), *s, n / 4);
        else
          k_pointwise_x4_f32<<<grid_for(n / 4, 256), 256, 0, st>>>(
              static_cast<const float*>(in), static_cast<float*>(out), *s, n / 4);
      } else if (out_type == FC_U8) {
        k_pointwise<uint8_t><<<grid_for(n, 256), 256, 0, st>>>(
            static_cast<const float*>(in), static_cast<uint8_t*>(out), *s, n);
      } else {
        k_pointwise<float><<<grid_for(n, 256), 256, 0, st>>>(
            static_cast<const float*>(in), static_cast<float*>(out), *s, n);
      }
      return status();
    case FC_BOX_MEAN:
      if (in_type != FC_F32 || out_type != FC_F32) return -1;
      k_box_mean<<<grid_for(n, 256), 256, 0, st>>>(
          static_cast<const float*>(in), static_cast<float*>(out), s->rx, s->ry,
          s->rt, d.width, d.height, d.frames);
      return status();
    default:
      return -1;
  }
}

int fc_stage_iir(const fc_stage* s, const float* in, float* out, fc_dims d,
                 int n_warm, const float* state_in, float* state_out,
                 void* stream) {
  long long hw = (long long)d.width * d.height;
  if (hw == 0 || d.frames == 0) return 0;
  float beta = 1.0f - s->alpha;  // host float arithmetic == reference's
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  auto aligned = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (hw % 4 == 0 && aligned(in) && aligned(out) && aligned(state_in) && aligned(state_out)) {
    const long long th = hw / 4;
    k_iir_x4<<<int((th + 127) / 128), 128, 0, st>>>(in, out, s->alpha, beta, hw, d.frames,
                                                     n_warm, state_in, state_out);
  } else {
    k_iir<<<int((hw + 127) / 128), 128, 0, st>>>(in, out, s->alpha, beta, hw, d.frames,
                                                 n_warm, state_in, state_out);
  }
  return status();
}

int fc_gray_iir_stream(const fc_stage* sg, const fc_stage* si, const void* video,
                       int in_type, float* out, fc_dims d, int n_warm,
                       const float* state_in, float* state_out, void* stream);  // fc_f12.cu

int fc_fused_gray_iir(const fc_stage* sg, const fc_stage* si, const void* video,
                      int in_type, float* out, fc_dims d, int n_warm,
                      const float* state_in, float* state_out, void* stream) {
  long long hw = (long long)d.width * d.height;
  if (hw == 0 || d.frames == 0) return 0;
  // streaming bulk-copy kernel for u8 video (fc_f12.cu); -1 = not applicable
  const int rc = fc_gray_iir_stream(sg, si, video, in_type, out, d, n_warm, state_in,
                                    state_out, stream);
  if (rc != -1) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  float beta = 1.0f - si->alpha;
  int grid = int((hw + 127) / 128);
  if (in_type == FC_U8)
    k_gray_iir<uint8_t><<<grid, 128, 0, st>>>(static_cast<const uint8_t*>(video),
                                              out, *sg, si->alpha, beta, hw,
                                              d.frames, n_warm, state_in, state_out);
  else
    k_gray_iir<float><<<grid, 128, 0, st>>>(static_cast<const float*>(video), out,
                                            *sg, si->alpha, beta, hw, d.frames,
                                            n_warm, state_in, state_out);
  return status();
}

int fc_fused_gauss_grad_thr(const fc_stage* sg, const fc_stage* /*sgrad*/,
                            const fc_stage* sthr, const float* in, void* out,
                            int out_type, fc_dims d, void* stream) {
  if ((long long)d.width * d.height * d.frames == 0) return 0;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const long long hw = (long long)d.width * d.height;
  const size_t osz = out_type == FC_U8 ? 1 : 4;
  GaussW gw;
  for (int i = 0; i < (2 * sg->g_radius + 1) * (2 * sg->g_radius + 1); ++i)
    gw.w[i] = double(sg->g_w[i]);
  // one CTA per (tile, frame): at most 65535 frames per launch (grid z)
  for (int f0 = 0; f0 < d.frames; f0 += 65535) {
  const int nf = std::min(65535, d.frames - f0);
  dim3 grid((d.width + FW - 1) / FW, (d.height + FH - 1) / FH, nf);
  const float* fin = in + f0 * hw;
  void* fout = static_cast<char*>(out) + size_t(f0) * hw * osz;
#define FC_GGT(R, T)                                                              \
  k_gauss_grad_thr<R, T><<<grid, FT, 0, st>>>(fin, static_cast<T*>(fout), gw,    \
                                              sthr->th, sthr->white, sthr->black, \
                                              d.width, d.height)
#define FC_GGT_R(T)            \
  switch (sg->g_radius) {      \
    case 0: FC_GGT(0, T); break; \
    case 1: FC_GGT(1, T); break; \
    case 2: FC_GGT(2, T); break; \
    case 3: FC_GGT(3, T); break; \
    case 4: FC_GGT(4, T); break; \
    default: return -1;        \
  }
  if (out_type == FC_U8) {
    FC_GGT_R(uint8_t)
  } else {
    FC_GGT_R(float)
  }
#undef FC_GGT_R
#undef FC_GGT
  if (const int rc = status()) return rc;
  }
  return 0;
}

// Exact streaming chain; the certified frame pipeline (fc_pipe.cu) is
// dispatched ahead of it by fc_fused_chain (fc_dispatch.cu).
int fc_chain_exact(const fc_stage* sgray, const fc_stage* si, const fc_stage* sg,
                   const fc_stage* sthr, const void* video, int in_type,
                   int gray_in, void* out, int out_type, fc_dims d, int n_warm,
                   const float* state_in, float* state_out, void* stream) {
  if ((long long)d.width * d.height * d.frames == 0) return 0;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  dim3 grid((d.width + FW - 1) / FW, (d.height + FH - 1) / FH);
  float beta = 1.0f - si->alpha;
  fc_stage gdummy = {};
  const fc_stage& sgr = sgray ? *sgray : gdummy;
  GaussW gw;
  for (int i = 0; i < (2 * sg->g_radius + 1) * (2 * sg->g_radius + 1); ++i)
    gw.w[i] = double(sg->g_w[i]);
#define FC_CH(R, IT, OT, GI)                                                     \
  k_chain_exact<R, IT, OT, GI><<<grid, FT, 0, st>>>(                            \
      static_cast<const IT*>(video), static_cast<OT*>(out), sgr, si->alpha,     \
      beta, gw, sthr->th, sthr->white, sthr->black, d.width, d.height,          \
      d.frames, n_warm, state_in, state_out)
#define FC_CH_GI(R, IT, OT) \
  if (gray_in) FC_CH(R, IT, OT, true); else FC_CH(R, IT, OT, false);
#define FC_CH_OT(R, IT) \
  if (out_type == FC_U8) { FC_CH_GI(R, IT, uint8_t) } else { FC_CH_GI(R, IT, float) }
#define FC_CH_IT(R) \
  if (in_type == FC_U8) { FC_CH_OT(R, uint8_t) } else { FC_CH_OT(R, float) }
  switch (sg->g_radius) {
    case 1: FC_CH_IT(1) break;
    case 2: FC_CH_IT(2) break;
    case 3: FC_CH_IT(3) break;
    default: return -1;
  }
#undef FC_CH_IT
#undef FC_CH_OT
#undef FC_CH_GI
#undef FC_CH
  return status();
}

int fc_hash_video_u8(uint8_t* out, fc_dims d, int channels, int t0,
                     uint64_t seed, void* stream) {
  long long n = (long long)d.width * d.height * d.frames * channels;
  if (n == 0) return 0;
  unsigned long long seed_term = (unsigned long long)seed * 0x9E3779B97F4A7C15ull;
  k_hash_video<<<grid_for((n + 15) / 16, 256), 256, 0,
                 static_cast<cudaStream_t>(stream)>>>(out, n, channels, d.height,
                                                      d.width, t0, seed_term);
  return status();
}

}  // extern "C"
