// F12345 certified fast path, FRAME-PAIR PIPELINE (the headline kernel).
//
// Arithmetic contract: exact S1+S2 (gray products fl(w c) from one FMA on a
// byte->float magic number, the IIR update in the reference's roundings),
// certified packed-FP32 S3-S5 (centre-normalised separable gaussian, Sobel,
// m compared with M* inside a rigorous error band, fccommon::certify_band_scaled)
// and an exact FP64 recheck (simulator.cpp:63-89 order) of every value inside
// the band.  The mask is bit-identical to run_sequential's
// (/root/reference/proj/src/simulator.cpp:158-177).
//
// Work decomposition (B200: the FP32 pipe, not HBM, bounds this chain; see
// DESIGN.md section 4).  A CTA owns a window of 128 columns x R = OUT + 6
// rows (outputs: the central 120 columns x OUT rows) and marches all frames.
// Every stencil value is a float2 pairing two consecutive FRAMES (t, t+1) of
// the same pixel, so each window row is computed exactly once per frame (the
// row-pair layout of fc_pipe.cu paired rows p and p + OH and recomputed the 6
// rows both halves share).  Warp roles, one CTA per SM:
//
//   stencil warps 0..3  one per SM sub-partition; warp w takes frame pairs
//                       w, w + 4, ... from the IIR ring and marches the
//                       window's rows: horizontal 5-tap pass, vertical 5-tap
//                       pass and Sobel in registers (skewed software
//                       pipeline), certified threshold, mask words straight
//                       to HBM (frame t and t+1), exact rechecks after the
//                       march from the pair's exact IIR planes in the slot;
//   IIR warps 4..11     each lane owns 4 columns of fixed window rows and
//                       keeps their exact IIR state in registers for the
//                       whole video; per frame: gray (packed over column
//                       pairs) + IIR update (scalar, so the two frames of a
//                       pixel land in one register pair), one STS.128 per 2
//                       columns x 2 frames into the pair slot; lane 0 of the
//                       last IIR warp also issues the R, G, B TMA copies
//                       (one frame ahead; alpha never leaves HBM).
//
// Pair slot layout (1 KB per window row): 64 16-byte chunks, chunk k holds
// columns 2k and 2k+1 as {IIR_t, IIR_t+1} each; even chunks at 0..31, odd
// chunks rotated by 4 at 32..63 (conflict-light STS.128 / LDS.128).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>
#include <type_traits>
#include <utility>
#include <vector>

#include "fc_common.cuh"
#include "fc_sobel.cuh"

namespace fcpipe2 {

using namespace fccommon;

constexpr int LC = 4;       // columns per stencil lane
// stencil warps per frame pair of the certified kernel (two warps splitting
// the window rows, with setmaxnreg 160 / 96, measured 1.06-1.19 vs 0.80 ms:
// the IIR warps fall behind; removed)
constexpr int WPF = 1;
constexpr int NPF = 4;      // frame pairs in flight in the stencil
constexpr int NS = WPF * NPF;  // stencil warps
constexpr int NI = 8;       // IIR warps (two per SM sub-partition)
constexpr int NWARP = NS + NI;
constexpr int NTHR = NWARP * 32;
constexpr int K2 = NPF + 1; // pair slots: one per pair in flight + one being written
#ifndef FP2_MRSPLIT
#define FP2_MRSPLIT 0  // 1: IIR row counts per warp at compile time (two code variants:
                       // 0.86 vs 0.80 ms, the instruction cache)
#endif
#ifndef FP2_NSF
#define FP2_NSF 3
#endif
// TMA RGB frame slots (3: a ring, two frames of prefetch; 2: output frame A
// of a pair in slot 0, B in slot 1 -- compile-time LDS offsets but one frame
// of prefetch: 0.88 vs 0.80 ms)
constexpr int NSF = FP2_NSF;
#ifndef FP2_STENCIL_HI
#define FP2_STENCIL_HI 1  // stencil warps at the high warp ids: scheduler priority (+3.7 %)
#endif
// named barriers: 1 + slot = "slot empty", 1 + K2 + slot = "slot full"; the
// pair's stencil warp(s) and every IIR warp take part
constexpr unsigned NB_THREADS = (NI + WPF) * 32;
// The exact pipeline runs two stencil warps per pair, one per frame (frame
// A on warps 0-3, frame B on warps 4-7 of the stencil group: two stencil
// warps per SM sub-partition hide the DFMA chains' latency); 16 warps at
// <= 128 registers.
constexpr int NS_X = 2 * NPF;
constexpr int NTHR_X = (NI + NS_X) * 32;
constexpr unsigned NB_THREADS_X = (NI + 2) * 32;
constexpr int SW = 120;     // output columns per strip (window 128 = SW + 8)
constexpr int BWB = 144;    // TMA box row bytes: 128 + worst-case 16-B alignment slack
constexpr int PROW = 1024;  // bytes per window row of a pair slot
constexpr int QC = 64;      // recheck queue records per stencil warp
constexpr int BODY = 6;     // steps per rolled body of the stencil march

struct Args {
  uint8_t* out;
  int W, H, n_frames, n_warm;
  int strips;
  unsigned rgb_bytes, rgb_stride;  // TMA bytes per frame, RGB slot pitch
  unsigned off_iir, iir_stride;    // pair ring base, pair slot pitch
  unsigned off_bar, off_taps, off_queue;
  const float* state_in;
  float* state_out;
  // time segments (see fc_pipe.cu Args): CTA b works on window b % n_windows
  // and output frames [s L, (s+1) L) of segment s = b / n_windows
  int n_windows, n_segs, seg_len, seg_warm;
  float* seg_end;
  float* seg_warm_out;
  int* fix_k;
  int* seg_k;
  unsigned long long* prof;  // FUSEPLAN_PIPE_PROFILE: per-CTA {start, end} globaltimer (ns)
  const float* planes;       // SRC (F345): the f32 IIR planes [t][y][x] the group reads
  int skip;    // timing experiments only (FUSEPLAN_PIPE_SKIP): 1 IIR math, 2 stencil math,
               // 4 no TMA, 8 no gray (IIR warps only hand off slots)
  int opitch;  // output row pitch in bytes (>= W, a multiple of 4)
  FastParams p;
  double dtaps[25];  // the reference taps widened once
  double dtap6[6];   // EXACT: the six distinct taps of the symmetric 5x5 gaussian, by
                     // (min, max) of (|dy|, |dx|): 00 01 02 11 12 22
};

struct Range {
  int f0;       // first input frame (video index)
  int n;        // frames processed
  int n_warm;   // leading warm-up frames (IIR state only)
  int out0;     // first output frame index (relative to `out`)
  const float* st_in;
  float* st_out;
  float* st_warm;
};

__shared__ Range fp2_rg;
__device__ unsigned long long g_rechecks2;
extern __shared__ __align__(128) unsigned char fp2_smem[];

// mbarriers: rgb_full[NSF] (TMA completion); every other hand-off is a
// named barrier
__device__ __forceinline__ uint64_t* bar_rgb_full(const Args& a, int i) {
  return reinterpret_cast<uint64_t*>(fp2_smem + a.off_bar) + i;
}

template <bool EXACT = false>
__device__ __forceinline__ void nb_sync(int id) {
  constexpr unsigned n = EXACT ? NB_THREADS_X : NB_THREADS;
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
template <bool EXACT = false>
__device__ __forceinline__ void nb_arrive(int id) {
  constexpr unsigned n = EXACT ? NB_THREADS_X : NB_THREADS;
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void nb_sync_n(int id, unsigned n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void nb_arrive_n(int id, unsigned n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_lane0(uint64_t* bar, int lane) {
  asm volatile(
      "{\n.reg .pred q;\nsetp.eq.u32 q, %1, 0;\n@q mbarrier.arrive.shared::cta.b64 _, [%0];\n}\n" ::
          "r"(smem_u32(bar)),
      "r"(unsigned(lane))
      : "memory");
}
__device__ __forceinline__ void wait_phase(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase), "r"(1000000u)
      : "memory");
}

__device__ __forceinline__ void sts_pred_u32(uint32_t* p, uint32_t v, bool on) {
  asm volatile(
      "{\n.reg .pred q;\nsetp.ne.u32 q, %2, 0;\n@q st.shared.b32 [%0], %1;\n}\n" ::"r"(
          smem_u32(p)),
      "r"(v), "r"(unsigned(on))
      : "memory");
}
__device__ __forceinline__ void st_pred_u16(void* p, uint32_t v, bool on) {
  asm volatile(
      "{\n.reg .pred q;\nsetp.ne.u32 q, %2, 0;\n@q st.global.b16 [%0], %1;\n}\n" ::"l"(p),
      "h"(uint16_t(v)), "r"(unsigned(on))
      : "memory");
}
// 0xFF where nd < 0 for two values -> the low 16 bits (sign-replicate PRMT)
__device__ __forceinline__ uint32_t pack_neg2(float a, float b) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, 0x00FB;" : "=r"(r) : "r"(__float_as_uint(a)), "r"(__float_as_uint(b)));
  return r;
}
__device__ __forceinline__ void st_pred_u32(void* p, uint32_t v, bool on) {
  asm volatile(
      "{\n.reg .pred q;\nsetp.ne.u32 q, %2, 0;\n@q st.global.b32 [%0], %1;\n}\n" ::"l"(p),
      "r"(v), "r"(unsigned(on))
      : "memory");
}

// byte offset of chunk k (columns 2k, 2k+1) inside a slot row
__device__ __forceinline__ unsigned chunk_off(int k) {
  return unsigned((k & 1) ? 32 + (((k >> 1) + 4) & 31) : (k >> 1)) << 4;
}
__device__ __forceinline__ float4 lds128(unsigned addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts128f(unsigned addr, float a, float b, float c, float d) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b), "f"(c),
               "f"(d)
               : "memory");
}

__device__ __forceinline__ float2 shfl_up2(float2 v) {
  return make_float2(__shfl_up_sync(0xffffffffu, v.x, 1), __shfl_up_sync(0xffffffffu, v.y, 1));
}
__device__ __forceinline__ float2 shfl_down2(float2 v) {
  return make_float2(__shfl_down_sync(0xffffffffu, v.x, 1),
                     __shfl_down_sync(0xffffffffu, v.y, 1));
}

// |a|, |b| folded into a running minimum: one FMNMX3
__device__ __forceinline__ float min3abs(float m, float a, float b) {
  float r;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(m), "f"(fabsf(a)), "f"(fabsf(b)));
  return r;
}

// ------------------------------------------------------------------ IIR warps

template <int N>
using ic = std::integral_constant<int, N>;

// RGB slot pitch for a window of R rows (R, G, B planes of BWB-byte rows)
__host__ __device__ constexpr unsigned rgb_stride_of(int R) { return (unsigned(3 * R * BWB) + 127u) / 128u * 128u; }

// RGB slot release on named barriers (IDs after the pair-slot ones): every
// IIR warp but the producer's arrives after reading a frame, the producer
// warp syncs before it issues the TMA copy into that slot
constexpr int NB_RGB = 1 + 2 * K2;
constexpr unsigned NB_RGB_THREADS = NI * 32;
static_assert(NB_RGB + NSF <= 16, "named barrier ids");

// MR: rows of this warp, p = iw + NI r for r < MR (all inside the window)
template <int OUT, bool HALF, int MR, bool EXACT>
__device__ __forceinline__ void iir_rows(const Args& a, const Range& rg, int iw, int lane,
                                         int bx, int by, int xoff, const CUtensorMap* tmap,
                                         int tx0) {
  constexpr int R = OUT + 6;
  const int W = a.W, H = a.H, n = rg.n, n_warm = rg.n_warm;
  const int n_out = n - n_warm;
  const int cplane = R * BWB;
  const int xl = bx + 4 * lane;
  const uint32_t k4b = a.p.k4b;
  const float wr = a.p.wr, wg = a.p.wg, wb = a.p.wb;
  const float wrm = a.p.wrm, wgm = a.p.wgm, wbm = a.p.wbm;
  const float ia = a.p.ia, ib = a.p.ib;

  int coloff = xoff + 4 * lane;
  // magic-float PRMT selectors: byte j of the word, or (lanes left / right
  // of the video) the edge byte in every cell
  uint32_t msel[4] = {0x7440u, 0x7441u, 0x7442u, 0x7443u};
  if (xl < 0 || xl > W - 1) {
    const int edge = xl < 0 ? 0 : W - 1;
    coloff = (edge & ~3) - bx + xoff;
#pragma unroll
    for (int j = 0; j < 4; ++j) msel[j] = 0x7440u + unsigned(edge & 3);
  }
  // rows past the window (FP2_MRSPLIT 0: every warp runs the longest row count)
  auto row_ok = [&](int r) { return FP2_MRSPLIT || r < MR - 1 || iw + NI * r < R; };
  int rowo[MR];  // RGB slot byte offset of the lane's word in row p (clamped row)
#pragma unroll
  for (int r = 0; r < MR; ++r) {
    const int p = iw + NI * r;
    rowo[r] = (clampi(min(by + p, by + R - 1), 0, H - 1) - by) * BWB + coloff;
  }
  const unsigned so0 = chunk_off(2 * lane), so1 = chunk_off(2 * lane + 1);

  // q[r][j] = {IIR of frame A of the current pair, exact IIR state}: the state
  // lives in .y; a pair computes .x = IIR(A) from .y, then .y = IIR(B) from .x,
  // and stores {q(c0), q(c1)} as one 16-byte chunk (no register moves)
  float2 q[MR][4];
  const bool fresh = rg.st_in == nullptr;
#pragma unroll
  for (int r = 0; r < MR; ++r) {
    const int p = iw + NI * r;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      q[r][j].x = 0.0f;
      q[r][j].y = fresh ? 0.0f
                        : rg.st_in[(long long)clampi(by + p, 0, H - 1) * W +
                                   clampi(xl + j, 0, W - 1)];
    }
  }
  // the lane's output cells (window rows 3 .. OUT + 2) -> a state plane
  auto write_state = [&](float* dst) {
    if (!dst || lane < 1 || lane > 30 || xl >= W) return;
#pragma unroll
    for (int r = 0; r < MR; ++r) {
      const int p = iw + NI * r;
      if (p < 3 || p > OUT + 2 || by + p >= H) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) dst[(long long)(by + p) * W + xl + j] = q[r][j].y;
    }
  };
  auto to_state = [&]() {  // frame A becomes the state (warm-up, odd tail)
#pragma unroll
    for (int r = 0; r < MR; ++r)
#pragma unroll
      for (int j = 0; j < 4; ++j) q[r][j].y = q[r][j].x;
  };

  const unsigned smem0 = smem_u32(fp2_smem);
  int islot = 0;
  // RGB slot of frame t: (t - n_warm) & 1, so every output pair's A frame
  // sits in slot 0 and its B frame in slot 1 (compile-time LDS offsets)
  constexpr unsigned RGB_STRIDE = rgb_stride_of(R);
  unsigned rph = 0;  // mbarrier phase bit of each RGB slot (bit s)
  int rs = 0;        // NSF > 2: ring slot of the next frame (frame t in slot t % NSF)
  // the last IIR warp is the producer: its lane 0 copies frame t + 1 into
  // the slot of frame t - 1 when it starts frame t, once every IIR warp has
  // released that slot (named barrier)
  const bool pwarp = iw == NI - 1;
  const int f0 = rg.f0;
  auto issue = [&](int tp, int slot) {  // producer warp only
    if (tp >= NSF) nb_sync_n(NB_RGB + slot, NB_RGB_THREADS);
    if (lane == 0) {
      if (a.skip & 4) {
        mbar_arrive(bar_rgb_full(a, slot));
      } else {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(bar_rgb_full(a, slot), a.rgb_bytes);
        tma_load_3d(fp2_smem + slot * RGB_STRIDE, tmap, bar_rgb_full(a, slot), tx0, by,
                    4 * (f0 + tp));
      }
    }
  };
  if (pwarp) {
    if (lane == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
    if (NSF == 2) {
      if (n > 0) issue(0, n_warm & 1);
    } else {
      for (int tp = 0; tp < NSF - 1 && tp < n; ++tp) issue(tp, tp);
    }
  }
  const unsigned rgb0 = smem0;  // shared-space address of RGB slot 0
  int rowa[MR];                 // + the lane's word in row p
#pragma unroll
  for (int r = 0; r < MR; ++r) rowa[r] = int(rgb0) + rowo[r];

  // gray of frame t for every cell: g[r][h] = {gray(col 2h), gray(col 2h+1)}
  // (x 0.5 when HALF: alpha folded into the weights), consumed row by row.
  // SLOT: the frame's RGB slot, 0 / 1, or -1 (warm-up frames: (t - n_warm) & 1)
  auto gray = [&](int t, auto slot_t, auto&& row_fn) {
    constexpr int SLOT = NSF == 2 ? decltype(slot_t)::value : -1;
    const int slot = NSF != 2 ? rs : SLOT >= 0 ? SLOT : ((t - n_warm) & 1);
    if (pwarp && t + NSF - 1 < n)
      issue(t + NSF - 1, NSF == 2 ? (slot ^ 1) : (slot == 0 ? NSF - 1 : slot - 1));
    wait_phase(bar_rgb_full(a, slot), (rph >> slot) & 1u);
    rph ^= 1u << slot;
    const unsigned soff = SLOT >= 0 ? unsigned(SLOT) * RGB_STRIDE : unsigned(slot) * RGB_STRIDE;
#pragma unroll
    for (int r = 0; r < MR; ++r) {
      if (!row_ok(r) || (a.skip & 8)) continue;  // skip 8: no gray at all (timing only)
      uint32_t w[3];
      float2 g[2];
#pragma unroll
      for (int c = 0; c < 3; ++c)
        asm volatile("ld.shared.b32 %0, [%1];"
                     : "=r"(w[c])
                     : "r"(unsigned(rowa[r]) + soff + unsigned(c * cplane)));
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float2 pr = wprod(f2(magic_rs(w[0], k4b, msel[2 * h]),
                                   magic_rs(w[0], k4b, msel[2 * h + 1])), wr, wrm);
        const float2 pg = wprod(f2(magic_rs(w[1], k4b, msel[2 * h]),
                                   magic_rs(w[1], k4b, msel[2 * h + 1])), wg, wgm);
        const float2 pb = wprod(f2(magic_rs(w[2], k4b, msel[2 * h]),
                                   magic_rs(w[2], k4b, msel[2 * h + 1])), wb, wbm);
        g[h] = __fadd2_rn(__fadd2_rn(pr, pg), pb);  // (wr r + wg g) + wb b
      }
      row_fn(r, g);  // consume the row at once (few live registers)
    }
    // the warp's RGB reads are done (values in registers): release the slot
    // to the producer warp's copy of frame t + 2 into it
    if (!pwarp && t + NSF < n) nb_arrive_n(NB_RGB + slot, NB_RGB_THREADS);
    if (NSF != 2) rs = rs == NSF - 1 ? 0 : rs + 1;
  };
  // IIR update y' from y and the cell's gray value x (simulator.cpp:57-62):
  // HALF: fl(0.5 x + fl(0.5 y)) == FMA(0.5, y, 0.5 x) (x = gray > 0 dwarfs
  // any rounding of 0.5 y; x = 0 gives fl(0.5 y) either way); otherwise
  // fl(fl(a x) + fl(b y)) in scalar .rn ops.  First frame: y' = gray.
  auto upd = [&](float yo, float gj, auto first_t) -> float {
    constexpr bool FIRST = decltype(first_t)::value;
    if (HALF) return FIRST ? __fadd_rn(gj, gj) : __fmaf_rn(0.5f, yo, gj);
    return FIRST ? gj : __fadd_rn(__fmul_rn(ia, gj), __fmul_rn(ib, yo));
  };
  // frame t into component A (.x, from the state .y) or B (.y, from .x)
  auto frame = [&](int t, auto to_b_t, auto first_t, auto slot_t) {
    constexpr bool TO_B = decltype(to_b_t)::value;
    const bool skip = (a.skip & 1) != 0;
    gray(t, slot_t, [&](int r, const float2 (&g)[2]) {
      if (skip) return;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float gj = (j & 1) ? g[j >> 1].y : g[j >> 1].x;
        if (TO_B)
          q[r][j].y = upd(q[r][j].x, gj, first_t);  // B never starts a recurrence
        else
          q[r][j].x = upd(q[r][j].y, gj, first_t);
      }
    });
  };
  int n_stored = 0;
  auto store_pair = [&]() {
    if (n_stored >= K2) nb_sync<EXACT>(1 + islot);  // the stencil released pair n_stored - K2
    const unsigned base = smem0 + a.off_iir + islot * a.iir_stride;
#pragma unroll
    for (int r = 0; r < MR; ++r) {
      const int p = iw + NI * r;
      if (!row_ok(r)) continue;
      if constexpr (EXACT) {  // frame planes: row p = {A: 128 floats, B: 128 floats}
        sts128f(base + p * PROW + 16 * lane, q[r][0].x, q[r][1].x, q[r][2].x, q[r][3].x);
        sts128f(base + p * PROW + 512 + 16 * lane, q[r][0].y, q[r][1].y, q[r][2].y,
                q[r][3].y);
      } else {
        sts128f(base + p * PROW + so0, q[r][0].x, q[r][0].y, q[r][1].x, q[r][1].y);
        sts128f(base + p * PROW + so1, q[r][2].x, q[r][2].y, q[r][3].x, q[r][3].y);
      }
    }
    nb_arrive<EXACT>(1 + K2 + islot);
    ++n_stored;
    if (++islot == K2) islot = 0;
  };
  const auto A = std::false_type{};
  const auto B = std::true_type{};
  const auto FIRST = std::true_type{};
  const auto NEXT = std::false_type{};
  const auto S0 = ic<0>{};
  const auto S1 = ic<1>{};
  const auto SR = ic<-1>{};

  // frame 0 of a fresh run starts the recurrence (y = gray): peeled, so the
  // loops below carry no first-frame test
  int t = 0;
  if (fresh && n > 0) {
    frame(0, A, FIRST, SR);
    to_state();
    t = 1;
  }
  // warm-up frames: state only
  for (; t < n_warm; ++t) {
    frame(t, A, NEXT, SR);
    to_state();
  }
  if (n_warm > 0) write_state(rg.st_warm);
  // output frames in pairs (A = t in RGB slot 0, B = t + 1 in slot 1); an
  // odd tail is stored {A, A}
  int k = 0;
  if (t > n_warm) {  // the peeled frame 0 is the first pair's A
    if (n_out > 1)
      frame(1, B, NEXT, S1);
    else
      to_state();
    store_pair();
    k = 2;
  }
  for (; k + 1 < n_out; k += 2) {
    frame(n_warm + k, A, NEXT, S0);
    frame(n_warm + k + 1, B, NEXT, S1);
    store_pair();
  }
  if (k < n_out) {
    frame(n_warm + k, A, NEXT, S0);
    to_state();
    store_pair();
  }
  write_state(rg.st_out);
}

template <int OUT, bool HALF, bool EXACT>
__device__ __forceinline__ void iir_role(const Args& a, const Range& rg, int iw, int lane,
                                         int bx, int by, int xoff, const CUtensorMap* tmap,
                                         int tx0) {
  constexpr int R = OUT + 6;
  constexpr int NR = (R + NI - 1) / NI;  // rows of the first R % NI warps (all, if 0)
  if (!FP2_MRSPLIT || R % NI == 0 || iw < R % NI)
    iir_rows<OUT, HALF, NR, EXACT>(a, rg, iw, lane, bx, by, xoff, tmap, tx0);
  else
    iir_rows<OUT, HALF, NR - 1, EXACT>(a, rg, iw, lane, bx, by, xoff, tmap, tx0);
}

// ------------------------------------------------------------------ stencil warps

// Exact IIR value of window cell (row rho, col c) of frame `comp` of the pair
__device__ __forceinline__ float iir_at(const unsigned char* base, int rho, int c, int comp) {
  return *reinterpret_cast<const float*>(base + rho * PROW + chunk_off(c >> 1) + (c & 1) * 8 +
                                         comp * 4);
}

// Exact reference threshold decision at video (x, y), frame `comp` of the
// pair: FP64 gaussian in dy/dx order at the 3x3 clamped centres, Sobel in
// the reference's float order, IEEE sqrt (simulator.cpp:63-89).
__device__ __noinline__ bool exact_white(const Args& a, const unsigned char* base,
                                         const double* taps, int bx, int by, int x, int y,
                                         int comp) {
  float g[3][3];
  for (int j = 0; j < 3; ++j)
    for (int i = 0; i < 3; ++i) {
      const int cx = clampi(x + i - 1, 0, a.W - 1), cy = clampi(y + j - 1, 0, a.H - 1);
      double acc = 0.0;
      for (int dy = -2; dy <= 2; ++dy) {
        const int ry = clampi(cy + dy, 0, a.H - 1) - by;
        for (int dx = -2; dx <= 2; ++dx) {
          const int rx = clampi(cx + dx, 0, a.W - 1) - bx;
          acc = __fma_rn(taps[(dy + 2) * 5 + dx + 2], double(iir_at(base, ry, rx, comp)), acc);
        }
      }
      g[j][i] = __double2float_rn(acc);
    }
  auto s = [&](int dx, int dy) { return g[dy + 1][dx + 1]; };
  const float gx =
      __fsub_rn(__fadd_rn(__fadd_rn(s(1, -1), __fmul_rn(2.0f, s(1, 0))), s(1, 1)),
                __fadd_rn(__fadd_rn(s(-1, -1), __fmul_rn(2.0f, s(-1, 0))), s(-1, 1)));
  const float gy =
      __fsub_rn(__fadd_rn(__fadd_rn(s(-1, 1), __fmul_rn(2.0f, s(0, 1))), s(1, 1)),
                __fadd_rn(__fadd_rn(s(-1, -1), __fmul_rn(2.0f, s(0, -1))), s(1, -1)));
  return __fsqrt_rn(__fadd_rn(__fmul_rn(gx, gx), __fmul_rn(gy, gy))) >= a.p.th_val;
}

// Stencil warp sw: frame pairs sw, sw + NS, ... of the pair ring.  Lane L
// owns window columns 4L .. 4L+3 (outputs: lanes 1..30).  The march over the
// window rows p = 0 .. R + 1 is a loop of 6-step bodies (ring indices are
// compile-time constants):
//   step p: H row p (4 x 16-byte loads: chunks 2L-1 .. 2L+2);
//           G row p - 3 (from H rows p-5 .. p-1); Sobel + threshold at row p - 5.
// Uncertain values are queued in shared memory (record: first row, lane,
// rows) and recomputed exactly after the march.
template <int OUT>
__device__ __forceinline__ void stencil_role(const Args& a, const Range& rg, int sw, int lane,
                                             int bx, int by0) {
  constexpr int OT = OUT;  // output rows of this warp: the whole window
  constexpr int NP = OT + 6;
  constexpr int r0 = 0;  // first window row of the march
  const int by = by0;    // origin of the march
  const int W = a.W, H = a.H;
  const int n_out = rg.n - rg.n_warm;
  const int n_pairs = (n_out + 1) / 2;
  const float mlo = a.p.mlo_n, band = a.p.band_n;  // scaled domain (normalised taps)
  const float g0 = a.p.g0, g1 = a.p.g1;
  const double* taps = reinterpret_cast<const double*>(fp2_smem + a.off_taps);
  uint32_t* queue = reinterpret_cast<uint32_t*>(fp2_smem + a.off_queue) + sw * QC;
  // lane columns 4L .. 4L+3 (outputs: lanes 1..30)
  const int fp0 = sw % NPF;
  const int k = 2 * lane;  // the lane's first chunk
  const int xl = bx + 2 * k;    // video column of the lane's first cell
  const bool outl = lane >= 1 && lane <= 30 && xl < W;
  const bool xlo = xl == 0, xhi = xl + LC - 1 == W - 1;  // Sobel x clamps (video edges)
  unsigned cch[LC / 2 + 2];
#pragma unroll
  for (int i = 0; i < LC / 2 + 2; ++i) cch[i] = chunk_off((k - 1 + i + 64) & 63);
  const unsigned smem0 = smem_u32(fp2_smem);
  const unsigned lt_mask = (1u << lane) - 1u;
  const int OW = a.opitch;
  const long long fstride = (long long)OW * H;

  int slot = fp0 % K2;
  for (int u = fp0; u < n_pairs; u += NPF) {
    nb_sync(1 + K2 + slot);  // the IIR warps stored pair u
    const unsigned sbase = smem0 + a.off_iir + slot * a.iir_stride;  // slot row 0
    const unsigned base = sbase + r0 * PROW;                         // march row 0
    const bool has_b = 2 * u + 1 < n_out;
    unsigned char* o = a.out + (long long)(rg.out0 + 2 * u) * fstride;
    unsigned char* ox = o + (long long)(by + 3) * OW + xl;  // frame A, window row 3
    const bool oka = outl, okb = outl && has_b;
    int nq = 0;
    float amin = __int_as_float(0x7f800000);

    float2 hr[6][LC];  // H row r at ring index r % 6 ({frame A, frame B})
    float2 gr[6][LC];  // G row r at ring index r % 6

    auto step = [&](auto pm_t, auto h_t, auto v_t, auto s_t, auto yb_t, int p) {
      constexpr int PM = decltype(pm_t)::value;  // p % 6
      constexpr bool DO_H = decltype(h_t)::value, DO_V = decltype(v_t)::value;
      constexpr bool DO_S = decltype(s_t)::value;
      constexpr int YB = decltype(yb_t)::value;
      if constexpr (DO_H) {
        const unsigned rb = base + p * PROW;
        float2 v[LC + 4];  // columns c-2 .. c+LC+1
#pragma unroll
        for (int i = 0; i < LC / 2 + 2; ++i) {
          const float4 q4 = lds128(rb + cch[i]);
          v[2 * i] = lo2(q4);
          v[2 * i + 1] = hi2(q4);
        }
#pragma unroll
        for (int j = 0; j < LC; ++j)
          hr[PM][j] = tap4n(v[j], v[j + 1], v[j + 2], v[j + 3], v[j + 4], g0, g1);
      }
      if constexpr (DO_V) {
#pragma unroll
        for (int j = 0; j < LC; ++j)
          gr[(PM + 3) % 6][j] = tap4n(hr[(PM + 1) % 6][j], hr[(PM + 2) % 6][j],
                                      hr[(PM + 3) % 6][j], hr[(PM + 4) % 6][j],
                                      hr[(PM + 5) % 6][j], g0, g1);
      }
      if constexpr (DO_S) {
        constexpr int QM = (PM + 1) % 6;  // q % 6
        const int yq = by + p - 5;        // video row of the Sobel centre
        float2 s2[LC], d2[LC];
#pragma unroll
        for (int j = 0; j < LC; ++j) {
          float2 gm = gr[(QM + 5) % 6][j], gc = gr[QM][j], gp = gr[(QM + 1) % 6][j];
          if (YB == 1 && yq == 0) gm = gc;      // top video row (band 0, first Sobel step)
          if (YB == 2 && yq == H - 1) gp = gc;  // bottom video row (last band, last step)
          s2[j] = __fadd2_rn(__ffma2_rn(splat(2.0f), gc, gm), gp);
          d2[j] = __ffma2_rn(splat(-1.0f), gm, gp);
        }
        float2 sl = shfl_up2(s2[LC - 1]), dl = shfl_up2(d2[LC - 1]);
        float2 sr = shfl_down2(s2[0]), dr = shfl_down2(d2[0]);
        if (xlo) sl = s2[0], dl = d2[0];
        if (xhi) sr = s2[LC - 1], dr = d2[LC - 1];
        float2 S[LC + 2], D[LC + 2];
        S[0] = sl, D[0] = dl, S[LC + 1] = sr, D[LC + 1] = dr;
#pragma unroll
        for (int j = 0; j < LC; ++j) S[j + 1] = s2[j], D[j + 1] = d2[j];
        float2 dm[LC];
#pragma unroll
        for (int j = 0; j < LC; ++j) {
          const float2 gx = __ffma2_rn(splat(-1.0f), S[j], S[j + 2]);
          const float2 gy = __fadd2_rn(__ffma2_rn(splat(2.0f), D[j + 1], D[j]), D[j + 2]);
          // nd = mlo - gy^2 - gx^2 (< 0 <=> white)
          const float2 ngx = f2(-gx.x, -gx.y), ngy = f2(-gy.x, -gy.y);
          dm[j] = __ffma2_rn(ngx, gx, __ffma2_rn(ngy, gy, splat(mlo)));
        }
        st_pred_u32(ox, pack_neg(dm[0].x, dm[1].x, dm[2].x, dm[3].x), oka);
        st_pred_u32(ox + fstride, pack_neg(dm[0].y, dm[1].y, dm[2].y, dm[3].y), okb);
        ox += OW;
#pragma unroll
        for (int j = 0; j < LC; ++j) amin = min3abs(amin, dm[j].x, dm[j].y);
      }
    };
    auto flush = [&](int q0, int nstep) {
      const bool amb = outl && amin <= band;
      const unsigned ballot = __ballot_sync(0xffffffffu, amb);
      if (ballot) {
        const int i = nq + __popc(ballot & lt_mask);
        sts_pred_u32(queue + min(i, QC - 1),
                     (unsigned(q0) << 16) | (lane << 8) | unsigned(nstep), amb && i < QC);
        nq += __popc(ballot);
        amin = __int_as_float(0x7f800000);
      }
    };

    const auto F = std::false_type{};
    const auto T = std::true_type{};
    if (!(a.skip & 2)) {
      const auto Y0 = ic<0>{};
      step(ic<0>{}, T, F, F, Y0, 0);
      step(ic<1>{}, T, F, F, Y0, 1);
      step(ic<2>{}, T, F, F, Y0, 2);
      step(ic<3>{}, T, F, F, Y0, 3);
      step(ic<4>{}, T, F, F, Y0, 4);
      step(ic<5>{}, T, T, F, Y0, 5);
      step(ic<0>{}, T, T, F, Y0, 6);
      step(ic<1>{}, T, T, F, Y0, 7);
      step(ic<2>{}, T, T, T, ic<1>{}, 8);  // Sobel row 3: the video's top row in band 0
      flush(3, 1);
#pragma unroll 1
      for (int p = 9; p + 6 <= NP; p += 6) {
        step(ic<3>{}, T, T, T, Y0, p);
        step(ic<4>{}, T, T, T, Y0, p + 1);
        step(ic<5>{}, T, T, T, Y0, p + 2);
        step(ic<0>{}, T, T, T, Y0, p + 3);
        step(ic<1>{}, T, T, T, Y0, p + 4);
        step(ic<2>{}, T, T, T, Y0, p + 5);
        flush(p - 5, BODY);
      }
      constexpr int PT = 9 + 6 * ((NP - 9) / 6);
      if constexpr (NP - PT >= 1) step(ic<3>{}, T, T, T, Y0, PT);
      if constexpr (NP - PT >= 2) step(ic<4>{}, T, T, T, Y0, PT + 1);
      if constexpr (NP - PT >= 3) step(ic<5>{}, T, T, T, Y0, PT + 2);
      if constexpr (NP - PT >= 4) step(ic<0>{}, T, T, T, Y0, PT + 3);
      if constexpr (NP - PT >= 5) step(ic<1>{}, T, T, T, Y0, PT + 4);
      if constexpr (NP - PT >= 1) flush(PT - 5, NP - PT);
      step(ic<NP % 6>{}, F, T, T, Y0, NP);
      step(ic<(NP + 1) % 6>{}, F, F, T, ic<2>{}, NP + 1);  // bottom row of the last band
      flush(NP - 5, 2);

      // ---- exact recheck of the queued uncertain values (rare)
      if (nq > QC) {
        // queue overflow (adversarial input): the exact decision for every
        // output pixel of this warp's pair
        __syncwarp();
        const unsigned char* sb = fp2_smem + (sbase - smem0);
        if (outl)
          for (int q = 3; q <= OT + 2; ++q)
            for (int c = 0; c < (has_b ? 2 : 1); ++c) {
              const int yy = by + q;
              if (yy >= H) continue;
              for (int j = 0; j < LC; ++j)
                o[c * fstride + (long long)yy * OW + xl + j] =
                    exact_white(a, sb, taps, bx, by0, xl + j, yy, c) ? 0xFF : 0x00;
            }
        if (lane == 0) atomicAdd(&g_rechecks2, (unsigned long long)(30 * LC * 2 * OT));
        __syncwarp();
      } else if (nq) {
        __syncwarp();
        const unsigned char* sb = fp2_smem + (sbase - smem0);
        unsigned cnt = 0;
        constexpr int PER = 2 * LC * BODY;  // values per record: rows x 2 frames x LC cols
        const int items = nq * PER;
        for (int it = lane; it < items; it += 32) {
          const uint32_t rec = queue[it / PER];
          const int e = it % PER, st = e / (2 * LC), c = (e / LC) & 1, j = e % LC;
          const int q0 = int(rec >> 16), L = int((rec >> 8) & 31), nstep = int(rec & 0xFFu);
          if (st >= nstep || (c == 1 && !has_b)) continue;
          const int x = bx + 4 * L + j;
          const int yy = by + q0 + st;
          if (yy >= H) continue;
          const bool wv = exact_white(a, sb, taps, bx, by0, x, yy, c);
          o[c * fstride + (long long)yy * OW + x] = wv ? 0xFF : 0x00;
          ++cnt;
        }
        for (int k2 = 16; k2 > 0; k2 >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, k2);
        if (lane == 0) atomicAdd(&g_rechecks2, (unsigned long long)cnt);
        __syncwarp();
      }
    }
    if (u + K2 < n_pairs) nb_arrive(1 + slot);  // the IIR warps wait for it
    slot += NPF;
    if (slot >= K2) slot -= K2;
  }
}

// ------------------------------------------------------------------ plane warps (F345)

// The F345 group (gaussian + Sobel + threshold on the f32 planes of an
// earlier group, e.g. the reference planner's `1-2,3-5`) on the exact
// pipeline: the IIR role becomes a plane loader -- each lane owns 4 columns of
// fixed window rows, loads them for both frames of a pair (float4 where the 4
// columns lie inside the video, clamped scalars at its edges; the next pair
// is loaded while the current one is stored) and writes the pair slot's frame
// planes.  Stateless: no warm-up, time segments are independent.  (The
// certified F345 stays on the row-pair pipeline's TMA ring: with the FP32
// stencil this loader's one pair of lookahead is too little, DESIGN 4.4.)
template <int OUT>
__device__ __forceinline__ void plane_role(const Args& a, const Range& rg, int iw, int lane,
                                           int bx, int by) {
  constexpr int R = OUT + 6;
  constexpr int NR = (R + NI - 1) / NI;
  const int W = a.W, H = a.H;
  const int n_out = rg.n;
  const int n_pairs = (n_out + 1) / 2;
  const int xl = bx + 4 * lane;
  const bool vec = (W & 3) == 0 && xl >= 0 && xl + 3 <= W - 1 &&
                   (reinterpret_cast<uintptr_t>(a.planes) & 15) == 0;
  int cols[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) cols[j] = clampi(xl + j, 0, W - 1);
  long long rowoff[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r)
    rowoff[r] = (long long)clampi(by + min(iw + NI * r, R - 1), 0, H - 1) * W;
  const long long hw = (long long)W * H;
  const float* base = a.planes + (long long)rg.f0 * hw;
  const unsigned smem0 = smem_u32(fp2_smem);

  auto load = [&](int u, float4 (&dst)[NR][2]) {
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      if (iw + NI * r >= R) continue;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int fr = 2 * u + c < n_out ? 2 * u + c : 2 * u;  // odd tail: {A, A}
        const float* row = base + fr * hw + rowoff[r];
        if (vec)
          dst[r][c] = __ldg(reinterpret_cast<const float4*>(row + xl));
        else
          dst[r][c] = make_float4(__ldg(row + cols[0]), __ldg(row + cols[1]),
                                  __ldg(row + cols[2]), __ldg(row + cols[3]));
      }
    }
  };
  float4 cur[NR][2], nxt[NR][2];
  if (n_pairs > 0) load(0, cur);
  int islot = 0;
  for (int u = 0; u < n_pairs; ++u) {
    if (u + 1 < n_pairs) load(u + 1, nxt);
    if (u >= K2) nb_sync<true>(1 + islot);  // the stencil released pair u - K2
    const unsigned sb = smem0 + a.off_iir + islot * a.iir_stride;
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const int p = iw + NI * r;
      if (p >= R) continue;
      const float4 A = cur[r][0], B = cur[r][1];
      sts128f(sb + p * PROW + 16 * lane, A.x, A.y, A.z, A.w);  // frame planes
      sts128f(sb + p * PROW + 512 + 16 * lane, B.x, B.y, B.z, B.w);
    }
    nb_arrive<true>(1 + K2 + islot);
    if (++islot == K2) islot = 0;
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      cur[r][0] = nxt[r][0];
      cur[r][1] = nxt[r][1];
    }
  }
}

// ------------------------------------------------------------------ exact stencil warps

// Reference-exact stencil role (the EXACT pipeline, variant "exact"): for each
// frame of the pair a march over the window rows computing the FP64 gaussian
// in the reference's dy-outer / dx-inner order, rounding it to float, the
// Sobel magnitude^2 in the reference's float order and `m >= M*` (==
// sqrtf(m) >= th, M* the smallest such float), simulator.cpp:63-89.  No
// certification, no rechecks: every operation is the reference's.
//
// Each loaded window row p (converted to double once) feeds the five gaussian
// rows g = p - 2 .. p + 2 that read it, as their dy = p - g + 2 term: the
// 25-term chain of G row g advances one tap row per step in the reference's
// order, and a step carries 5 rows x 4 columns = 20 independent DFMA chains
// (a per-row 25-deep chain would leave the FP64 pipe latency-bound).  G row
// g completes at step g + 2; the Sobel of row q = p - 3 runs at step p.
// Lane L owns window columns 4L .. 4L+3 (outputs: lanes 1..30).
template <int OUT>
__device__ __forceinline__ void exact_stencil_role(const Args& a, const Range& rg, int sw,
                                                   int lane, int bx, int by) {
  constexpr int R = OUT + 6;
  static_assert(R >= 10, "window too short for the exact march");
  const int W = a.W, H = a.H;
  const int n_out = rg.n - rg.n_warm;
  const int n_pairs = (n_out + 1) / 2;
  const float mstar = a.p.mstar;
  const int k = 2 * lane;
  const int xl = bx + 2 * k;
  const bool outl = lane >= 1 && lane <= 30 && xl < W;
  const bool xlo = xl == 0, xhi = xl + LC - 1 == W - 1;
  const unsigned smem0 = smem_u32(fp2_smem);
  const int OW = a.opitch;
  const long long fstride = (long long)OW * H;

  const int fp0 = sw % NPF, c = sw / NPF;  // pair phase, frame of the pair (A / B)
  // the six distinct taps in registers (the symmetric gaussian; exact_params
  // checked the symmetry bit for bit)
  double t6[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) t6[i] = a.dtap6[i];
  auto tap = [&](int dy, int dx) -> double {  // compile-time dy, dx after unrolling
    const int p = dy < 2 ? 2 - dy : dy - 2, q = dx < 2 ? 2 - dx : dx - 2;
    const int lo = p < q ? p : q, hi = p < q ? q : p;
    return t6[lo == 0 ? hi : (lo == 1 ? 2 + hi : 5)];
  };
  const unsigned mcol = 16u * unsigned(lane);
  int slot = fp0 % K2;
  for (int u = fp0; u < n_pairs; u += NPF) {
    nb_sync<true>(1 + K2 + slot);  // the IIR warps stored pair u
    const unsigned base = smem0 + a.off_iir + slot * a.iir_stride;
    if (c == 0 || 2 * u + 1 < n_out) {
      unsigned char* ox =
          a.out + (long long)(rg.out0 + 2 * u + c) * fstride + (long long)(by + 3) * OW + xl;
      const unsigned cbase = base + 512 * c;  // frame c's plane of every slot row
      double acc[5][LC];    // gaussian row g at ring index g % 5
      float gq[5][LC + 2];  // G row g at ring index g % 5; cols 4L-1 .. 4L+4

      // step p (PM = p % 5): tap rows k in [KMIN, KMAX] of G rows p + 2 - k;
      // DONE: G row p - 2 completes (k = 4); SOB: Sobel of row p - 3
      // YC: the first / last Sobel step, where the video's top / bottom row may
      // clamp G in y (no other step can)
      auto step = [&](auto pm_t, auto kmin_t, auto kmax_t, auto done_t, auto sob_t, int p,
                      auto yc_t) {
        constexpr int PM = decltype(pm_t)::value;
        constexpr int KMIN = decltype(kmin_t)::value, KMAX = decltype(kmax_t)::value;
        constexpr bool DONE = decltype(done_t)::value, SOB = decltype(sob_t)::value;
        constexpr bool YC = decltype(yc_t)::value;
        double v[LC + 4];  // window row p, cols 4L-2 .. 4L+5 (frame c's plane)
        {
          const unsigned rb = cbase + p * PROW;
          // the lane's 4 columns from shared memory, the 2 + 2 halo columns
          // from the neighbouring lanes by shuffle (lane 0 / 31 wrap: their
          // outputs are not stored)
          const float4 qm = lds128(rb + mcol);
          float4 ql, qr;
          ql.z = __shfl_sync(0xffffffffu, qm.z, (lane + 31) & 31);
          ql.w = __shfl_sync(0xffffffffu, qm.w, (lane + 31) & 31);
          qr.x = __shfl_sync(0xffffffffu, qm.x, (lane + 1) & 31);
          qr.y = __shfl_sync(0xffffffffu, qm.y, (lane + 1) & 31);
          v[0] = double(ql.z);
          v[1] = double(ql.w);
          v[2] = double(qm.x);
          v[3] = double(qm.y);
          v[4] = double(qm.z);
          v[5] = double(qm.w);
          v[6] = double(qr.x);
          v[7] = double(qr.y);
        }
#pragma unroll
        for (int kk = KMIN; kk <= KMAX; ++kk) {
          constexpr int dummy = 0;
          (void)dummy;
          const int gi = (PM + 2 - kk + 5) % 5;  // compile-time after unrolling
#pragma unroll
          for (int j = 0; j < LC; ++j) {
            double t = kk == 0 ? 0.0 : acc[gi][j];
#pragma unroll
            for (int dx = 0; dx < 5; ++dx) t = __fma_rn(tap(kk, dx), v[j + dx], t);
            acc[gi][j] = t;
          }
        }
        if constexpr (DONE) {
          constexpr int GM = (PM + 3) % 5;  // (p - 2) % 5
          float gv[LC];
#pragma unroll
          for (int j = 0; j < LC; ++j) gv[j] = __double2float_rn(acc[GM][j]);
          float l = __shfl_up_sync(0xffffffffu, gv[LC - 1], 1);
          float r = __shfl_down_sync(0xffffffffu, gv[0], 1);
          if (xlo) l = gv[0];       // the Sobel reads G clamped to the video (x = -1 -> 0)
          if (xhi) r = gv[LC - 1];  // (x = W -> W - 1)
          gq[GM][0] = l;
#pragma unroll
          for (int j = 0; j < LC; ++j) gq[GM][j + 1] = gv[j];
          gq[GM][LC + 1] = r;
        }
        if constexpr (SOB) {
          constexpr int QM = (PM + 2) % 5;  // (p - 3) % 5
          const int yq = by + p - 3;        // video row of the Sobel centre
          const bool ytop = YC && yq == 0, ybot = YC && yq == H - 1;  // G clamped in y
          float rm[LC + 2], rc[LC + 2], rp[LC + 2];
#pragma unroll
          for (int i = 0; i < LC + 2; ++i) {
            rc[i] = gq[QM][i];
            rm[i] = ytop ? rc[i] : gq[(QM + 4) % 5][i];
            rp[i] = ybot ? rc[i] : gq[(QM + 1) % 5][i];
          }
          float m[LC];
          sobel_m4(rm, rc, rp, m);  // fc_sobel.cuh: packed, the reference's rounding
          uint32_t word = 0;
#pragma unroll
          for (int j = 0; j < LC; ++j) word |= (m[j] >= mstar ? 0xFFu : 0u) << (8 * j);
          st_pred_u32(ox, word, outl);
          ox += OW;
        }
      };
      const auto F = std::false_type{};
      const auto T = std::true_type{};
      // head: rows 0..5 start G rows 2 .. 7; G rows 2, 3 complete at steps 4, 5
      step(ic<0>{}, ic<0>{}, ic<0>{}, F, F, 0, F);
      step(ic<1>{}, ic<0>{}, ic<1>{}, F, F, 1, F);
      step(ic<2>{}, ic<0>{}, ic<2>{}, F, F, 2, F);
      step(ic<3>{}, ic<0>{}, ic<3>{}, F, F, 3, F);
      step(ic<4>{}, ic<0>{}, ic<4>{}, T, F, 4, F);
      step(ic<0>{}, ic<0>{}, ic<4>{}, T, F, 5, F);
      // step 6: the first Sobel (row 3: the video's top row in band 0); body
      // steps 7 .. R - 5 update all five rows; then the tail R - 4 .. R - 1
      // (no G rows past R - 3; the last Sobel may be the video's bottom row)
      static_assert(R - 4 > 6, "exact march layout");
      step(ic<1>{}, ic<0>{}, ic<4>{}, T, T, 6, T);
      constexpr int NB = R - 11;  // full steps from p = 7
#pragma unroll 1
      for (int p = 7; p + 5 <= 7 + NB; p += 5) {
        step(ic<2>{}, ic<0>{}, ic<4>{}, T, T, p, F);
        step(ic<3>{}, ic<0>{}, ic<4>{}, T, T, p + 1, F);
        step(ic<4>{}, ic<0>{}, ic<4>{}, T, T, p + 2, F);
        step(ic<0>{}, ic<0>{}, ic<4>{}, T, T, p + 3, F);
        step(ic<1>{}, ic<0>{}, ic<4>{}, T, T, p + 4, F);
      }
      constexpr int PR = 7 + 5 * (NB / 5);  // first remaining full step
      if constexpr (7 + NB - PR >= 1) step(ic<2>{}, ic<0>{}, ic<4>{}, T, T, PR, F);
      if constexpr (7 + NB - PR >= 2) step(ic<3>{}, ic<0>{}, ic<4>{}, T, T, PR + 1, F);
      if constexpr (7 + NB - PR >= 3) step(ic<4>{}, ic<0>{}, ic<4>{}, T, T, PR + 2, F);
      if constexpr (7 + NB - PR >= 4) step(ic<0>{}, ic<0>{}, ic<4>{}, T, T, PR + 3, F);
      step(ic<(R - 4) % 5>{}, ic<1>{}, ic<4>{}, T, T, R - 4, F);
      step(ic<(R - 3) % 5>{}, ic<2>{}, ic<4>{}, T, T, R - 3, F);
      step(ic<(R - 2) % 5>{}, ic<3>{}, ic<4>{}, T, T, R - 2, F);
      step(ic<(R - 1) % 5>{}, ic<4>{}, ic<4>{}, T, T, R - 1, T);
    }
    if (u + K2 < n_pairs) nb_arrive<true>(1 + slot);  // the IIR warps wait for it
    slot += NPF;
    if (slot >= K2) slot -= K2;
  }
}

// ------------------------------------------------------------------ kernel

template <int OUT, bool HALF, bool EXACT, bool SRC>
__global__ void __launch_bounds__(EXACT ? NTHR_X : NTHR, 1)
    k_chain_pair(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ Args a) {
  constexpr int R = OUT + 6;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int win = blockIdx.x % a.n_windows, seg = blockIdx.x / a.n_windows;
  const int strip = win % a.strips, band = win / a.strips;
  Range rg{0, a.n_frames, a.n_warm, 0, a.state_in, a.state_out, nullptr};
  {
    const long long hwl = (long long)a.W * a.H;
    const int n_out = a.n_frames - a.n_warm;
    if (a.fix_k) {  // fix-up: re-run every window from the first wrong segment
      const int k = *a.fix_k;
      if (k >= a.n_segs) return;
      rg.out0 = k * a.seg_len;
      rg.f0 = rg.out0;
      rg.n = n_out - rg.out0;
      rg.n_warm = 0;
      rg.st_in = a.seg_end + (long long)(k - 1) * hwl;
    } else if (a.n_segs > 1) {
      rg.out0 = seg * a.seg_len;
      const int e = min(rg.out0 + a.seg_len, n_out);
      rg.f0 = max(0, rg.out0 - a.seg_warm);
      rg.n_warm = rg.out0 - rg.f0;
      rg.n = e - rg.f0;
      rg.st_in = nullptr;
      rg.st_out = seg < a.n_segs - 1 ? (a.seg_end ? a.seg_end + (long long)seg * hwl : nullptr)
                                     : a.state_out;
      rg.st_warm = seg > 0 && a.seg_warm_out ? a.seg_warm_out + (long long)seg * hwl : nullptr;
    }
    if (rg.n <= 0 || rg.n_warm > rg.n) return;
    if (a.fix_k == nullptr && a.n_segs > 1 && blockIdx.x == 0 && tid == 0 && a.seg_k)
      *a.seg_k = a.n_segs;
  }
  // the last band ends exactly at row H - 1 (overlapping the band above it;
  // both write identical values): the Sobel y clamps sit at fixed steps
  const int bands = a.n_windows / a.strips;
  const int x0 = strip * SW, y0 = band == bands - 1 ? max(0, a.H - OUT) : band * OUT;
  const int bx = x0 - 4, by = y0 - 3;
  const int tx0 = bx >= 0 ? (bx & ~15) : -((-bx + 15) & ~15);
  double* taps = reinterpret_cast<double*>(fp2_smem + a.off_taps);
  if (tid == 0) {
    for (int i = 0; i < NSF; ++i) mbar_init(bar_rgb_full(a, i), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < 25) taps[tid] = double(a.p.taps[tid]);
  if (tid == 0) fp2_rg = rg;
  if (a.prof && tid == 0) a.prof[2 * blockIdx.x] = globaltimer();
  __syncthreads();  // the only CTA-wide barrier: roles run decoupled from here
  (void)R;
  const int sw = FP2_STENCIL_HI ? warp - NI : warp;  // stencil warp index (or < 0)
  if (sw >= 0 && sw < (EXACT ? NS_X : NS)) {
    if constexpr (EXACT)
      exact_stencil_role<OUT>(a, fp2_rg, sw, lane, bx, by);
    else
      stencil_role<OUT>(a, fp2_rg, sw, lane, bx, by);
  } else {
    if constexpr (SRC)
      plane_role<OUT>(a, fp2_rg, FP2_STENCIL_HI ? warp : warp - NS_X, lane, bx, by);
    else
      iir_role<OUT, HALF, EXACT>(a, fp2_rg, FP2_STENCIL_HI ? warp : warp - NS, lane, bx, by,
                                 bx - tx0, &tmap, tx0);
  }
  if (a.prof && lane == 0) atomicMax(&a.prof[2 * blockIdx.x + 1], globaltimer());
}

// ------------------------------------------------------------------ host

// tap (dy, dx) of the 5x5 grid holding distinct value i (see Args::dtap6)
inline int tap6_index(int i) {
  static const int idx[6] = {2 * 5 + 2, 2 * 5 + 1, 2 * 5 + 0, 1 * 5 + 1, 1 * 5 + 0, 0};
  return idx[i];
}

// the exact stencil role reads six distinct taps: the 5x5 grid must be the
// symmetric gaussian bit for bit
inline bool taps_symmetric(const float* w) {
  for (int dy = 0; dy < 5; ++dy)
    for (int dx = 0; dx < 5; ++dx) {
      const int p = dy < 2 ? 2 - dy : dy - 2, q = dx < 2 ? 2 - dx : dx - 2;
      const int lo = p < q ? p : q, hi = p < q ? q : p;
      const int i = lo == 0 ? hi : (lo == 1 ? 2 + hi : 5);
      if (w[dy * 5 + dx] != w[tap6_index(i)]) return false;
    }
  return true;
}

size_t layout(int out_rows, Args* a) {
  const int R = out_rows + 6;
  const size_t rgb = size_t(3) * R * BWB;
  const size_t rgb_stride = rgb_stride_of(R);
  size_t off = NSF * rgb_stride;
  const size_t off_iir = off;
  const size_t iir_stride = size_t(R) * PROW;
  off += K2 * iir_stride;
  const size_t off_bar = off;
  off += NSF * 8;
  const size_t off_taps = (off + 7) / 8 * 8;
  off = off_taps + 25 * 8;
  const size_t off_queue = off;
  off += size_t(NS) * QC * 4;
  if (a) {
    a->off_queue = unsigned(off_queue);
    a->rgb_bytes = unsigned(rgb);
    a->rgb_stride = unsigned(rgb_stride);
    a->off_iir = unsigned(off_iir);
    a->iir_stride = unsigned(iir_stride);
    a->off_bar = unsigned(off_bar);
    a->off_taps = unsigned(off_taps);
  }
  return off;
}

using KernelFn = void (*)(CUtensorMap, Args);

#define FP2_OUT_LIST(X) X(6) X(10) X(14) X(18) X(22) X(26) X(29)  // 30 rows exceed 227 KB

KernelFn kernel_for(int out_rows, bool half, bool exact, bool src = false) {
  switch (out_rows) {
#define FP2_CASE(N)                                                                        \
  case N:                                                                                  \
    if (src) return k_chain_pair<N, true, true, true>; /* exact F345 on f32 planes */      \
    return exact ? (half ? k_chain_pair<N, true, true, false> : k_chain_pair<N, false, true, false>) \
                 : (half ? k_chain_pair<N, true, false, false>                             \
                         : k_chain_pair<N, false, false, false>);
    FP2_OUT_LIST(FP2_CASE)
#undef FP2_CASE
  }
  return nullptr;
}

struct PairPlan {
  int W = -1, H = -1, dev = -1, frames = -1, force_out = 0, force_segs = 0;
  bool segs_ok = false;
  int out_rows = 0, strips = 0, bands = 0, n_segs = 1, seg_len = 0;
  size_t smem = 0;
};

constexpr int SEG_WARM = 48;  // IIR warm-up of a time segment (verified + fixed up)

// An SM's time ~ (CTAs it runs) x (window rows) x (frames of a CTA, warm-up
// frames at ~0.4 of a full frame).  Pick (OUT, segments) minimising the
// busiest SM's load; ties go to the taller window.
bool choose(int W, int H, int frames, bool segs_ok, int dev, int force, int force_segs,
            PairPlan* pp, bool stateless = false) {
  int sms = 0, optin = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const int strips = (W + SW - 1) / SW;
  double best = 1e300;
  const int outs[] = {
#define FP2_ITEM(N) N,
      FP2_OUT_LIST(FP2_ITEM)
#undef FP2_ITEM
  };
  const bool dbg = fc_get_knobs()->debug != 0;
  for (int o : outs) {
    if (force && o != force) continue;
    const size_t smem = layout(o, nullptr);
    if (smem > size_t(optin) || o > H) continue;  // the last band must fit the video
    cudaError_t e = cudaSuccess;
    for (int h = 0; h < 5 && e == cudaSuccess; ++h)
      e = cudaFuncSetAttribute(kernel_for(o, (h & 1) != 0, (h & 2) != 0, h == 4),
                               cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    int per_sm = 0;
    if (e == cudaSuccess)
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel_for(o, true, false), NTHR,
                                                        smem);
    if (dbg)
      std::fprintf(stderr, "fc_pipe2 choose: out=%d smem=%zu optin=%d err=%s per_sm=%d\n", o,
                   smem, optin, cudaGetErrorString(e), per_sm);
    if (e != cudaSuccess || per_sm < 1) {
      cudaGetLastError();
      continue;
    }
    const long long bands = (H + o - 1) / o;
    const long long windows = strips * bands;
    const int max_segs = segs_ok ? 16 : 1;
    for (int segs = 1; segs <= max_segs; ++segs) {
      if (force_segs && segs_ok && segs != force_segs) continue;
      const long long L = (frames + segs - 1) / segs;
      // segments that actually hold frames (16 asked of 161 frames: L = 11,
      // 15 segments); an empty trailing segment would march warm-up frames
      // past the end of its range
      const int nseg = L > 0 ? int((frames + L - 1) / L) : 1;
      if (!force_segs && !stateless && segs > 1 && L < 2 * SEG_WARM) break;
      if (segs > 1 && L < 2) break;
      const long long ctas = windows * nseg;
      const long long per_busiest = (ctas + sms - 1) / sms;
      const double cta_frames = double(L) + (segs > 1 && !stateless ? 0.4 * SEG_WARM : 0.0);
      const double cost = double(per_busiest) * (o + 6) * cta_frames * (1.0 - 1e-4 * o);
      if (cost < best) {
        best = cost;
        pp->out_rows = o;
        pp->strips = strips;
        pp->bands = int(bands);
        pp->smem = smem;
        pp->n_segs = nseg;
        pp->seg_len = int(L);
      }
    }
  }
  if (best >= 1e300 && force_segs)
    return choose(W, H, frames, segs_ok, dev, force, 0, pp, stateless);
  if (dbg && best < 1e300)
    std::fprintf(stderr, "fc_pipe2 choose: -> out=%d segs=%d seg_len=%d\n", pp->out_rows,
                 pp->n_segs, pp->seg_len);
  return best < 1e300;
}

__global__ void k_verify_segments(const float* __restrict__ warm, const float* __restrict__ end,
                                  long long hw, int n_segs, int* k) {
  const long long total = (long long)(n_segs - 1) * hw;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int s = int(i / hw) + 1;
    const long long px = i % hw;
    if (__float_as_uint(warm[s * hw + px]) != __float_as_uint(end[(s - 1) * hw + px]))
      atomicMin(k, s);
  }
}

struct SegScratch {
  float* buf = nullptr;
  size_t cap = 0;
  int* k = nullptr;
};

// per (device, stream): launches on one stream are ordered, so they may share
std::mutex& seg_mu() {
  static std::mutex mu;
  return mu;
}
std::map<std::pair<int, cudaStream_t>, SegScratch>& seg_all() {
  static std::map<std::pair<int, cudaStream_t>, SegScratch> all;
  return all;
}

SegScratch& seg_scratch(int dev, cudaStream_t st) {
  std::lock_guard<std::mutex> lock(seg_mu());
  return seg_all()[{dev, st}];
}

// frees a stream's scratch (a CUDA graph captured on it is gone; the caller
// synchronised the device)
void release_scratch(int dev, cudaStream_t st) {
  std::lock_guard<std::mutex> lock(seg_mu());
  auto it = seg_all().find({dev, st});
  if (it == seg_all().end()) return;
  if (it->second.buf) cudaFree(it->second.buf);
  if (it->second.k) cudaFree(it->second.k);
  seg_all().erase(it);
}

// src: `in` are f32 planes (the exact F345 group: stateless, no TMA, no seam check)
int launch(const FastParams& fp, const void* in, void* out, fc_dims d, int n_warm,
           const float* state_in, float* state_out, void* stream, int pitch, int opitch,
           bool exact, bool src = false) {
  if (d.frames == 0) return 0;
  int dev = 0;
  cudaGetDevice(&dev);
  const fc_knobs& kn = *fc_get_knobs();
  const bool segs_ok = state_in == nullptr && n_warm == 0;
  const int force_out = kn.pipe_out, force_segs = kn.pipe_segs;
  // plans per (device, shape, frames, segment eligibility, forcing knobs): a
  // host thread driving several devices or executors does not re-plan (and
  // re-set the kernels' shared-memory attributes) on every launch
  using Key = std::tuple<int, int, int, int, int, bool, int, int, bool>;
  static thread_local std::map<Key, PairPlan> plans;
  const Key key{dev, d.width, d.height, d.frames, n_warm, segs_ok, force_out, force_segs, src};
  auto it = plans.find(key);
  if (it == plans.end()) {
    PairPlan pp;
    if (!choose(d.width, d.height, d.frames - n_warm, segs_ok, dev, force_out, force_segs, &pp,
                src))
      return -1;
    if (plans.size() > 256) plans.clear();
    it = plans.emplace(key, pp).first;
  }
  const PairPlan& cache = it->second;
  Args a;
  std::memset(&a, 0, sizeof a);
  layout(cache.out_rows, &a);
  a.out = static_cast<uint8_t*>(out);
  a.opitch = opitch ? opitch : d.width;
  a.W = d.width;
  a.H = d.height;
  a.n_frames = d.frames;
  a.n_warm = n_warm;
  a.strips = cache.strips;
  a.n_windows = cache.strips * cache.bands;
  a.n_segs = cache.n_segs;
  a.seg_len = cache.seg_len;
  a.seg_warm = src ? 0 : (kn.pipe_seg_warm > 0 ? kn.pipe_seg_warm : SEG_WARM);
  a.planes = src ? static_cast<const float*>(in) : nullptr;
  const long long hwl = (long long)d.width * d.height;
  const bool verify = cache.n_segs > 1 && !src;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (verify) {
    SegScratch& sc = seg_scratch(dev, st);
    const size_t need = size_t(2 * cache.n_segs) * size_t(hwl);
    if (need > sc.cap) {
      if (sc.buf) cudaFree(sc.buf);
      sc.buf = nullptr;
      sc.cap = 0;
      if (cudaMalloc(&sc.buf, need * sizeof(float)) != cudaSuccess) return int(cudaGetLastError());
      sc.cap = need;
    }
    if (!sc.k && cudaMalloc(&sc.k, sizeof(int)) != cudaSuccess) return int(cudaGetLastError());
    a.seg_end = sc.buf;
    a.seg_warm_out = sc.buf + size_t(cache.n_segs) * size_t(hwl);
    a.seg_k = sc.k;
  }
  a.state_in = state_in;
  a.state_out = state_out;
  a.p = fp;
  for (int i = 0; i < 25; ++i) a.dtaps[i] = double(fp.taps[i]);
  for (int i = 0; i < 6; ++i) a.dtap6[i] = double(fp.taps[tap6_index(i)]);
  a.skip = kn.pipe_skip;
  if (kn.band_scale > 0.0f) a.p.band_n *= kn.band_scale;  // tests / diagnostics only
  CUtensorMap map;
  std::memset(&map, 0, sizeof map);  // src: the plane warps load with LDG, no TMA
  if (!src && !rgb_tensor_map(&map, in, d, BWB, cache.out_rows + 6, pitch ? pitch : d.width))
    return -1;
  const int grid = cache.strips * cache.bands * cache.n_segs;
  KernelFn fn = kernel_for(cache.out_rows, fp.alpha_half != 0, exact, src);
  const int nthr = exact ? NTHR_X : NTHR;
  if (kn.profile) {
    cudaMalloc(&a.prof, sizeof(unsigned long long) * 2 * grid);
    cudaMemsetAsync(a.prof, 0, sizeof(unsigned long long) * 2 * grid, st);
  }
  fn<<<grid, nthr, cache.smem, st>>>(map, a);
  int rc = int(cudaGetLastError());
  if (kn.profile && a.prof) {  // per-CTA spans (diagnostics)
    std::vector<unsigned long long> h(size_t(2) * grid);
    cudaStreamSynchronize(st);
    cudaMemcpy(h.data(), a.prof, h.size() * sizeof(h[0]), cudaMemcpyDeviceToHost);
    cudaFree(a.prof);
    a.prof = nullptr;
    unsigned long long t0 = ~0ull, t1 = 0;
    double sum = 0, mx = 0, mn = 1e30;
    for (int b = 0; b < grid; ++b) {
      t0 = std::min(t0, h[2 * b]);
      t1 = std::max(t1, h[2 * b + 1]);
      const double span = double(h[2 * b + 1] - h[2 * b]) / 1e3;
      sum += span;
      mx = std::max(mx, span);
      mn = std::min(mn, span);
    }
    std::fprintf(stderr, "fc_pipe2 out=%d segs=%d grid=%d exact=%d: kernel span %.1f us, CTA span "
                 "avg %.1f min %.1f max %.1f us\n", cache.out_rows, cache.n_segs, grid, int(exact),
                 double(t1 - t0) / 1e3, sum / grid, mn, mx);
    if (kn.profile == 2)
      for (int b = 0; b < grid; ++b)
        std::fprintf(stderr, "  cta %4d win(%d,%d) start %+.2f us span %.1f us\n", b,
                     (b % a.n_windows) % cache.strips, (b % a.n_windows) / cache.strips,
                     double(h[2 * b] - t0) / 1e3, double(h[2 * b + 1] - h[2 * b]) / 1e3);
  }
  if (rc == 0 && verify) {
    k_verify_segments<<<296, 256, 0, st>>>(a.seg_warm_out, a.seg_end, hwl, cache.n_segs,
                                           a.seg_k);
    Args f = a;
    f.fix_k = a.seg_k;
    f.seg_k = nullptr;
    fn<<<cache.strips * cache.bands, nthr, cache.smem, st>>>(map, f);
    rc = int(cudaGetLastError());
  }
  return rc;
}

// Host entry of both pipelines (certified / exact).
int entry(const fc_stage* sgray, const fc_stage* si, const fc_stage* sg, const fc_stage* sthr,
          const void* video, int in_type, int gray_in, void* out, int out_type, fc_dims d,
          int n_warm, const float* state_in, float* state_out, int pitch, int opitch,
          void* stream, bool exact) {
  FastParams fp;
  if (pitch == 0) pitch = d.width;
  if (opitch == 0) opitch = d.width;
  if (opitch < d.width || opitch % 4 != 0 || reinterpret_cast<uintptr_t>(out) % 4 != 0)
    return -1;
  if (d.height < 6) return -1;
  const bool ok = exact ? exact_params(sgray, si, sg, sthr, video, in_type, gray_in, out_type, d,
                                       pitch, &fp)
                        : fast_params(sgray, si, sg, sthr, video, in_type, gray_in, out_type, d,
                                      pitch, &fp);
  if (!ok || (exact && !taps_symmetric(fp.taps))) return -1;
  return launch(fp, video, out, d, n_warm, state_in, state_out, stream, pitch, opitch, exact);
}

}  // namespace fcpipe2

// Same contract as fc_chain_pipe (fc_pipe.cu): -1 when the chain or the
// layout is outside the certified path.
extern "C" int fc_chain_pipe2(const fc_stage* sgray, const fc_stage* si, const fc_stage* sg,
                              const fc_stage* sthr, const void* video, int in_type, int gray_in,
                              void* out, int out_type, fc_dims d, int n_warm,
                              const float* state_in, float* state_out, int pitch, int opitch,
                              void* stream) {
  return fcpipe2::entry(sgray, si, sg, sthr, video, in_type, gray_in, out, out_type, d, n_warm,
                        state_in, state_out, pitch, opitch, stream, false);
}

// The exact frame-pair pipeline (FP64 gaussian in the reference's order, no
// certification): -1 when the chain or the layout is outside it.
extern "C" int fc_chain_pipe2_exact(const fc_stage* sgray, const fc_stage* si,
                                    const fc_stage* sg, const fc_stage* sthr, const void* video,
                                    int in_type, int gray_in, void* out, int out_type, fc_dims d,
                                    int n_warm, const float* state_in, float* state_out,
                                    int pitch, int opitch, void* stream) {
  return fcpipe2::entry(sgray, si, sg, sthr, video, in_type, gray_in, out, out_type, d, n_warm,
                        state_in, state_out, pitch, opitch, stream, true);
}

// The exact F345 group (FP64 gaussian in the reference's order, float Sobel,
// m >= M*) on f32 planes: the exact frame-pair pipeline with the plane
// loader role.  -1 when outside it (the caller runs the FP64 tiles).
extern "C" int fc_f345_pair_exact(const fc_stage* sg, const fc_stage* sthr, const float* in,
                                  void* out, int out_type, fc_dims d, void* stream) {
  using namespace fcpipe2;
  FastParams fp;
  std::memset(&fp, 0, sizeof fp);
  if (d.width % 4 != 0 || d.height < 6 || reinterpret_cast<uintptr_t>(out) % 4 != 0) return -1;
  if (out_type != FC_U8 || sg->g_radius != 2 || !(sthr->th > 0.0f)) return -1;
  if (sthr->white != 255.0f || sthr->black != 0.0f) return -1;
  std::memcpy(fp.taps, sg->g_w, sizeof fp.taps);
  if (!taps_symmetric(fp.taps)) return -1;
  fp.th_val = sthr->th;
  fp.mstar = threshold_mstar(sthr->th);
  fp.mlo = std::nextafter(fp.mstar, 0.0f);
  return launch(fp, in, out, d, 0, nullptr, nullptr, stream, 0, 0, true, true);
}

extern "C" int fc_chain_pipe2_exact_applies(const fc_stage* sgray, const fc_stage* si,
                                            const fc_stage* sg, const fc_stage* sthr,
                                            int in_type, int gray_in, int out_type, fc_dims d,
                                            int pitch) {
  using namespace fcpipe2;
  FastParams fp;
  alignas(16) static const unsigned char probe[16] = {};
  return d.height >= 6 &&
         exact_params(sgray, si, sg, sthr, probe, in_type, gray_in, out_type, d, pitch, &fp) &&
         taps_symmetric(fp.taps);
}

extern "C" void fc_pipe2_release_scratch(int device, void* stream) {
  fcpipe2::release_scratch(device, static_cast<cudaStream_t>(stream));
}

extern "C" long long fc_pipe2_recheck_count(void) {
  unsigned long long v = 0;
  if (cudaMemcpyFromSymbol(&v, fcpipe2::g_rechecks2, sizeof v) != cudaSuccess) return -1;
  return (long long)v;
}
