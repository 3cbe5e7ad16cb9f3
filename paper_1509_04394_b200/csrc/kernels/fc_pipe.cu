// F12345 certified fast path, ROW-PAIR PIPELINE (the round-1 headline kernel,
// superseded by the frame-pair pipeline fc_pipe2.cu; this
// one still runs the certified F345 group of two-fusion plans and, with
// FUSEPLAN_PIPE_IMPL=1, the whole chain).
//
// Arithmetic contract: exact S1+S2, certified packed-FP32 S3-S5, exact FP64
// recheck inside the error band (fc_common.cuh certify_band /
// certify_band_scaled; tests/test_certified_band.py).  What changes is the work
// decomposition, built around the one serial dependency of the chain: only
// the IIR (S2) carries state across frames; S3-S5 of different frames are
// independent once the frame's IIR plane exists.  A CTA owns a spatial window
// and runs three warp roles connected by mbarrier rings in shared memory:
//
//   producer warp   one lane streams the window's R, G, B planes of every
//                   frame into an NSF-slot TMA ring (alpha never leaves HBM);
//   IIR warps (NI)  each lane owns fixed cells of the window and keeps their
//                   exact IIR state in registers for the whole march: gray +
//                   IIR (exact) per frame, the IIR plane written into a
//                   K-slot ring of IIR frames;
//   stencil warps   warps 2f, 2f+1 take frames f, f+NF, ... from the IIR ring
//   (2 NF)          (one 64-column half of the window each) and march the
//                   frame's window rows top to bottom:
//                   horizontal 5-tap pass, vertical 5-tap pass and Sobel all
//                   in registers (sliding row windows), certified threshold,
//                   mask bytes straight to HBM, exact rechecks read the
//                   frame's exact IIR plane still held in the ring.
//
// Geometry.  Window = 128 columns (lane L owns columns 4L..4L+3) x R = 2 OH + 6
// rows; outputs = the central 120 columns x 2 OH rows (halo: 3 rows and 4
// columns each side for gaussian r=2 + Sobel r=1).  Every value is a float2
// pairing window rows (p, p + OH): the top and bottom halves of the window run
// in lock-step, so every stencil op and the IIR update is one FFMA2 / FADD2 /
// FMUL2.  Pair-row p (0 <= p < OH + 6) of an IIR slot holds, for all 128
// columns, the float2 {IIR(row p), IIR(row p + OH)}; a pair-row is 1 KB laid
// out as 64 16-byte chunks (two columns each), even chunks first, odd chunks
// second, so every warp-wide 16-byte access below touches 512 contiguous
// bytes (conflict-free).
//
// Video borders (BORDER instantiation): window rows / 4-column groups outside
// the video read the clamped RGB row / replicate the edge byte, so the IIR and
// H values hold clamp-to-edge values (simulator.cpp:202-210); Sobel clamps its
// G rows / columns at the first and last video row / column.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <type_traits>
#include <utility>
#include <vector>

#include "fc_common.cuh"

// Warp-role counts (compile-time; a tuning build may predefine them together
// with FP_NAMESPACE / FP_ENTRY to compile a second layout alongside).
// The shipped layout: one stencil warp per frame (4-column lanes, 168
// registers), 6 frames in flight, 5 IIR warps + the producer warp (12 warps),
// 3 TMA slots, 8 IIR slots (measured 940 k vs 904 k frames/s for two 2-column
// warps per frame, 5 frames, 16 warps at 128 registers).  Each count can be
// overridden with -D for A/B builds (build.py FUSEPLAN_NVCC_EXTRA).
#ifndef FP_LC
#define FP_LC 4
#endif
#ifndef FP_NF
#define FP_NF 6
#endif
#ifndef FP_NI
#define FP_NI 5
#endif
#ifndef FP_KSLACK
#define FP_KSLACK 2
#endif
#ifndef FP_NSF
#define FP_NSF 3
#endif
#ifndef FP_SPECIALISE
#define FP_SPECIALISE 0  // one code path: 978 k vs 950 k (per-CTA variants slow
                         // the SMs around them -- instruction caches)
#endif
#ifndef FP_NAMESPACE
#define FP_NAMESPACE fcpipe
#define FP_ENTRY fc_chain_pipe
#define FP_F345_ENTRY fc_f345_pipe
#define FP_RECHECKS fc_pipe_recheck_count
#endif
#ifndef FP_WAIT_HINT
#define FP_WAIT_HINT ", %2"  // suspend-time hint operand of try_wait ("" = none)
#endif
#ifndef FP_WAIT_SLEEP
#define FP_WAIT_SLEEP 0  // > 0: poll with plain try_wait + __nanosleep(ns) back-off
#endif
// FP_SPECIALISE 1: interior / border variants of every role per CTA; 0: the
// general (border) variant everywhere; 2: IIR / plane roles specialised, one
// stencil path (measured: 0 is fastest in the 12-warp layout).
#ifndef FP_IIR_TMA
#define FP_IIR_TMA 1  // all-fused mode: the TMA producer warp is also an IIR warp
#endif

namespace FP_NAMESPACE {

using namespace fccommon;

constexpr int LC = FP_LC;   // columns per stencil lane: 2 (two warps per frame) or 4 (one)
constexpr int WPF = 4 / LC; // stencil warps per frame
constexpr int NF = FP_NF;   // frames in flight in the stencil
constexpr int NS = WPF * NF;  // stencil warps
constexpr int NI = FP_NI;   // IIR warps
// warps sharing the IIR rows in the all-fused mode: with FP_IIR_TMA the
// producer warp takes rows too (lane 0 still issues the TMA copies), so the
// slowest IIR warp has ceil(NP / (NI + 1)) pair-rows instead of ceil(NP / NI)
constexpr int NIE = NI + (FP_IIR_TMA ? 1 : 0);
constexpr int NWARP = NS + NI + 1;
constexpr int NTHR = NWARP * 32;
constexpr int K = NF + FP_KSLACK;  // IIR frame slots (slack: frames the IIR may run ahead)
constexpr int NSF = FP_NSF; // TMA RGB frame slots
constexpr int SW = 120;     // output columns per strip (window 128 = SW + 8)
constexpr int BWB = 144;    // TMA box row bytes: 128 + worst-case 16-B alignment slack
constexpr int PROW = 1024;  // bytes per IIR pair-row
constexpr int QC = 64;      // recheck queue records per stencil warp
constexpr int BODY = 6;     // steps per rolled body of the stencil march (= max rows per record)

struct Args {
  uint8_t* out;
  int W, H, n_frames, n_warm;
  int strips;
  unsigned rgb_bytes, rgb_stride;  // TMA bytes per frame, RGB slot pitch
  unsigned off_iir, iir_stride;    // IIR ring base, IIR slot pitch
  unsigned off_bar, off_taps, off_queue;
  const float* state_in;
  float* state_out;
  // Time segments (small frames): CTA b works on window b % n_windows and
  // segment b / n_windows of seg_len output frames; chain segments s > 0
  // restart the IIR seg_warm frames early, publish their warm state to
  // seg_warm_out[s] and their end state to seg_end[s] for verification; a
  // fix-up launch (fix_k != null) re-runs every window from segment *fix_k.
  int n_windows, n_segs, seg_len, seg_warm;
  float* seg_end;
  float* seg_warm_out;
  int* fix_k;
  int* seg_k;  // main segmented launch: reset to n_segs by CTA 0 (read by verify / fix-up)
  long long* dbg;  // optional per-CTA timing (FUSEPLAN_PIPE_PROFILE), 8 slots per CTA
  int skip;        // timing experiments only (FUSEPLAN_PIPE_SKIP): 1 IIR math, 2 stencil math
  int opitch;      // output row pitch in bytes (>= W, a multiple of 4)
  int dbg_x, dbg_y, dbg_t;  // diagnostics (FUSEPLAN_PIPE_DEBUG_PX=x,y,t): dump the
  float* dbg_px;            // recheck's 7x7 IIR neighbourhood + decision
  FastParams p;
};

// The frames one CTA processes (see Args: time segments / fix-up)
struct Range {
  int f0;       // first input frame (video / plane index)
  int n;        // frames processed
  int n_warm;   // leading warm-up frames (IIR state only)
  int out0;     // first output frame index (relative to `out`)
  const float* st_in;
  float* st_out;
  float* st_warm;  // state after the warm-up frames (segments s > 0)
};

// The CTA's Range lives in shared memory: the roles read each field where
// they use it, so the segment bookkeeping costs no registers in the marches.
__shared__ Range fp_rg;

__device__ unsigned long long g_rechecks;
extern __shared__ __align__(128) unsigned char fp_smem[];

// mbarrier layout: rgb_full[NSF], rgb_empty[NSF], iir_full[K], iir_empty[K]
__device__ __forceinline__ uint64_t* bar_rgb_full(const Args& a, int i) {
  return reinterpret_cast<uint64_t*>(fp_smem + a.off_bar) + i;
}
__device__ __forceinline__ uint64_t* bar_rgb_empty(const Args& a, int i) {
  return reinterpret_cast<uint64_t*>(fp_smem + a.off_bar) + NSF + i;
}
__device__ __forceinline__ uint64_t* bar_iir_full(const Args& a, int i) {
  return reinterpret_cast<uint64_t*>(fp_smem + a.off_bar) + 2 * NSF + i;
}
__device__ __forceinline__ uint64_t* bar_iir_empty(const Args& a, int i) {
  return reinterpret_cast<uint64_t*>(fp_smem + a.off_bar) + 2 * NSF + K + i;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// one arrive per warp (lane 0) without a divergent branch
__device__ __forceinline__ void mbar_arrive_lane0(uint64_t* bar, int lane) {
  asm volatile(
      "{\n.reg .pred q;\nsetp.eq.u32 q, %1, 0;\n@q mbarrier.arrive.shared::cta.b64 _, [%0];\n}\n" ::
          "r"(smem_u32(bar)),
      "r"(unsigned(lane))
      : "memory");
}

// Blocking wait: the suspend-time hint parks the warp in the barrier unit
// instead of spinning through issue slots the working warps need.
__device__ __forceinline__ void wait_phase(uint64_t* bar, unsigned phase) {
#if FP_WAIT_SLEEP
  // variant: plain try_wait, then a software back-off between polls
  for (;;) {
    unsigned ok;
    asm volatile(
        "{\n.reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    if (ok) return;
    __nanosleep(FP_WAIT_SLEEP);
  }
#endif
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1" FP_WAIT_HINT ";\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase), "r"(1000000u)
      : "memory");
}

__device__ __forceinline__ long long clk() { return clock64(); }

__device__ __forceinline__ void sts_pred_u32(uint32_t* p, uint32_t v, bool on) {
  asm volatile(
      "{\n.reg .pred q;\nsetp.ne.u32 q, %2, 0;\n@q st.shared.b32 [%0], %1;\n}\n" ::"r"(
          smem_u32(p)),
      "r"(v), "r"(unsigned(on))
      : "memory");
}

__device__ __forceinline__ void st_pred_u32(void* p, uint32_t v, bool on) {
  asm volatile(
      "{\n.reg .pred q;\nsetp.ne.u32 q, %2, 0;\n@q st.global.b32 [%0], %1;\n}\n" ::"l"(p),
      "r"(v), "r"(unsigned(on))
      : "memory");
}

// Byte offset of chunk k (columns 2k, 2k+1; 16 bytes) inside a pair-row:
// even chunks at positions 0..31, odd chunks at 32 + ((k >> 1) + 4) % 32.
// IIR lanes store chunks 2L and 2L+1 (each store: 32 consecutive positions);
// stencil lanes load chunks b + L (8 lanes per wavefront: 4 even + 4 odd
// chunks, the rotation by 4 puts the two groups on disjoint banks).
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
__device__ __forceinline__ void sts128(unsigned addr, float2 a, float2 b) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a.x), "f"(a.y),
               "f"(b.x), "f"(b.y)
               : "memory");
}

// 0xFF where nd < 0 for two values -> the low 16 bits (sign-replicate PRMT)
__device__ __forceinline__ uint32_t pack_neg2(float a, float b) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, 0x00FB;" : "=r"(r) : "r"(__float_as_uint(a)), "r"(__float_as_uint(b)));
  return r;
}

__device__ __forceinline__ float2 shfl_up2(float2 v) {
  return make_float2(__shfl_up_sync(0xffffffffu, v.x, 1), __shfl_up_sync(0xffffffffu, v.y, 1));
}
__device__ __forceinline__ float2 shfl_down2(float2 v) {
  return make_float2(__shfl_down_sync(0xffffffffu, v.x, 1),
                     __shfl_down_sync(0xffffffffu, v.y, 1));
}

// ------------------------------------------------------------------ IIR warps

template <int OH, bool BX, bool BY, bool HALF>
__device__ __forceinline__ void iir_role(const Args& a, const Range& rg, int iw, int lane,
                                         int bx, int by, int xoff, const CUtensorMap* tmap,
                                         int tx0) {
  constexpr int NP = OH + 6;               // pair-rows
  constexpr int NR = (NP + NIE - 1) / NIE; // pair-rows of this warp: p = iw + NIE r
  constexpr int R = 2 * OH + 6;
  const int W = a.W, H = a.H, n = rg.n, n_warm = rg.n_warm;
  const int cplane = R * BWB;
  const int xl = bx + 4 * lane;
  const uint32_t k4b = a.p.k4b;
  const float wr = a.p.wr, wg = a.p.wg, wb = a.p.wb;
  const float wrm = a.p.wrm, wgm = a.p.wgm, wbm = a.p.wbm;
  const float ia = a.p.ia, ib = a.p.ib;

  int rowx[NR], rowy[NR];  // RGB slot byte offsets of the two window rows
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const int p = iw + NIE * r;
    const int rx = p, ry = p + OH;
    rowx[r] = (BY ? clampi(by + rx, 0, H - 1) - by : rx) * BWB;
    rowy[r] = (BY ? clampi(by + ry, 0, H - 1) - by : ry) * BWB;
  }
  int coloff = xoff + 4 * lane;
  // magic-float PRMT selectors of the lane's 4 cells: byte j of the word, or
  // (lanes left / right of the video) the edge byte in every cell -- a
  // register selector, so the x clamp costs no instruction per frame
  uint32_t msel[4] = {0x7440u, 0x7441u, 0x7442u, 0x7443u};
  if (BX && (xl < 0 || xl > W - 1)) {
    const int edge = xl < 0 ? 0 : W - 1;
    coloff = (edge & ~3) - bx + xoff;
#pragma unroll
    for (int j = 0; j < 4; ++j) msel[j] = 0x7440u + unsigned(edge & 3);
  }
  const unsigned so0 = chunk_off(2 * lane), so1 = chunk_off(2 * lane + 1);

  // exact IIR state of the lane's cells: v[r][j] = {row p, row p + OH}, col 4L + j
  float2 v[NR][4];
  const bool fresh = rg.st_in == nullptr;
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const int p = iw + NIE * r;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (fresh || p >= NP) {
        v[r][j] = make_float2(0.0f, 0.0f);
      } else {
        const int cx = clampi(xl + j, 0, W - 1);
        v[r][j].x = rg.st_in[(long long)clampi(by + p, 0, H - 1) * W + cx];
        v[r][j].y = rg.st_in[(long long)clampi(by + p + OH, 0, H - 1) * W + cx];
      }
    }
  }

  // the lane's output cells (rows 3 .. OH+2 of both halves) -> a state plane
  auto write_state = [&](float* dst) {
    if (!dst || lane < 1 || lane > 30 || xl >= W) return;
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const int p = iw + NIE * r;
      if (p < 3 || p > OH + 2) continue;  // output rows of both halves
      const int yx = by + p, yy = by + p + OH;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (yx < H) dst[(long long)yx * W + xl + j] = v[r][j].x;
        if (yy < H) dst[(long long)yy * W + xl + j] = v[r][j].y;
      }
    }
  };
  const unsigned smem0 = smem_u32(fp_smem);
  int rslot = 0, islot = 0;
  unsigned rpar = 0, ipar = 0;
  long long w_rgb = 0, w_slot = 0;
  const long long t_begin = clk();
  // FP_IIR_TMA: lane 0 of warp NI keeps NSF - 1 frames of RGB in flight; the
  // slot of frame t + NSF - 1 is that of frame t - 1, which every IIR warp
  // (this one included) has released before this warp starts frame t
  const bool prod = FP_IIR_TMA && iw == NI && lane == 0;
  int pslot = 0;
  unsigned ppar = 0;
  const int f0 = rg.f0;
  auto issue = [&](int tp) {
    wait_phase(bar_rgb_empty(a, pslot), ppar ^ 1u);
    if (a.skip & 4) {  // timing experiment: no RGB transfer (stale slot contents)
      mbar_arrive(bar_rgb_full(a, pslot));
    } else {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(bar_rgb_full(a, pslot), a.rgb_bytes);
      tma_load_3d(fp_smem + pslot * a.rgb_stride, tmap, bar_rgb_full(a, pslot), tx0, by,
                  4 * (f0 + tp));
    }
    if (++pslot == NSF) {
      pslot = 0;
      ppar ^= 1u;
    }
  };
  if (prod) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
    for (int tp = 0; tp < NSF - 1 && tp < n; ++tp) issue(tp);
  }
  for (int t = 0; t < n; ++t) {
    if (prod && t + NSF - 1 < n) issue(t + NSF - 1);
    if (a.dbg) {
      const long long c0 = clk();
      wait_phase(bar_rgb_full(a, rslot), rpar);
      w_rgb += clk() - c0;
    } else {
      wait_phase(bar_rgb_full(a, rslot), rpar);
    }
    const unsigned char* f = fp_smem + rslot * a.rgb_stride;
    auto body = [&](auto first_tag) {
      constexpr bool FIRST = decltype(first_tag)::value;
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        if (iw + NIE * r >= NP) continue;
        uint32_t wx[3], wy[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          wx[c] = *reinterpret_cast<const uint32_t*>(f + c * cplane + rowx[r] + coloff);
          wy[c] = *reinterpret_cast<const uint32_t*>(f + c * cplane + rowy[r] + coloff);
        }
#define FP_MG(W_, J) (BX ? magic_rs(W_, k4b, msel[J]) : magic_r<J>(W_, k4b))
#define FP_CELL(J)                                                                          \
  {                                                                                         \
    const float2 g = __fadd2_rn(                                                            \
        __fadd2_rn(wprod(f2(FP_MG(wx[0], J), FP_MG(wy[0], J)), wr, wrm),                    \
                   wprod(f2(FP_MG(wx[1], J), FP_MG(wy[1], J)), wg, wgm)),                   \
        wprod(f2(FP_MG(wx[2], J), FP_MG(wy[2], J)), wb, wbm));                              \
    /* HALF: g = 0.5 gray exactly; IIR y = fl(0.5 x + fl(0.5 y)) == FMA(0.5, y, g); */     \
    /* else g = gray and y = fl(fl(a x) + fl(b y)) (simulator.cpp:57-62) in scalar */      \
    /* ops: ptxas contracts mul.rn.f32x2 followed by add.rn.f32x2 into FFMA2 despite */       \
    /* the .rn (measured), which would drop a rounding; scalar .rn ops are kept */            \
    if (HALF)                                                                               \
      v[r][J] = FIRST ? __fadd2_rn(g, g) : __ffma2_rn(splat(0.5f), v[r][J], g);             \
    else                                                                                    \
      v[r][J] = FIRST ? g                                                                   \
                      : f2(__fadd_rn(__fmul_rn(ia, g.x), __fmul_rn(ib, v[r][J].x)),         \
                           __fadd_rn(__fmul_rn(ia, g.y), __fmul_rn(ib, v[r][J].y)));        \
  }
        FP_CELL(0) FP_CELL(1) FP_CELL(2) FP_CELL(3)
#undef FP_CELL
#undef FP_MG
      }
    };
    if (a.skip & 1) {
    } else if (t == 0 && fresh)
      body(std::true_type{});
    else
      body(std::false_type{});
    __syncwarp();  // the warp's RGB reads are done (values in registers)
    mbar_arrive_lane0(bar_rgb_empty(a, rslot), lane);
    if (++rslot == NSF) {
      rslot = 0;
      rpar ^= 1u;
    }
    if (t < n_warm) {  // warm-up frame: state only
      if (t == n_warm - 1) write_state(rg.st_warm);
      continue;
    }
    if (a.dbg) {
      const long long c0 = clk();
      wait_phase(bar_iir_empty(a, islot), ipar ^ 1u);
      w_slot += clk() - c0;
    } else {
      wait_phase(bar_iir_empty(a, islot), ipar ^ 1u);
    }
    const unsigned base = smem0 + a.off_iir + islot * a.iir_stride;
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const int p = iw + NIE * r;
      if (p >= NP) continue;
      sts128(base + p * PROW + so0, v[r][0], v[r][1]);
      sts128(base + p * PROW + so1, v[r][2], v[r][3]);
    }
    __syncwarp();  // the warp's IIR stores precede the release arrive
    mbar_arrive_lane0(bar_iir_full(a, islot), lane);
    if (++islot == K) {
      islot = 0;
      ipar ^= 1u;
    }
  }

  if (a.dbg && lane == 0) {
    long long* d = a.dbg + 8 * blockIdx.x;
    atomicAdd(reinterpret_cast<unsigned long long*>(d + 3), (unsigned long long)w_rgb);
    atomicAdd(reinterpret_cast<unsigned long long*>(d + 4), (unsigned long long)w_slot);
    atomicAdd(reinterpret_cast<unsigned long long*>(d + 6), (unsigned long long)(clk() - t_begin));
  }
  write_state(rg.st_out);
}

// F345 mode: the "IIR" warps load the frame's f32 input plane window (TMA
// slot, row-major, 512 B per row) and repack it into the pair-row layout; no
// state.  Window cells outside the video take the clamped row / edge column.
template <int OH, bool BX, bool BY>
__device__ __forceinline__ void plane_role(const Args& a, const Range& rg, int iw, int lane,
                                           int bx, int by) {
  constexpr int NP = OH + 6;
  constexpr int NR = (NP + NI - 1) / NI;
  const int W = a.W, H = a.H, n = rg.n;
  const int xl = bx + 4 * lane;
  int colb = 16 * lane, comp = -1;  // byte offset of the lane's 4 floats in a slot row
  if (BX && (xl < 0 || xl > W - 1)) {
    const int edge = xl < 0 ? 0 : W - 1;
    colb = ((edge & ~3) - bx) * 4;
    comp = edge & 3;  // replicate this component
  }
  const unsigned so0 = chunk_off(2 * lane), so1 = chunk_off(2 * lane + 1);
  const unsigned smem0 = smem_u32(fp_smem);
  int rslot = 0, islot = 0;
  unsigned rpar = 0, ipar = 0;
  for (int t = 0; t < n; ++t) {
    wait_phase(bar_rgb_full(a, rslot), rpar);
    const unsigned char* f = fp_smem + rslot * a.rgb_stride;
    float2 v[NR][4];
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const int p = iw + NI * r;
      if (p >= NP) continue;
      const int rx = BY ? clampi(by + p, 0, H - 1) - by : p;
      const int ry = BY ? clampi(by + p + OH, 0, H - 1) - by : p + OH;
      float4 qx = *reinterpret_cast<const float4*>(f + rx * 512 + colb);
      float4 qy = *reinterpret_cast<const float4*>(f + ry * 512 + colb);
      if (BX && comp >= 0) {
        const float ex = comp == 0 ? qx.x : comp == 1 ? qx.y : comp == 2 ? qx.z : qx.w;
        const float ey = comp == 0 ? qy.x : comp == 1 ? qy.y : comp == 2 ? qy.z : qy.w;
        qx = make_float4(ex, ex, ex, ex);
        qy = make_float4(ey, ey, ey, ey);
      }
      v[r][0] = f2(qx.x, qy.x);
      v[r][1] = f2(qx.y, qy.y);
      v[r][2] = f2(qx.z, qy.z);
      v[r][3] = f2(qx.w, qy.w);
    }
    __syncwarp();
    mbar_arrive_lane0(bar_rgb_empty(a, rslot), lane);
    if (++rslot == NSF) {
      rslot = 0;
      rpar ^= 1u;
    }
    wait_phase(bar_iir_empty(a, islot), ipar ^ 1u);
    const unsigned base = smem0 + a.off_iir + islot * a.iir_stride;
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const int p = iw + NI * r;
      if (p >= NP) continue;
      sts128(base + p * PROW + so0, v[r][0], v[r][1]);
      sts128(base + p * PROW + so1, v[r][2], v[r][3]);
    }
    __syncwarp();
    mbar_arrive_lane0(bar_iir_full(a, islot), lane);
    if (++islot == K) {
      islot = 0;
      ipar ^= 1u;
    }
  }
}

// ------------------------------------------------------------------ stencil warps

// Exact IIR value of window cell (window row rho, col c) in the slot at `base`.
template <int OH>
__device__ __forceinline__ float iir_at(const unsigned char* base, int rho, int c, int half) {
  const int p = rho - half * OH;
  return *reinterpret_cast<const float*>(base + p * PROW + chunk_off(c >> 1) + (c & 1) * 8 +
                                         half * 4);
}

// Exact reference threshold decision at video (x, y) whose window row lies in
// half `half` (rows p + half OH): FP64 gaussian in dy/dx order at the 3x3
// clamped centres, Sobel in the reference's float order, IEEE sqrt
// (simulator.cpp:63-89).
template <int OH>
__device__ __noinline__ bool exact_white(const Args& a, const unsigned char* base,
                                         const double* taps, int bx, int by, int x, int y,
                                         int half) {
  float g[3][3];
  for (int j = 0; j < 3; ++j)
    for (int i = 0; i < 3; ++i) {
      const int cx = clampi(x + i - 1, 0, a.W - 1), cy = clampi(y + j - 1, 0, a.H - 1);
      double acc = 0.0;
      for (int dy = -2; dy <= 2; ++dy) {
        const int ry = clampi(cy + dy, 0, a.H - 1) - by;
        for (int dx = -2; dx <= 2; ++dx) {
          const int rx = clampi(cx + dx, 0, a.W - 1) - bx;
          acc = __fma_rn(taps[(dy + 2) * 5 + dx + 2], double(iir_at<OH>(base, ry, rx, half)),
                         acc);
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

template <int N>
using ic = std::integral_constant<int, N>;

// Stencil warps 2f + side: frames f, f + NF, ... of the IIR ring, side 0 the
// window columns 2..65 (outputs 4..63), side 1 columns 62..125 (outputs
// 64..123); lane L owns the column pair c = 2k, 2k + 1 with k = 1 + 30 side + L.
// The march over the frame's pair-rows p = 0 .. OH + 5 is a loop of 5-step
// bodies (the H and G row rings have period 5, so every ring index is a
// compile-time constant and the code stays small for the instruction cache):
//   step p: H row p (3 x 16-byte loads: chunks k-1, k, k+1);
//           G row p - 2 (p >= 4); Sobel + threshold at pair-row p - 3 (p >= 6).
// Uncertain values are queued in shared memory (record: pair-row, lane,
// 4 value bits) and recomputed exactly after the march.
template <int OH, bool BORDER>
__device__ __forceinline__ void stencil_role(const Args& a, const Range& rg, int sw, int lane,
                                             int bx, int by) {
  constexpr int NP = OH + 6;
  const int W = a.W, H = a.H;
  const int n_out = rg.n - rg.n_warm;
  const long long hw = (long long)W * H;
  const float mlo = a.p.mlo_n, band = a.p.band_n;  // scaled domain (normalised taps)
  const float g0 = a.p.g0, g1 = a.p.g1;
  const double* taps = reinterpret_cast<const double*>(fp_smem + a.off_taps);
  uint32_t* queue = reinterpret_cast<uint32_t*>(fp_smem + a.off_queue) + sw * QC;
  // LC = 2: warps 2f, 2f+1 share frame f (64-column halves, lane chunk
  // k = 1 + 30 side + L); LC = 4: warp f alone, lane columns 4L .. 4L+3
  const int f0 = sw / WPF, side = sw % WPF;
  const int k = LC == 2 ? 1 + 30 * side + lane : 2 * lane;  // the lane's first chunk
  const int xl = bx + 2 * k;           // video column of the lane's first cell
  const bool outl = lane >= 1 && lane <= 30 && xl < W;
  // loaded chunks: k-1 .. k + LC/2 (the edge lanes of LC = 4 wrap around the
  // row; those values only feed non-output columns)
  unsigned cch[LC / 2 + 2];
#pragma unroll
  for (int i = 0; i < LC / 2 + 2; ++i) cch[i] = chunk_off((k - 1 + i + 64) & 63);
  const unsigned smem0 = smem_u32(fp_smem);
  const unsigned lt_mask = (1u << lane) - 1u;

  int slot = f0 % K;
  unsigned par = (f0 / K) & 1u;
  long long w_full = 0;
  const long long t_begin = clk();
  for (int u = f0; u < n_out; u += NF) {
    if (a.dbg) {
      const long long c0 = clk();
      wait_phase(bar_iir_full(a, slot), par);
      w_full += clk() - c0;
    } else {
      wait_phase(bar_iir_full(a, slot), par);
    }
    const unsigned base = smem0 + a.off_iir + slot * a.iir_stride;
    const int OW = a.opitch;  // output rows: opitch bytes apart, frames opitch * H
    unsigned char* o = a.out + (long long)(rg.out0 + u) * OW * H;
    unsigned char* ox = o + (long long)(by + 3) * OW + xl;  // pair-row 3, top half
    unsigned char* oy = ox + (long long)OH * OW;              // bottom half
    int nq = 0;                                              // queued records
    float amin = __int_as_float(0x7f800000);                 // running min |nd|

    float2 hr[6][LC];  // H row r at ring index r % 6
    float2 gr[6][LC];  // G row r at ring index r % 6

    // Step p of the skewed march: H row p, G row p - 3 (from H rows p-5..p-1)
    // and Sobel at pair-row p - 5 (G rows p-6..p-4) are mutually
    // independent, so the scheduler overlaps the loads and the three
    // dependency chains of a step.
    // YB: the video's top row (1: window row 3 of band 0, the first Sobel
    // step) or bottom row (2: the last band ends at row H - 1, so it is the
    // bottom half of the last Sobel step) may be in this step's Sobel rows;
    // every other step needs no y clamp
    auto step = [&](auto pm_t, auto h_t, auto v_t, auto s_t, auto yb_t, int p) {
      constexpr int PM = decltype(pm_t)::value;  // p % 6
      constexpr bool DO_H = decltype(h_t)::value, DO_V = decltype(v_t)::value;
      constexpr bool DO_S = decltype(s_t)::value;
      constexpr int YB = decltype(yb_t)::value;
      // ---- horizontal pass of pair-row p
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
      // ---- vertical pass: G row p - 3
      if constexpr (DO_V) {
#pragma unroll
        for (int j = 0; j < LC; ++j)
          gr[(PM + 3) % 6][j] = tap4n(hr[(PM + 1) % 6][j], hr[(PM + 2) % 6][j],
                                      hr[(PM + 3) % 6][j], hr[(PM + 4) % 6][j],
                                      hr[(PM + 5) % 6][j], g0, g1);
      }
      // ---- Sobel + certified threshold at pair-row q = p - 5 (G rows q-1..q+1)
      if constexpr (DO_S) {
        constexpr int QM = (PM + 1) % 6;  // q % 6
        const int q = p - 5;
        const int yx = by + q, yy = by + q + OH;  // video rows of the two halves
        float2 s2[LC], d2[LC];
#pragma unroll
        for (int j = 0; j < LC; ++j) {
          float2 gm = gr[(QM + 5) % 6][j], gc = gr[QM][j], gp = gr[(QM + 1) % 6][j];
          if (YB == 1 && yx == 0) gm.x = gc.x;      // predicated selects: the step
          if (YB == 2 && yy == H - 1) gp.y = gc.y;  // stays one basic block
          s2[j] = __fadd2_rn(__ffma2_rn(splat(2.0f), gc, gm), gp);
          d2[j] = __ffma2_rn(splat(-1.0f), gm, gp);
        }
        float2 sl = shfl_up2(s2[LC - 1]), dl = shfl_up2(d2[LC - 1]);
        float2 sr = shfl_down2(s2[0]), dr = shfl_down2(d2[0]);
        if (BORDER) {
          if (xl == 0) sl = s2[0], dl = d2[0];
          if (xl + LC - 1 == W - 1) sr = s2[LC - 1], dr = d2[LC - 1];
        }
        float2 S[LC + 2], D[LC + 2];
        S[0] = sl, D[0] = dl, S[LC + 1] = sr, D[LC + 1] = dr;
#pragma unroll
        for (int j = 0; j < LC; ++j) S[j + 1] = s2[j], D[j + 1] = d2[j];
        float2 dm[LC];
#pragma unroll
        for (int j = 0; j < LC; ++j) {
          const float2 gx = __ffma2_rn(splat(-1.0f), S[j], S[j + 2]);
          const float2 gy = __fadd2_rn(__ffma2_rn(splat(2.0f), D[j + 1], D[j]), D[j + 2]);
          // nd = mlo - gy^2 - gx^2 (< 0 <=> white); certify_band's 2u (M* + m) term
          const float2 ngx = f2(-gx.x, -gx.y), ngy = f2(-gy.x, -gy.y);
          dm[j] = __ffma2_rn(ngx, gx, __ffma2_rn(ngy, gy, splat(mlo)));
        }
        // rows are inside the video: the last band is aligned to end at H - 1
        const bool okx = outl, oky = outl;
        if constexpr (LC == 2) {
          if (okx) *reinterpret_cast<uint16_t*>(ox) = uint16_t(pack_neg2(dm[0].x, dm[1].x));
          if (oky) *reinterpret_cast<uint16_t*>(oy) = uint16_t(pack_neg2(dm[0].y, dm[1].y));
        } else {
          // predicated stores (no branch: the next step's shuffles then need
          // no reconvergence / divergence checks)
          st_pred_u32(ox, pack_neg(dm[0].x, dm[1].x, dm[2].x, dm[3].x), okx);
          st_pred_u32(oy, pack_neg(dm[0].y, dm[1].y, dm[2].y, dm[3].y), oky);
        }
        ox += OW;  // running row pointers
        oy += OW;
        // running min of |nd| over the lane's output values (branch-free;
        // checked once per 6-step body; values of rows below the video only
        // cause a harmless extra recheck)
#pragma unroll
        for (int j = 0; j < LC; ++j) amin = fminf(amin, fminf(fabsf(dm[j].x), fabsf(dm[j].y)));
      }
    };
    // After a body of steps whose Sobel rows are q0 .. q0 + nstep - 1: lanes
    // whose running min fell inside the band queue those rows for the exact
    // recheck (all four values of each row; rare)
    auto flush = [&](int q0, int nstep) {
      const bool amb = outl && amin <= band;
      const unsigned ballot = __ballot_sync(0xffffffffu, amb);
      if (ballot) {
        const int i = nq + __popc(ballot & lt_mask);
        sts_pred_u32(queue + min(i, QC - 1),
                     (unsigned(q0) << 16) | (lane << 8) | unsigned(nstep), amb && i < QC);
        nq += __popc(ballot);  // nq > QC: overflow, handled after the march
        amin = __int_as_float(0x7f800000);
      }
    };

    const auto F = std::false_type{};
    const auto T = std::true_type{};
    if (!(a.skip & 2)) {
    // Steps p = 0 .. NP + 1: H while p < NP, V for 5 <= p <= NP, Sobel for
    // 8 <= p <= NP + 1.  Prologue p < 8, a rolled loop of 6-step bodies,
    // then a compile-time tail.
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
    for (int p = 9; p + 6 <= NP; p += 6) {  // p % 6 == 3 at the top
      step(ic<3>{}, T, T, T, Y0, p);
      step(ic<4>{}, T, T, T, Y0, p + 1);
      step(ic<5>{}, T, T, T, Y0, p + 2);
      step(ic<0>{}, T, T, T, Y0, p + 3);
      step(ic<1>{}, T, T, T, Y0, p + 4);
      step(ic<2>{}, T, T, T, Y0, p + 5);
      flush(p - 5, BODY);
    }
    constexpr int PT = 9 + 6 * ((NP - 9) / 6);  // tail: full steps PT .. NP - 1
    if constexpr (NP - PT >= 1) step(ic<3>{}, T, T, T, Y0, PT);
    if constexpr (NP - PT >= 2) step(ic<4>{}, T, T, T, Y0, PT + 1);
    if constexpr (NP - PT >= 3) step(ic<5>{}, T, T, T, Y0, PT + 2);
    if constexpr (NP - PT >= 4) step(ic<0>{}, T, T, T, Y0, PT + 3);
    if constexpr (NP - PT >= 5) step(ic<1>{}, T, T, T, Y0, PT + 4);
    if constexpr (NP - PT >= 1) flush(PT - 5, NP - PT);  // <= 5 rows per record
    step(ic<NP % 6>{}, F, T, T, Y0, NP);
    step(ic<(NP + 1) % 6>{}, F, F, T, ic<2>{}, NP + 1);  // bottom row of the last band
    flush(NP - 5, 2);

    // ---- exact recheck of the queued uncertain values (rare)
    if (nq > QC) {
      // queue overflow (adversarial input: many values inside the band): the
      // exact decision for every output pixel of this warp's half-window
      __syncwarp();
      const unsigned char* sb = fp_smem + (base - smem0);
      if (outl)
        for (int q = 3; q <= OH + 2; ++q)
          for (int half = 0; half < 2; ++half) {
            const int y = by + q + half * OH;
            if (y >= H) continue;
            for (int j = 0; j < LC; ++j)
              o[(long long)y * OW + xl + j] =
                  exact_white<OH>(a, sb, taps, bx, by, xl + j, y, half) ? 0xFF : 0x00;
          }
      if (lane == 0) atomicAdd(&g_rechecks, (unsigned long long)(30 * LC * 2 * OH));
      __syncwarp();
    } else if (nq) {
      __syncwarp();  // queue records and the warp's mask stores are visible
      const unsigned char* sb = fp_smem + (base - smem0);
      unsigned cnt = 0;
      // work items: record r, row q0 + s, half h, column j -> one exact
      // decision each, spread over the lanes (latency ~ items / 32 calls)
      constexpr int PER = 2 * LC * BODY;  // values per record: rows x 2 halves x LC cols
      const int items = nq * PER;
      for (int it = lane; it < items; it += 32) {
        const uint32_t rec = queue[it / PER];
        const int e = it % PER, st = e / (2 * LC), half = (e / LC) & 1, j = e % LC;
        const int q0 = int(rec >> 16), L = int((rec >> 8) & 31), nstep = int(rec & 0xFFu);
        if (st >= nstep) continue;
        const int x = bx + 2 * (LC == 2 ? 1 + 30 * side + L : 2 * L) + j;
        const int y = by + q0 + st + half * OH;
        if (y >= H) continue;
        const bool wv = exact_white<OH>(a, sb, taps, bx, by, x, y, half);
        o[(long long)y * OW + x] = wv ? 0xFF : 0x00;
        ++cnt;
        if (a.dbg_px && x == a.dbg_x && y == a.dbg_y && u == a.dbg_t) {
          for (int dy = -3; dy <= 3; ++dy)
            for (int dx = -3; dx <= 3; ++dx)
              a.dbg_px[(dy + 3) * 7 + dx + 3] =
                  iir_at<OH>(sb, clampi(y + dy, 0, H - 1) - by, clampi(x + dx, 0, W - 1) - bx,
                             half);
          a.dbg_px[49] = wv ? 1.0f : 0.0f;
          a.dbg_px[50] = float(half);
          a.dbg_px[51] = 1.0f;
        }
      }
      for (int k2 = 16; k2 > 0; k2 >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, k2);
      if (lane == 0) atomicAdd(&g_rechecks, (unsigned long long)cnt);
      __syncwarp();  // queue reads done before the next frame reuses it
    }
    }
    __syncwarp();  // the warp's slot reads (and rechecks) are done
    mbar_arrive_lane0(bar_iir_empty(a, slot), lane);
    slot += NF;
    if (slot >= K) {
      slot -= K;
      par ^= 1u;
    }
  }
  if (a.dbg && lane == 0) {
    long long* d = a.dbg + 8 * blockIdx.x;
    atomicAdd(reinterpret_cast<unsigned long long*>(d + 2), (unsigned long long)w_full);
    atomicAdd(reinterpret_cast<unsigned long long*>(d + 5), (unsigned long long)(clk() - t_begin));
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    atomicMax(reinterpret_cast<unsigned long long*>(d + 1), now);
  }
}

// ------------------------------------------------------------------ kernel

__device__ __forceinline__ long long interior_flag(const Args& a, int bx, int by, int R) {
  return (bx >= 0 && bx + 127 <= a.W - 1 ? 1 : 0) + (by >= 0 && by + R - 1 <= a.H - 1 ? 2 : 0);
}

// SRC_F32 = false: the SPEC chain from the u8 RGBA video (F12345);
// SRC_F32 = true:  gaussian + gradient + threshold from f32 planes (F345).
template <int OH, bool SRC_F32, bool HALF>
__global__ void __launch_bounds__(NTHR, 1)
    k_chain_pipe(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ Args a) {
  constexpr int R = 2 * OH + 6;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int win = blockIdx.x % a.n_windows, seg = blockIdx.x / a.n_windows;
  const int strip = win % a.strips, band = win / a.strips;
  // this CTA's frames (Args: time segments / fix-up)
  Range rg{0, a.n_frames, a.n_warm, 0, a.state_in, a.state_out, nullptr};
  {
    const long long hwl = (long long)a.W * a.H;
    const int n_out = a.n_frames - a.n_warm;
    if (a.fix_k) {  // fix-up: re-run every window from the first wrong segment
      const int k = *a.fix_k;
      if (k >= a.n_segs) return;  // all segment warm states were exact
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
      *a.seg_k = a.n_segs;  // verification result slot (reset before verify runs)
  }
  // the last band ends exactly at row H - 1 (it overlaps the band above it;
  // both write identical values): the y clamps of the stencil march then
  // sit at compile-time steps (choose() keeps 2 OH <= H)
  const int bands = a.n_windows / a.strips;
  const int x0 = strip * SW,
            y0 = band == bands - 1 ? max(0, a.H - 2 * OH) : band * (2 * OH);
  const int bx = x0 - 4, by = y0 - 3;
  const int tx0 = bx >= 0 ? (bx & ~15) : -((-bx + 15) & ~15);
  double* taps = reinterpret_cast<double*>(fp_smem + a.off_taps);
  if (tid == 0) {
    for (int i = 0; i < NSF; ++i) {
      mbar_init(bar_rgb_full(a, i), 1);
      mbar_init(bar_rgb_empty(a, i), SRC_F32 ? NI : NIE);  // one arrive per IIR warp
    }
    for (int i = 0; i < K; ++i) {
      mbar_init(bar_iir_full(a, i), SRC_F32 ? NI : NIE);
      mbar_init(bar_iir_empty(a, i), WPF);  // the frame's stencil warps
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < 25) taps[tid] = double(a.p.taps[tid]);
  if (a.dbg && tid == 0) {
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    a.dbg[8 * blockIdx.x] = (long long)now;
    a.dbg[8 * blockIdx.x + 7] = (interior_flag(a, bx, by, 2 * OH + 6));
  }
  if (tid == 0) fp_rg = rg;
  __syncthreads();  // the only CTA-wide barrier: roles run decoupled from here

  const bool in_x = bx >= 0 && bx + 127 <= a.W - 1, in_y = by >= 0 && by + R - 1 <= a.H - 1;
  const bool interior = FP_SPECIALISE && in_x && in_y;
  // FP_SPECIALISE 2: IIR / plane roles specialised per CTA, one stencil path
  const bool interior_iir = (FP_SPECIALISE != 0) && in_x && in_y;
  if (warp < NS) {
    if (FP_SPECIALISE == 1 && interior)
      stencil_role<OH, false>(a, fp_rg, warp, lane, bx, by);
    else
      stencil_role<OH, true>(a, fp_rg, warp, lane, bx, by);
  } else if (warp < NS + NI && SRC_F32) {
    const int iw = warp - NS;
    if (interior_iir)
      plane_role<OH, false, false>(a, fp_rg, iw, lane, bx, by);
    else if (FP_SPECIALISE && in_x)
      plane_role<OH, false, true>(a, fp_rg, iw, lane, bx, by);
    else if (FP_SPECIALISE && in_y)
      plane_role<OH, true, false>(a, fp_rg, iw, lane, bx, by);
    else
      plane_role<OH, true, true>(a, fp_rg, iw, lane, bx, by);
  } else if (warp < NS + NIE && !SRC_F32) {
    const int iw = warp - NS, xoff = bx - tx0;
    if (interior_iir)
      iir_role<OH, false, false, HALF>(a, fp_rg, iw, lane, bx, by, xoff, &tmap, tx0);
    else if (FP_SPECIALISE && in_x)
      iir_role<OH, false, true, HALF>(a, fp_rg, iw, lane, bx, by, xoff, &tmap, tx0);
    else if (FP_SPECIALISE && in_y)
      iir_role<OH, true, false, HALF>(a, fp_rg, iw, lane, bx, by, xoff, &tmap, tx0);
    else
      iir_role<OH, true, true, HALF>(a, fp_rg, iw, lane, bx, by, xoff, &tmap, tx0);
  } else if (lane == 0) {
    // producer: frame t -> RGB slot t % NSF once the IIR warps released it
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap) : "memory");
    int slot = 0;
    unsigned par = 0;
    const int n = fp_rg.n, f0 = fp_rg.f0;
    for (int t = 0; t < n; ++t) {
      wait_phase(bar_rgb_empty(a, slot), par ^ 1u);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(bar_rgb_full(a, slot), a.rgb_bytes);
      if (SRC_F32)  // f32 plane window: x start bx is a multiple of 4 (16-byte aligned)
        tma_load_3d(fp_smem + slot * a.rgb_stride, &tmap, bar_rgb_full(a, slot), bx, by,
                    f0 + t);
      else
        tma_load_3d(fp_smem + slot * a.rgb_stride, &tmap, bar_rgb_full(a, slot), tx0, by,
                    4 * (f0 + t));
      if (++slot == NSF) {
        slot = 0;
        par ^= 1u;
      }
    }
  }
}

// ------------------------------------------------------------------ host

size_t layout(int oh, bool src_f32, Args* a) {
  const int R = 2 * oh + 6;
  const size_t rgb = src_f32 ? size_t(R) * 512 : size_t(3) * R * BWB;
  const size_t rgb_stride = (rgb + 127) / 128 * 128;
  size_t off = NSF * rgb_stride;
  const size_t off_iir = off;
  const size_t iir_stride = size_t(oh + 6) * PROW;
  off += K * iir_stride;
  const size_t off_bar = off;
  off += (2 * NSF + 2 * K) * 8;
  const size_t off_taps = (off + 7) / 8 * 8;
  off = off_taps + 25 * 8;
  const size_t off_queue = off;  // per stencil warp: QC records
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

#define FP_OH_LIST(X) X(3) X(4) X(5) X(8) X(10) X(12) X(15)

// src_f32: F345 (no IIR role; HALF irrelevant, one instantiation)
KernelFn kernel_for(int oh, bool src_f32, bool half = true) {
  switch (oh) {
#define FP_CASE(N)                                                          \
  case N:                                                                   \
    return src_f32 ? k_chain_pipe<N, true, true>                            \
                   : (half ? k_chain_pipe<N, false, true> : k_chain_pipe<N, false, false>);
    FP_OH_LIST(FP_CASE)
#undef FP_CASE
  }
  return nullptr;
}

struct PipePlan {
  int W = -1, H = -1, dev = -1, frames = -1, force_oh = 0, force_segs = 0;
  bool segs_ok = false;
  int oh = 0, strips = 0, bands = 0, n_segs = 1, seg_len = 0;
  size_t smem = 0;
};

constexpr int SEG_WARM = 48;  // IIR warm-up of a time segment (48 -> no mismatch;
                              // the seam check + fix-up keep any length exact)

// Every CTA marches its frames; an SM's time is ~ (CTAs it runs) x (pair-rows
// of a window) x (frames of a CTA, warm-up frames at ~0.4 of a full frame).
// Small frames leave SMs idle with one CTA per window, so the frames may be
// split into time segments (chain: restarted SEG_WARM frames early and
// verified, see Args).  Pick (OH, segments) minimising the busiest SM's load;
// ties go to the larger window.  The knobs pipe_oh / pipe_segs force.
bool choose(int W, int H, int frames, bool segs_ok, int dev, bool src_f32, int force,
            int force_segs, PipePlan* pp) {
  int sms = 0, optin = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const int strips = (W + SW - 1) / SW;
  double best = 1e300;
  const int ohs[] = {
#define FP_ITEM(N) N,
      FP_OH_LIST(FP_ITEM)
#undef FP_ITEM
  };
  const bool dbg = fc_get_knobs()->debug != 0;
  const double warm_cost = src_f32 ? 0.0 : 0.4;
  for (int oh : ohs) {
    if (force && oh != force) continue;
    const size_t smem = layout(oh, src_f32, nullptr);
    if (smem > size_t(optin) || 2 * oh > H) continue;  // the last band must fit the video
    KernelFn fn = kernel_for(oh, src_f32);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(smem));
    if (e == cudaSuccess && !src_f32)  // the general-alpha IIR variant of the same window
      e = cudaFuncSetAttribute(kernel_for(oh, false, false),
                               cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    int per_sm = 0;
    if (e == cudaSuccess)
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, NTHR, smem);
    if (dbg)
      std::fprintf(stderr, "fc_pipe choose: oh=%d smem=%zu optin=%d err=%s per_sm=%d\n", oh,
                   smem, optin, cudaGetErrorString(e), per_sm);
    if (e != cudaSuccess || per_sm < 1) {
      cudaGetLastError();
      continue;
    }
    const long long bands = (H + 2 * oh - 1) / (2 * oh);
    const long long windows = strips * bands;
    const int max_segs = segs_ok ? 16 : 1;
    for (int segs = 1; segs <= max_segs; ++segs) {
      if (force_segs && segs_ok && segs != force_segs) continue;
      const long long L = (frames + segs - 1) / segs;
      // segments that actually hold frames (16 asked of 161 frames: L = 11,
      // 15 segments); an empty trailing segment would march warm-up frames
      // past the end of its range
      const int nseg = L > 0 ? int((frames + L - 1) / L) : 1;
      if (!force_segs && segs > 1 && !src_f32 && L < 2 * SEG_WARM) break;  // warm-up dominates
      if (segs > 1 && L < 2) break;
      const long long ctas = windows * nseg;
      const long long per_busiest = (ctas + sms - 1) / sms;
      const double cta_frames = double(L) + (segs > 1 ? warm_cost * SEG_WARM : 0.0);
      const double cost = double(per_busiest) * (oh + 6) * cta_frames * (1.0 - 1e-4 * oh);
      if (cost < best) {
        best = cost;
        pp->oh = oh;
        pp->strips = strips;
        pp->bands = int(bands);
        pp->smem = smem;
        pp->n_segs = nseg;
        pp->seg_len = int(L);
      }
    }
  }
  if (best >= 1e300 && force_segs)  // a forced segment count the frames cannot take
    return choose(W, H, frames, segs_ok, dev, src_f32, force, 0, pp);
  if (dbg && best < 1e300)
    std::fprintf(stderr, "fc_pipe choose: -> oh=%d segs=%d seg_len=%d\n", pp->oh, pp->n_segs,
                 pp->seg_len);
  return best < 1e300;
}

// Chain segments: first segment s >= 1 whose warm state differs from the end
// state of segment s-1 (bitwise), atomically minimised into *k.
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

// Scratch of the segmented launches, per (device, stream).
struct SegScratch {
  float* buf = nullptr;
  size_t cap = 0;
  int* k = nullptr;
  float* dbg_px = nullptr;
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
    if (it->second.dbg_px) cudaFree(it->second.dbg_px);
  seg_all().erase(it);
}

// Shared launcher of both modes (src_f32: F345 from f32 planes).
int launch_pipe(bool src_f32, const FastParams& fp, const void* in, void* out, fc_dims d,
                int n_warm, const float* state_in, float* state_out, void* stream,
                int pitch = 0, int opitch = 0) {
  if (d.frames == 0) return 0;
  int dev = 0;
  cudaGetDevice(&dev);
  static thread_local PipePlan caches[2];
  PipePlan& cache = caches[src_f32 ? 1 : 0];
  const fc_knobs& kn = *fc_get_knobs();
  // time segments only for self-contained launches (no carried state in,
  // no launch-level warm-up): their CTAs may restart the IIR anywhere
  const bool segs_ok = src_f32 || (state_in == nullptr && n_warm == 0);
  const int force_oh = kn.pipe_oh;
  const int force_segs = kn.pipe_segs;
  if (cache.W != d.width || cache.H != d.height || cache.dev != dev ||
      cache.frames != d.frames || cache.segs_ok != segs_ok || cache.force_oh != force_oh ||
      cache.force_segs != force_segs) {
    PipePlan pp;
    if (!choose(d.width, d.height, d.frames - n_warm, segs_ok, dev, src_f32, force_oh,
                force_segs, &pp))
      return -1;
    pp.force_oh = force_oh;
    pp.force_segs = force_segs;
    pp.W = d.width;
    pp.H = d.height;
    pp.dev = dev;
    pp.frames = d.frames;
    pp.segs_ok = segs_ok;
    cache = pp;
  }
  Args a;
  std::memset(&a, 0, sizeof a);
  layout(cache.oh, src_f32, &a);
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
  a.seg_warm = src_f32 ? 0 : (kn.pipe_seg_warm > 0 ? kn.pipe_seg_warm : SEG_WARM);
  const long long hwl = (long long)d.width * d.height;
  const bool verify = !src_f32 && cache.n_segs > 1;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (verify) {  // per-segment end / warm state planes and the verdict slot
    // Owned by (device, stream): launches on one stream are ordered, so a
    // segmented launch never sees another's seams; two streams (two
    // executors, or device-pointer runs on two streams) get two buffers.
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
  a.skip = kn.pipe_skip;
  if (kn.band_scale > 0.0f) a.p.band_n *= kn.band_scale;  // tests / diagnostics only
  if (kn.dbg_px_on) {
    SegScratch& sc = seg_scratch(dev, st);
    if (!sc.dbg_px && cudaMalloc(&sc.dbg_px, 64 * sizeof(float)) != cudaSuccess)
      return int(cudaGetLastError());
    cudaMemsetAsync(sc.dbg_px, 0, 64 * sizeof(float), st);
    a.dbg_x = kn.dbg_px[0];
    a.dbg_y = kn.dbg_px[1];
    a.dbg_t = kn.dbg_px[2];
    a.dbg_px = sc.dbg_px;
  }
  CUtensorMap map;
  if (src_f32 ? !plane_tensor_map(&map, in, d, 128, 2 * cache.oh + 6)
              : !rgb_tensor_map(&map, in, d, BWB, 2 * cache.oh + 6, pitch ? pitch : d.width))
    return -1;
  const int grid = cache.strips * cache.bands * cache.n_segs;
  const bool profile = kn.profile != 0;
  if (profile) {
    cudaMalloc(&a.dbg, sizeof(long long) * 8 * grid);
    cudaMemsetAsync(a.dbg, 0, sizeof(long long) * 8 * grid, st);
  }
  const bool half = src_f32 || fp.alpha_half;
  kernel_for(cache.oh, src_f32, half)<<<grid, NTHR, cache.smem, st>>>(map, a);
  int rc = int(cudaGetLastError());
  if (rc == 0 && verify) {
    // verify the segment seams, then (device-side decision) re-run every
    // window from the first wrong segment; a no-op launch when all matched
    k_verify_segments<<<296, 256, 0, st>>>(a.seg_warm_out, a.seg_end, hwl, cache.n_segs,
                                           a.seg_k);
    Args f = a;
    f.fix_k = a.seg_k;
    f.seg_k = nullptr;
    kernel_for(cache.oh, src_f32, half)<<<cache.strips * cache.bands, NTHR, cache.smem, st>>>(
        map, f);
    rc = int(cudaGetLastError());
  }
  if (profile && a.dbg) {  // per-CTA span and per-role wait shares
    std::vector<long long> h(size_t(8) * grid);
    cudaStreamSynchronize(st);
    cudaMemcpy(h.data(), a.dbg, h.size() * sizeof(long long), cudaMemcpyDeviceToHost);
    cudaFree(a.dbg);
    long long t0 = h[0], t1 = 0;
    for (int b = 0; b < grid; ++b) t0 = std::min(t0, h[size_t(b) * 8]);
    double cls[4][6] = {};
    for (int b = 0; b < grid; ++b) {
      const long long* r = &h[size_t(b) * 8];
      t1 = std::max(t1, r[1]);
      double* c = cls[r[7] & 3];
      c[0] += 1;
      c[1] += double(r[1] - r[0]) / 1e3;
      c[2] += double(r[2]) / double(r[5]);  // stencil wait share
      c[3] += double(r[3]) / double(r[6]);  // IIR rgb wait share
      c[4] += double(r[4]) / double(r[6]);  // IIR slot wait share
      c[5] = std::max(c[5], double(r[1] - r[0]) / 1e3);
    }
    std::fprintf(stderr, "fc_pipe oh=%d grid=%d NF=%d NI=%d K=%d: kernel span %.1f us\n",
                 cache.oh, grid, NF, NI, K, double(t1 - t0) / 1e3);
    const char* names[4] = {"corner", "x-interior", "y-interior", "interior"};
    for (int k = 0; k < 4; ++k)
      if (cls[k][0] > 0)
        std::fprintf(stderr,
                     "  %-10s ctas %3.0f  span avg %.1f max %.1f us  stencil wait %.2f  "
                     "iir wait rgb %.2f slot %.2f\n",
                     names[k], cls[k][0], cls[k][1] / cls[k][0], cls[k][5],
                     cls[k][2] / cls[k][0], cls[k][3] / cls[k][0], cls[k][4] / cls[k][0]);
    if (kn.profile == 2) {  // every CTA: start, span, waits
      for (int b = 0; b < grid; ++b) {
        const long long* r = &h[size_t(b) * 8];
        std::fprintf(stderr, "  cta %4d win(%d,%d) class %lld start %+.2f us span %.1f us  "
                     "stencil wait %.3f  iir rgb %.3f slot %.3f\n",
                     b, b % cache.strips, (b / cache.strips) % cache.bands, r[7] & 3,
                     double(r[0] - t0) / 1e3, double(r[1] - r[0]) / 1e3,
                     double(r[2]) / double(r[5]), double(r[3]) / double(r[6]),
                     double(r[4]) / double(r[6]));
      }
    }
  }
  if (a.dbg_px) {
    float h[64];
    cudaStreamSynchronize(st);
    cudaMemcpy(h, a.dbg_px, sizeof h, cudaMemcpyDeviceToHost);
    std::fprintf(stderr, "fc_pipe debug px (%d,%d,%d): seen %g half %g white %g\n", a.dbg_x,
                 a.dbg_y, a.dbg_t, h[51], h[50], h[49]);
    for (int r = 0; r < 7; ++r) {
      for (int c = 0; c < 7; ++c) std::fprintf(stderr, " %.9g", h[r * 7 + c]);
      std::fprintf(stderr, "\n");
    }
  }
  return rc;
}

}  // namespace FP_NAMESPACE

using namespace FP_NAMESPACE;

extern "C" void fc_pipe_release_scratch(int device, void* stream) {
  release_scratch(device, static_cast<cudaStream_t>(stream));
}

// pitch: the video's row pitch in bytes (0 = width); the planes stay
// [t][4][H][pitch].  -1: the chain or the layout is outside the certified path.
// opitch: the mask's row pitch in bytes (0 = width): the stencil warps store
// 4 mask bytes at a time, so rows must start 4-byte aligned.
extern "C" int FP_ENTRY(const fc_stage* sgray, const fc_stage* si, const fc_stage* sg,
                        const fc_stage* sthr, const void* video, int in_type, int gray_in,
                        void* out, int out_type, fc_dims d, int n_warm,
                        const float* state_in, float* state_out, int pitch, int opitch,
                        void* stream) {
  FastParams fp;
  if (pitch == 0) pitch = d.width;
  if (opitch == 0) opitch = d.width;
  if (opitch < d.width || opitch % 4 != 0 || reinterpret_cast<uintptr_t>(out) % 4 != 0)
    return -1;
  if (!fast_params(sgray, si, sg, sthr, video, in_type, gray_in, out_type, d, pitch, &fp))
    return -1;
  return launch_pipe(false, fp, video, out, d, n_warm, state_in, state_out, stream, pitch,
                     opitch);
}

extern "C" int fc_chain_pipe_applies(const fc_stage* sgray, const fc_stage* si,
                                     const fc_stage* sg, const fc_stage* sthr, int in_type,
                                     int gray_in, int out_type, fc_dims d, int pitch) {
  FastParams fp;
  alignas(16) static const unsigned char probe[16] = {};
  return fast_params(sgray, si, sg, sthr, probe, in_type, gray_in, out_type, d, pitch, &fp) &&
         2 * 3 <= d.height;
}

// F345 (gaussian r=2 + Sobel + threshold) on f32 planes whose values lie in
// [0, in_max] (in_max from the executor's range analysis; <= 0: unknown ->
// -1, the caller runs the exact kernel).
extern "C" int FP_F345_ENTRY(const fc_stage* sg, const fc_stage* sthr, const float* in,
                             void* out, int out_type, fc_dims d, double in_max,
                             void* stream) {
  FastParams fp;
  std::memset(&fp, 0, sizeof fp);
  if (d.width % 4 != 0 || reinterpret_cast<uintptr_t>(in) % 16 != 0) return -1;
  if (!stencil_params(sg, sthr, out_type, in_max, &fp)) return -1;
  return launch_pipe(true, fp, in, out, d, 0, nullptr, nullptr, stream);
}

extern "C" long long FP_RECHECKS(void) {
  unsigned long long v = 0;
  if (cudaMemcpyFromSymbol(&v, g_rechecks, sizeof v) != cudaSuccess) return -1;
  return (long long)v;
}
