// F12345 certified fast path, STRIP MARCH (the headline kernel).
//
// Same arithmetic contract as fc_fast.cu (exact S1+S2, certified packed-FP32
// S3-S5, exact FP64 recheck inside the error band; see that file's header and
// fccommon::certify_band), re-organised so that stencil intermediates live in
// REGISTERS instead of shared-memory planes:
//
//   * a CTA owns a window of 128 columns x R = 4 * nw rows of the video (nw
//     warps) and marches it over all frames carrying the exact IIR state; the
//     window's outputs are its central 120 columns x (R - 6) rows (3-row /
//     4-column halo for gaussian r=2 + Sobel r=1);
//   * lane L of warp w owns the 4 x 4 pixel block (cols 4L..4L+3, rows
//     4w..4w+3): its IIR state stays in 16 registers for the whole march;
//   * horizontal neighbours come from the adjacent lanes (SHFL), vertical
//     neighbours from the lane's own rows, and only the 3 boundary rows of the
//     horizontal-pass plane cross warps, through shared memory (one CTA
//     barrier per frame pair, double-buffered planes);
//   * frames are processed in pairs (t, t+1) so every stencil value is a
//     float2 and every stencil op one FFMA2 / FADD2 / FMUL2;
//   * input: a TMA ring of NSF frames, one 3-D copy per frame (R, G, B planes
//     of the window; alpha never leaves HBM).
//
// Per frame pair, per warp:
//   1  S1+S2 exact for its 16 pixels x 2 frames (state in registers), store
//      the IIR values (needed only by the rare exact recheck), horizontal
//      5-tap pass with 8 SHFL per row -> H rows kept in registers + stored;
//   -- __syncthreads (H planes of the pair complete; TMA slots consumed)
//   2  vertical 5-tap pass over own + 6 halo H rows -> G (6 rows), Sobel with
//      SHFL for the x-neighbours, m - M*, packed mask stores; pixels inside
//      the certified band are recomputed exactly from the IIR plane.
//
// Video borders (BORDER instantiation): rows / 4-column groups outside the
// video read the clamped RGB row / replicate the edge byte, so the IIR and H
// planes hold clamp-to-edge values (simulator.cpp:202-210); Sobel then clamps
// its G rows / columns at the first and last video row / column.
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "fc_common.cuh"

namespace fcstrip {

using namespace fccommon;

constexpr int RY = 4;      // rows per warp
constexpr int NWMAX = 9;   // warps per CTA (bounded by shared memory)
constexpr int NSF = 4;     // TMA frame slots (two frame pairs in flight)
constexpr int SW = 120;    // output columns per strip (window 128 = SW + 8)
constexpr int BWB = 144;   // TMA box row bytes: 128 + worst-case 16-B alignment slack
constexpr int ROWB = 1024; // bytes per plane row: 4 cell slots x 32 lanes x float2

struct Args {
  uint8_t* out;
  int W, H, n_frames, n_warm;
  int R, strips;                     // window rows (4 nw), strips across W
  unsigned slot_bytes, slot_stride;  // TMA bytes per frame, slot pitch
  unsigned off_iir, off_h, buf_bytes, off_bar, off_taps;
  const float* state_in;
  float* state_out;
  FastParams p;
};

__device__ unsigned long long g_rechecks;
extern __shared__ __align__(128) unsigned char fs_smem[];

__device__ __forceinline__ float2 shfl_up2(float2 v) {
  return make_float2(__shfl_up_sync(0xffffffffu, v.x, 1), __shfl_up_sync(0xffffffffu, v.y, 1));
}
__device__ __forceinline__ float2 shfl_down2(float2 v) {
  return make_float2(__shfl_down_sync(0xffffffffu, v.x, 1),
                     __shfl_down_sync(0xffffffffu, v.y, 1));
}

// Plane cell (row r, cell j of every lane L = window col 4L + j), this lane:
// slot j of a row is a contiguous float2[32] (conflict-free 8-byte accesses).
__device__ __forceinline__ float2* pcell(unsigned off, int r, int j, int lane) {
  return reinterpret_cast<float2*>(fs_smem + off + r * ROWB + j * 256) + lane;
}

// Frame component f of IIR cell (window row r, window col c).
__device__ __forceinline__ float iir_cell(unsigned off, int r, int c, int f) {
  return *reinterpret_cast<const float*>(fs_smem + off + r * ROWB + (c & 3) * 256 +
                                         (c >> 2) * 8 + f * 4);
}

// Exact reference threshold decision at (x, y), frame component f, from the
// exact IIR plane (simulator.cpp:63-89): FP64 gaussian in dy/dx order at the
// 3x3 clamped centres, Sobel in the reference's float order, IEEE sqrt.
__device__ __forceinline__ bool exact_white(const Args& a, unsigned iir_off, const double* taps,
                                         int bx, int by, int x, int y, int f) {
  float g[3][3];
  for (int j = 0; j < 3; ++j)
    for (int i = 0; i < 3; ++i) {
      int cx = clampi(x + i - 1, 0, a.W - 1), cy = clampi(y + j - 1, 0, a.H - 1);
      double acc = 0.0;
      for (int dy = -2; dy <= 2; ++dy) {
        int ry = clampi(cy + dy, 0, a.H - 1) - by;
        for (int dx = -2; dx <= 2; ++dx) {
          int rx = clampi(cx + dx, 0, a.W - 1) - bx;
          acc = __fma_rn(taps[(dy + 2) * 5 + dx + 2], double(iir_cell(iir_off, ry, rx, f)), acc);
        }
      }
      g[j][i] = __double2float_rn(acc);
    }
  auto s = [&](int dx, int dy) { return g[dy + 1][dx + 1]; };
  float gx = __fsub_rn(__fadd_rn(__fadd_rn(s(1, -1), __fmul_rn(2.0f, s(1, 0))), s(1, 1)),
                       __fadd_rn(__fadd_rn(s(-1, -1), __fmul_rn(2.0f, s(-1, 0))), s(-1, 1)));
  float gy = __fsub_rn(__fadd_rn(__fadd_rn(s(-1, 1), __fmul_rn(2.0f, s(0, 1))), s(1, 1)),
                       __fadd_rn(__fadd_rn(s(-1, -1), __fmul_rn(2.0f, s(0, -1))), s(1, -1)));
  return __fsqrt_rn(__fadd_rn(__fmul_rn(gx, gx), __fmul_rn(gy, gy))) >= a.p.th_val;
}

template <bool BORDER>
__device__ __forceinline__ void march(const CUtensorMap& tmap, const Args& a, int x0, int y0) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int W = a.W, H = a.H, n = a.n_frames, R = a.R;
  const int bx = x0 - 4, by = y0 - 3;
  const int tx0 = bx >= 0 ? (bx & ~15) : -((-bx + 15) & ~15);
  const int xoff = bx - tx0;
  const int r0 = warp * RY;
  const int xl = bx + 4 * lane;  // video column of this lane's first cell
  const bool fresh = a.state_in == nullptr;
  const long long hw = (long long)W * H;
  const float h0 = a.p.h0, h1 = a.p.h1, h2 = a.p.h2;
  const int cplane = R * BWB;  // bytes of one colour plane in a slot
  uint64_t* bar = reinterpret_cast<uint64_t*>(fs_smem + a.off_bar);
  const double* taps = reinterpret_cast<const double*>(fs_smem + a.off_taps);

  // RGB word offsets of the lane's rows (clamped rows in BORDER windows) and
  // column (an out-of-video group replicates the edge byte)
  int rowoff[RY];
#pragma unroll
  for (int i = 0; i < RY; ++i)
    rowoff[i] = (BORDER ? clampi(by + r0 + i, 0, H - 1) - by : r0 + i) * BWB;
  int coloff = xoff + 4 * lane;
  unsigned sel = 0x3210u;
  if (BORDER && (xl < 0 || xl > W - 1)) {
    const int edge = xl < 0 ? 0 : W - 1;
    coloff = (edge & ~3) - bx + xoff;
    sel = unsigned(edge & 3) * 0x1111u;
  }
  const bool outl = lane >= 1 && lane <= 30 && xl < W;
  bool outr[RY];
#pragma unroll
  for (int i = 0; i < RY; ++i) outr[i] = r0 + i >= 3 && r0 + i <= R - 4 && by + r0 + i < H;

  // IIR values of the lane's 16 cells for the current pair (frame t, t+1);
  // .y is the exact carried state
  float2 sv[RY][4];
#pragma unroll
  for (int i = 0; i < RY; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
      sv[i][j].y = fresh ? 0.0f
                         : a.state_in[(long long)clampi(by + r0 + i, 0, H - 1) * W +
                                      clampi(xl + j, 0, W - 1)];
  uint32_t orow[RY];  // mask offset of the lane's first cell in each row
#pragma unroll
  for (int i = 0; i < RY; ++i) orow[i] = uint32_t((by + r0 + i) * W + xl);
  const uint32_t k4b = a.p.k4b;

  float2 hreg[RY][4];  // horizontal-pass values of the lane's cells
  int slot = 0;
  unsigned parity = 0;
  for (int t = 0; t < n; t += 2) {
    const bool has1 = t + 1 < n;
    mbar_wait(&bar[slot], parity);
    if (has1) mbar_wait(&bar[slot + 1], parity);
    const unsigned char* f0 = fs_smem + slot * a.slot_stride;
    const unsigned char* f1 = f0 + a.slot_stride;
    const unsigned pb = ((t >> 1) & 1) * a.buf_bytes;
    const unsigned iir_off = a.off_iir + pb, h_off = a.off_h + pb;

    // ---------------- 1: S1+S2 exact, horizontal pass
    auto phase1 = [&](auto steady_tag) {
      constexpr bool STEADY = decltype(steady_tag)::value;
#pragma unroll
      for (int i = 0; i < RY; ++i) {
        uint32_t w0[3], w1[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          w0[c] = *reinterpret_cast<const uint32_t*>(f0 + c * cplane + rowoff[i] + coloff);
          w1[c] = *reinterpret_cast<const uint32_t*>(f1 + c * cplane + rowoff[i] + coloff);
          if (BORDER) {
            w0[c] = __byte_perm(w0[c], 0, sel);
            w1[c] = __byte_perm(w1[c], 0, sel);
          }
        }
        float2* v = sv[i];
#define FS_CELL(J)                                                                          \
  {                                                                                         \
    const float2 g = __fadd2_rn(                                                            \
        __fadd2_rn(wprod(f2(magic_r<J>(w0[0], k4b), magic_r<J>(w1[0], k4b)), a.p.wr, a.p.wrm), \
                   wprod(f2(magic_r<J>(w0[1], k4b), magic_r<J>(w1[1], k4b)), a.p.wg, a.p.wgm)), \
        wprod(f2(magic_r<J>(w0[2], k4b), magic_r<J>(w1[2], k4b)), a.p.wb, a.p.wbm));          \
    /* g = 0.5 * gray, exactly; y = fl(0.5 x + fl(0.5 y)) == FMA(0.5, y, g) */             \
    if (STEADY) {                                                                           \
      v[J].x = __fmaf_rn(0.5f, v[J].y, g.x);                                                \
      v[J].y = __fmaf_rn(0.5f, v[J].x, g.y);                                                \
    } else {                                                                                \
      v[J].x = (fresh && t == 0) ? __fadd_rn(g.x, g.x) : __fmaf_rn(0.5f, v[J].y, g.x);      \
      v[J].y = has1 ? __fmaf_rn(0.5f, v[J].x, g.y) : v[J].x;                                \
    }                                                                                       \
  }
        FS_CELL(0) FS_CELL(1) FS_CELL(2) FS_CELL(3)
#undef FS_CELL
#pragma unroll
        for (int j = 0; j < 4; ++j) *pcell(iir_off, r0 + i, j, lane) = v[j];
        const float2 l2 = shfl_up2(v[2]), l1 = shfl_up2(v[3]);
        const float2 q1 = shfl_down2(v[0]), q2 = shfl_down2(v[1]);
        hreg[i][0] = tap5(l2, l1, v[0], v[1], v[2], h0, h1, h2);
        hreg[i][1] = tap5(l1, v[0], v[1], v[2], v[3], h0, h1, h2);
        hreg[i][2] = tap5(v[0], v[1], v[2], v[3], q1, h0, h1, h2);
        hreg[i][3] = tap5(v[1], v[2], v[3], q1, q2, h0, h1, h2);
#pragma unroll
        for (int j = 0; j < 4; ++j) *pcell(h_off, r0 + i, j, lane) = hreg[i][j];
      }
    };
    if (has1 && !(fresh && t == 0))
      phase1(std::true_type{});
    else
      phase1(std::false_type{});
    __syncthreads();  // H / IIR planes of this pair complete; RGB slots consumed

    if (tid == 0) {  // refill the two slots with frames t+NSF, t+NSF+1
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      for (int q = 0; q < 2; ++q) {
        const int tf = t + q + NSF;
        if (tf < n) {
          mbar_expect_tx(&bar[slot + q], a.slot_bytes);
          tma_load_3d(fs_smem + (slot + q) * a.slot_stride, &tmap, &bar[slot + q], tx0, by,
                      4 * tf);
        }
      }
    }
    slot += 2;
    if (slot == NSF) {
      slot = 0;
      parity ^= 1u;
    }
    const bool out0 = t >= a.n_warm, out1 = has1 && t + 1 >= a.n_warm;
    if (!out0 && !out1) continue;  // warm-up pair: state only

    // ---------------- 2: vertical pass, Sobel, certified threshold
    float2 hh[RY + 6][4];  // H rows r0-3 .. r0+6
#pragma unroll
    for (int k = 0; k < RY + 6; ++k) {
      if (k >= 3 && k < 3 + RY) {
#pragma unroll
        for (int j = 0; j < 4; ++j) hh[k][j] = hreg[k - 3][j];
      } else {
        const int r = clampi(r0 - 3 + k, 0, R - 1);
#pragma unroll
        for (int j = 0; j < 4; ++j) hh[k][j] = *pcell(h_off, r, j, lane);
      }
    }
    float2 g[RY + 2][4];  // G rows r0-1 .. r0+4
#pragma unroll
    for (int m = 0; m < RY + 2; ++m)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        g[m][j] = tap5(hh[m][j], hh[m + 1][j], hh[m + 2][j], hh[m + 3][j], hh[m + 4][j], h0,
                       h1, h2);

    unsigned char* o0p = a.out + (long long)(t - a.n_warm) * hw;
    unsigned char* o1p = o0p + hw;
    const float mlo = a.p.mlo, band = a.p.band;
    const bool st0 = outl && out0, st1 = outl && out1;
    float2 dm[RY][4];  // mlo - m per cell and frame
    float amin = INFINITY;
#pragma unroll
    for (int i = 0; i < RY; ++i) {
      float2 s[4], d[4];
      const int y = by + r0 + i;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float2 gm = g[i][j], gc = g[i + 1][j], gp = g[i + 2][j];
        if (BORDER) {
          if (y == 0) gm = gc;
          if (y == H - 1) gp = gc;
        }
        s[j] = __fadd2_rn(__ffma2_rn(splat(2.0f), gc, gm), gp);
        d[j] = __ffma2_rn(splat(-1.0f), gm, gp);
      }
      float2 sl = shfl_up2(s[3]), dl = shfl_up2(d[3]);
      float2 sr = shfl_down2(s[0]), dr = shfl_down2(d[0]);
      if (BORDER) {
        if (xl == 0) sl = s[0], dl = d[0];
        if (xl + 3 == W - 1) sr = s[3], dr = d[3];
      }
      const float2 S[6] = {sl, s[0], s[1], s[2], s[3], sr};
      const float2 D[6] = {dl, d[0], d[1], d[2], d[3], dr};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 gx = __ffma2_rn(splat(-1.0f), S[j], S[j + 2]);
        const float2 gy = __fadd2_rn(__ffma2_rn(splat(2.0f), D[j + 1], D[j]), D[j + 2]);
        // nd = mlo - gy^2 - gx^2 (< 0 <=> white); two roundings, covered by
        // certify_band's 2u (M* + m) term
        const float2 ngx = f2(-gx.x, -gx.y), ngy = f2(-gy.x, -gy.y);
        dm[i][j] = __ffma2_rn(ngx, gx, __ffma2_rn(ngy, gy, splat(mlo)));
      }
      if (outr[i]) {
        if (st0)
          *reinterpret_cast<uint32_t*>(o0p + orow[i]) =
              pack_neg(dm[i][0].x, dm[i][1].x, dm[i][2].x, dm[i][3].x);
        if (st1)
          *reinterpret_cast<uint32_t*>(o1p + orow[i]) =
              pack_neg(dm[i][0].y, dm[i][1].y, dm[i][2].y, dm[i][3].y);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          amin = fminf(amin, fminf(fabsf(dm[i][j].x), fabsf(dm[i][j].y)));
      }
    }
    // ---------------- exact recheck of the uncertain pixels (rare)
    const bool amb = outl && amin <= band;
    if (__any_sync(0xffffffffu, amb)) {
      unsigned cnt = 0;
      if (amb) {
        unsigned bits = 0;  // bit 8i + 4f + j: cell (row i, col j), frame f uncertain
#pragma unroll
        for (int i = 0; i < RY; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (outr[i]) {
              if (out0 && fabsf(dm[i][j].x) <= band) bits |= 1u << (8 * i + j);
              if (out1 && fabsf(dm[i][j].y) <= band) bits |= 1u << (8 * i + 4 + j);
            }
        while (bits) {
          const int b = __ffs(bits) - 1;
          bits &= bits - 1;
          const int i = b >> 3, f = (b >> 2) & 1, j = b & 3;
          const int y = by + r0 + i;
          const bool wv = exact_white(a, iir_off, taps, bx, by, xl + j, y, f);
          o0p[(f ? hw : 0) + (long long)y * W + xl + j] = wv ? 0xFF : 0x00;
          ++cnt;
        }
      }
      for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
      if (lane == 0) atomicAdd(&g_rechecks, (unsigned long long)cnt);
    }
  }

  if (a.state_out && outl)
#pragma unroll
    for (int i = 0; i < RY; ++i)
      if (outr[i])
#pragma unroll
        for (int j = 0; j < 4; ++j)
          a.state_out[(long long)(by + r0 + i) * W + xl + j] = sv[i][j].y;
}

__global__ void __launch_bounds__(NWMAX * 32, 1)
    k_chain_strip(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ Args a) {
  const int tid = threadIdx.x;
  const int strip = blockIdx.x % a.strips, band = blockIdx.x / a.strips;
  const int x0 = strip * SW, y0 = band * (a.R - 6);
  const int bx = x0 - 4, by = y0 - 3;
  const int tx0 = bx >= 0 ? (bx & ~15) : -((-bx + 15) & ~15);
  uint64_t* bar = reinterpret_cast<uint64_t*>(fs_smem + a.off_bar);
  double* taps = reinterpret_cast<double*>(fs_smem + a.off_taps);
  if (tid == 0) {
    for (int i = 0; i < NSF; ++i) mbar_init(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap) : "memory");
  }
  if (tid < 25) taps[tid] = double(a.p.taps[tid]);
  __syncthreads();
  if (tid == 0)
    for (int t = 0; t < NSF && t < a.n_frames; ++t) {
      mbar_expect_tx(&bar[t], a.slot_bytes);
      tma_load_3d(fs_smem + t * a.slot_stride, &tmap, &bar[t], tx0, by, 4 * t);
    }
  const bool interior = bx >= 0 && bx + 127 <= a.W - 1 && by >= 0 && by + a.R - 1 <= a.H - 1;
  if (interior)
    march<false>(tmap, a, x0, y0);
  else
    march<true>(tmap, a, x0, y0);
}

// ------------------------------------------------------------------ host

size_t layout(int R, Args* a) {
  const size_t slot = size_t(3) * R * BWB, stride = (slot + 127) / 128 * 128;
  size_t off = NSF * stride;
  const size_t buf = size_t(R) * ROWB;
  const size_t off_iir = off;
  off += 2 * buf;
  const size_t off_h = off;
  off += 2 * buf;
  const size_t off_bar = off;
  off += NSF * 8;
  const size_t off_taps = (off + 7) / 8 * 8;
  off = off_taps + 25 * 8;
  if (a) {
    a->R = R;
    a->slot_bytes = unsigned(slot);
    a->slot_stride = unsigned(stride);
    a->off_iir = unsigned(off_iir);
    a->off_h = unsigned(off_h);
    a->buf_bytes = unsigned(buf);
    a->off_bar = unsigned(off_bar);
    a->off_taps = unsigned(off_taps);
  }
  return off;
}

struct StripPlan {
  int W = -1, H = -1, dev = -1;
  int nw = 0, strips = 0, bands = 0;
  size_t smem = 0;
};

// Every CTA marches the whole video, so an SM's time is (CTAs it runs) x
// (rows per CTA); pick the warps per CTA minimising the busiest SM's rows.
// FUSEPLAN_STRIP_NW forces the choice (tuning).
bool choose(int W, int H, int dev, StripPlan* sp) {
  int sms = 0, optin = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (cudaFuncSetAttribute(k_chain_strip, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(std::min<size_t>(size_t(optin), layout(4 * NWMAX, nullptr)))) !=
      cudaSuccess)
    return false;
  int force = 0;
  if (const char* env = std::getenv("FUSEPLAN_STRIP_NW")) force = std::atoi(env);
  const int strips = (W + SW - 1) / SW;
  double best = 1e300;
  for (int nw = 2; nw <= NWMAX; ++nw) {
    if (force && nw != force) continue;
    const int R = 4 * nw;
    const size_t smem = layout(R, nullptr);
    if (smem > size_t(optin)) continue;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_chain_strip, 32 * nw, smem) !=
            cudaSuccess ||
        per_sm < 1)
      continue;
    const long long bands = (H + (R - 6) - 1) / (R - 6);
    const long long ctas = strips * bands;
    const long long waves = (ctas + (long long)sms * per_sm - 1) / ((long long)sms * per_sm);
    const double cost = double(waves) * std::min<long long>(per_sm, (ctas + sms - 1) / sms) * R;
    if (cost < best) {
      best = cost;
      sp->nw = nw;
      sp->strips = strips;
      sp->bands = int(bands);
      sp->smem = smem;
    }
  }
  return best < 1e300;
}

}  // namespace fcstrip

using namespace fcstrip;

extern "C" int fc_chain_strip(const fc_stage* sgray, const fc_stage* si, const fc_stage* sg,
                              const fc_stage* sthr, const void* video, int in_type, int gray_in,
                              void* out, int out_type, fc_dims d, int n_warm,
                              const float* state_in, float* state_out, void* stream) {
  FastParams fp;
  if (!fast_params(sgray, si, sg, sthr, video, in_type, gray_in, out_type, d, &fp)) return -1;
  if (d.frames == 0) return 0;
  int dev = 0;
  cudaGetDevice(&dev);
  static thread_local StripPlan cache;
  if (cache.W != d.width || cache.H != d.height || cache.dev != dev) {
    StripPlan sp;
    if (!choose(d.width, d.height, dev, &sp)) return -1;
    sp.W = d.width;
    sp.H = d.height;
    sp.dev = dev;
    cache = sp;
  }
  Args a;
  std::memset(&a, 0, sizeof a);
  layout(4 * cache.nw, &a);
  a.out = static_cast<uint8_t*>(out);
  a.W = d.width;
  a.H = d.height;
  a.n_frames = d.frames;
  a.n_warm = n_warm;
  a.strips = cache.strips;
  a.state_in = state_in;
  a.state_out = state_out;
  a.p = fp;
  CUtensorMap map;
  if (!rgb_tensor_map(&map, video, d, BWB, a.R)) return -1;
  const int grid = cache.strips * cache.bands;
  k_chain_strip<<<grid, 32 * cache.nw, cache.smem, static_cast<cudaStream_t>(stream)>>>(map, a);
  return int(cudaGetLastError());
}

extern "C" long long fc_strip_recheck_count(void) {
  unsigned long long v = 0;
  if (cudaMemcpyFromSymbol(&v, g_rechecks, sizeof v) != cudaSuccess) return -1;
  return (long long)v;
}
