// GPU restatement of the reference's tiled-fused executor semantics
// (run_group_box / run_tiled, /root/reference/proj/src/simulator.cpp:202-333)
// for fp_simulate.
//
// The production kernels never under-stage a halo, so their output equals
// run_sequential's; the reference's run_tiled, however, reproduces what a
// plan with a SHORT halo (halo_mode PaperMax: per-side maxima instead of the
// cumulative sums) or a recurrence split across boxes (tile.t < frames)
// would compute: every member stage runs over the whole staged box and reads
// its input clamped to the video FIRST and to the staged box SECOND, so
// values near box edges erode, and the IIR restarts at each box's first
// staged frame.  fp_simulate reports those differences (interior vs
// boundary, simulator.cpp:335-368); this kernel computes them on the device:
// one CTA per output box, the staged box and its stage-to-stage successor in
// a per-CTA global scratch slot, reference arithmetic for every op
// (apply_stencil_at, simulator.cpp:48-108).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "fc_kernels.h"

namespace fctiled {

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return min(max(v, lo), hi); }

struct Geo {
  int W, H, F;
  int tx, ty, tt;                       // tile (output box) shape
  int xlo, xhi, ylo, yhi, tlo, thi;     // group halo
  int nbx, nby, nbt;                    // boxes per axis
  long long box_elems;                  // staged elements x max channels
};

struct Box {
  int x0, y0, t0, ex, ey, et, ch;
  const float* p;
  // StagedBox::read_global (simulator.cpp:202-210): clamp to the video, then
  // to the staged extent
  __device__ float at(const Geo& g, int gx, int gy, int gt, int c) const {
    gx = clampi(gx, 0, g.W - 1);
    gy = clampi(gy, 0, g.H - 1);
    gt = clampi(gt, 0, g.F - 1);
    const int ix = clampi(gx - x0, 0, ex - 1), iy = clampi(gy - y0, 0, ey - 1),
              it = clampi(gt - t0, 0, et - 1);
    return p[(((long long)it * ch + c) * ey + iy) * ex + ix];
  }
};

// apply_stencil_at for the frame-local / box ops (the IIR is scanned apart)
__device__ float apply_at(const fc_stage& s, const Geo& g, const Box& b, int x, int y, int t,
                          int c) {
  switch (s.op) {
    case FC_RGBA2GRAY:  // simulator.cpp:51-56
      return __fadd_rn(__fadd_rn(__fmul_rn(s.wr, b.at(g, x, y, t, 0)),
                                 __fmul_rn(s.wg, b.at(g, x, y, t, 1))),
                       __fmul_rn(s.wb, b.at(g, x, y, t, 2)));
    case FC_GAUSSIAN: {  // :63-74, FP64 accumulation dy outer, dx inner
      const int r = s.g_radius, d = 2 * r + 1;
      double acc = 0.0;
      for (int dy = -r; dy <= r; ++dy)
        for (int dx = -r; dx <= r; ++dx)
          acc = __fma_rn(double(s.g_w[(dy + r) * d + dx + r]),
                         double(b.at(g, x + dx, y + dy, t, c)), acc);
      return __double2float_rn(acc);
    }
    case FC_GRADIENT: {  // :75-83
      auto q = [&](int dx, int dy) { return b.at(g, x + dx, y + dy, t, c); };
      const float gx =
          __fsub_rn(__fadd_rn(__fadd_rn(q(1, -1), __fmul_rn(2.0f, q(1, 0))), q(1, 1)),
                    __fadd_rn(__fadd_rn(q(-1, -1), __fmul_rn(2.0f, q(-1, 0))), q(-1, 1)));
      const float gy =
          __fsub_rn(__fadd_rn(__fadd_rn(q(-1, 1), __fmul_rn(2.0f, q(0, 1))), q(1, 1)),
                    __fadd_rn(__fadd_rn(q(-1, -1), __fmul_rn(2.0f, q(0, -1))), q(1, -1)));
      return __fsqrt_rn(__fadd_rn(__fmul_rn(gx, gx), __fmul_rn(gy, gy)));
    }
    case FC_THRESHOLD:  // :84-89
      return b.at(g, x, y, t, c) >= s.th ? s.white : s.black;
    case FC_SCALE_OFFSET:  // :91-95
      return __fadd_rn(__fmul_rn(s.scale, b.at(g, x, y, t, c)), s.offset);
    case FC_BOX_MEAN: {  // :96-106
      double acc = 0.0;
      for (int dt = -s.rt; dt <= s.rt; ++dt)
        for (int dy = -s.ry; dy <= s.ry; ++dy)
          for (int dx = -s.rx; dx <= s.rx; ++dx)
            acc = __dadd_rn(acc, double(b.at(g, x + dx, y + dy, t + dt, c)));
      const int vol = (2 * s.rx + 1) * (2 * s.ry + 1) * (2 * s.rt + 1);
      return __double2float_rn(__ddiv_rn(acc, double(vol)));
    }
    default:  // identity (:90)
      return b.at(g, x, y, t, c);
  }
}

// run_group_box (simulator.cpp:229-294) for boxes blockIdx.x, +gridDim.x, ...
// in: [t][c][y][x] with in_ch channels (u8 or f32); out: [t][y][x] f32 (the
// group's members end single-channel).
template <typename InT>
__global__ void __launch_bounds__(256) k_tiled_group(const fc_stage* __restrict__ st, int n_st,
                                                     const InT* __restrict__ in, int in_ch,
                                                     float* __restrict__ out, Geo g,
                                                     float* __restrict__ scratch) {
  float* A = scratch + (long long)blockIdx.x * 2 * g.box_elems;
  float* B = A + g.box_elems;
  const long long n_boxes = (long long)g.nbx * g.nby * g.nbt;
  for (long long bi = blockIdx.x; bi < n_boxes; bi += gridDim.x) {
    const int bxi = int(bi % g.nbx), byi = int((bi / g.nbx) % g.nby), bti = int(bi / ((long long)g.nbx * g.nby));
    const int bx0 = bxi * g.tx, by0 = byi * g.ty, bt0 = bti * g.tt;
    const int ox = min(g.tx, g.W - bx0), oy = min(g.ty, g.H - by0), ot = min(g.tt, g.F - bt0);
    Box cur{bx0 - g.xlo, by0 - g.ylo, bt0 - g.tlo, ox + g.xlo + g.xhi, oy + g.ylo + g.yhi,
            ot + g.tlo + g.thi, in_ch, A};
    const long long vol = (long long)cur.ex * cur.ey * cur.et;
    // stage the haloed input box: out-of-video cells hold the clamped edge
    for (long long i = threadIdx.x; i < vol * in_ch; i += blockDim.x) {
      const int ix = int(i % cur.ex);
      const int iy = int((i / cur.ex) % cur.ey);
      const int c = int((i / ((long long)cur.ex * cur.ey)) % in_ch);
      const int it = int(i / ((long long)cur.ex * cur.ey * in_ch));
      const int gx = clampi(cur.x0 + ix, 0, g.W - 1), gy = clampi(cur.y0 + iy, 0, g.H - 1),
                gt = clampi(cur.t0 + it, 0, g.F - 1);
      A[i] = float(in[((long long)gt * in_ch + c) * g.H * g.W + (long long)gy * g.W + gx]);
    }
    __syncthreads();
    for (int k = 0; k < n_st; ++k) {
      const fc_stage s = st[k];
      Box nxt = cur;
      nxt.ch = 1;
      nxt.p = cur.p == A ? B : A;
      float* dst = const_cast<float*>(nxt.p);
      if (s.op == FC_IIR_TEMPORAL) {
        // each (x, y) scans the staged t extent; the recurrence restarts at
        // global frame 0 or at the staged box's first frame (:256-268)
        const int i0 = max(0, -cur.t0);
        const float beta = 1.0f - s.alpha;  // float(1 - alpha), as the reference
        for (long long i = threadIdx.x; i < (long long)cur.ex * cur.ey; i += blockDim.x) {
          const int ix = int(i % cur.ex), iy = int(i / cur.ex);
          float prev = 0.0f;
          for (int it = 0; it < cur.et; ++it) {
            const float x = cur.at(g, cur.x0 + ix, cur.y0 + iy, cur.t0 + it, 0);
            prev = it <= i0 ? x : __fadd_rn(__fmul_rn(s.alpha, x), __fmul_rn(beta, prev));
            dst[((long long)it * cur.ey + iy) * cur.ex + ix] = prev;
          }
        }
      } else {
        for (long long i = threadIdx.x; i < vol; i += blockDim.x) {
          const int ix = int(i % cur.ex), iy = int((i / cur.ex) % cur.ey),
                    it = int(i / ((long long)cur.ex * cur.ey));
          dst[i] = apply_at(s, g, cur, cur.x0 + ix, cur.y0 + iy, cur.t0 + it, 0);
        }
      }
      __syncthreads();
      cur = nxt;
    }
    // write-back of the output box through read_global (:287-293)
    for (long long i = threadIdx.x; i < (long long)ox * oy * ot; i += blockDim.x) {
      const int x = bx0 + int(i % ox), y = by0 + int((i / ox) % oy),
                t = bt0 + int(i / ((long long)ox * oy));
      out[((long long)t * g.H + y) * g.W + x] = cur.at(g, x, y, t, 0);
    }
    __syncthreads();
  }
}

}  // namespace fctiled

using namespace fctiled;

// stages: device array of n_stages fc_stage (host copy in `host_stages` for
// the channel bookkeeping); halo = {x_lo, x_hi, y_lo, y_hi, t_lo, t_hi}.
// scratch: device memory of at least fc_tiled_scratch_bytes(...).
extern "C" long long fc_tiled_scratch_bytes(int tile_x, int tile_y, int tile_t,
                                            const int* halo, int in_ch, int ctas) {
  const long long e = (long long)(tile_x + halo[0] + halo[1]) * (tile_y + halo[2] + halo[3]) *
                      (tile_t + halo[4] + halo[5]) * std::max(in_ch, 1);
  return 2 * e * ctas * (long long)sizeof(float);
}

extern "C" int fc_tiled_group(const fc_stage* dev_stages, int n_stages, const void* in,
                              int in_type, int in_ch, float* out, fc_dims d, int tile_x,
                              int tile_y, int tile_t, const int* halo, float* scratch,
                              int ctas, void* stream) {
  if ((long long)d.width * d.height * d.frames == 0) return 0;
  Geo g;
  g.W = d.width;
  g.H = d.height;
  g.F = d.frames;
  g.tx = tile_x;
  g.ty = tile_y;
  g.tt = tile_t;
  g.xlo = halo[0];
  g.xhi = halo[1];
  g.ylo = halo[2];
  g.yhi = halo[3];
  g.tlo = halo[4];
  g.thi = halo[5];
  g.nbx = (d.width + tile_x - 1) / tile_x;
  g.nby = (d.height + tile_y - 1) / tile_y;
  g.nbt = (d.frames + tile_t - 1) / tile_t;
  g.box_elems = (long long)(tile_x + halo[0] + halo[1]) * (tile_y + halo[2] + halo[3]) *
                (tile_t + halo[4] + halo[5]) * std::max(in_ch, 1);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (in_type == FC_U8)
    k_tiled_group<uint8_t><<<ctas, 256, 0, st>>>(dev_stages, n_stages,
                                                 static_cast<const uint8_t*>(in), in_ch, out, g,
                                                 scratch);
  else
    k_tiled_group<float><<<ctas, 256, 0, st>>>(dev_stages, n_stages,
                                               static_cast<const float*>(in), in_ch, out, g,
                                               scratch);
  return int(cudaGetLastError());
}
