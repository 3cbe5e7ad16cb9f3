// T-shard carry verification: how far into a shard does a
// wrong start state reach?
//
// A shard of frames [lo, hi) runs from a warm state s_warm (its IIR restarted
// W frames early).  When the true carry s_true from the previous shard
// differs, only the frames whose IIR plane differs need recomputing: the
// recurrence y = fl(a x + fl(b y)) is deterministic, so once the trajectory
// started from s_true and the one started from s_warm coincide at a pixel
// they stay equal there.  This kernel re-runs S1+S2 ONLY for the pixels whose
// two start states differ (bitwise), both trajectories side by side, and
// returns k = the number of leading frames in which some pixel still
// differs (atomicMax of each pixel's first coincidence frame; 0 when the
// states agree everywhere, n when some pixel never converges inside the
// shard -- then the shard's end state changes too).  Frames >= k of the
// shard's output are already exact, so the fix-up recomputes S1-S5 over
// frames [lo, lo + k) only.  Reference arithmetic: simulator.cpp:51-62.
#include <cuda_runtime.h>

#include <cstdint>

#include "fc_kernels.h"

namespace fcshard {

template <typename InT>
__device__ __forceinline__ float load_px(const InT* p) {
  return float(*p);
}

template <typename InT, bool GRAY_IN>
__global__ void k_iir_converge(const InT* __restrict__ video, fc_stage sg, float alpha,
                               float beta, long long hw, int n_frames,
                               const float* __restrict__ s_true,
                               const float* __restrict__ s_warm, int* __restrict__ k_out) {
  constexpr int C = GRAY_IN ? 1 : 4;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < hw;
       p += (long long)gridDim.x * blockDim.x) {
    float a = s_true[p], b = s_warm[p];
    if (__float_as_uint(a) == __float_as_uint(b)) continue;
    int t = 0;
    for (; t < n_frames; ++t) {
      const InT* f = video + (long long)t * C * hw + p;
      float x;
      if (GRAY_IN) {
        x = load_px(f);
      } else {
        x = __fadd_rn(__fadd_rn(__fmul_rn(sg.wr, load_px(f)), __fmul_rn(sg.wg, load_px(f + hw))),
                      __fmul_rn(sg.wb, load_px(f + 2 * hw)));
      }
      a = __fadd_rn(__fmul_rn(alpha, x), __fmul_rn(beta, a));
      b = __fadd_rn(__fmul_rn(alpha, x), __fmul_rn(beta, b));
      if (__float_as_uint(a) == __float_as_uint(b)) break;
    }
    // frames 0 .. t-1 differ at this pixel (t = n: never converged)
    atomicMax(k_out, t < n_frames ? t : n_frames);
  }
}

}  // namespace fcshard

using namespace fcshard;

extern "C" int fc_iir_converge(const fc_stage* sgray, const fc_stage* si, const void* video,
                               int in_type, int gray_in, fc_dims d, const float* s_true,
                               const float* s_warm, int* k_dev, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (cudaMemsetAsync(k_dev, 0, sizeof(int), st) != cudaSuccess) return int(cudaGetLastError());
  const long long hw = (long long)d.width * d.height;
  if (hw == 0 || d.frames == 0) return 0;
  const float beta = 1.0f - si->alpha;  // host float arithmetic == the reference's
  fc_stage g = {};
  if (sgray) g = *sgray;
  const int grid = int((hw + 255) / 256 < 148 * 8 ? (hw + 255) / 256 : 148 * 8);
  if (in_type == FC_U8) {
    if (gray_in)
      k_iir_converge<uint8_t, true><<<grid, 256, 0, st>>>(
          static_cast<const uint8_t*>(video), g, si->alpha, beta, hw, d.frames, s_true, s_warm,
          k_dev);
    else
      k_iir_converge<uint8_t, false><<<grid, 256, 0, st>>>(
          static_cast<const uint8_t*>(video), g, si->alpha, beta, hw, d.frames, s_true, s_warm,
          k_dev);
  } else {
    if (gray_in)
      k_iir_converge<float, true><<<grid, 256, 0, st>>>(static_cast<const float*>(video), g,
                                                        si->alpha, beta, hw, d.frames, s_true,
                                                        s_warm, k_dev);
    else
      k_iir_converge<float, false><<<grid, 256, 0, st>>>(static_cast<const float*>(video), g,
                                                         si->alpha, beta, hw, d.frames, s_true,
                                                         s_warm, k_dev);
  }
  return int(cudaGetLastError());
}
