// Throughput of FFMA vs FFMA2 (and FADD2) on one SM: independent chains.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float* out, long long* cyc, int iters) {
  float a[16];
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i;
  const float x = 0.999f, y = 1e-3f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = __fmaf_rn(a[i], x, y);
    } else if (MODE == 1) {
#pragma unroll
      for (int i = 0; i < 16; i += 2) {
        float2 v = make_float2(a[i], a[i + 1]);
        v = __ffma2_rn(v, make_float2(x, x), make_float2(y, y));
        a[i] = v.x; a[i + 1] = v.y;
      }
    } else if (MODE == 2) {
#pragma unroll
      for (int i = 0; i < 16; i += 2) {
        float2 v = make_float2(a[i], a[i + 1]);
        v = __fadd2_rn(v, make_float2(y, y));
        a[i] = v.x; a[i + 1] = v.y;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = __fadd_rn(a[i], y);
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* out; long long* cyc;
  cudaMalloc(&out, 1 << 24); cudaMalloc(&cyc, 8 * 1024);
  const char* names[4] = {"FFMA", "FFMA2", "FADD2", "FADD"};
  for (int mode = 0; mode < 4; ++mode)
    for (int warps : {4, 8, 16, 32}) {
      int iters = 4096;
      auto launch = [&]() {
        if (mode == 0) k<0><<<1, warps * 32>>>(out, cyc, iters);
        if (mode == 1) k<1><<<1, warps * 32>>>(out, cyc, iters);
        if (mode == 2) k<2><<<1, warps * 32>>>(out, cyc, iters);
        if (mode == 3) k<3><<<1, warps * 32>>>(out, cyc, iters);
      };
      launch(); cudaDeviceSynchronize(); launch();
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      const double insts = double(iters) * (mode == 1 || mode == 2 ? 8 : 16) * warps;  // warp-instr
      const double lane_ops = insts * 32 * (mode == 1 || mode == 2 ? 2 : 1);
      printf("%-6s warps %2d: %.3f warp-instr/clk/SM  %.1f lane-ops/clk/SM\n", names[mode], warps,
             insts / c, lane_ops / c);
    }
  return 0;
}
