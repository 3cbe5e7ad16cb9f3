// Dependent-chain latency of FFMA, FFMA2, SHFL, LDS (one warp).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(float* out, long long* cyc, int iters) {
  __shared__ float sm[1024];
  sm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  float a = threadIdx.x * 1e-3f; float2 b = make_float2(a, a + 1);
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) a = __fmaf_rn(a, 0.999f, 1e-3f);
  long long t1 = clock64();
  for (int i = 0; i < iters; ++i) b = __ffma2_rn(b, make_float2(0.999f, 0.999f), make_float2(1e-3f, 1e-3f));
  long long t2 = clock64();
  float c = a;
  for (int i = 0; i < iters; ++i) c = __shfl_down_sync(0xffffffffu, c, 1) + 0.0f;
  long long t3 = clock64();
  int idx = threadIdx.x;
  for (int i = 0; i < iters; ++i) idx = (int)sm[idx & 1023];
  long long t4 = clock64();
  out[threadIdx.x] = a + b.x + b.y + c + idx;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 4096); cudaMalloc(&cyc, 64);
  int iters = 4096;
  k<<<1, 32>>>(out, cyc, iters); cudaDeviceSynchronize(); k<<<1, 32>>>(out, cyc, iters);
  long long c[4]; cudaMemcpy(c, cyc, 32, cudaMemcpyDeviceToHost);
  printf("latency cycles: FFMA %.2f  FFMA2 %.2f  SHFL(+FADD) %.2f  LDS(+cvt) %.2f\n", c[0] / (double)iters,
         c[1] / (double)iters, c[2] / (double)iters, c[3] / (double)iters);
}
