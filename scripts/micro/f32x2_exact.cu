#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ uint32_t hsh(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }
__device__ float rf(uint32_t s) { return (hsh(s) & 0xFFFFFF) * (1.0f / 65536.0f) - 128.0f; }
__global__ void k(unsigned long long* bad) {
  unsigned long long b0 = 0, b1 = 0, b2 = 0, b3 = 0;
  for (int it = 0; it < 256; ++it) {
    uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) * 256 + it;
    float a = rf(6 * i), b = rf(6 * i + 1), c = rf(6 * i + 2), d = rf(6 * i + 3), e = rf(6 * i + 4), f = rf(6 * i + 5);
    float2 x = make_float2(a, b), y = make_float2(c, d), z = make_float2(e, f);
    float2 r = __fadd2_rn(x, y);
    if (r.x != __fadd_rn(a, c) || r.y != __fadd_rn(b, d)) ++b0;
    r = __fmul2_rn(x, y);
    if (r.x != __fmul_rn(a, c) || r.y != __fmul_rn(b, d)) ++b1;
    r = __ffma2_rn(x, y, z);
    if (r.x != __fmaf_rn(a, c, e) || r.y != __fmaf_rn(b, d, f)) ++b2;
    r = __fadd2_rn(__fmul2_rn(x, x), __fmul2_rn(y, y));
    if (r.x != __fadd_rn(__fmul_rn(a, a), __fmul_rn(c, c)) || r.y != __fadd_rn(__fmul_rn(b, b), __fmul_rn(d, d))) ++b3;
  }
  atomicAdd(&bad[0], b0); atomicAdd(&bad[1], b1); atomicAdd(&bad[2], b2); atomicAdd(&bad[3], b3);
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 32); cudaMemset(d, 0, 32);
  k<<<1184, 256>>>(d);
  unsigned long long h[4]; cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
  printf("fadd2 %llu  fmul2 %llu  ffma2 %llu  mul2+add2 %llu  of %llu\n", h[0], h[1], h[2], h[3], 1184ull * 256 * 256);
}
