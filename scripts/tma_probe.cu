// Probe: which TMA 3-D tiled loads of a u8 tensor are legal (x alignment, negative x).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
__global__ void k(const __grid_constant__ CUtensorMap map, int x, int y, int z, unsigned bytes, int* out) {
  __shared__ __align__(128) unsigned char buf[16384];
  __shared__ __align__(8) uint64_t bar;
  unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
  unsigned d = (unsigned)__cvta_generic_to_shared(buf);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      :: "r"(d), "l"(&map), "r"(x), "r"(y), "r"(z), "r"(b) : "memory");
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" :: "r"(b) : "memory");
    out[0] = buf[0]; out[1] = buf[1]; out[2] = buf[3];
  }
}
int main(int argc, char** argv) {
  int W = 64, H = 48, F = 4, BW = atoi(argv[1]), BH = atoi(argv[2]), x = atoi(argv[3]), y = atoi(argv[4]);
  unsigned char* v; cudaMalloc(&v, W * H * F * 4);
  unsigned char* h = (unsigned char*)malloc(W*H*F*4); for (int i = 0; i < W*H*F*4; ++i) h[i] = i & 255;
  cudaMemcpy(v, h, W*H*F*4, cudaMemcpyHostToDevice);
  int* out; cudaMallocManaged(&out, 16);
  void* p; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
  CUtensorMap map;
  cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)(4 * F)};
  cuuint64_t strides[2] = {(cuuint64_t)W, (cuuint64_t)W * H};
  cuuint32_t box[3] = {(cuuint32_t)BW, (cuuint32_t)BH, 3};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, v, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  k<<<1, 32>>>(map, x, y, 0, BW * BH * 3, out);
  cudaError_t e = cudaDeviceSynchronize();
  printf("box %dx%d at (%d,%d): encode=%d run=%s out=%d,%d,%d\n", BW, BH, x, y, (int)r, cudaGetErrorString(e), out[0], out[1], out[2]);
  return 0;
}
