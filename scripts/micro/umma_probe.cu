// tcgen05 probe (sm_100a): (1) SWIZZLE_NONE smem descriptor layouts for
// K-major / MN-major f16 operands, checked against a host GEMM; (2) issue
// throughput of M=128 x N x K=16 MMAs for small N (the banded stencil GEMMs
// of fc_tc.cu use N = 16..64).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_probe umma_probe.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e = (x);                                                           \
    if (e != cudaSuccess) {                                                        \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      std::exit(1);                                                                \
    }                                                                              \
  } while (0)

__device__ __forceinline__ unsigned su32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// byte offset of element (mn, k) of a SWIZZLE_NONE canonical layout
__host__ __device__ inline unsigned off_kmaj(int mn, int k, unsigned sbo, unsigned lbo) {
  return (mn / 8) * sbo + (k / 8) * lbo + (mn % 8) * 16 + (k % 8) * 2;
}
__host__ __device__ inline unsigned off_mnmaj(int mn, int k, unsigned sbo, unsigned lbo) {
  return (mn / 8) * sbo + (k / 8) * lbo + (k % 8) * 16 + (mn % 8) * 2;
}

__device__ __forceinline__ uint64_t sdesc(unsigned addr, unsigned lbo, unsigned sbo) {
  uint64_t d = 0;
  d |= uint64_t((addr >> 4) & 0x3FFF);
  d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;  // version (Blackwell)
  return d;                 // base offset 0, SWIZZLE_NONE
}

__host__ __device__ constexpr uint32_t idesc_f16(int M, int N, int amaj, int bmaj) {
  return (1u << 4) /*f32 acc*/ | (0u << 7) /*a f16*/ | (0u << 10) /*b f16*/ |
         (uint32_t(amaj) << 15) | (uint32_t(bmaj) << 16) | (uint32_t(N >> 3) << 17) |
         (uint32_t(M >> 4) << 24);
}

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                        int acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   su32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned ph) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W_%=;\n}\n" ::"r"(su32(bar)),
      "r"(ph)
      : "memory");
}

// A: M=128 x K (f16), B: K x N; layouts: amaj/bmaj 0 = K-major, 1 = MN-major
// D[m][n] = sum_k A[m][k] B[k][n]  (A given as a[m*K+k], B as b[k*N+n])
__global__ void k_gemm(const __half* a, const __half* b, float* d, int K, int N, int amaj,
                       int bmaj, unsigned a_sbo, unsigned a_lbo, unsigned b_sbo, unsigned b_lbo,
                       unsigned a_bytes) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  unsigned char* sa = sm;
  unsigned char* sb = sm + a_bytes;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 128 * K; i += blockDim.x) {
    const int m = i / K, k = i % K;
    const unsigned o = amaj ? off_mnmaj(m, k, a_sbo, a_lbo) : off_kmaj(m, k, a_sbo, a_lbo);
    *reinterpret_cast<__half*>(sa + o) = a[i];
  }
  for (int i = tid; i < K * N; i += blockDim.x) {
    const int k = i / N, n = i % N;
    const unsigned o = bmaj ? off_mnmaj(n, k, b_sbo, b_lbo) : off_kmaj(n, k, b_sbo, b_lbo);
    *reinterpret_cast<__half*>(sb + o) = b[i];
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  if (tid == 0) {
    const uint32_t id = idesc_f16(128, N, amaj, bmaj);
    for (int ks = 0; ks < K / 16; ++ks) {
      // advance by 16 k = 2 core matrices in K
      const unsigned ao = amaj ? off_mnmaj(0, 16 * ks, a_sbo, a_lbo) : off_kmaj(0, 16 * ks, a_sbo, a_lbo);
      const unsigned bo = bmaj ? off_mnmaj(0, 16 * ks, b_sbo, b_lbo) : off_kmaj(0, 16 * ks, b_sbo, b_lbo);
      mma_f16(tm, sdesc(su32(sa) + ao, a_lbo, a_sbo), sdesc(su32(sb) + bo, b_lbo, b_sbo), id, ks > 0);
    }
    commit(&bar);
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp < 4) {
    for (int c = 0; c < N; c += 16) {
      uint32_t r[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
            "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
            "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
          : "r"(tm + ((32u * warp) << 16) + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      const int m = 32 * warp + lane;
      for (int j = 0; j < 16; ++j) d[m * N + c + j] = __uint_as_float(r[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
}

// throughput: one thread issues `iters` batches of 8 MMAs (M x N x 16);
// amaj selects the A layout; acc chains into 4 accumulators round robin
template <int M, int N, int AMAJ>
__global__ void k_rate(int iters, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  if (tid == 0) {
    constexpr uint32_t id = idesc_f16(M, N, AMAJ, 0);
    // A: M x 16 -> K-major: lbo 128 (k chunks), sbo 256 (8-row groups);
    //    MN-major: sbo 128 (8-col groups), lbo M/8*128 (k chunks)
    const uint64_t da = AMAJ ? sdesc(su32(sm), (M / 8) * 128, 128) : sdesc(su32(sm), 128, 256);
    const uint64_t db = sdesc(su32(sm) + 32768, 128, 256);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int j = 0; j < 8; ++j) mma_f16(tm + (j & 3) * N, da, db, id, 1);
    }
    commit(&bar);
    mbar_wait(&bar, 0);
    cyc[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int M, int N, int AMAJ>
void rate(long long* dc) {
  CK(cudaFuncSetAttribute(k_rate<M, N, AMAJ>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
  const int iters = 512;
  k_rate<M, N, AMAJ><<<1, 128, 64 * 1024>>>(iters, dc);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  long long h;
  CK(cudaMemcpy(&h, dc, sizeof h, cudaMemcpyDeviceToHost));
  const double n = 8.0 * iters;
  std::printf("rate M=%d N=%3d amaj=%d: %.1f cycles/MMA, %.0f MAC/clk/SM\n", M, N, AMAJ,
              double(h) / n, double(M) * N * 16 * n / double(h));
}

int main() {
  int fails = 0;
  for (int N : {16, 32, 64}) {
    const int K = 48;
    std::vector<__half> ha(128 * K), hb(K * N);
    std::vector<float> fa(128 * K), fb(K * N);
    for (int i = 0; i < 128 * K; ++i) {
      fa[i] = float((i * 37 + 11) % 23) - 11.0f;
      ha[i] = __float2half(fa[i]);
    }
    for (int i = 0; i < K * N; ++i) {
      fb[i] = float((i * 53 + 5) % 17) - 8.0f;
      hb[i] = __float2half(fb[i]);
    }
    std::vector<double> ref(128 * N, 0.0);
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < N; ++n)
        for (int k = 0; k < K; ++k) ref[m * N + n] += double(fa[m * K + k]) * fb[k * N + n];
    __half *da, *db;
    float* dd;
    CK(cudaMalloc(&da, ha.size() * 2));
    CK(cudaMalloc(&db, hb.size() * 2));
    CK(cudaMalloc(&dd, 128 * N * 4));
    CK(cudaMemcpy(da, ha.data(), ha.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(db, hb.data(), hb.size() * 2, cudaMemcpyHostToDevice));
    for (int amaj = 0; amaj < 2; ++amaj)
      for (int bmaj = 0; bmaj < 2; ++bmaj) {
        // A: 128 rows (16 groups of 8) x K (K/8 chunks): K-major: core matrices
        // along K contiguous (lbo = 128), mn groups at sbo = K/8 * 128;
        // MN-major: mn groups contiguous (sbo = 128), k groups at lbo = 16 * 128
        unsigned a_sbo, a_lbo, b_sbo, b_lbo;
        if (amaj == 0) { a_lbo = 128; a_sbo = (K / 8) * 128; }
        else { a_sbo = 128; a_lbo = 16 * 128; }
        if (bmaj == 0) { b_lbo = 128; b_sbo = (K / 8) * 128; }
        else { b_sbo = 128; b_lbo = (N / 8) * 128; }
        const unsigned a_bytes = 128 * K * 2;
        CK(cudaMemset(dd, 0, 128 * N * 4));
        CK(cudaFuncSetAttribute(k_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
        k_gemm<<<1, 128, 64 * 1024>>>(da, db, dd, K, N, amaj, bmaj, a_sbo, a_lbo, b_sbo, b_lbo,
                                      a_bytes);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        std::vector<float> hd(128 * N);
        CK(cudaMemcpy(hd.data(), dd, hd.size() * 4, cudaMemcpyDeviceToHost));
        int bad = 0;
        double maxe = 0;
        for (int i = 0; i < 128 * N; ++i) {
          maxe = std::max(maxe, std::fabs(hd[i] - ref[i]));
          if (hd[i] != float(ref[i])) ++bad;
        }
        std::printf("gemm N=%d amaj=%d bmaj=%d: mismatches %d / %d (max err %g) d[0]=%g ref %g\n",
                    N, amaj, bmaj, bad, 128 * N, maxe, hd[0], ref[0]);
        fails += bad != 0;
      }
    cudaFree(da);
    cudaFree(db);
    cudaFree(dd);
  }
  long long* dc;
  CK(cudaMalloc(&dc, 148 * sizeof(long long)));
  rate<128, 16, 0>(dc); rate<128, 16, 1>(dc);
  rate<128, 32, 0>(dc); rate<128, 32, 1>(dc);
  rate<128, 64, 0>(dc); rate<128, 64, 1>(dc);
  rate<128, 128, 0>(dc); rate<128, 128, 1>(dc);
  rate<128, 256, 0>(dc); rate<128, 256, 1>(dc);
  rate<64, 32, 0>(dc); rate<64, 64, 0>(dc); rate<64, 128, 0>(dc); rate<64, 256, 0>(dc);
  std::printf("%s\n", fails ? "LAYOUT FAILURES" : "all layouts ok");
  return 0;
}
