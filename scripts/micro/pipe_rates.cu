// Issue / pipe throughput of the instruction forms the frame pipeline uses
// (B200, one CTA per SM, 16 independent chains per thread).  Prints warp
// instructions and lane operations per clock per SM for each form.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CH 16

template <int OP>
__device__ __forceinline__ void step(float* a, uint32_t* u, float x, float y, uint32_t s) {
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    if (OP == 0) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(x), "f"(y));
    if (OP == 1) asm volatile("fma.rn.f32 %0, %0, 0f3F7FBE77, %1;" : "+f"(a[i]) : "f"(y));
    if (OP == 2) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(y));
    if (OP == 3) asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(x));
    if (OP == 4) asm volatile("add.rn.f32 %0, %0, 0f3A83126F;" : "+f"(a[i]));
    if (OP == 5 && (i & 1) == 0) {
      asm volatile(
          "{.reg .b64 p, q, r;\n mov.b64 p, {%0, %1};\n mov.b64 q, {%2, %2};\n mov.b64 r, {%3, %3};\n"
          " fma.rn.f32x2 p, p, q, r;\n mov.b64 {%0, %1}, p;}"
          : "+f"(a[i]), "+f"(a[i + 1])
          : "f"(x), "f"(y));
    }
    if (OP == 6 && (i & 1) == 0) {
      asm volatile(
          "{.reg .b64 p, r;\n mov.b64 p, {%0, %1};\n mov.b64 r, {%2, %2};\n"
          " add.rn.f32x2 p, p, r;\n mov.b64 {%0, %1}, p;}"
          : "+f"(a[i]), "+f"(a[i + 1])
          : "f"(y));
    }
    if (OP == 7 && (i & 1) == 0) {  // f32x2 with both operands distinct pairs
      asm volatile(
          "{.reg .b64 p, q, r;\n mov.b64 p, {%0, %1};\n mov.b64 q, {%1, %0};\n mov.b64 r, {%2, %3};\n"
          " fma.rn.f32x2 p, p, r, q;\n mov.b64 {%0, %1}, p;}"
          : "+f"(a[i]), "+f"(a[i + 1])
          : "f"(x), "f"(y));
    }
    if (OP == 8) asm volatile("prmt.b32 %0, %0, %1, 0x7440;" : "+r"(u[i]) : "r"(s));
    if (OP == 9) asm volatile("add.u32 %0, %0, %1;" : "+r"(u[i]) : "r"(s));
    if (OP == 10) asm volatile("lop3.b32 %0, %0, %1, 0x5A, 0x96;" : "+r"(u[i]) : "r"(s));
    if (OP == 11) asm volatile("min.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(x));
    if (OP == 12) asm volatile("shfl.sync.down.b32 %0, %0, 1, 31, -1;" : "+f"(a[i]));
    if (OP == 13) {  // FFMA-imm + PRMT interleaved
      asm volatile("fma.rn.f32 %0, %0, 0f3F7FBE77, %1;" : "+f"(a[i]) : "f"(y));
      asm volatile("prmt.b32 %0, %0, %1, 0x7440;" : "+r"(u[i]) : "r"(s));
    }
    if (OP == 14 && (i & 1) == 0) {  // FFMA2 + 2 PRMT
      asm volatile(
          "{.reg .b64 p, q, r;\n mov.b64 p, {%0, %1};\n mov.b64 q, {%2, %2};\n mov.b64 r, {%3, %3};\n"
          " fma.rn.f32x2 p, p, q, r;\n mov.b64 {%0, %1}, p;}"
          : "+f"(a[i]), "+f"(a[i + 1])
          : "f"(x), "f"(y));
      asm volatile("prmt.b32 %0, %0, %1, 0x7440;" : "+r"(u[i]) : "r"(s));
      asm volatile("prmt.b32 %0, %0, %1, 0x7440;" : "+r"(u[i + 1]) : "r"(s));
    }
    if (OP == 15) {  // FFMA RRR + FFMA imm interleaved
      if (i & 1)
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(x), "f"(y));
      else
        asm volatile("fma.rn.f32 %0, %0, 0f3F7FBE77, %1;" : "+f"(a[i]) : "f"(y));
    }
    if (OP == 16) asm volatile("ld.shared.f32 %0, [%1];" : "=f"(a[i]) : "r"(s + 4 * i));
    if (OP == 17 && (i & 3) == 0)
      asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                   : "=f"(a[i]), "=f"(a[i + 1]), "=f"(a[i + 2]), "=f"(a[i + 3])
                   : "r"(s + 16 * i));
    if (OP == 18) asm volatile("fma.rn.f32 %0, %0, %0, %1;" : "+f"(a[i]) : "f"(y));  // RRR, 2 distinct
    if (OP == 19) asm volatile("sub.f32 %0, %1, %0;" : "+f"(a[i]) : "f"(x));
    if (OP == 20 && (i & 1) == 0)  // DFMA on a register pair
      asm volatile(
          "{.reg .f64 p, q;\n mov.b64 p, {%0, %1};\n mov.b64 q, {%2, %3};\n"
          " fma.rn.f64 p, p, q, q;\n mov.b64 {%0, %1}, p;}"
          : "+f"(a[i]), "+f"(a[i + 1])
          : "f"(x), "f"(y));
    if (OP == 21 && (i & 3) == 0) {  // 2 FFMA2 + 1 DFMA interleaved
      asm volatile(
          "{.reg .b64 p, q, r;\n mov.b64 p, {%0, %1};\n mov.b64 q, {%2, %2};\n mov.b64 r, {%3, %3};\n"
          " fma.rn.f32x2 p, p, q, r;\n mov.b64 {%0, %1}, p;}"
          : "+f"(a[i]), "+f"(a[i + 1])
          : "f"(x), "f"(y));
      asm volatile(
          "{.reg .f64 p, q;\n mov.b64 p, {%0, %1};\n mov.b64 q, {%2, %3};\n"
          " fma.rn.f64 p, p, q, q;\n mov.b64 {%0, %1}, p;}"
          : "+f"(a[i + 2]), "+f"(a[i + 3])
          : "f"(x), "f"(y));
    }
    if (OP == 22 && (i & 1) == 0)  // cvt.f64.f32
      asm volatile("{.reg .f64 p;\n cvt.f64.f32 p, %0;\n mov.b64 {%0, %1}, p;}"
                   : "+f"(a[i]), "+f"(a[i + 1]));
    if (OP == 23 && (i & 1) == 0)  // cvt.rn.f32.f64
      asm volatile("{.reg .f64 p;\n mov.b64 p, {%0, %1};\n cvt.rn.f32.f64 %0, p;}"
                   : "+f"(a[i]), "+f"(a[i + 1]));
    if (OP == 24)  // HFMA2 (two halves per lane)
      asm volatile("fma.rn.f16x2 %0, %0, %1, %1;" : "+r"(u[i]) : "r"(s));
    if (OP == 25 && (i & 1) == 0) {  // FFMA2 + FMNMX3 (alu) interleaved
      asm volatile(
          "{.reg .b64 p, q, r;\n mov.b64 p, {%0, %1};\n mov.b64 q, {%2, %2};\n mov.b64 r, {%3, %3};\n"
          " fma.rn.f32x2 p, p, q, r;\n mov.b64 {%0, %1}, p;}"
          : "+f"(a[i]), "+f"(a[i + 1])
          : "f"(x), "f"(y));
      asm volatile("min.f32 %0, %0, %1, %2;" : "+r"(u[i]) : "r"(s), "r"(u[i + 1]));
    }
    if (OP == 26 && (i & 1) == 0) {  // FFMA2 + LDS.64
      asm volatile(
          "{.reg .b64 p, q, r;\n mov.b64 p, {%0, %1};\n mov.b64 q, {%2, %2};\n mov.b64 r, {%3, %3};\n"
          " fma.rn.f32x2 p, p, q, r;\n mov.b64 {%0, %1}, p;}"
          : "+f"(a[i]), "+f"(a[i + 1])
          : "f"(x), "f"(y));
      asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(u[i]), "=r"(u[i + 1]) : "r"(s + 8 * i));
    }
    if (OP == 28) asm volatile("cvt.rn.f32.u32 %0, %1;" : "=f"(a[i]) : "r"(u[i] ^ s));  // I2FP (+LOP)
    if (OP == 29) {  // I2F.U8 from the low byte
      asm volatile("{.reg .u16 h;\n cvt.u16.u32 h, %1;\n cvt.rn.f32.u8 %0, h;}" : "=f"(a[i]) : "r"(u[i]));
      u[i] += 1;
    }
    if (OP == 30) asm volatile("shr.b32 %0, %0, 1;" : "+r"(u[i]));
    if (OP == 31) asm volatile("{.reg .pred p;\n setp.ne.u32 p, %2, 0;\n selp.f32 %0, %0, %1, p;}" : "+f"(a[i]) : "f"(x), "r"(s));
    if (OP == 32) asm volatile("min.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(x), "f"(y));
    if (OP == 33) asm volatile("mad.lo.u32 %0, %0, %1, %1;" : "+r"(u[i]) : "r"(s));
    if (OP == 34) {  // HADD2.F32: half -> float
      asm volatile("{.reg .f16 h;\n mov.b32 {h, _}, %1;\n cvt.f32.f16 %0, h;}" : "=f"(a[i]) : "r"(u[i]));
      u[i] += 1;
    }
    if (OP == 35 && (i & 1) == 0) {  // FFMA2 + FSEL
      asm volatile(
          "{.reg .b64 p, q, r;\n mov.b64 p, {%0, %1};\n mov.b64 q, {%2, %2};\n mov.b64 r, {%3, %3};\n"
          " fma.rn.f32x2 p, p, q, r;\n mov.b64 {%0, %1}, p;}"
          : "+f"(a[i]), "+f"(a[i + 1])
          : "f"(x), "f"(y));
      asm volatile("{.reg .pred p;\n setp.ne.u32 p, %1, 0;\n selp.b32 %0, %0, %1, p;}" : "+r"(u[i]) : "r"(s));
    }
    if (OP == 36) asm volatile("add.u32 %0, %0, %1;\n add.u32 %0, %0, %2;" : "+r"(u[i]) : "r"(s), "r"(u[(i + 1) % CH]));  // IADD3
    if (OP == 37) asm volatile("shf.r.wrap.b32 %0, %0, %1, 8;" : "+r"(u[i]) : "r"(s));  // funnel shift
    if (OP == 38) {  // mixed f16 x f16 + f32 (sm_100 FFMA with f16 sources)
      asm volatile("{.reg .f16 h;\n mov.b32 {h, _}, %1;\n fma.rn.f32.f16 %0, h, h, %0;}" : "+f"(a[i]) : "r"(s));
    }
    if ((OP == 39 || OP == 40) && (i & 7) == 0) {  // 3 DFMA + 1 F2F (f32 -> f64 / f64 -> f32)
#pragma unroll
      for (int k = 0; k < 6; k += 2)
        asm volatile(
            "{.reg .f64 p, q;\n mov.b64 p, {%0, %1};\n mov.b64 q, {%2, %3};\n"
            " fma.rn.f64 p, p, q, q;\n mov.b64 {%0, %1}, p;}"
            : "+f"(a[i + k]), "+f"(a[i + k + 1])
            : "f"(x), "f"(y));
      if (OP == 39)
        asm volatile("{.reg .f64 p;\n cvt.f64.f32 p, %0;\n mov.b64 {%0, %1}, p;}"
                     : "+f"(a[i + 6]), "+f"(a[i + 7]));
      else
        asm volatile("{.reg .f64 p;\n mov.b64 p, {%0, %1};\n cvt.rn.f32.f64 %0, p;}"
                     : "+f"(a[i + 6]), "+f"(a[i + 7]));
    }
    if (OP == 41 && (i & 1) == 0) {  // DFMA + IADD interleaved
      asm volatile(
          "{.reg .f64 p, q;\n mov.b64 p, {%0, %1};\n mov.b64 q, {%2, %3};\n"
          " fma.rn.f64 p, p, q, q;\n mov.b64 {%0, %1}, p;}"
          : "+f"(a[i]), "+f"(a[i + 1])
          : "f"(x), "f"(y));
      asm volatile("add.u32 %0, %0, %1;" : "+r"(u[i]) : "r"(s));
    }
    if (OP == 27 && (i & 1) == 0) {  // FFMA2 + SHFL
      asm volatile(
          "{.reg .b64 p, q, r;\n mov.b64 p, {%0, %1};\n mov.b64 q, {%2, %2};\n mov.b64 r, {%3, %3};\n"
          " fma.rn.f32x2 p, p, q, r;\n mov.b64 {%0, %1}, p;}"
          : "+f"(a[i]), "+f"(a[i + 1])
          : "f"(x), "f"(y));
      asm volatile("shfl.sync.down.b32 %0, %0, 1, 31, -1;" : "+r"(u[i]));
    }
  }
}

template <int OP>
__global__ void k(float* out, long long* cyc, int iters, float px, float py, uint32_t ps) {
  __shared__ float sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i;
  float a[CH];
  uint32_t u[CH];
  const float x = px + threadIdx.x * 1e-9f, y = py * (1.0f + threadIdx.x * 1e-9f);
  uint32_t s = ps ^ threadIdx.x;
  if (OP == 16 || OP == 17 || OP == 26) s = (unsigned)__cvta_generic_to_shared(sm) + 16 * (threadIdx.x & 31) * 0;
  for (int i = 0; i < CH; ++i) {
    a[i] = threadIdx.x * 1e-3f + i;
    u[i] = threadIdx.x * 77 + i;
  }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) step<OP>(a, u, x, y, s);
  __syncthreads();
  long long t1 = clock64();
  float acc = 0;
  for (int i = 0; i < CH; ++i) acc += a[i] + __uint_as_float(u[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, double instr_per_step, double lanes_per_instr, float* out, long long* cyc) {
  for (int warps : {4, 8, 12, 16, 32}) {
    const int iters = 2048;
    k<OP><<<148, warps * 32>>>(out, cyc, iters, 0.999f, 1e-3f, 0x4B000000u);
    k<OP><<<148, warps * 32>>>(out, cyc, iters, 0.999f, 1e-3f, 0x4B000000u);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
    long long c[148];
    cudaMemcpy(c, cyc, sizeof c, cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < 148; ++i) mx = c[i] > mx ? c[i] : mx;
    const double winstr = double(iters) * instr_per_step * warps;
    printf("%-22s warps %2d: %.3f warp-instr/clk/SM  %6.1f lane-ops/clk/SM\n", name, warps,
           winstr / mx, winstr * 32 * lanes_per_instr / mx);
  }
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  run<0>("FFMA RRR", CH, 1, out, cyc);
  run<18>("FFMA R,R,R(a*a+y)", CH, 1, out, cyc);
  run<1>("FFMA R,imm,R", CH, 1, out, cyc);
  run<2>("FADD RR", CH, 1, out, cyc);
  run<19>("FADD R-R (sub)", CH, 1, out, cyc);
  run<3>("FMUL RR", CH, 1, out, cyc);
  run<4>("FADD R,imm", CH, 1, out, cyc);
  run<5>("FFMA2 splat RRR", CH / 2, 2, out, cyc);
  run<7>("FFMA2 pairs RRR", CH / 2, 2, out, cyc);
  run<6>("FADD2 splat", CH / 2, 2, out, cyc);
  run<8>("PRMT", CH, 1, out, cyc);
  run<9>("IADD", CH, 1, out, cyc);
  run<10>("LOP3", CH, 1, out, cyc);
  run<11>("FMNMX", CH, 1, out, cyc);
  run<12>("SHFL", CH, 1, out, cyc);
  run<13>("FFMAimm+PRMT", 2 * CH, 1, out, cyc);
  run<14>("FFMA2+2PRMT", CH / 2 * 3, 1, out, cyc);
  run<15>("FFMA RRR+imm", CH, 1, out, cyc);
  run<16>("LDS.32", CH, 1, out, cyc);
  run<17>("LDS.128", CH / 4, 4, out, cyc);
  run<20>("DFMA", CH / 2, 1, out, cyc);
  run<21>("2 FFMA2 + DFMA", CH / 4 * 3, 1, out, cyc);
  run<22>("F2F.F64.F32", CH / 2, 1, out, cyc);
  run<23>("F2F.F32.F64", CH / 2, 1, out, cyc);
  run<24>("HFMA2", CH, 2, out, cyc);
  run<25>("FFMA2 + FMNMX3", CH, 1, out, cyc);
  run<26>("FFMA2 + LDS.64", CH, 1, out, cyc);
  run<27>("FFMA2 + SHFL", CH, 1, out, cyc);
  run<28>("I2FP.F32.U32", CH, 1, out, cyc);
  run<29>("I2F.U8", CH, 1, out, cyc);
  run<30>("SHF.R", CH, 1, out, cyc);
  run<31>("FSEL", CH, 1, out, cyc);
  run<32>("FMNMX3", CH, 1, out, cyc);
  run<33>("IMAD", CH, 1, out, cyc);
  run<34>("HADD2.F32 (f16->f32)", CH, 1, out, cyc);
  run<35>("FFMA2 + SEL", CH, 1, out, cyc);
  run<36>("IADD3 (2 adds)", CH, 1, out, cyc);
  run<37>("SHF funnel", CH, 1, out, cyc);
  run<38>("FFMA f32.f16", CH, 1, out, cyc);
  run<39>("3 DFMA + F2F.F64.F32", CH / 2, 1, out, cyc);
  run<40>("3 DFMA + F2F.F32.F64", CH / 2, 1, out, cyc);
  run<41>("DFMA + IADD", CH, 1, out, cyc);
  return 0;
}
