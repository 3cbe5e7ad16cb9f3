// The reference's float Sobel magnitude term (simulator.cpp:75-83) for four
// adjacent columns, on column pairs in packed f32x2 ops (sm_100): each lane
// of a pair is rounded exactly as the reference's scalar op, because
// a + 2 b == FMA(2, b, a) and a - b == FMA(-1, b, a) (2 b and -b are exact);
// no packed multiply feeds a packed add (ptxas would contract the pair).
//   S_i  = (rm_i + 2 rc_i) + rp_i              gx_j = S_{j+2} - S_j
//   T_j(r) = (r_j + 2 r_{j+1}) + r_{j+2}       gy_j = T_j(rp) - T_j(rm)
//   m_j  = gx_j * gx_j + gy_j * gy_j
// rm / rc / rp: the rows above / at / below, columns x-1 .. x+4 (clamped by
// the caller); m[j] for output column x + j.
#pragma once
#include <cuda_runtime.h>

__device__ __forceinline__ void sobel_m4(const float (&rm)[6], const float (&rc)[6],
                                         const float (&rp)[6], float (&m)[4]) {
  const float2 two = make_float2(2.0f, 2.0f), neg = make_float2(-1.0f, -1.0f);
  auto p2 = [](float a, float b) { return make_float2(a, b); };
  float2 S[3];
#pragma unroll
  for (int h = 0; h < 3; ++h)
    S[h] = __fadd2_rn(__ffma2_rn(two, p2(rc[2 * h], rc[2 * h + 1]), p2(rm[2 * h], rm[2 * h + 1])),
                      p2(rp[2 * h], rp[2 * h + 1]));
#pragma unroll
  for (int h = 0; h < 2; ++h) {  // outputs 2h, 2h + 1
    const float2 gx = __ffma2_rn(neg, S[h], S[h + 1]);
    const float2 tp = __fadd2_rn(
        __ffma2_rn(two, p2(rp[2 * h + 1], rp[2 * h + 2]), p2(rp[2 * h], rp[2 * h + 1])),
        p2(rp[2 * h + 2], rp[2 * h + 3]));
    const float2 tm = __fadd2_rn(
        __ffma2_rn(two, p2(rm[2 * h + 1], rm[2 * h + 2]), p2(rm[2 * h], rm[2 * h + 1])),
        p2(rm[2 * h + 2], rm[2 * h + 3]));
    const float2 gy = __ffma2_rn(neg, tm, tp);
    // m in scalar .rn ops: ptxas contracts mul.rn.f32x2 + add.rn.f32x2 into
    // FFMA2 despite the .rn (scripts/micro/f32x2_exact.cu: 30 % of random
    // inputs then differ), which would drop the reference's rounding of gx^2
    m[2 * h] = __fadd_rn(__fmul_rn(gx.x, gx.x), __fmul_rn(gy.x, gy.x));
    m[2 * h + 1] = __fadd_rn(__fmul_rn(gx.y, gx.y), __fmul_rn(gy.y, gy.y));
  }
}
