// K6: centroid-in-ROI measurement + constant-velocity Kalman tracking
// (reference: proj/src/tracking.cpp:40-128, capi.cpp:366-381) on the device
// mask.  One CTA per marker marches the frames: the ROI of frame t is
// recentred on the Kalman prediction from frame t-1, so frames are serial per
// marker; inside a frame the CTA's threads reduce the ROI (pixel count and
// coordinate sums, exact in 64-bit integers == the reference's double sums of
// integer coordinates), then one thread runs the Kalman predict / update in
// FP64 with explicit round-to-nearest operations (no contraction).
//
// Matrix products follow the textbook order (sum over k ascending, starting
// from the k = 0 product), the 2x2 inverse is the closed form
// 1 / (a d - c b) x [d -b; -c a]; oracle/tracking_oracle.py restates exactly
// this arithmetic (the reference's Eigen build is not available here, so the
// restatement is checked against the reference's own behavioural tests).
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

#include "fc_kernels.h"

namespace fctrack {

constexpr int NT = 128;
constexpr int PTS = 23;  // measured, meas_x, meas_y, est_x, est_y, est_vx, est_vy, cov[16]

struct Params {
  double q, r, p0;
};

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }

// C[m x n] = A[m x k] B[k x n], row-major, sum over k ascending
template <int M, int K, int N>
__device__ __forceinline__ void matmul(const double* A, const double* B, double* C) {
#pragma unroll
  for (int i = 0; i < M; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) {
      double acc = dmul(A[i * K], B[j]);
#pragma unroll
      for (int k = 1; k < K; ++k) acc = dadd(acc, dmul(A[i * K + k], B[k * N + j]));
      C[i * N + j] = acc;
    }
}

template <int M, int N>
__device__ __forceinline__ void transpose(const double* A, double* T) {
#pragma unroll
  for (int i = 0; i < M; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) T[j * M + i] = A[i * N + j];
}

// tracking.cpp:72-75 (recenter): lround, then integer halving of the extent
__device__ __forceinline__ int lround_d(double v) { return int(llround(v)); }

template <typename T>
__device__ __forceinline__ bool is_set(T v);
template <>
__device__ __forceinline__ bool is_set<uint8_t>(uint8_t v) {
  return v > 127;  // float(v) > 127.0f
}
template <>
__device__ __forceinline__ bool is_set<float>(float v) {
  return v > 127.0f;
}

template <typename T>
__global__ void __launch_bounds__(NT) k_track(const T* __restrict__ mask, int W, int H, int F,
                                               const int* __restrict__ rois, Params prm,
                                               double* __restrict__ out) {
  __shared__ long long red_n[NT / 32], red_x[NT / 32], red_y[NT / 32];
  __shared__ int roi_s[6];
  const int m = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // Kalman state lives in thread 0's registers; roi broadcast through smem
  double state[4], cov[16], f[16], q[16];
  int roi[4];
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) roi[i] = rois[4 * m + i];
#pragma unroll
    for (int i = 0; i < 16; ++i) f[i] = (i % 5 == 0) ? 1.0 : 0.0;  // identity
    f[0 * 4 + 2] = 1.0;
    f[1 * 4 + 3] = 1.0;
#pragma unroll
    for (int i = 0; i < 16; ++i) q[i] = 0.0;
#pragma unroll
    for (int axis = 0; axis < 2; ++axis) {  // tracking.cpp:28-38
      const int p = axis, v = axis + 2;
      q[p * 4 + p] = dmul(0.25, prm.q);
      q[p * 4 + v] = dmul(0.5, prm.q);
      q[v * 4 + p] = dmul(0.5, prm.q);
      q[v * 4 + v] = prm.q;
    }
    // tracking.cpp:95-96: state at the ROI centre, cov = p0 I
    state[0] = dadd(double(roi[0]), __ddiv_rn(double(roi[2]), 2.0));
    state[1] = dadd(double(roi[1]), __ddiv_rn(double(roi[3]), 2.0));
    state[2] = 0.0;
    state[3] = 0.0;
#pragma unroll
    for (int i = 0; i < 16; ++i) cov[i] = (i % 5 == 0) ? prm.p0 : 0.0;
  }
  for (int t = 0; t < F; ++t) {
    if (tid == 0) {
      if (t > 0) {  // predict: state = F state; cov = F cov F^T + Q
        double ns[4], fc[16], ft[16], fcf[16];
        matmul<4, 4, 1>(f, state, ns);
#pragma unroll
        for (int i = 0; i < 4; ++i) state[i] = ns[i];
        matmul<4, 4, 4>(f, cov, fc);
        transpose<4, 4>(f, ft);
        matmul<4, 4, 4>(fc, ft, fcf);
#pragma unroll
        for (int i = 0; i < 16; ++i) cov[i] = dadd(fcf[i], q[i]);
      }
      roi[0] = lround_d(state[0]) - roi[2] / 2;
      roi[1] = lround_d(state[1]) - roi[3] / 2;
#pragma unroll
      for (int i = 0; i < 4; ++i) roi_s[i] = roi[i];
      // the next frame's ROI, assuming the update moves the prediction by
      // < 2 px: warm L2 with a 2-px margin while this frame is reduced
      if (t + 1 < F) {
        const int gx = lround_d(dadd(state[0], state[2])) - roi[2] / 2 - 2;
        const int gy = lround_d(dadd(state[1], state[3])) - roi[3] / 2 - 2;
        roi_s[4] = gx, roi_s[5] = gy;
      } else {
        roi_s[4] = roi_s[5] = INT_MIN;
      }
    }
    __syncthreads();
    if (roi_s[4] != INT_MIN) {  // one prefetch per row of the guessed window
      const int gy = roi_s[5] + tid, gx = max(roi_s[4], 0);
      if (tid < roi_s[3] + 4 && gy >= 0 && gy < H && gx < W)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(mask + ((long long)(t + 1) * H + gy) * W +
                                                        gx));
    }
    // centroid over the clipped ROI (tracking.cpp:54-70)
    const int x0 = max(roi_s[0], 0), y0 = max(roi_s[1], 0);
    const int x1 = min(roi_s[0] + roi_s[2], W), y1 = min(roi_s[1] + roi_s[3], H);
    long long n = 0, sx = 0, sy = 0;
    const int rw = max(x1 - x0, 0), rh = max(y1 - y0, 0);
    const T* fr = mask + (long long)t * W * H;
    for (int i = tid; i < rw * rh; i += NT) {
      const int y = y0 + i / rw, x = x0 + i % rw;
      if (is_set<T>(fr[(long long)y * W + x])) {
        ++n;
        sx += x;
        sy += y;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      n += __shfl_xor_sync(0xffffffffu, n, o);
      sx += __shfl_xor_sync(0xffffffffu, sx, o);
      sy += __shfl_xor_sync(0xffffffffu, sy, o);
    }
    if (lane == 0) red_n[warp] = n, red_x[warp] = sx, red_y[warp] = sy;
    __syncthreads();
    if (tid == 0) {
      n = sx = sy = 0;
      for (int w = 0; w < NT / 32; ++w) n += red_n[w], sx += red_x[w], sy += red_y[w];
      double* pt = out + ((long long)m * F + t) * PTS;
      pt[0] = n > 0 ? 1.0 : 0.0;
      pt[1] = pt[2] = 0.0;
      if (n > 0) {
        const double zx = __ddiv_rn(double(sx), double(n)), zy = __ddiv_rn(double(sy), double(n));
        if (t == 0) {  // tracking.cpp:107-110: initialise the position
          state[0] = zx;
          state[1] = zy;
        } else {
          // S = H cov H^T + R (the leading 2x2 of cov plus r I)
          double s[4] = {dadd(cov[0], prm.r), dadd(cov[1], 0.0), dadd(cov[4], 0.0),
                         dadd(cov[5], prm.r)};
          const double det = dsub(dmul(s[0], s[3]), dmul(s[2], s[1]));
          const double inv = __ddiv_rn(1.0, det);
          const double si[4] = {dmul(s[3], inv), dmul(-s[1], inv), dmul(-s[2], inv),
                                dmul(s[0], inv)};
          // K = (cov H^T) S^-1, cov H^T = the first two columns of cov
          double ch[8], k[8];
          for (int i = 0; i < 4; ++i) ch[2 * i] = cov[4 * i], ch[2 * i + 1] = cov[4 * i + 1];
          matmul<4, 2, 2>(ch, si, k);
          // state += K (z - H state)
          const double y[2] = {dsub(zx, state[0]), dsub(zy, state[1])};
          double ky[4];
          matmul<4, 2, 1>(k, y, ky);
          for (int i = 0; i < 4; ++i) state[i] = dadd(state[i], ky[i]);
          // cov = (I - K H) cov
          double ikh[16], nc[16];
          for (int i = 0; i < 4; ++i)
            for (int j = 0; j < 4; ++j) {
              const double kh = j < 2 ? k[2 * i + j] : 0.0;
              ikh[4 * i + j] = dsub(i == j ? 1.0 : 0.0, kh);
            }
          matmul<4, 4, 4>(ikh, cov, nc);
          for (int i = 0; i < 16; ++i) cov[i] = nc[i];
        }
        pt[1] = zx;
        pt[2] = zy;
      }
      pt[3] = state[0];
      pt[4] = state[1];
      pt[5] = state[2];
      pt[6] = state[3];
      for (int i = 0; i < 16; ++i) pt[7 + i] = cov[i];
    }
    __syncthreads();
  }
}

}  // namespace fctrack

using namespace fctrack;

extern "C" int fc_track_features(const void* mask, int elem_type, int W, int H, int F,
                                 const int* rois_dev, int n_rois, double q, double r,
                                 double p0, double* points_dev, void* stream) {
  if (n_rois <= 0 || F <= 0) return 0;
  Params prm{q, r, p0};
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (elem_type == FC_U8)
    k_track<uint8_t><<<n_rois, NT, 0, st>>>(static_cast<const uint8_t*>(mask), W, H, F,
                                            rois_dev, prm, points_dev);
  else
    k_track<float><<<n_rois, NT, 0, st>>>(static_cast<const float*>(mask), W, H, F, rois_dev,
                                          prm, points_dev);
  return int(cudaGetLastError());
}
