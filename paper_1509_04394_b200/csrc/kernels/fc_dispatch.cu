// Variant dispatch for the streaming all-fused chain (F12345).
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>

#include "fc_kernels.h"

#define FC_CHAIN_ARGS                                                          \
  const fc_stage *sgray, const fc_stage *si, const fc_stage *sg,               \
      const fc_stage *sthr, const void *video, int in_type, int gray_in,       \
      void *out, int out_type, fc_dims d, int n_warm, const float *state_in,   \
      float *state_out, void *stream

extern "C" int fc_chain_exact(FC_CHAIN_ARGS);  // fc_exact.cu: FP64 everywhere
extern "C" int fc_chain_pipe(FC_CHAIN_ARGS);   // fc_pipe.cu: certified, headline
extern "C" int fc_chain_pipe63(FC_CHAIN_ARGS); // fc_pipe_cfg63.cu: role-count variant
extern "C" int fc_chain_strip(FC_CHAIN_ARGS);  // fc_strip.cu: certified, strip march
extern "C" int fc_chain_tile(FC_CHAIN_ARGS);   // fc_fast.cu: certified, tile march
extern "C" int fc_f345_pipe(const fc_stage* sg, const fc_stage* sthr, const float* in,
                            void* out, int out_type, fc_dims d, double in_max, void* stream);
extern "C" int fc_f345_pipe63(const fc_stage* sg, const fc_stage* sthr, const float* in,
                              void* out, int out_type, fc_dims d, double in_max, void* stream);
extern "C" long long fc_strip_recheck_count(void);
extern "C" long long fc_pipe_recheck_count(void);
extern "C" long long fc_pipe63_recheck_count(void);
extern "C" long long fc_tile_recheck_count(void);

// variant: 0 auto (certified kernel when covered, else exact), 1 exact,
//          2 fast (certified kernel or -1), 3 fast_tile (tile kernel or -1).
// The certified kernel of 0 / 2 is the frame pipeline (fc_pipe.cu);
// FUSEPLAN_FAST_KERNEL=strip selects the strip march (comparison runs).
extern "C" int fc_fused_chain(const fc_stage* sgray, const fc_stage* si,
                              const fc_stage* sg, const fc_stage* sgrad,
                              const fc_stage* sthr, const void* video,
                              int in_type, int gray_in, void* out, int out_type,
                              fc_dims d, int n_warm, const float* state_in,
                              float* state_out, int variant, void* stream) {
  (void)sgrad;
  if (variant == 3)
    return fc_chain_tile(sgray, si, sg, sthr, video, in_type, gray_in, out,
                         out_type, d, n_warm, state_in, state_out, stream);
  if (variant == 2 || variant == 0) {
    const char* k = std::getenv("FUSEPLAN_FAST_KERNEL");
    const bool strip = k && std::strcmp(k, "strip") == 0;
    const char* cfg = std::getenv("FUSEPLAN_PIPE_CFG");
    auto* pipe = (cfg && std::strcmp(cfg, "63") == 0) ? fc_chain_pipe63 : fc_chain_pipe;
    int rc = strip ? fc_chain_strip(sgray, si, sg, sthr, video, in_type, gray_in, out,
                                    out_type, d, n_warm, state_in, state_out, stream)
                   : pipe(sgray, si, sg, sthr, video, in_type, gray_in, out, out_type, d,
                          n_warm, state_in, state_out, stream);
    if (rc != -1) return rc;  // -1: parameters not covered
    if (variant == 2)  // frames lower than 6 rows: the certified tile march
      return fc_chain_tile(sgray, si, sg, sthr, video, in_type, gray_in, out, out_type, d,
                           n_warm, state_in, state_out, stream);
  }
  return fc_chain_exact(sgray, si, sg, sthr, video, in_type, gray_in, out,
                        out_type, d, n_warm, state_in, state_out, stream);
}

extern "C" long long fc_last_recheck_count(void) {
  long long a = fc_strip_recheck_count(), b = fc_tile_recheck_count();
  long long c = fc_pipe_recheck_count(), e = fc_pipe63_recheck_count();
  return (a < 0 || b < 0 || c < 0 || e < 0) ? -1 : a + b + c + e;
}

extern "C" int fc_fused_gauss_grad_thr_v(const fc_stage* sg, const fc_stage* sgrad,
                                         const fc_stage* sthr, const float* in, void* out,
                                         int out_type, fc_dims d, int variant, double in_max,
                                         void* stream) {
  if (variant != 1 && in_max > 0.0) {
    const char* cfg = std::getenv("FUSEPLAN_PIPE_CFG");
    auto* f345 = (cfg && std::strcmp(cfg, "63") == 0) ? fc_f345_pipe63 : fc_f345_pipe;
    const int rc = f345(sg, sthr, in, out, out_type, d, in_max, stream);
    if (rc != -1) return rc;  // -1: parameters not covered -> exact
  }
  return fc_fused_gauss_grad_thr(sg, sgrad, sthr, in, out, out_type, d, stream);
}
