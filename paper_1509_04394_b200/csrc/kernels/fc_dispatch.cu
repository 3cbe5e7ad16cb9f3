// Variant dispatch for the streaming all-fused chain (F12345).
#include <cuda_runtime.h>

#include "fc_kernels.h"

extern "C" int fc_chain_exact(const fc_stage* sgray, const fc_stage* si,
                              const fc_stage* sg, const fc_stage* sthr,
                              const void* video, int in_type, int gray_in,
                              void* out, int out_type, fc_dims d, int n_warm,
                              const float* state_in, float* state_out,
                              void* stream);

extern "C" int fc_chain_fast(const fc_stage* sgray, const fc_stage* si,
                             const fc_stage* sg, const fc_stage* sthr,
                             const void* video, int in_type, int gray_in,
                             void* out, int out_type, fc_dims d, int n_warm,
                             const float* state_in, float* state_out,
                             void* stream);

extern "C" int fc_fused_chain(const fc_stage* sgray, const fc_stage* si,
                              const fc_stage* sg, const fc_stage* sgrad,
                              const fc_stage* sthr, const void* video,
                              int in_type, int gray_in, void* out, int out_type,
                              fc_dims d, int n_warm, const float* state_in,
                              float* state_out, int variant, void* stream) {
  (void)sgrad;
  if (variant == 2 || variant == 0) {
    int rc = fc_chain_fast(sgray, si, sg, sthr, video, in_type, gray_in, out,
                           out_type, d, n_warm, state_in, state_out, stream);
    if (rc != -1 || variant == 2) return rc;  // -1: parameters not covered
  }
  return fc_chain_exact(sgray, si, sg, sthr, video, in_type, gray_in, out,
                        out_type, d, n_warm, state_in, state_out, stream);
}
