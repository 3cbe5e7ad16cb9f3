// Tuning variant of the frame pipeline: 4-column stencil lanes (one warp
// per frame), 6 frames in flight, 3 IIR warps, 1 slack IIR slot.
// FUSEPLAN_PIPE_CFG=63 selects it.
#define FP_LC 4
#define FP_NF 6
#define FP_NI 3
#define FP_KSLACK 1
#define FP_NAMESPACE fcpipe63
#define FP_ENTRY fc_chain_pipe63
#define FP_F345_ENTRY fc_f345_pipe63
#define FP_RECHECKS fc_pipe63_recheck_count
#include "fc_pipe.cu"
