// Tuning variant of the frame pipeline (FUSEPLAN_PIPE_CFG=63 selects it):
// the earlier 16-warp layout -- two 2-column stencil warps per frame, 5
// frames in flight, 128 registers, 4 TMA slots, IIR code specialised per
// window -- kept for A/B runs.
#define FP_SPECIALISE 2
#define FP_LC 2
#define FP_NF 5
#define FP_NI 5
#define FP_KSLACK 2
#define FP_NSF 4
#define FP_NAMESPACE fcpipe63
#define FP_ENTRY fc_chain_pipe63
#define FP_F345_ENTRY fc_f345_pipe63
#define FP_RECHECKS fc_pipe63_recheck_count
#include "fc_pipe.cu"
