// Tuning variant of the frame pipeline (FUSEPLAN_PIPE_CFG=63 selects it):
// separate TMA producer warp (the IIR rows shared by the 5 IIR warps only),
// the layout before the producer warp took IIR rows -- kept for A/B runs.
#define FP_SPECIALISE 2
#define FP_NF 5
#define FP_NI 5
#define FP_KSLACK 2
#define FP_IIR_TMA 0
#define FP_NAMESPACE fcpipe63
#define FP_ENTRY fc_chain_pipe63
#define FP_F345_ENTRY fc_f345_pipe63
#define FP_RECHECKS fc_pipe63_recheck_count
#include "fc_pipe.cu"
