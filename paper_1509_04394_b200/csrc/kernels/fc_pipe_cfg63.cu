// Tuning variant of the frame pipeline (FUSEPLAN_PIPE_CFG=63 selects it):
// mbarrier waits poll with a software back-off instead of the suspend hint.
#define FP_SPECIALISE 2
#define FP_NF 5
#define FP_NI 5
#define FP_KSLACK 2
#define FP_WAIT_SLEEP 64
#define FP_NAMESPACE fcpipe63
#define FP_ENTRY fc_chain_pipe63
#define FP_F345_ENTRY fc_f345_pipe63
#define FP_RECHECKS fc_pipe63_recheck_count
#include "fc_pipe.cu"
