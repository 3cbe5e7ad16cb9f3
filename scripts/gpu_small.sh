# config-1 plan study: auto plan (FUSEPLAN_DEBUG shows it), forced window
# heights / segment counts, and the launch list of the auto plan
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
FUSEPLAN_DEBUG=1 python scripts/small_frames.py 2>&1 | grep -E "choose: ->|fps"
for o in 10 14 18 22 26 29; do for s in 1 2 3 4 5 6; do FUSEPLAN_PIPE_OUT=$o FUSEPLAN_PIPE_SEGS=$s python scripts/small_frames.py 2>&1 | grep fps; done; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/small_frames.py 2>/dev/null | grep -E "k_chain_pair|k_verify" | tail -6
