# A/B of in-tree library builds: parity on assorted shapes + timing (pair_ab.py),
# then the pipe-rate microbenchmark
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python scripts/pair_ab.py "$@" 2>&1 | tee gpurun_out/ab.txt
if [ -x scripts/micro/pipe_rates ]; then timeout 120 scripts/micro/pipe_rates > gpurun_out/pipe_rates2.txt 2>&1; fi
