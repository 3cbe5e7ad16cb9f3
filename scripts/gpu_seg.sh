cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "segments" 2>&1 | tail -5
timeout 300 python scripts/bench_configs.py 1 2 2>&1 | tail -8
for s in 1 2 4 6 8; do FUSEPLAN_DEBUG=1 FUSEPLAN_PIPE_SEGS=$s timeout 120 python scripts/tile_sweep.py 192 432 600 2>&1 | grep -E "\->|fps" | tail -2; done
