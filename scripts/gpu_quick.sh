# quick iteration: headline + small-frame timings, segment / F12 parity
cd $GRAFT_REPO_ROOT
for i in 1 2 3; do timeout 120 python scripts/tile_sweep.py 800 600 1000 2>&1 | tail -1; done
timeout 120 python scripts/tile_sweep.py 192 432 600 2>&1 | tail -1
timeout 300 python scripts/bench_configs.py 1 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "segments or golden or f12 or carry or shard" 2>&1 | tail -2
