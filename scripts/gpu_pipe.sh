# frame-pipeline kernel iteration: parity (fast subset), sweeps vs strip
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
FUSEPLAN_PIPE_CFG=55 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fast or golden or dense or carry" 2>&1 | tail -2
for cfg in 63 55; do
  export FUSEPLAN_PIPE_CFG=$cfg; echo "cfg $cfg"
  timeout 120 python scripts/tile_sweep.py 800 600 300 2>&1 | tail -1
  timeout 120 python scripts/tile_sweep.py 800 600 1000 2>&1 | tail -1
  timeout 120 python scripts/tile_sweep.py 192 432 600 2>&1 | tail -1
  timeout 120 python scripts/tile_sweep.py 2048 2048 200 2>&1 | tail -1
done
