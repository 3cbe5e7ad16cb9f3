# Exact pipeline timing (configs 2, 3) and its parity tests.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for i in 1 2; do
  FUSEPLAN_VARIANT=exact timeout 120 python scripts/tile_sweep.py 800 600 1000
  FUSEPLAN_VARIANT=exact timeout 120 python scripts/tile_sweep.py 192 432 600
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider --timeout 300 \
  -k "f345_exact or pair_exact" 2>&1 | tail -3
