for cfg in 63 55; do
  export FUSEPLAN_PIPE_CFG=$cfg
  FUSEPLAN_PIPE_PROFILE=1 timeout 120 python scripts/tile_sweep.py 800 600 1000 2>&1 | tail -6
done
