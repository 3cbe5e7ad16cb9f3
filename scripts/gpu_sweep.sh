timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
FUSEPLAN_FAST_PROFILE=1 FUSEPLAN_FAST_TILE=64,30 timeout 120 python scripts/tile_sweep.py 800 600 300 2>&1 | tail -2
for t in auto 48,38 64,30 80,22 96,22 128,18 160,22 160,14; do
  FUSEPLAN_FAST_TILE=$t timeout 120 python scripts/tile_sweep.py 800 600 300 2>&1 | tail -1
done
