for t in auto 32,36 32,28 48,40 48,30 64,36 64,28 80,43 80,21 96,22 128,18 160,22 32,64 48,20 64,20; do
  FUSEPLAN_FAST_TILE=$t timeout 120 python scripts/tile_sweep.py 800 600 300 2>&1 | tail -1
done
