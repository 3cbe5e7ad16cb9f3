# HEAD check: full gpu suite, strip-kernel sweep, bench line
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
for nw in auto 8; do
  if [ $nw = auto ]; then unset FUSEPLAN_STRIP_NW; else export FUSEPLAN_STRIP_NW=$nw; fi
  timeout 120 python scripts/tile_sweep.py 800 600 300 2>&1 | tail -1
done
unset FUSEPLAN_STRIP_NW
timeout 120 python scripts/tile_sweep.py 800 600 1000 2>&1 | tail -1
timeout 120 python scripts/tile_sweep.py 192 432 600 2>&1 | tail -1
timeout 120 python scripts/tile_sweep.py 2048 2048 200 2>&1 | tail -1
timeout 300 python bench.py --steps 10 --warmup 3 --e2e-steps 2 2>&1 | tail -1
