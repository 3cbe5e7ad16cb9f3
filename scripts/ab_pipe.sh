# A/B timing of pipe-kernel layout variants (FUSEPLAN_LIB), 800x600x1000 and
# 2048x2048x200, 3 alternating rounds; per-CTA role waits for each variant.
cd $GRAFT_REPO_ROOT
for round in 1 2 3; do
for lib in "$@"; do
  echo "== $lib $(FUSEPLAN_LIB=$PWD/paper_1509_04394_b200/$lib python scripts/tile_sweep.py 800 600 1000 | cut -d: -f2)"
done
done
for lib in "$@"; do
  echo "== $lib 2048: $(FUSEPLAN_LIB=$PWD/paper_1509_04394_b200/$lib python scripts/tile_sweep.py 2048 2048 200 | cut -d: -f2)"
  FUSEPLAN_LIB=$PWD/paper_1509_04394_b200/$lib FUSEPLAN_PIPE_PROFILE=1 python scripts/tile_sweep.py 800 600 1000 2>&1 >/dev/null | grep -E "interior   ctas" | tail -1
done
