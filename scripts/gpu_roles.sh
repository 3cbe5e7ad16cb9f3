# Role isolation timings of the headline pipe kernel (800x600x1000) for each
# library variant given: full, stencil math skipped (IIR alone), IIR math
# skipped (stencil alone), no RGB transfer, and combinations.
cd $GRAFT_REPO_ROOT
for lib in "$@"; do
  for skip in 0 2 4 6 1 5; do
    echo "== $lib skip=$skip $(FUSEPLAN_LIB=$PWD/paper_1509_04394_b200/$lib FUSEPLAN_PIPE_SKIP=$skip python scripts/tile_sweep.py 800 600 1000 | cut -d: -f2)"
  done
  FUSEPLAN_LIB=$PWD/paper_1509_04394_b200/$lib FUSEPLAN_PIPE_PROFILE=1 python scripts/tile_sweep.py 800 600 1000 2>&1 >/dev/null | grep -E "interior   ctas" | tail -1
done
