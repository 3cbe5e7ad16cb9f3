# Role isolation timings of the frame-pair kernel (800x600x1000) for each
# library given: full, IIR math skipped (stencil alone), stencil math skipped
# (IIR alone), 8 = IIR warps only hand off slots (stencil alone), no RGB transfer
cd $GRAFT_REPO_ROOT
for lib in "$@"; do
  for skip in 0 8 2 1 4; do
    echo "== $lib skip=$skip $(FUSEPLAN_LIB=$PWD/paper_1509_04394_b200/$lib FUSEPLAN_PIPE_SKIP=$skip python scripts/tile_sweep.py 800 600 1000 | cut -d: -f2)"
  done
done
