# strip-kernel iteration: fast-path parity, nw sweep, ncu counters + full capture
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fast or state_carry or golden_partitions or dense" 2>&1 | tail -2
for nw in auto 8 7; do
  if [ $nw = auto ]; then unset FUSEPLAN_STRIP_NW; else export FUSEPLAN_STRIP_NW=$nw; fi
  timeout 120 python scripts/tile_sweep.py 800 600 300 2>&1 | tail -1
done
unset FUSEPLAN_STRIP_NW
timeout 120 python scripts/tile_sweep.py 800 600 1000 2>&1 | tail -1
timeout 900 ncu --set full --import-source on -k regex:k_chain_strip -c 1 -o gpurun_out/strip_full python scripts/tile_sweep.py 800 600 300 > /dev/null 2>&1
ls -la gpurun_out/
