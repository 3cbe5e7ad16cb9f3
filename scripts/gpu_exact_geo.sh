# exact pipeline geometry A/B: default (8 IIR warps, 4 pairs) vs 4 IIR warps with 5 / 4 pairs
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for L in libX.so libY.so; do
  echo "== parity $L"
  FUSEPLAN_LIB=$PWD/paper_1509_04394_b200/$L timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider --timeout 120 -x -k "pair_exact or f345_exact or threshold_at_exact" 2>&1 | tail -2
done
timeout 600 python scripts/exact_ab.py libA.so libX.so libY.so
