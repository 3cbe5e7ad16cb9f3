# GPU test suite (per-test timeout, durations) + the frame-pair kernel profile
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 240 --durations 15 > gpurun_out/tests.txt 2>&1
tail -30 gpurun_out/tests.txt
bash scripts/gpu_pair_prof.sh pair0
