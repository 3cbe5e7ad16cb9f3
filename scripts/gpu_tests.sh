# GPU test suite with a per-test timeout and the slowest tests listed
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 --durations 15 ${@} > gpurun_out/tests.txt 2>&1
tail -40 gpurun_out/tests.txt
