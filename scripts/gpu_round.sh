# Round evidence on one B200: GPU tests, smoke, bench line (N=1), launch list,
# frame-pair kernel ncu capture, BASELINE configs
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 --durations 10 > gpurun_out/tests.txt 2>&1
tail -15 gpurun_out/tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 1500 gpurun_out/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-parity > /dev/null 2>&1
bash scripts/gpu_pair_prof.sh pairF > /dev/null 2>&1
if [ "$1" = "configs" ]; then timeout 1500 python scripts/bench_configs.py 1 2 3 4 5 > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; fi
ls gpurun_out
