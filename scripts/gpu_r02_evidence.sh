# Round-2 evidence on one B200: GPU test suite, bench line (N=1), the bench
# command's launch list (ncu, cold / serialised), every BASELINE config with
# full-volume oracle checks, the multi-rank path emulated on one GPU.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ev2_tests.txt 2>&1
tail -3 gpurun_out/ev2_tests.txt
timeout 900 python bench.py > gpurun_out/ev2_bench.json 2> gpurun_out/ev2_bench.err
tail -c 2500 gpurun_out/ev2_bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev2_launches.csv python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-parity > /dev/null 2>&1
timeout 1500 python scripts/bench_configs.py 1 2 3 4 5 > gpurun_out/ev2_configs.jsonl 2> gpurun_out/ev2_configs.err
tail -3 gpurun_out/ev2_configs.err
bash scripts/gpu_multi.sh > gpurun_out/ev2_multi.txt 2>&1
ls -la gpurun_out/ev2_*
