# Round evidence: bench line, launch list of the bench command, full ncu of the
# headline kernel on the bench workload (-> traffic), gpu test suite.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/ev_tests.log
timeout 600 python bench.py > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev_launches.csv python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chain_pipe -c 1 -o gpurun_out/ev_full python scripts/tile_sweep.py 800 600 1000 > /dev/null 2>&1
ncu -i gpurun_out/ev_full.ncu-rep --page raw --csv > gpurun_out/ev_full_raw.csv 2>&1
ncu -i gpurun_out/ev_full.ncu-rep --page details --csv > gpurun_out/ev_full_details.csv 2>&1
ncu -i gpurun_out/ev_full.ncu-rep --page source --print-source sass --csv > gpurun_out/ev_full_sass.csv 2>&1
cat gpurun_out/ev_tests.log; tail -c 3000 gpurun_out/ev_bench.json
timeout 900 python scripts/bench_configs.py 1 2 3 5 > gpurun_out/ev_configs.jsonl 2> gpurun_out/ev_configs.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_cfg1_launches.csv python scripts/bench_configs.py 1 > /dev/null 2>&1
tail -c 1500 gpurun_out/ev_configs.jsonl
