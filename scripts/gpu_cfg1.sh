cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python scripts/bench_configs.py 1 2>&1 | tail -1
FUSEPLAN_F12_LEGACY=1 timeout 300 python scripts/bench_configs.py 1 2>&1 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/q_cfg1_launches.csv python scripts/bench_configs.py 1 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "golden or f12 or carry or shard or segments" 2>&1 | tail -2
