# Exact F345 on the frame-pair pipeline: its parity tests, the exact pair
# tests next to it, and the configs table rows for cfg2/cfg3.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider --timeout 300 \
  -k "f345_exact or pair_exact or forced_rechecks or time_segments" > gpurun_out/f345x_tests.txt 2>&1
tail -15 gpurun_out/f345x_tests.txt
timeout 600 python scripts/bench_configs.py 2 3 > gpurun_out/f345x_configs.jsonl 2> gpurun_out/f345x_configs.err
python - <<'P'
import json
for l in open("gpurun_out/f345x_configs.jsonl"):
    try: r = json.loads(l)
    except Exception: continue
    print(r["config"], r["scene"], r["partition"], r["variant"], round(r["ms"], 3), int(r["fps"]), r["oracle_mismatches"])
P
tail -3 gpurun_out/f345x_configs.err
