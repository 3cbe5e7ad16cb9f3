# CUDA graph capture: parity tests + configs table with graph timings
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider --timeout 300 -k "graph" 2>&1 | tail -15
timeout 1200 python scripts/bench_configs.py 1 2 3 5 > gpurun_out/graph_configs.jsonl 2> gpurun_out/graph_configs.err
python - <<'P'
import json
for l in open("gpurun_out/graph_configs.jsonl"):
    try: r = json.loads(l)
    except Exception: continue
    print(r["config"], r["scene"], r["partition"], r["variant"], "ms %.4f single %.4f | graph %.4f single %.4f same=%s" % (r["ms"], r["ms_single_run"], r["ms_graph"], r["ms_graph_single_run"], r["graph_output_identical"]), int(r["fps"]), int(r["fps_graph"]), r["oracle_mismatches"])
P
tail -3 gpurun_out/graph_configs.err
