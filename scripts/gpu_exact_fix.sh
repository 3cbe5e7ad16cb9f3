cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
scripts/micro/f32x2_exact
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 2>&1 | tail -3
timeout 900 python scripts/bench_configs.py 2 3 > gpurun_out/uf_configs.jsonl 2> gpurun_out/uf_configs.err
python - <<'P'
import json
for l in open("gpurun_out/uf_configs.jsonl"):
    try: r = json.loads(l)
    except Exception: continue
    print(r["config"], r["partition"], r["variant"], "%.4f" % r["ms"], int(r["fps"]), int(r["fps_graph"]), r["oracle_mismatches"])
P
