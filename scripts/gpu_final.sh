# Round-end numbers: bench line + BASELINE configs table
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 400 gpurun_out/bench.json
timeout 1500 python scripts/bench_configs.py 1 2 3 4 5 > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
python - <<'P'
import json
for l in open("gpurun_out/configs.jsonl"):
    try: r = json.loads(l)
    except Exception: continue
    print(r["config"], r.get("scene"), r.get("partition"), r.get("variant"), "%.4f" % r.get("ms", 0), int(r["fps"]), int(r.get("fps_graph", 0)), "%.3f" % r.get("roofline_frac", 0), r["oracle_mismatches"])
P
