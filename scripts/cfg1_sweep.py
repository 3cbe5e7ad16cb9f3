"""Window height x time-segment sweep of the frame-pair pipeline at config 1
(192x432x600), CUDA-graph replay timing (the chooser's pick = out 0 segs 0)."""
import json, os, subprocess, sys
code = r'''
import json, os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_1509_04394_b200 import fuseplan as fp
W, H, F = 192, 432, 600
pipe = fp.Pipeline(json.dumps(fp.spec_chain(W, H, F)))
ex = fp.Executor(pipe, fp.Plan(pipe, fp.Device.load("b200"), {"force_partition": "1-5"}))
v = torch.empty((F, 4, H, W), dtype=torch.uint8, device="cuda")
fp.synth_hash_u8(v, seed=1234)
ref = ex.run(v).clone()
g = ex.capture(v)
for _ in range(3): g.launch()
torch.cuda.synchronize()
ts = []
for _ in range(5):
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(20): g.launch()
    e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e) / 20)
ts.sort()
print(json.dumps({"ms": ts[2], "same": bool(torch.equal(g.out, ref))}))
'''
OUTS = [int(x) for x in os.environ.get("SWEEP_OUTS", "0,10,14,18,22,26,29").split(",")]
SEGS = [int(x) for x in os.environ.get("SWEEP_SEGS", "0,1,2,3,4,5,6").split(",")]
for out in OUTS:
    for segs in SEGS:
        env = dict(os.environ)
        if out: env["FUSEPLAN_PIPE_OUT"] = str(out)
        if segs: env["FUSEPLAN_PIPE_SEGS"] = str(segs)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        res = r.stdout.strip().splitlines()[-1] if r.returncode == 0 and r.stdout.strip() else r.stderr[-3000:]
        print(f"out {out:2d} segs {segs}: {res}", flush=True)
