"""A/B of library builds (FUSEPLAN_LIB per process) on the unfused chain
(partition 1,2,3,4,5) at configs 2 and 3, rounds interleaved."""
import os, subprocess, sys
code = r'''
import json, os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_1509_04394_b200 import fuseplan as fp
res = []
for W, H, F in ((800, 600, 1000), (192, 432, 600)):
    pipe = fp.Pipeline(json.dumps(fp.spec_chain(W, H, F)))
    ex = fp.Executor(pipe, fp.Plan(pipe, fp.Device.load("b200"), {"force_partition": "1,2,3,4,5"}))
    v = torch.empty((F, 4, H, W), dtype=torch.uint8, device="cuda")
    fp.synth_hash_u8(v, seed=1)
    out = torch.empty((F, H, W), dtype=torch.uint8, device="cuda")
    for _ in range(2): ex.run(v, out=out)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        for _ in range(5): ex.run(v, out=out)
        e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e) / 5)
    ts.sort()
    res.append(f"{W}x{H}x{F} {ts[2]:.4f} ms")
print(" | ".join(res))
'''
for rnd in range(3):
    for lib in sys.argv[1:]:
        env = dict(os.environ, FUSEPLAN_LIB=os.path.abspath(f"paper_1509_04394_b200/{lib}"))
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        print(f"== {lib}: {r.stdout.strip() if r.returncode == 0 else r.stderr[-300:]}", flush=True)
