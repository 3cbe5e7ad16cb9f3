"""Small-frame (config 1, 192x432x600) timing of the all-fused chain with the
frame-pair kernel's plan printed (FUSEPLAN_DEBUG), for plan / segment studies."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1509_04394_b200 import fuseplan as fp
W, H, F = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (192, 432, 600)))
pipe = fp.Pipeline(json.dumps(fp.spec_chain(W, H, F)))
ex = fp.Executor(pipe, fp.Plan(pipe, fp.Device.load("b200"), {"force_partition": "1-5"}))
v = torch.empty((F, 4, H, W), dtype=torch.uint8, device="cuda")
fp.synth_hash_u8(v, seed=1)
out = torch.empty((F, H, W), dtype=torch.uint8, device="cuda")
for _ in range(3):
    ex.run(v, out=out)
ts = []
for _ in range(9):
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record(); ex.run(v, out=out); e.record(); torch.cuda.synchronize()
    ts.append(s.elapsed_time(e))
ts.sort()
print(f"{W}x{H}x{F} out={os.environ.get('FUSEPLAN_PIPE_OUT','auto')} segs={os.environ.get('FUSEPLAN_PIPE_SEGS','auto')}: "
      f"{ts[4]:.4f} ms {F / ts[4] * 1e3:.0f} fps", flush=True)
