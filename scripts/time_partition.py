"""Times one partition of the SPEC chain on a W x H x F hash video (device resident)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1509_04394_b200 import fuseplan as fp
W, H, F, part = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
pipe = fp.Pipeline(json.dumps(fp.spec_chain(W, H, F)))
opts = None if part == "plan" else {"force_partition": part}
ex = fp.Executor(pipe, fp.Plan(pipe, fp.Device.load("b200"), opts),
                 variant=os.environ.get("FUSEPLAN_VARIANT", "auto"))
v = torch.empty((F, 4, H, W), dtype=torch.uint8, device="cuda")
fp.synth_hash_u8(v, seed=1)
out = torch.empty((F, H, W), dtype=torch.uint8, device="cuda")
for _ in range(2):
    ex.run(v, out=out)
ts = []
for _ in range(5):
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record(); ex.run(v, out=out); e.record(); torch.cuda.synchronize()
    ts.append(s.elapsed_time(e))
ts.sort()
print(f"{part} {W}x{H}x{F}: {ts[2]:.3f} ms {F / ts[2] * 1e3:.0f} fps")
