"""Times the certified fused kernel for one tile shape (FUSEPLAN_FAST_TILE)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1509_04394_b200 import fuseplan as fp
W, H, F = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
pipe = fp.Pipeline(json.dumps(fp.spec_chain(W, H, F)))
ex = fp.Executor(pipe, fp.Plan(pipe, fp.Device.load("b200"), {"force_partition": "1-5"}),
                 variant=os.environ.get("FUSEPLAN_VARIANT", "fast"))
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
ms = ts[2]
print(f"{os.environ.get("FUSEPLAN_VARIANT", "fast")} nw={os.environ.get("FUSEPLAN_STRIP_NW","auto")} tile={os.environ.get("FUSEPLAN_FAST_TILE","auto")} {W}x{H}x{F}: {ms:.3f} ms "
      f"{F/ms*1e3:.0f} fps {4*W*H*F/ms/1e6:.0f} GB/s")
