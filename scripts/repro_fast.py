import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1509_04394_b200 import fuseplan as fp
W, H, F = [int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (64, 48, 4))]
pipe = fp.spec_chain(W, H, F, th=24.0)
p = fp.Pipeline(json.dumps(pipe))
ex = fp.Executor(p, fp.Plan(p, fp.Device.load("b200"), {"force_partition": "1-5"}), variant="fast")
v = torch.from_numpy(fp.hash_video_u8(F, 4, H, W, 1)).cuda()
out = ex.run(v)
torch.cuda.synchronize()
print("ok", out.float().mean().item())
