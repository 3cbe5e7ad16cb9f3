"""One run of the unfused SPEC chain (partition 1,2,3,4,5) at 800x600x100 (ncu target)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1509_04394_b200 import fuseplan as fp
W, H, F = 800, 600, 100
pipe = fp.Pipeline(json.dumps(fp.spec_chain(W, H, F)))
ex = fp.Executor(pipe, fp.Plan(pipe, fp.Device.load("b200"), {"force_partition": "1,2,3,4,5"}))
v = torch.empty((F, 4, H, W), dtype=torch.uint8, device="cuda")
fp.synth_hash_u8(v, seed=1)
out = ex.run(v)
torch.cuda.synchronize()
print(out.shape)
