import json, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_1509_04394_b200 import fuseplan as fp
W, H, F = 136, 61, 9
pipe = fp.Pipeline(json.dumps(fp.spec_chain(W, H, F, th=30.0)))
ex = fp.Executor(pipe, fp.Plan(pipe, fp.Device.load("b200"), {"force_partition": "1-2,3-5"}))
v = torch.empty((F, 4, H, W), dtype=torch.uint8, device="cuda")
fp.synth_hash_u8(v, seed=3)
out = ex.run(v)
torch.cuda.synchronize()
print("ok")
