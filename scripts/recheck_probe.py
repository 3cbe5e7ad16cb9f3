"""Runs the fused chain once and prints the exact-recheck count."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1509_04394_b200 import fuseplan as fp
W, H, F = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
pipe = fp.Pipeline(json.dumps(fp.spec_chain(W, H, F)))
ex = fp.Executor(pipe, fp.Plan(pipe, fp.Device.load("b200"), {"force_partition": "1-5"}),
                 variant="fast")
v = torch.empty((F, 4, H, W), dtype=torch.uint8, device="cuda")
fp.synth_hash_u8(v, seed=1)
out = ex.run(v)
torch.cuda.synchronize()
d = ex.describe()
print("rechecks", d.get("exact_rechecks_total"), "white", int((out == 255).sum()))
