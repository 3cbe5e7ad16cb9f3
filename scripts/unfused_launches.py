"""One unfused (1,2,3,4,5) run of the SPEC chain at 800x600xF for a launch list."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1509_04394_b200 import fuseplan as fp
W, H, F = 800, 600, int(sys.argv[1]) if len(sys.argv) > 1 else 200
pipe = fp.Pipeline(json.dumps(fp.spec_chain(W, H, F)))
ex = fp.Executor(pipe, fp.Plan(pipe, fp.Device.load("b200"), {"force_partition": "1,2,3,4,5"}),
                 variant="exact")
v = torch.empty((F, 4, H, W), dtype=torch.uint8, device="cuda")
fp.synth_hash_u8(v, seed=1)
out = torch.empty((F, H, W), dtype=torch.uint8, device="cuda")
for _ in range(2):
    ex.run(v, out=out)
torch.cuda.synchronize()
