import json, sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from oracle import oracle as O
from paper_1509_04394_b200 import fuseplan as fp
from paper_1509_04394_b200.fuseplan import hash_video_u8, spec_chain
W, H, F = 256, 96, 30
pipe = spec_chain(W, H, F, alpha=0.3, th=30.0)
v = hash_video_u8(F, 4, H, W, 17)
want = O.orc_chain(pipe, v)
p = fp.Pipeline(json.dumps(pipe))
ex = fp.Executor(p, fp.Plan(p, fp.Device.load("b200"), {"force_partition": "1-5"}), variant="fast")
out = ex.run(torch.from_numpy(v).cuda()).cpu().numpy().astype(np.float32)
torch.cuda.synchronize()
print("scale", os.environ.get("FUSEPLAN_PIPE_BAND_SCALE"), "mism", np.argwhere(out != want).tolist(),
      "got", out[24, 71, 178], "want", want[24, 71, 178], "rechecks", ex.describe()["exact_rechecks_total"], flush=True)
iir = O.orc_chain(dict(pipe, kernels=pipe["kernels"][:2]), v)
np.set_printoptions(precision=9)
print("exact IIR 7x7 at t=24:\n", iir[24, 68:75, 175:182])
