"""Debug: the certified pipe with a general IIR alpha; locate mismatches and
compare the kernel's decision inputs with exact values."""
import json, sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from oracle import oracle as O
from paper_1509_04394_b200 import fuseplan as fp
from paper_1509_04394_b200.fuseplan import hash_video_u8, spec_chain
W, H, F = 256, 96, 30
for alpha in (0.3, 0.3001, 0.7, 0.25):
    for seed in (17, 18):
        pipe = spec_chain(W, H, F, alpha=alpha, th=30.0)
        v = hash_video_u8(F, 4, H, W, seed)
        want = O.orc_chain(pipe, v)
        p = fp.Pipeline(json.dumps(pipe))
        res = {}
        for variant in ("fast", "exact"):
            ex = fp.Executor(p, fp.Plan(p, fp.Device.load("b200"), {"force_partition": "1-5"}),
                             variant=variant)
            out = ex.run(torch.from_numpy(v).cuda()).cpu().numpy().astype(np.float32)
            res[variant] = np.argwhere(out != want)
        iir = O.orc_chain(dict(pipe, kernels=pipe["kernels"][:2]), v)
        # the GPU's IIR planes (1-2 group through the F12 kernel)
        p2 = fp.Pipeline(json.dumps(dict(pipe, kernels=pipe["kernels"][:2])))
        e2 = fp.Executor(p2, fp.Plan(p2, fp.Device.load("b200"), {"force_partition": "1-2"}))
        g_iir = e2.run(torch.from_numpy(v).cuda()).cpu().numpy()
        print(alpha, seed, "fast mism", res["fast"][:5].tolist(), "exact mism", len(res["exact"]),
              "F12 iir diffs", int((g_iir.view(np.uint32) != iir.view(np.uint32)).sum()), flush=True)
        for (t, y, x) in res["fast"][:3]:
            g = O.orc_chain(dict(pipe, kernels=pipe["kernels"][:4]), v)[t, y, x]
            print("   px", t, y, x, "grad", g, "th", 30.0)
