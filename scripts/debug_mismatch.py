"""Locates mask mismatches vs the oracle for a W x H x F hash video and
prints the reference gradient magnitude around them."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import oracle as O
from paper_1509_04394_b200 import fuseplan as fp
W, H, F = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
variant = sys.argv[4] if len(sys.argv) > 4 else "auto"
seed = int(sys.argv[5]) if len(sys.argv) > 5 else 1234
spec = fp.spec_chain(W, H, F, kalman=True)
pipe = fp.Pipeline(json.dumps(spec))
ex = fp.Executor(pipe, fp.Plan(pipe, fp.Device.load("b200"), {"force_partition": "1-5,6"}),
                 variant=variant)
v = torch.empty((F, 4, H, W), dtype=torch.uint8, device="cuda")
fp.synth_hash_u8(v, seed=seed)
m = ex.run(v).cpu().numpy().astype(np.float32)
vh = v.cpu().numpy()
want, st = O.orc_chain(spec, vh, return_state=True)
bad = np.argwhere(m != want)
print("variant", variant, "mismatches", len(bad), "rechecks", ex.describe().get("exact_rechecks_total"))
# reference gradient planes via the per-stage oracle for the frames involved
for t, y, x in bad[:10]:
    print(f"t={t} y={y} x={x} got={m[t,y,x]} want={want[t,y,x]}  strip={x//120} band={y//30}")
if len(bad):
    t0 = int(bad[0][0])
    k = spec["kernels"]
    vol = vh[:t0 + 1].astype(np.float32)
    g = O.orc_apply_stage(k[0], vol)[:, None]
    i = O.orc_apply_stage(k[1], g)[:, None]
    s3 = O.orc_apply_stage(k[2], i)[:, None]
    s4 = O.orc_apply_stage(k[3], s3)
    for t, y, x in bad[:10]:
        if t == t0:
            print(f"  gradient at ({y},{x}) = {s4[t, y, x]!r} (threshold {k[4]['params']})")
    # the oracle's IIR (= gray at t=0) neighbourhood of the first mismatch
    t, y, x = [int(q) for q in bad[0]]
    print("oracle IIR neighbourhood:")
    for dy in range(-3, 4):
        print(" ".join(f"{i[t, 0, min(max(y+dy,0),H-1), min(max(x+dx,0),W-1)]:.9g}" for dx in range(-3, 4)))
