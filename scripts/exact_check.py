"""Exact variant (FP64 frame-pair pipeline) vs the oracle on assorted shapes,
then device timings at configs 2 and 3 (scratch check, GPU)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1509_04394_b200 import fuseplan as fp
from oracle import oracle as O


def run(W, H, F, th=128.0, seed=1, alpha=0.5, check=True, variant="exact"):
    pipe = fp.spec_chain(W, H, F, th=th)
    pipe["kernels"][1].setdefault("params", {})["alpha"] = alpha
    p = fp.Pipeline(json.dumps(pipe))
    ex = fp.Executor(p, fp.Plan(p, fp.Device.load("b200"), {"force_partition": "1-5"}),
                     variant=variant)
    v = torch.empty((F, 4, H, W), dtype=torch.uint8, device="cuda")
    fp.synth_hash_u8(v, seed=seed)
    out = torch.empty((F, H, W), dtype=torch.uint8, device="cuda")
    ex.run(v, out=out)
    torch.cuda.synchronize()
    bad = -1
    if check:
        want = O.orc_chain(pipe, v.cpu().numpy())
        bad = int((out.cpu().numpy().astype(np.float32) != want).sum())
    return ex, v, out, bad


def timeit(ex, v, out, reps=10):
    for _ in range(2):
        ex.run(v, out=out)
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(reps):
        ex.run(v, out=out)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


if __name__ == "__main__":
    for (W, H, F, th) in [(800, 600, 24, 128.0), (800, 600, 17, 20.0), (192, 432, 60, 40.0),
                          (160, 96, 24, 24.0), (144, 40, 9, 30.0), (256, 64, 7, 10.0),
                          (800, 600, 1, 60.0)]:
        ex, v, out, bad = run(W, H, F, th=th)
        print(f"exact {W}x{H}x{F} th={th}: mismatches {bad}  {ex.describe()['last_chain_kernel']}",
              flush=True)
    ex, v, out, bad = run(256, 128, 21, th=30.0, alpha=0.3)
    print(f"exact alpha 0.3: mismatches {bad}", flush=True)
    for (W, H, F) in [(192, 432, 600), (800, 600, 1000)]:
        for variant in ("exact", "auto"):
            ex, v, out, _ = run(W, H, F, check=False, variant=variant)
            ms = timeit(ex, v, out)
            print(f"{variant} {W}x{H}x{F}: {ms:.3f} ms {F / ms * 1e3:.0f} fps "
                  f"({ex.describe()['last_chain_kernel']})", flush=True)
