"""Frame-pair pipeline (fc_pipe2.cu) vs the oracle on assorted shapes, then
timing of both pipelines at 800x600x1000 (scratch check, GPU)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1509_04394_b200 import fuseplan as fp
from oracle import oracle as O


def run(W, H, F, impl, th=128.0, seed=1, alpha=0.5, band=None, check=True):
    os.environ["FUSEPLAN_PIPE_IMPL"] = str(impl)
    if band: os.environ["FUSEPLAN_PIPE_BAND_SCALE"] = str(band)
    else: os.environ.pop("FUSEPLAN_PIPE_BAND_SCALE", None)
    pipe = fp.spec_chain(W, H, F, th=th)
    pipe["kernels"][1].setdefault("params", {})["alpha"] = alpha
    p = fp.Pipeline(json.dumps(pipe))
    ex = fp.Executor(p, fp.Plan(p, fp.Device.load("b200"), {"force_partition": "1-5"}), variant="fast")
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


def timeit(W, H, F, impl):
    ex, v, out, _ = run(W, H, F, impl, check=False)
    ts = []
    for _ in range(7):
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); ex.run(v, out=out); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[3]


if __name__ == "__main__":
    cases = [(800, 600, 40), (800, 600, 33), (192, 432, 60), (160, 96, 24), (132, 40, 9),
             (256, 64, 7), (800, 600, 1)]
    for (W, H, F) in cases:
        for impl in (2,):
            ex, v, out, bad = run(W, H, F, impl)
            print(f"impl{impl} {W}x{H}x{F}: mismatches {bad} kernel {ex.describe()['groups'][0].get('kernel') if isinstance(ex.describe(), dict) else ''}", flush=True)
    ex, v, out, bad = run(800, 600, 40, 2, th=20.0, band=64.0)
    print(f"impl2 dense rechecks 800x600x40 th=20 band x64: mismatches {bad}", flush=True)
    ex, v, out, bad = run(256, 128, 21, 2, alpha=0.3)
    print(f"impl2 alpha 0.3 256x128x21: mismatches {bad}", flush=True)
    for impl in (1, 2):
        ms = timeit(800, 600, 1000, impl)
        print(f"impl{impl} 800x600x1000: {ms:.3f} ms {1000/ms*1e3:.0f} fps {1.92/ms*1e3:.0f} GB/s", flush=True)
    for impl in (1, 2):
        ms = timeit(2048, 2048, 200, impl)
        print(f"impl{impl} 2048x2048x200: {ms:.3f} ms {200/ms*1e3:.0f} fps", flush=True)
