"""Times K6 tracking on the GPU mask of the SPEC chain (800x600x1000 marker
scene rendered by the counter-hash video + square markers)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1509_04394_b200 import fuseplan as fp
F, H, W, n = 1000, 600, 800, int(sys.argv[1]) if len(sys.argv) > 1 else 8
mask = torch.zeros((F, H, W), dtype=torch.uint8, device="cuda")
rois = []
for i in range(n):
    x0, y0 = 50 + 80 * i, 100 + 40 * i
    for t in range(0, F):
        cx, cy = (x0 + t // 4) % (W - 10), (y0 + t // 7) % (H - 10)
        mask[t, cy:cy + 5, cx:cx + 5] = 255
    rois.append((x0 - 5, y0 - 5, 15, 15))
torch.cuda.synchronize()
fp.track_features(mask, rois, csv=False)
ts = []
for _ in range(3):
    t0 = time.perf_counter(); pts, _ = fp.track_features(mask, rois, csv=False); ts.append(time.perf_counter() - t0)
print(json.dumps({"tracking": f"{n} markers x {F} frames on a device mask", "ms": min(ts) * 1e3,
                  "frames_per_s": F / min(ts), "measured_frac": float(pts[:, :, 0].mean())}))
