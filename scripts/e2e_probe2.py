"""e2e (host pointers) variance probe: repeated fp_exec_run on pinned buffers,
per call wall times, next to plain pinned copies of the same bytes."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1509_04394_b200 import fuseplan as fp
W, H, F = 800, 600, 1000
pipe = fp.Pipeline(json.dumps(fp.spec_chain(W, H, F)))
plan = fp.Plan(pipe, fp.Device.load("b200"), {"force_partition": "1-5"})
v = torch.empty((F, 4, H, W), dtype=torch.uint8, device="cuda")
fp.synth_hash_u8(v, seed=1)
hv = torch.empty((F, 4, H, W), dtype=torch.uint8, pin_memory=True)
hv.copy_(v.cpu())
hm = torch.empty((F, H, W), dtype=torch.uint8, pin_memory=True)
for chunk in [int(c) for c in sys.argv[1:]] or [0]:
    ex = fp.Executor(pipe, plan, host_chunk_frames=chunk)
    ts = []
    for _ in range(6):
        t0 = time.perf_counter(); ex.run(hv.numpy(), out=hm.numpy()); ts.append(time.perf_counter() - t0)
    print(f"chunk {chunk}: " + " ".join(f"{t*1e3:.1f}" for t in ts) + " ms")
t0 = time.perf_counter(); v.copy_(hv, non_blocking=True); torch.cuda.synchronize()
print(f"plain H2D of the RGBA video: {(time.perf_counter()-t0)*1e3:.1f} ms")
