"""Host-pointer (e2e) timing of the fused chain for a few chunk sizes."""
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
    ex.run(hv.numpy(), out=hm.numpy())
    t0 = time.perf_counter(); ex.run(hv.numpy(), out=hm.numpy()); dt = time.perf_counter() - t0
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    out = torch.empty((F, H, W), dtype=torch.uint8, device="cuda")
    s.record(); ex.run(v, out=out); e.record(); torch.cuda.synchronize()
    print(f"chunk {chunk}: host e2e {dt*1e3:.1f} ms ({F/dt:.0f} fps), device {s.elapsed_time(e):.2f} ms")
