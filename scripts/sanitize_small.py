"""Small runs of every kernel family for compute-sanitizer (memcheck /
racecheck / synccheck): certified and exact frame-pair pipelines (segments
included), unfused stages, two-fusion groups."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1509_04394_b200 import fuseplan as fp
for (W, H, F, part, variant) in [(136, 61, 9, "1-5", "auto"), (136, 61, 9, "1-5", "exact"),
                                 (192, 96, 130, "1-5", "auto"), (196, 50, 6, "1-5", "exact"),
                                 (136, 61, 9, "1,2,3,4,5", "exact"), (136, 61, 9, "1-2,3-5", "auto"),
                                 (136, 61, 9, "1-2,3-5", "exact"), (196, 50, 7, "1-2,3-5", "exact")]:
    pipe = fp.Pipeline(json.dumps(fp.spec_chain(W, H, F, th=30.0)))
    ex = fp.Executor(pipe, fp.Plan(pipe, fp.Device.load("b200"), {"force_partition": part}),
                     variant=variant)
    v = torch.empty((F, 4, H, W), dtype=torch.uint8, device="cuda")
    fp.synth_hash_u8(v, seed=3)
    out = ex.run(v)
    torch.cuda.synchronize()
    print(W, H, F, part, variant, ex.describe()["last_chain_kernel"], int(out.float().sum().item()))
