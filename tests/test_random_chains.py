"""The reference's own randomized bit-exactness suites (test_simulator.cpp:
228-243, seed 2024 x 25 chains; acceptance.cpp:276-293, seed 606 x 30
chains) with their exact chains and videos, expected outputs from the
reference itself (tests/golden/random_chains.npz, make_random_chains.py):
the CPU restatement (oracle) and the GPU executor under the optimizer's plan
(the reference's make_device: 48 KB shared memory, 13 SMs = k20_like) and
under the unfused partition must reproduce them bit for bit."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN


def _cases():
    z = np.load(os.path.join(GOLDEN, "random_chains.npz"))
    meta = json.loads(str(z["meta"]))
    vo = oo = 0
    for m in meta:
        v = m["pipeline"]["video"]
        n = v["width"] * v["height"] * v["frames"]
        video = z["videos"][vo:vo + n].reshape(v["frames"], 1, v["height"], v["width"])
        want = z["outputs"][oo:oo + n].reshape(v["frames"], v["height"], v["width"])
        vo += n
        oo += n
        yield m, video, want


def test_oracle_reproduces_reference_random_suites(oracle):
    n = 0
    for m, video, want in _cases():
        got = oracle.orc_run_sequential(m["pipeline"], video)[-1]
        np.testing.assert_array_equal(got, want, err_msg=f"{m['suite']} {m['trial']}")
        n += 1
    assert n == 55


@pytest.mark.gpu
def test_gpu_executor_reproduces_reference_random_suites(fp, cuda):
    import torch
    for m, video, want in _cases():
        p = fp.Pipeline(json.dumps(m["pipeline"]))
        k = len(m["pipeline"]["kernels"])
        for opts in (None, {"force_partition": ",".join(str(i + 1) for i in range(k))}):
            ex = fp.Executor(p, fp.Plan(p, fp.Device.load("k20_like"), opts))
            out = ex.run(torch.from_numpy(np.ascontiguousarray(video)).to(cuda))
            torch.cuda.synchronize()
            np.testing.assert_array_equal(out.cpu().numpy().astype(np.float32), want,
                                          err_msg=f"{m['suite']} {m['trial']} {opts}")
