"""Regenerates tests/golden/random_chains.npz: the reference's own randomized
bit-exactness suites (test_simulator.cpp:228-243, seed 2024 x 25 chains;
acceptance.cpp:276-293, seed 606 x 30 chains) with their exact chains and
videos (gen_random_chains.cpp restates helpers.hpp:67-120 call for call, so
libstdc++'s generators produce the same values), and the expected outputs from
the reference ITSELF (oracle/_ref run_sequential, simulator.cpp:158-177).

    python tests/golden/make_random_chains.py     # build container only
"""
import json
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

PARAMS = {  # helpers.hpp:81-107
    "identity": {}, "scale_offset": {"scale": 1.5, "offset": 3.0},
    "gaussian": {"radius": 1, "sigma": 1.0}, "gradient": {}, "threshold": {"th": 32.0},
    "box_mean": {"radius_x": 1, "radius_y": 1, "radius_t": 1},
    "iir_temporal": {"alpha": 0.25},
}


def main():
    exe, vid = "/tmp/gen_random_chains", "/tmp/random_chain_videos.f32"
    subprocess.run(["g++", "-O2", "-std=c++17", os.path.join(HERE, "gen_random_chains.cpp"),
                    "-o", exe], check=True)
    lines = subprocess.run([exe, vid], check=True, capture_output=True,
                           text=True).stdout.split("\n")
    raw = np.fromfile(vid, np.float32)
    meta, videos, outs, off = [], [], [], 0
    for ln in lines:
        if not ln.strip():
            continue
        suite, trial, w, h, f, ops = ln.split()
        w, h, f = int(w), int(h), int(f)
        n = w * h * f
        v = raw[off:off + n].reshape(f, 1, h, w)
        off += n
        pipe = {"video": {"width": w, "height": h, "frames": f, "channels": 1},
                "kernels": [{"name": f"k{i + 1}", "stencil_op": op, "params": PARAMS[op]}
                            for i, op in enumerate(ops.split(","))]}
        final, _ = O.ref_run_sequential(json.dumps(pipe), v)
        meta.append({"suite": suite, "trial": int(trial), "pipeline": pipe})
        videos.append(v.ravel())
        outs.append(np.asarray(final, np.float32).ravel())
    assert off == raw.size
    np.savez_compressed(os.path.join(HERE, "random_chains.npz"),
                        meta=np.array(json.dumps(meta)), videos=np.concatenate(videos),
                        outputs=np.concatenate(outs))
    print(f"{len(meta)} chains")


if __name__ == "__main__":
    main()
