"""Regenerates the golden fixtures in tests/golden/ from the REFERENCE ITSELF.

Run in the build container (needs /root/reference and oracle/_ref built):

    python tests/golden/make_golden.py

Every output vector below is produced by the reference's own code compiled
unmodified (oracle/_ref/libfuseplan_ref.so): run_sequential
(/root/reference/proj/src/simulator.cpp:158-177), synth_video
(synth.cpp:35-78) + FPVD u8 truncation (video.cpp:46-94), and plan /
render_plan (planner.cpp:342-442).  The GPU box has no /root/reference; tests
there read these committed files.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

DATA = os.path.join(ROOT, "paper_1509_04394_b200", "data")


def spec_chain(w, h, f, alpha=0.5, radius=2, sigma=1.0, th=128.0, kalman=False,
               channels=4):
    ks = []
    if channels == 4:
        ks.append({"name": "rgba_to_gray", "stencil_op": "rgba2gray"})
    ks += [
        {"name": "temporal_denoise", "stencil_op": "iir_temporal",
         "params": {"alpha": alpha}},
        {"name": "gaussian_smooth", "stencil_op": "gaussian",
         "params": {"radius": radius, "sigma": sigma}},
        {"name": "gradient_magnitude", "stencil_op": "gradient"},
        {"name": "binarize", "stencil_op": "threshold", "params": {"th": th}},
    ]
    if kalman:
        ks.append({"name": "kalman_tracking", "stencil_op": "kalman_track"})
    return {"video": {"width": w, "height": h, "frames": f, "fps": 1,
                      "channels": channels}, "kernels": ks}


def hash_video(f, c, h, w, seed):
    """Counter-hash uniform u8 video; mirrored by
    paper_1509_04394_b200.synth.hash_video_u8 and the device generator."""
    t = np.arange(f, dtype=np.uint64)[:, None, None, None]
    ch = np.arange(c, dtype=np.uint64)[None, :, None, None]
    y = np.arange(h, dtype=np.uint64)[None, None, :, None]
    x = np.arange(w, dtype=np.uint64)[None, None, None, :]
    idx = (((t * np.uint64(c) + ch) * np.uint64(h) + y) * np.uint64(w) + x)
    with np.errstate(over="ignore"):
        z = idx + np.uint64((seed * 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(56)).astype(np.uint8)


MARKERS = [
    {"x": 20, "y": 20, "vx": 1.0, "vy": 0.0, "radius": 3, "intensity": 255},
    {"x": 40, "y": 30, "vx": 0.5, "vy": 0.5, "radius": 3, "intensity": 255},
]


def chain_case(name, pipe, video, stages=False):
    pj = json.dumps(pipe)
    final, st = O.ref_run_sequential(pj, video, stages=stages)
    arrays = {"video": video, "final": final}
    if stages:
        arrays["stages"] = st
    np.savez_compressed(os.path.join(HERE, f"chain_{name}.npz"),
                        pipeline=np.array(pj), **arrays)
    print(f"chain_{name}: video {video.shape} white={(final == 255).sum()}")


def main():
    O.build()
    # 1. reference-faithful marker scene, bundled chain
    spec = {"width": 64, "height": 48, "frames": 20, "channels": 4,
            "noise_sigma": 8.0, "seed": 1234, "markers": MARKERS}
    chain_case("synth_64x48x20", spec_chain(64, 48, 20, kalman=True),
               O.ref_synth_u8(spec))
    # 2. tiny ragged uniform video with every stage output
    rng = np.random.default_rng(7)
    chain_case("tiny_13x11x7", spec_chain(13, 11, 7),
               rng.integers(0, 256, (7, 4, 11, 13), dtype=np.uint8), stages=True)
    # 3. counter-hash adversarial video, threshold lowered so masks are dense
    chain_case("hash_40x36x16_th24", spec_chain(40, 36, 16, th=24.0),
               hash_video(16, 4, 36, 40, 5150))
    # 4. non-default parameters (alpha, radius, sigma, th)
    chain_case("params_33x17x9", spec_chain(33, 17, 9, alpha=0.25, radius=1,
                                            sigma=1.5, th=40.0),
               hash_video(9, 4, 17, 33, 1234), stages=True)
    # 5. degenerate shapes: single column, single row, single pixel, one frame
    for (w, h, f) in [(1, 9, 5), (9, 1, 5), (1, 1, 4), (10, 8, 1)]:
        chain_case(f"edge_{w}x{h}x{f}", spec_chain(w, h, f, th=8.0),
                   hash_video(f, 4, h, w, 99), stages=True)
    # 6. single-channel (gray) video: chain starts at the IIR
    chain_case("gray_24x20x6", spec_chain(24, 20, 6, th=20.0, channels=1),
               hash_video(6, 1, 20, 24, 3))

    # 7. planner known answers through the reference planner
    devices = {n: open(os.path.join(DATA, n + ".json")).read()
               for n in ("k20_like", "c1060_like", "b200")}
    bundled = open(os.path.join(DATA, "vision_pipeline.json")).read()
    cases = []

    def plan_case(pipe_json, dev, opts=None):
        try:
            out = O.ref_plan_json(pipe_json, devices[dev], opts)
            cases.append({"pipeline": pipe_json, "device": dev, "options": opts,
                          "status": 0, "plan": out})
        except O.RefError as e:
            cases.append({"pipeline": pipe_json, "device": dev, "options": opts,
                          "status": e.code, "plan": None})

    for dev in devices:
        plan_case(bundled, dev)
        for (w, h, f) in [(192, 432, 600), (800, 600, 1000), (800, 600, 16000),
                          (2048, 2048, 1000), (64, 64, 32), (13, 11, 7)]:
            plan_case(json.dumps(spec_chain(w, h, f, kalman=True)), dev)
        for part in ([[1, 1], [2, 2], [3, 3], [4, 4], [5, 5], [6, 6]],
                     [[1, 2], [3, 5], [6, 6]], [[1, 5], [6, 6]],
                     [[1, 3], [4, 5], [6, 6]], [[2, 4]], [[1, 4], [5, 6]]):
            plan_case(bundled, dev, {"force_partition": part})
            plan_case(json.dumps(spec_chain(192, 432, 600, kalman=True)), dev,
                      {"force_partition": part})
        plan_case(bundled, dev, {"halo_mode": "paper-max"})
        plan_case(bundled, dev, {"transfer_variant": "paper"})
        plan_case(bundled, dev, {"force_partition": [[1, 5], [6, 6]],
                                 "tile": {"x": 32, "y": 32, "t": 8}})
    # random single-channel chains over the catalog (helpers.hpp:67-112 ops)
    rng = np.random.default_rng(2024)
    pool = [("identity", {}), ("scale_offset", {"scale": 1.5, "offset": 3.0}),
            ("gaussian", {"radius": 1, "sigma": 1.0}), ("gradient", {}),
            ("threshold", {"th": 32.0}),
            ("box_mean", {"radius_x": 1, "radius_y": 1, "radius_t": 1}),
            ("iir_temporal", {"alpha": 0.25})]
    for trial in range(40):
        sizes = [8, 16, 24, 32]
        w, h, f = (int(rng.choice(sizes)), int(rng.choice(sizes)),
                   int(rng.choice(sizes)) // 2)
        n = int(rng.integers(2, 6))
        ks = []
        for i in range(n):
            op, params = pool[int(rng.integers(0, len(pool)))]
            ks.append({"name": f"{op}_{i + 1}", "stencil_op": op, "params": params})
        pipe = {"video": {"width": w, "height": h, "frames": f, "channels": 1},
                "kernels": ks}
        plan_case(json.dumps(pipe), "k20_like")
        plan_case(json.dumps(pipe), "c1060_like", {"halo_mode": "paper-max"})
    with open(os.path.join(HERE, "plans.json"), "w") as fh:
        json.dump(cases, fh, indent=1)
    print(f"plans.json: {len(cases)} cases, "
          f"{sum(c['status'] != 0 for c in cases)} errors")


if __name__ == "__main__":
    main()
