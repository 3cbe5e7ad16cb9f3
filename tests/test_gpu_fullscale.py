"""Full-volume GPU parity at the BASELINE configurations.

The reference's contract for the path is "GPU mask == run_sequential(p,
v).final_output" (/root/reference/proj/src/simulator.cpp:158-177, SURVEY.md
8(c)).  These tests check EVERY frame of the BASELINE shapes -- not a sample
-- against the streaming C restatement (oracle/fusechain_oracle.c, pinned to
the reference build by tests/test_oracle.py), run in chunks with the IIR
state carried from chunk to chunk (the restatement's state_in / state_out).

They also cover the edge cases the certified kernels rely on: IIR decay into
subnormals (no FTZ anywhere), and a dense-recheck volume where a large share
of pixels fall inside the certification band and take the exact FP64 path.
"""
import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

MARKERS = [  # two markers, r = 3, intensity 255
    {"x": 20.0, "y": 30.0, "vx": 1.0, "vy": 0.0, "radius": 3.0, "intensity": 255.0},
    {"x": 100.0, "y": 200.0, "vx": 0.5, "vy": 0.5, "radius": 3.0, "intensity": 255.0},
]


def _executor(fp, pipe, partition, variant="auto"):
    p = fp.Pipeline(json.dumps(pipe))
    opts = None if partition == "plan" else {"force_partition": partition}
    return fp.Executor(p, fp.Plan(p, fp.Device.load("b200"), opts), variant=variant)


def _oracle_mismatches(oracle, pipe, video_dev, mask_dev, chunk=100, state=None,
                       first=0, count=None):
    """Compare mask_dev[first : first+count] with the oracle, chunk by chunk
    with the IIR state carried.  `state` is the oracle IIR state before frame
    `first` (None: frame `first` starts the recurrence, i.e. first == 0).
    Returns (frames checked, mismatching pixels, state after the last frame)."""
    F = int(video_dev.shape[0]) if count is None else first + count
    bad = 0
    checked = 0
    for a in range(first, F, chunk):
        b = min(F, a + chunk)
        v = video_dev[a:b].cpu().numpy()
        want, state = oracle.orc_chain(pipe, v, state_in=state, return_state=True)
        got = mask_dev[a:b].cpu().numpy()
        bad += int(np.count_nonzero(got.astype(np.float32) != want))
        checked += b - a
    return checked, bad, state


def _iir_state(oracle, pipe, video_dev, lo, hi, chunk=100, state=None):
    """Oracle gray+IIR state after frames [lo, hi) (state: before lo)."""
    sub = dict(pipe, kernels=pipe["kernels"][:2])
    for a in range(lo, hi, chunk):
        b = min(hi, a + chunk)
        _, state = oracle.orc_chain(sub, video_dev[a:b].cpu().numpy(), state_in=state,
                                    return_state=True)
    return state


@pytest.mark.parametrize("partition", ["plan", "1-2,3-5,6"])
def test_cfg3_800x600x1000_every_frame(fp, cuda, oracle, partition):
    """BASELINE config 3 (the headline workload): all 1000 frames, bit-exact."""
    import torch
    W, H, F = 800, 600, 1000
    pipe = fp.spec_chain(W, H, F, kalman=True)
    video = torch.empty((F, 4, H, W), dtype=torch.uint8, device=cuda)
    fp.synth_hash_u8(video, seed=1234)
    ex = _executor(fp, pipe, partition)
    mask = ex.run(video)
    torch.cuda.synchronize()
    checked, bad, _ = _oracle_mismatches(oracle, pipe, video, mask)
    assert checked == F and bad == 0, f"{bad} mismatching pixels over {checked} frames"


def _ref_scene(oracle, W, H, F):
    if not oracle.ref_available():
        pytest.skip("oracle/_ref (the reference build) is not present")
    spec = {"width": W, "height": H, "frames": F, "channels": 4, "noise_sigma": 8.0,
            "seed": 1234, "markers": MARKERS}
    return oracle.ref_synth_u8(spec)


@pytest.mark.parametrize("scene", ["hash", "reference_synth"])
@pytest.mark.parametrize("partition", ["plan", "1-2,3-5,6", "1,2,3,4,5,6"])
def test_cfg1_192x432x600_every_frame(fp, cuda, oracle, scene, partition):
    """BASELINE configs 1-2: the optimizer's partition on the b200 profile
    (all-fused 1-5 under the streaming cost model), the reference model's
    1-2,3-5 and the unfused chain,
    on the counter-hash video and on the reference's own marker scene
    (synth_video, synth.cpp:35-78, quantised through FPVD, video.cpp:57)."""
    import torch
    W, H, F = 192, 432, 600
    pipe = fp.spec_chain(W, H, F, kalman=True)
    if scene == "hash":
        video = torch.empty((F, 4, H, W), dtype=torch.uint8, device=cuda)
        fp.synth_hash_u8(video, seed=5150)
    else:
        video = torch.from_numpy(_ref_scene(oracle, W, H, F)).to(cuda)
    ex = _executor(fp, pipe, partition)
    mask = ex.run(video)
    torch.cuda.synchronize()
    checked, bad, _ = _oracle_mismatches(oracle, pipe, video, mask, chunk=200)
    assert checked == F and bad == 0, f"{bad} mismatching pixels over {checked} frames"
    if scene == "reference_synth":
        assert int((mask == 255).sum()) > 0  # the markers' rims are found


def test_cfg5_2048x2048_long_march_windows(fp, cuda, oracle):
    """BASELINE config 5 (2048x2048x1000): the first 64 frames and two
    16-frame windows deep in the march (frames 500-515 and 984-999), the
    oracle resumed there from its own gray+IIR state."""
    import torch
    W, H, F = 2048, 2048, 1000
    pipe = fp.spec_chain(W, H, F, kalman=True)
    video = torch.empty((F, 4, H, W), dtype=torch.uint8, device=cuda)
    fp.synth_hash_u8(video, seed=1234)
    ex = _executor(fp, pipe, "1-5,6")
    mask = ex.run(video)
    torch.cuda.synchronize()
    total = 0
    c, bad, st = _oracle_mismatches(oracle, pipe, video, mask, chunk=16, count=64)
    assert bad == 0, f"frames 0-63: {bad} mismatching pixels"
    total += c
    st = _iir_state(oracle, pipe, video, 64, 500, state=st)
    c, bad, st = _oracle_mismatches(oracle, pipe, video, mask, chunk=16, state=st,
                                    first=500, count=16)
    assert bad == 0, f"frames 500-515: {bad} mismatching pixels"
    total += c
    st = _iir_state(oracle, pipe, video, 516, 984, state=st)
    c, bad, _ = _oracle_mismatches(oracle, pipe, video, mask, chunk=16, state=st,
                                   first=984, count=16)
    assert bad == 0, f"frames 984-999: {bad} mismatching pixels"
    assert total + c == 96


def test_cfg4_800x600x16000_every_frame(fp, cuda, oracle):
    """BASELINE config 4's length: 16000 frames (16 s at 1000 fps) in one
    device launch, every frame checked against the oracle with its IIR state
    carried across 160 chunks."""
    import torch
    W, H, F = 800, 600, 16000
    pipe = fp.spec_chain(W, H, F, kalman=True)
    video = torch.empty((F, 4, H, W), dtype=torch.uint8, device=cuda)
    fp.synth_hash_u8(video, seed=2024)
    p = fp.Pipeline(json.dumps(pipe))
    plan = fp.Plan(p, fp.Device.load("b200"), {"force_partition": "1-5,6",
                                                "iir_streaming": True})
    ex = fp.Executor(p, plan)
    mask = ex.run(video)
    torch.cuda.synchronize()
    checked, bad, _ = _oracle_mismatches(oracle, pipe, video, mask, chunk=200)
    assert checked == F and bad == 0, f"{bad} mismatching pixels over {checked} frames"


@pytest.mark.parametrize("partition", ["1-5,6", "1-2,3-5,6", "1,2,3,4,5,6"])
def test_iir_decays_into_subnormals_exactly(fp, cuda, oracle, partition):
    """A bright frame followed by 200 black frames: the IIR state halves
    every frame and passes through the float subnormal range (frames ~130-160)
    down to zero.  Any flush-to-zero or reassociation would change the state
    planes and, through the later bright frames, the masks."""
    import torch
    W, H, F = 256, 128, 232
    rng = np.random.default_rng(11)
    v = np.zeros((F, 4, H, W), np.uint8)
    v[0] = rng.integers(0, 256, (4, H, W), dtype=np.uint8)
    v[0, :, 40:80, 100:160] = 255
    v[201:] = rng.integers(0, 256, (F - 201, 4, H, W), dtype=np.uint8)
    pipe = fp.spec_chain(W, H, F, th=2.0, kalman=True)
    # the state planes themselves: gray + IIR only, every frame
    sub = dict(pipe, kernels=pipe["kernels"][:2])
    want_iir = oracle.orc_chain(sub, v)
    assert (np.abs(want_iir[150]) < np.finfo(np.float32).tiny).any()  # subnormals occur
    assert (want_iir[150] > 0).any()
    ex12 = _executor(fp, sub, "1-2")
    got_iir = ex12.run(torch.from_numpy(v).to(cuda))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(got_iir.cpu().numpy().view(np.uint32),
                                  want_iir.view(np.uint32))
    want = oracle.orc_chain(pipe, v)
    ex = _executor(fp, pipe, partition)
    got = ex.run(torch.from_numpy(v).to(cuda))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(got.cpu().numpy().astype(np.float32), want)


def test_dense_rechecks_full_frame_exact(fp, cuda, oracle):
    """800x600 frames with the threshold at the median gradient: a large share
    of all pixels lies inside the certification band and takes the exact
    FP64 recheck; every decision must still be the reference's."""
    import torch
    W, H, F = 800, 600, 48
    video = torch.empty((F, 4, H, W), dtype=torch.uint8, device=cuda)
    fp.synth_hash_u8(video, seed=31)
    v = video.cpu().numpy()
    pipe = fp.spec_chain(W, H, F)
    grads = oracle.orc_chain(dict(pipe, kernels=pipe["kernels"][:4]), v[:8])
    th = float(np.float32(np.median(grads[4:])))
    pipe = fp.spec_chain(W, H, F, th=th, kalman=True)
    ex = _executor(fp, pipe, "1-5,6")
    before = ex.describe()["exact_rechecks_total"]
    mask = ex.run(video)
    torch.cuda.synchronize()
    after = ex.describe()["exact_rechecks_total"]
    assert after - before > 0.001 * W * H * F, f"only {after - before} rechecks"
    checked, bad, _ = _oracle_mismatches(oracle, pipe, video, mask, chunk=16)
    assert checked == F and bad == 0, f"{bad} mismatching pixels"
