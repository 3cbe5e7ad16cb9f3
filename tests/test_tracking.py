"""K6 tracking: the oracle restatement against the
reference's own behavioural tests (CPU), and the device kernel against the
restatement bit for bit (GPU)."""
import json
import math
import os

import numpy as np
import pytest

from conftest import ROOT


@pytest.fixture(scope="module")
def tro():
    from oracle import tracking_oracle
    return tracking_oracle


def scene(oracle, spec):
    """Reference synth_video (u8 FPVD round trip) of a 1-channel scene."""
    return oracle.ref_synth_u8(spec)[:, 0]


def threshold_mask(oracle, video, th=128.0, smooth_r=0):
    F, H, W = video.shape
    ks = []
    if smooth_r:
        ks.append({"name": "s", "stencil_op": "gaussian", "params": {"radius": smooth_r,
                                                                    "sigma": 1.0}})
    ks.append({"name": "t", "stencil_op": "threshold", "params": {"th": th}})
    pipe = {"video": {"width": W, "height": H, "frames": F, "channels": 1}, "kernels": ks}
    return oracle.orc_run_sequential(pipe, video[:, None])[-1]


def static_case(oracle):
    spec = {"width": 64, "height": 64, "frames": 30, "channels": 1,
            "markers": [{"x": 31.0, "y": 24.0, "vx": 0.0, "vy": 0.0, "radius": 3.0}]}
    return threshold_mask(oracle, scene(oracle, spec)), [(25, 18, 15, 15)]


def two_marker_case(oracle, frames=200):
    spec = {"width": 64, "height": 64, "frames": frames, "channels": 1, "noise_sigma": 8.0,
            "seed": 1234,
            "markers": [{"x": 10.0, "y": 10.0, "vx": 1.0, "vy": 0.0, "radius": 3.0},
                        {"x": 20.0, "y": 30.0, "vx": 0.5, "vy": 0.5, "radius": 3.0}]}
    return spec, threshold_mask(oracle, scene(oracle, spec), smooth_r=1)


def test_static_marker_converges(oracle, tro):
    """test_tracking.cpp:103-117: an off-centre ROI snaps onto a static marker."""
    if not oracle.ref_available():
        pytest.skip("reference build not available")
    mask, rois = static_case(oracle)
    pts = tro.track_features(mask, rois)
    last = pts[0, -1]
    assert last[0] == 1.0
    assert abs(last[3] - 31.0) < 0.5 and abs(last[4] - 24.0) < 0.5
    assert abs(last[5]) < 0.1


def test_acceptance_tracking_rmse(oracle, tro):
    """acceptance.cpp:440-480: two moving markers in noise, gaussian r1 +
    threshold 128 mask, worst per-frame RMSE <= 1.5 px after frame 20."""
    if not oracle.ref_available():
        pytest.skip("reference build not available")
    spec, mask = two_marker_case(oracle)
    rois = tro.marker_rois(spec["markers"])
    pts = tro.track_features(mask, rois)
    truth = tro.truth_centers(spec)
    worst = 0.0
    for t in range(21, spec["frames"]):
        sq = sum((pts[i, t, 3] - truth[i][t][0]) ** 2 + (pts[i, t, 4] - truth[i][t][1]) ** 2
                 for i in range(2))
        worst = max(worst, math.sqrt(sq / 2))
    assert worst <= 1.5, worst


def test_csv_format(tro):
    """trajectories_to_csv: header, 1-based marker ids, empty measurement
    columns on missing frames, %.9g numbers."""
    pts = np.zeros((1, 2, 23))
    pts[0, 0, :7] = [1.0, 1.5, 2.25, 1.0 / 3.0, 4.0, 0.0, -1e-5]
    pts[0, 1, 3:7] = [10.0, 11.0, 0.5, 0.25]
    csv = tro.trajectories_csv(pts)
    lines = csv.splitlines()
    assert lines[0] == "frame,marker_id,meas_x,meas_y,est_x,est_y,est_vx,est_vy"
    assert lines[1] == "0,1,1.5,2.25,0.333333333,4,0,-1e-05"
    assert lines[2] == "1,1,,,10,11,0.5,0.25"


def test_lround_matches_cpp(tro):
    for v, want in [(2.5, 3), (-2.5, -3), (2.4999999999999996, 2), (-0.5, -1), (0.5, 1),
                    (7.0, 7), (-7.2, -7), (1e6 + 0.5, 1000001)]:
        assert tro._lround(v) == want, v


@pytest.mark.gpu
def test_device_tracking_matches_oracle(fp, cuda, oracle, tro):
    """Device K6 == restatement, every field of every point, on the static
    and the two-marker scenes, u8 and f32 masks, host and device pointers."""
    import torch
    from paper_1509_04394_b200.fuseplan import track_features
    if not oracle.ref_available():
        pytest.skip("reference build not available")
    mask, rois = static_case(oracle)
    want = tro.track_features(mask, rois)
    got, csv = track_features(mask.astype(np.uint8), rois)
    np.testing.assert_array_equal(got, want)
    assert csv == tro.trajectories_csv(want)
    spec, mask2 = two_marker_case(oracle)
    rois2 = tro.marker_rois(spec["markers"])
    want2 = tro.track_features(mask2, rois2)
    for m in (mask2.astype(np.float32), torch.from_numpy(mask2.astype(np.uint8)).to(cuda)):
        got2, csv2 = track_features(m, rois2)
        np.testing.assert_array_equal(got2, want2)
        assert csv2 == tro.trajectories_csv(want2)


@pytest.mark.gpu
def test_device_tracking_edges(fp, cuda, tro):
    """ROIs partly / wholly outside the frame, a marker that disappears (no
    measurement -> prediction only), parameters other than the defaults."""
    from paper_1509_04394_b200.fuseplan import track_features
    rng = np.random.default_rng(5)
    F, H, W = 40, 48, 80
    mask = np.zeros((F, H, W), np.uint8)
    for t in range(F):
        if t < 25:
            cx, cy = 5 + t, 3 + t // 3
            mask[t, max(cy - 2, 0):cy + 3, max(cx - 2, 0):cx + 3] = 255
        mask[t] |= (rng.random((H, W)) < 0.01).astype(np.uint8) * 255
    rois = [(-4, -4, 13, 13), (70, 40, 15, 15), (100, 100, 5, 5)]
    want = tro.track_features(mask, rois, q=0.05, r=0.5, p0=3.0)
    got, _ = track_features(mask, rois, q=0.05, r=0.5, p0=3.0)
    np.testing.assert_array_equal(got, want)
    assert (want[0, 25:, 0] == 0).any()  # the marker vanished


@pytest.mark.gpu
def test_simulate_writes_track_csv(fp, cuda, tmp_path, tro, oracle):
    """fp_simulate with a tracking stage writes the reference's CSV
    (test_capi.cpp:162-185), equal to the restatement on the GPU mask."""
    import ctypes
    pipe = {"video": {"width": 32, "height": 32, "frames": 6, "channels": 1},
            "kernels": [{"name": "smooth", "stencil_op": "gaussian",
                         "params": {"radius": 1, "sigma": 1.0}},
                        {"name": "bin", "stencil_op": "threshold", "params": {"th": 100}},
                        {"name": "track", "stencil_op": "kalman_track"}]}
    synth = {"width": 32, "height": 32, "frames": 6, "channels": 1, "noise_sigma": 4.0,
             "seed": 7, "markers": [{"x": 12.0, "y": 14.0, "vx": 1.0, "vy": 0.5,
                                     "radius": 3.0}]}
    p = fp.Pipeline(json.dumps(pipe))
    d = fp.Device.load("k20_like")
    csv = tmp_path / "track.csv"
    out = ctypes.c_void_p()
    L = fp.lib()
    st = L.fp_simulate(p.ptr, d.ptr, None, None, json.dumps(synth).encode(),
                       str(csv).encode(), b"json", 0, ctypes.byref(out))
    assert st == 0, L.fp_last_error()
    L.fp_string_free(out)
    text = csv.read_text()
    assert text.startswith("frame,marker_id,")
    if oracle.ref_available():
        video = oracle.ref_synth_u8(synth)[:, 0]
        mask = oracle.orc_run_sequential(pipe, video[:, None])[-1]
        want = tro.trajectories_csv(tro.track_features(mask, tro.marker_rois(synth["markers"])))
        assert text == want
