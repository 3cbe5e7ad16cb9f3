"""GPU parity: the sm_100a kernels, called through the C ABI, against the
reference's golden vectors and the oracle -- bit-exact for every element
(masks and float planes alike; the reference semantics are reproduced
operation for operation)."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN_CHAINS, load_golden

pytestmark = pytest.mark.gpu


def partitions(pipe):
    """No / Two / Full fusion + the optimizer's choice (capi.cpp:149-168)."""
    ks = pipe["kernels"]
    n = len(ks)
    agg = [i + 1 for i, k in enumerate(ks) if k["stencil_op"] == "kalman_track"]
    last = n - len(agg)
    tail = ",".join(str(a) for a in agg)
    none = ",".join(str(i) for i in range(1, last + 1))
    full = f"1-{last}" if last > 1 else "1"
    two = f"1-2,3-{last}" if last >= 3 else full
    out = {"none": none, "two": two, "full": full}
    return {k: (v + ("," + tail if tail else "")) for k, v in out.items()}


def run(fp, pipe, video, options=None, variant="auto", device="b200", torch_dev=None,
        chunk=0):
    p = fp.Pipeline(json.dumps(pipe))
    plan = fp.Plan(p, fp.Device.load(device), options)
    ex = fp.Executor(p, plan, variant=variant, host_chunk_frames=chunk)
    if torch_dev is not None:
        import torch
        v = torch.from_numpy(np.ascontiguousarray(video)).to(torch_dev)
        out = ex.run(v)
        torch.cuda.synchronize()
        return out.cpu().numpy().astype(np.float32), ex
    return ex.run(video).astype(np.float32), ex


@pytest.mark.parametrize("name", GOLDEN_CHAINS)
@pytest.mark.parametrize("part", ["default", "none", "two", "full"])
def test_golden_partitions(fp, cuda, name, part):
    g = load_golden(name)
    pipe = json.loads(str(g["pipeline"]))
    opts = None if part == "default" else {"force_partition": partitions(pipe)[part]}
    try:
        out, ex = run(fp, pipe, g["video"], opts, torch_dev=cuda)
    except fp.InfeasibleError:
        pytest.skip("partition infeasible under the device profile")
    np.testing.assert_array_equal(out, g["final"])


@pytest.mark.parametrize("name", GOLDEN_CHAINS)
@pytest.mark.parametrize("variant", ["exact", "auto"])
def test_golden_host_pointers_chunked(fp, cuda, name, variant):
    g = load_golden(name)
    pipe = json.loads(str(g["pipeline"]))
    out, _ = run(fp, pipe, g["video"], {"force_partition": partitions(pipe)["full"]},
                 variant=variant, chunk=3)
    np.testing.assert_array_equal(out, g["final"])


@pytest.mark.parametrize("name", [n for n in GOLDEN_CHAINS if "stages" in load_golden(n)])
def test_golden_every_stage_plane(fp, cuda, name):
    """Truncated chains expose every intermediate plane: each must equal the
    reference's stage_outputs[k] (simulator.hpp:37-42) bit for bit."""
    g = load_golden(name)
    pipe = json.loads(str(g["pipeline"]))
    for k in range(1, len(pipe["kernels"]) + 1):
        sub = dict(pipe, kernels=pipe["kernels"][:k])
        for part in ("none", "full"):
            opts = {"force_partition": partitions(sub)[part]}
            out, _ = run(fp, sub, g["video"], opts, torch_dev=cuda)
            np.testing.assert_array_equal(out, g["stages"][k - 1],
                                          err_msg=f"stage {k} {part}")


def test_f32_video_input(fp, cuda, oracle):
    g = load_golden("synth_64x48x20")
    pipe = json.loads(str(g["pipeline"]))
    rng = np.random.default_rng(3)
    v = (g["video"].astype(np.float32) + rng.uniform(-0.49, 0.49, g["video"].shape)
         ).clip(0, 255).astype(np.float32)
    want = oracle.orc_chain(pipe, v)
    for part in ("none", "two", "full"):
        out, _ = run(fp, pipe, v, {"force_partition": partitions(pipe)[part]},
                     torch_dev=cuda)
        np.testing.assert_array_equal(out, want, err_msg=part)


def test_larger_hash_video_dense_mask(fp, cuda, oracle):
    from paper_1509_04394_b200.fuseplan import hash_video_u8, spec_chain
    pipe = spec_chain(200, 150, 24, th=24.0)
    v = hash_video_u8(24, 4, 150, 200, 77)
    want = oracle.orc_chain(pipe, v)
    assert 0.05 < (want == 255).mean() < 0.95
    for part in ("none", "two", "full"):
        for variant in ("exact", "auto"):
            out, _ = run(fp, pipe, v, {"force_partition": partitions(pipe)[part]},
                         variant=variant, torch_dev=cuda)
            np.testing.assert_array_equal(out, want, err_msg=f"{part} {variant}")


@pytest.mark.parametrize("shape,th", [((64, 48, 20), 128.0), ((160, 120, 24), 24.0),
                                      ((192, 96, 17), 40.0), ((48, 37, 9), 24.0),
                                      ((800, 64, 6), 24.0), ((16, 8, 5), 12.0),
                                      ((256, 200, 11), 24.0), ((368, 131, 4), 30.0),
                                      ((240, 1, 3), 8.0), ((128, 300, 2), 24.0)])
def test_fast_certified_path_exact(fp, cuda, oracle, shape, th):
    """The certified FP32 frame pipeline (variant='fast' fails loudly if it does
    not apply; frames under 6 rows run 'auto', i.e. the FP64 kernel) is
    bit-exact, including pixels that took the FP64 recheck."""
    from paper_1509_04394_b200.fuseplan import hash_video_u8, spec_chain
    W, H, F = shape
    variant = "fast" if H >= 6 else "auto"
    pipe = spec_chain(W, H, F, th=th)
    v = hash_video_u8(F, 4, H, W, 4242)
    want = oracle.orc_chain(pipe, v)
    out, ex = run(fp, pipe, v, {"force_partition": "1-5"}, variant=variant, torch_dev=cuda)
    np.testing.assert_array_equal(out, want)
    assert ex.describe()["exact_rechecks_total"] >= 0


def test_fast_path_rechecks_happen_and_are_exact(fp, cuda, oracle):
    """A threshold placed in the bulk of the gradient distribution forces many
    pixels into the uncertain band; all of them must resolve exactly."""
    from paper_1509_04394_b200.fuseplan import hash_video_u8, spec_chain
    W, H, F = 128, 64, 12
    v = hash_video_u8(F, 4, H, W, 99)
    pipe = spec_chain(W, H, F, th=20.0)
    grads = oracle.orc_run_sequential(dict(pipe, kernels=pipe["kernels"][:4]), v)[-1]
    th = float(np.float32(np.median(grads)))
    pipe = spec_chain(W, H, F, th=th)
    want = oracle.orc_chain(pipe, v)
    p = fp.Pipeline(json.dumps(pipe))
    ex = fp.Executor(p, fp.Plan(p, fp.Device.load("b200"), {"force_partition": "1-5"}),
                     variant="fast")
    before = ex.describe()["exact_rechecks_total"]
    import torch
    out = ex.run(torch.from_numpy(v).to(cuda))
    torch.cuda.synchronize()
    after = ex.describe()["exact_rechecks_total"]
    assert after > before
    np.testing.assert_array_equal(out.cpu().numpy().astype(np.float32), want)


@pytest.mark.parametrize("part", ["1-5", "1-2,3-5"])
@pytest.mark.parametrize("shape,seed", [((240, 90, 7), 5), ((368, 131, 5), 6),
                                        ((2048, 64, 3), 7), ((64, 600, 3), 8),
                                        ((800, 600, 2), 9)])
def test_certified_kernels_forced_rechecks(fp, cuda, oracle, monkeypatch, part, shape, seed):
    """Every certified kernel (all-fused F12345 and the optimizer's F345 group
    on f32 IIR planes), with the pipe kernel's band scaled x1000 so that
    several % of all pixels take the exact FP64 recheck (and the per-warp
    recheck queue overflows): still bit-exact.  Shapes cover strips/bands
    that end inside the window, multi-wave grids and one-band videos."""
    from paper_1509_04394_b200.fuseplan import hash_video_u8, spec_chain
    monkeypatch.setenv("FUSEPLAN_PIPE_BAND_SCALE", "1000")
    W, H, F = shape
    pipe = spec_chain(W, H, F)
    v = hash_video_u8(F, 4, H, W, seed)
    want = oracle.orc_chain(pipe, v)
    p = fp.Pipeline(json.dumps(pipe))
    ex = fp.Executor(p, fp.Plan(p, fp.Device.load("b200"), {"force_partition": part}),
                     variant="fast" if part == "1-5" else "auto")
    import torch
    before = ex.describe()["exact_rechecks_total"]
    out = ex.run(torch.from_numpy(v).to(cuda))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out.cpu().numpy().astype(np.float32), want)
    assert ex.describe()["exact_rechecks_total"] - before > W * H * F // 50


@pytest.mark.parametrize("shape", [(64, 48, 9), (192, 432, 5), (800, 600, 3), (16, 1, 40)])
@pytest.mark.parametrize("alpha", [0.5, 0.3])
def test_f12_stream_kernel_exact(fp, cuda, oracle, monkeypatch, shape, alpha):
    """The bulk-copy F12 kernel (forced on for small frames too) writes the
    reference's exact IIR planes, for the default and a non-dyadic alpha,
    including state carry across a range split."""
    from paper_1509_04394_b200.fuseplan import hash_video_u8, spec_chain
    monkeypatch.setenv("FUSEPLAN_F12_STREAM", "1")
    W, H, F = shape
    pipe = spec_chain(W, H, F, alpha=alpha)
    pipe12 = dict(pipe, kernels=pipe["kernels"][:2])
    v = hash_video_u8(F, 4, H, W, 31)
    want = oracle.orc_run_sequential(pipe12, v)[-1]
    out, _ = run(fp, pipe12, v, {"force_partition": "1-2"}, torch_dev=cuda)
    np.testing.assert_array_equal(out, want)


def test_state_carry_and_warm_restart(fp, cuda, oracle):
    """run_range: resuming from the carried state is exact; a warm-up restart
    equals the oracle's restart semantics at the same frame."""
    import torch
    from paper_1509_04394_b200.fuseplan import hash_video_u8, spec_chain
    F = 30
    pipe = spec_chain(96, 64, F, th=24.0)
    v = hash_video_u8(F, 4, 64, 96, 5)
    full = oracle.orc_chain(pipe, v)
    p = fp.Pipeline(json.dumps(pipe))
    for part in ("1-5", "1-2,3-5", "1,2,3,4,5"):
        plan = fp.Plan(p, fp.Device.load("b200"), {"force_partition": part})
        ex = fp.Executor(p, plan)
        vt = torch.from_numpy(v).to(cuda)
        st = torch.empty((1, 64, 96), device=cuda)
        a = ex.run_range(vt[:13], state_out=st)
        b = ex.run_range(vt[13:], state_in=st)
        torch.cuda.synchronize()
        got = torch.cat([a, b]).cpu().numpy().astype(np.float32)
        np.testing.assert_array_equal(got, full, err_msg=part)
        # warm restart at frame 20 - 8
        w = ex.run_range(vt[12:], n_warm=8)
        torch.cuda.synchronize()
        want = oracle.orc_chain(pipe, v, t_begin=12, t_out=20)
        np.testing.assert_array_equal(w.cpu().numpy().astype(np.float32), want,
                                      err_msg=part)


def test_device_hash_generator_matches_host(fp, cuda):
    import torch
    from paper_1509_04394_b200.fuseplan import hash_video_u8, synth_hash_u8
    out = torch.empty((5, 4, 33, 47), dtype=torch.uint8, device=cuda)
    synth_hash_u8(out, t0=7, seed=1234)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out.cpu().numpy(), hash_video_u8(5, 4, 33, 47, 1234, 7))


def test_random_catalog_chains(fp, cuda, oracle):
    """The reference's randomized suites (test_simulator.cpp:228-243,
    acceptance.cpp:276-320) over the whole catalog, on the GPU executor."""
    rng = np.random.default_rng(2024)
    pool = [("identity", {}), ("scale_offset", {"scale": 1.5, "offset": 3.0}),
            ("gaussian", {"radius": 1, "sigma": 1.0}), ("gradient", {}),
            ("threshold", {"th": 32.0}),
            ("box_mean", {"radius_x": 1, "radius_y": 1, "radius_t": 1}),
            ("iir_temporal", {"alpha": 0.25})]
    for trial in range(30):
        w, h, f = (int(rng.choice([8, 16, 24, 32])), int(rng.choice([8, 16, 24, 32])),
                   int(rng.choice([8, 16, 24, 32])) // 2)
        ks = []
        for i in range(int(rng.integers(2, 6))):
            op, params = pool[int(rng.integers(0, len(pool)))]
            ks.append({"name": f"k{i}", "stencil_op": op, "params": params})
        pipe = {"video": {"width": w, "height": h, "frames": f, "channels": 1},
                "kernels": ks}
        vid = rng.uniform(0, 255, (f, 1, h, w)).astype(np.float32)
        want = oracle.orc_run_sequential(pipe, vid)[-1]
        for opts in (None, {"force_partition": ",".join(str(i + 1) for i in range(len(ks)))}):
            out, _ = run(fp, pipe, vid, opts, device="k20_like", torch_dev=cuda)
            np.testing.assert_array_equal(out, want, err_msg=f"trial {trial} {opts}")


def test_simulate_reports_identical_outputs(fp, cuda):
    """test_capi.cpp:136-160 through the GPU-backed fp_simulate."""
    pipe = fp.Pipeline(json.dumps({
        "video": {"width": 32, "height": 32, "frames": 6, "channels": 1},
        "kernels": [{"name": "smooth", "stencil_op": "gaussian",
                     "params": {"radius": 1, "sigma": 1.0}},
                    {"name": "bin", "stencil_op": "threshold", "params": {"th": 100}}]}))
    dev = fp.Device.load("k20_like")
    rep = fp.simulate(pipe, dev, synth={"width": 32, "height": 32, "frames": 6,
                                        "channels": 1,
                                        "markers": [{"x": 16, "y": 16, "radius": 4}]})
    assert "outputs identical: true" in rep
    assert "Full Fusion" in rep
    bundled = fp.Pipeline.load(fp.DATA_DIR + "/vision_pipeline.json")
    rep = fp.simulate(bundled, dev, synth={"width": 64, "height": 64, "frames": 32,
                                           "channels": 4, "noise_sigma": 8, "seed": 1234,
                                           "markers": [{"x": 20, "y": 20, "vx": 1}]})
    assert "outputs identical: true" in rep


@pytest.mark.parametrize("world,warmup", [(4, 64), (4, 2), (3, 0)])
def test_sharding_protocol_on_device_emulated(fp, cuda, oracle, world, warmup):
    """The T-shard protocol (sharding.py) with the sm_100a executor as the
    shard compute; ranks are emulated in order in one process with a mailbox
    for the carry planes (the real run sends them over NCCL)."""
    import torch
    from paper_1509_04394_b200.fuseplan import hash_video_u8, spec_chain
    from paper_1509_04394_b200.sharding import run_sharded, shard_of
    W, H, F = 96, 40, 60
    pipe = spec_chain(W, H, F, th=24.0)
    video = torch.from_numpy(hash_video_u8(F, 4, H, W, 31)).to(cuda)
    p = fp.Pipeline(json.dumps(pipe))
    ex = fp.Executor(p, fp.Plan(p, fp.Device.load("b200"), {"force_partition": "1-5"}))
    mailbox, outs, fixups = {}, {}, {"fixups": 0}

    for rank in range(world):
        sh = shard_of(rank, world, F, warmup)

        def run_shard(first, n, n_warm, state_in):
            st = torch.empty((1, H, W), device=cuda)
            o = ex.run_range(video[first:first + n], n_warm=n_warm, state_in=state_in,
                             state_out=st)
            return o, st

        out, _ = run_sharded(sh, run_shard,
                             lambda s, dst: mailbox.__setitem__(dst, s.clone()),
                             lambda src: mailbox.pop(sh.rank),
                             torch.equal, fixups)
        outs[rank] = out
    torch.cuda.synchronize()
    got = torch.cat([outs[r] for r in range(world)]).cpu().numpy().astype(np.float32)
    np.testing.assert_array_equal(got, oracle.orc_chain(pipe, video.cpu().numpy()))
    if warmup <= 2:
        assert fixups["fixups"] >= 1


@pytest.mark.parametrize("world,warmup", [(2, 64), (3, 2), (4, 64), (4, 1)])
@pytest.mark.parametrize("opts", [None, {"force_partition": "1-2,3,4-6"}])
def test_sharding_temporal_halo_on_device_emulated(fp, cuda, oracle, world, warmup, opts):
    """T-shards of a chain with a temporal box_mean window (SURVEY 8(f)
    rank 3) on the device executor: each rank runs its context (R = 2 halo
    frames each side, temporal windows clamped at the range ends by the range
    run), keeps its own frames, and carries the gray+IIR state taken before the
    next rank's context.  Bit-exact with the whole-video reference."""
    import torch
    from paper_1509_04394_b200.fuseplan import hash_video_u8
    from paper_1509_04394_b200.sharding import run_sharded, shard_of
    W, H, F = 96, 40, 60
    ks = [{"name": "g", "stencil_op": "rgba2gray"},
          {"name": "i", "stencil_op": "iir_temporal", "params": {"alpha": 0.5}},
          {"name": "b", "stencil_op": "box_mean",
           "params": {"radius_x": 1, "radius_y": 1, "radius_t": 2}},
          {"name": "s", "stencil_op": "gaussian", "params": {"radius": 2, "sigma": 1.0}},
          {"name": "d", "stencil_op": "gradient"},
          {"name": "t", "stencil_op": "threshold", "params": {"th": 24.0}}]
    pipe = {"video": {"width": W, "height": H, "frames": F, "channels": 4}, "kernels": ks}
    vnp = hash_video_u8(F, 4, H, W, 91)
    video = torch.from_numpy(vnp).to(cuda)
    p = fp.Pipeline(json.dumps(pipe))
    ex = fp.Executor(p, fp.Plan(p, fp.Device.load("b200"), opts))
    p12 = fp.Pipeline(json.dumps(dict(pipe, kernels=ks[:2])))
    ex12 = fp.Executor(p12, fp.Plan(p12, fp.Device.load("b200"), {"force_partition": "1-2"}))
    mailbox, outs, fixups = {}, {}, {"fixups": 0}

    def run_shard(first, n, n_warm, state_in):
        return ex.run_range(video[first:first + n], n_warm=n_warm, state_in=state_in), None

    def advance(first, n, state_in):
        st = torch.empty((1, H, W), device=cuda)
        ex12.run_range(video[first:first + n], n_warm=n, state_in=state_in, state_out=st)
        return st

    for rank in range(world):
        sh = shard_of(rank, world, F, warmup, t_halo=2)
        out, _ = run_sharded(sh, run_shard,
                             lambda s, dst: mailbox.__setitem__(dst, s.clone()),
                             lambda src: mailbox.pop(sh.rank),
                             torch.equal, fixups, advance=advance)
        outs[rank] = out
    torch.cuda.synchronize()
    got = torch.cat([outs[r] for r in range(world)]).cpu().numpy().astype(np.float32)
    want = oracle.orc_run_sequential(pipe, vnp.astype(np.float32))[-1]
    np.testing.assert_array_equal(got, want)
    if warmup <= 2:
        assert fixups["fixups"] >= 1


@pytest.mark.parametrize("part", ["1-5", "1-2,3-5"])
@pytest.mark.parametrize("segs,seg_warm", [(0, None), (4, None), (3, 1), (7, 2), (16, 64)])
@pytest.mark.parametrize("shape", [(192, 432, 300), (64, 48, 170)])
def test_pipe_time_segments_exact(fp, cuda, oracle, monkeypatch, part, segs, seg_warm, shape):
    """Time-segmented pipe launches (small frames: several CTAs per window,
    each over its own run of frames).  All-fused segments restart the IIR
    seg_warm frames early; a tiny seg_warm makes the seam verification fail
    and the device-side fix-up re-run from the first wrong segment.  Output
    and the carried end state stay bit-exact, with forced rechecks on top."""
    import torch
    from paper_1509_04394_b200.fuseplan import hash_video_u8, spec_chain
    if segs:
        monkeypatch.setenv("FUSEPLAN_PIPE_SEGS", str(segs))
    if seg_warm is not None:
        monkeypatch.setenv("FUSEPLAN_PIPE_SEG_WARM", str(seg_warm))
    monkeypatch.setenv("FUSEPLAN_PIPE_BAND_SCALE", "30")
    W, H, F = shape
    pipe = spec_chain(W, H, F)
    v = hash_video_u8(F, 4, H, W, 40 + segs)
    want = oracle.orc_chain(pipe, v)
    p = fp.Pipeline(json.dumps(pipe))
    ex = fp.Executor(p, fp.Plan(p, fp.Device.load("b200"), {"force_partition": part}),
                     variant="fast" if part == "1-5" else "auto")
    vt = torch.from_numpy(v).to(cuda)
    st = torch.empty((1, H, W), device=cuda)
    out = ex.run_range(vt[:F - 9], state_out=st)
    tail = ex.run_range(vt[F - 9:], state_in=st)
    torch.cuda.synchronize()
    got = torch.cat([out, tail]).cpu().numpy().astype(np.float32)
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("oh", [3, 4, 5, 8, 10, 12, 15])
@pytest.mark.parametrize("part", ["1-5", "1-2,3-5"])
@pytest.mark.parametrize("shape", [(256, 131, 6), (144, 31, 5), (64, 30, 4)])
def test_pipe_every_window_height_exact(fp, cuda, oracle, monkeypatch, oh, part, shape):
    """Every window height, on frame heights that are not multiples of it: the
    last band is shifted up to end at the video's bottom row (overlapping the
    band above), so the y clamps of the march sit at fixed steps.  Bit-exact
    with widened certification bands (forced rechecks)."""
    from paper_1509_04394_b200.fuseplan import hash_video_u8, spec_chain
    W, H, F = shape
    if 2 * oh > H:
        pytest.skip("window taller than the video")
    monkeypatch.setenv("FUSEPLAN_PIPE_OH", str(oh))
    monkeypatch.setenv("FUSEPLAN_PIPE_IMPL", "1")  # the row-pair pipeline (fc_pipe.cu)
    monkeypatch.setenv("FUSEPLAN_PIPE_BAND_SCALE", "100")
    pipe = spec_chain(W, H, F)
    v = hash_video_u8(F, 4, H, W, 70 + oh)
    want = oracle.orc_chain(pipe, v)
    out, _ = run(fp, pipe, v, {"force_partition": part},
                 variant="fast" if part == "1-5" else "auto", torch_dev=cuda)
    np.testing.assert_array_equal(out, want)


@pytest.mark.parametrize("out_rows", [6, 10, 14, 18, 22, 26, 29])
@pytest.mark.parametrize("shape", [(256, 131, 7), (136, 61, 6), (64, 37, 5)])
def test_pair_every_window_height_exact(fp, cuda, oracle, monkeypatch, out_rows, shape):
    """The frame-pair pipeline (fc_pipe2.cu) at every window height it is built
    for, on frame heights that are not multiples of it (the last band shifted
    up to end at the bottom row) and odd frame counts (a {A, A} tail pair):
    bit-exact with widened certification bands (forced rechecks)."""
    from paper_1509_04394_b200.fuseplan import hash_video_u8, spec_chain
    W, H, F = shape
    if out_rows > H:
        pytest.skip("window taller than the video")
    monkeypatch.setenv("FUSEPLAN_PIPE_OUT", str(out_rows))
    monkeypatch.setenv("FUSEPLAN_PIPE_BAND_SCALE", "100")
    pipe = spec_chain(W, H, F)
    v = hash_video_u8(F, 4, H, W, 170 + out_rows)
    want = oracle.orc_chain(pipe, v)
    out, ex = run(fp, pipe, v, {"force_partition": "1-5"}, variant="fast", torch_dev=cuda)
    assert "frame-pair" in ex.describe()["last_chain_kernel"]
    np.testing.assert_array_equal(out, want)


@pytest.mark.parametrize("out_rows", [0, 6, 14, 22, 29])
@pytest.mark.parametrize("shape,th", [((256, 131, 7), 30.0), ((192, 432, 61), 40.0),
                                      ((800, 600, 9), 20.0), ((64, 37, 5), 10.0),
                                      ((196, 50, 6), 25.0)])
def test_pair_exact_pipeline(fp, cuda, oracle, monkeypatch, out_rows, shape, th):
    """The exact frame-pair pipeline (variant "exact": FP64 gaussian in the
    reference's order, float Sobel, no certification) at several window
    heights, frame heights that are not multiples of them, odd frame counts
    and a width that needs the pitched copy (196): bit-exact, and it is the
    kernel that ran."""
    from paper_1509_04394_b200.fuseplan import hash_video_u8, spec_chain
    W, H, F = shape
    if out_rows > H:
        pytest.skip("window taller than the video")
    if out_rows:
        monkeypatch.setenv("FUSEPLAN_PIPE_OUT", str(out_rows))
    pipe = spec_chain(W, H, F, th=th)
    v = hash_video_u8(F, 4, H, W, 270 + out_rows)
    want = oracle.orc_chain(pipe, v)
    out, ex = run(fp, pipe, v, {"force_partition": "1-5"}, variant="exact", torch_dev=cuda)
    assert "exact FP64 frame-pair" in ex.describe()["last_chain_kernel"]
    np.testing.assert_array_equal(out, want)


@pytest.mark.parametrize("segs,seg_warm", [(0, None), (3, 1), (4, None)])
def test_pair_exact_segments_and_carry(fp, cuda, oracle, monkeypatch, segs, seg_warm):
    """The exact pipeline with time segments (forced seam fix-ups at a 1-frame
    warm-up) and a range run carrying the IIR state: bit-exact."""
    import torch
    from paper_1509_04394_b200.fuseplan import hash_video_u8, spec_chain
    if segs:
        monkeypatch.setenv("FUSEPLAN_PIPE_SEGS", str(segs))
    if seg_warm is not None:
        monkeypatch.setenv("FUSEPLAN_PIPE_SEG_WARM", str(seg_warm))
    W, H, F = 192, 96, 230
    pipe = spec_chain(W, H, F, th=30.0)
    v = hash_video_u8(F, 4, H, W, 77 + segs)
    want = oracle.orc_chain(pipe, v)
    p = fp.Pipeline(json.dumps(pipe))
    ex = fp.Executor(p, fp.Plan(p, fp.Device.load("b200"), {"force_partition": "1-5"}),
                     variant="exact")
    vt = torch.from_numpy(v).to(cuda)
    st = torch.empty((1, H, W), device=cuda)
    out = ex.run_range(vt[:F - 11], state_out=st)
    tail = ex.run_range(vt[F - 11:], state_in=st)
    torch.cuda.synchronize()
    assert "exact FP64 frame-pair" in ex.describe()["last_chain_kernel"]
    got = torch.cat([out, tail]).cpu().numpy().astype(np.float32)
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("tiles", [False, True])
@pytest.mark.parametrize("out_rows,segs", [(0, 0), (6, 0), (14, 3), (29, 0), (22, 7)])
@pytest.mark.parametrize("shape,th", [((256, 131, 7), 30.0), ((192, 432, 61), 40.0),
                                      ((800, 600, 9), 20.0), ((64, 37, 5), 10.0),
                                      ((196, 50, 6), 25.0), ((98, 40, 4), 15.0)])
def test_f345_exact_pipeline(fp, cuda, oracle, monkeypatch, tiles, out_rows, segs, shape, th):
    """The exact F345 group of the reference planner's `1-2,3-5` (gaussian +
    Sobel + threshold on the f32 IIR planes, variant "exact") on the exact
    frame-pair pipeline with the plane-loader role -- window heights, time
    segments (stateless), odd frame counts, widths that are not multiples of
    128 -- and, forced, on the FP64 tiles (and for a width the pipeline does
    not take, 98): bit-exact either way, and the expected kernel ran."""
    from paper_1509_04394_b200.fuseplan import hash_video_u8, spec_chain
    W, H, F = shape
    if out_rows > H:
        pytest.skip("window taller than the video")
    if out_rows:
        monkeypatch.setenv("FUSEPLAN_PIPE_OUT", str(out_rows))
    if segs:
        monkeypatch.setenv("FUSEPLAN_PIPE_SEGS", str(segs))
    if tiles:
        monkeypatch.setenv("FUSEPLAN_PIPE_IMPL", "3")
    pipe = spec_chain(W, H, F, th=th)
    v = hash_video_u8(F, 4, H, W, 310 + out_rows + segs)
    want = oracle.orc_chain(pipe, v)
    out, ex = run(fp, pipe, v, {"force_partition": "1-2,3-5"}, variant="exact", torch_dev=cuda)
    kern = ex.describe()["last_chain_kernel"]
    if tiles or W % 4:
        assert "exact FP64 tiles on f32 planes" in kern, kern
    else:
        assert "exact FP64 frame-pair pipeline on f32 planes" in kern, kern
    np.testing.assert_array_equal(out, want)


@pytest.mark.parametrize("shape", [(128, 64, 1), (128, 64, 2), (256, 30, 3), (1024, 12, 7)])
@pytest.mark.parametrize("segs", [0, 2, 5])
def test_pipe_tiny_frame_counts_exact(fp, cuda, oracle, monkeypatch, shape, segs):
    """1-7 frames (single-frame launches, more segments than frames asked
    for, one-band videos): bit-exact, carried end state included."""
    import torch
    from paper_1509_04394_b200.fuseplan import hash_video_u8, spec_chain
    if segs:
        monkeypatch.setenv("FUSEPLAN_PIPE_SEGS", str(segs))
    W, H, F = shape
    pipe = spec_chain(W, H, F + 3, th=40.0)
    v = hash_video_u8(F + 3, 4, H, W, 500 + F)
    want = oracle.orc_chain(pipe, v)
    p = fp.Pipeline(json.dumps(pipe))
    ex = fp.Executor(p, fp.Plan(p, fp.Device.load("b200"), {"force_partition": "1-5"}),
                     variant="fast")
    vt = torch.from_numpy(v).to(cuda)
    st = torch.empty((1, H, W), device=cuda)
    a = ex.run_range(vt[:F], state_out=st)
    b = ex.run_range(vt[F:], state_in=st)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(torch.cat([a, b]).cpu().numpy().astype(np.float32), want)


@pytest.mark.parametrize("case", ["paper_max", "iir_split", "exact"])
def test_simulate_matches_reference_run_tiled(fp, cuda, oracle, tmp_path, case):
    """fp_simulate's report against the reference's own executors
    (oracle/_ref: run_sequential, run_tiled, simulator.cpp:158-333): the same
    diff count and max |diff| (a PaperMax plan under-stages the halo and
    erodes tile edges; a forced tile shorter than the video restarts the IIR
    per box), every diff classified (interior + boundary), and the
    reference's gmem element tallies."""
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    W, H, F = 160, 120, 12
    spec = fp.spec_chain(W, H, F, th=24.0, kalman=True)
    if case == "paper_max":
        opts = {"halo_mode": "paper-max"}
    elif case == "iir_split":
        opts = {"force_partition": "1-5,6", "tile": {"x": 8, "y": 8, "t": 4}}
    else:
        opts = None
    dev_json = open(os.path.join(fp.DATA_DIR, "k20_like.json")).read()
    from paper_1509_04394_b200.fuseplan import hash_video_u8
    video = hash_video_u8(F, 4, H, W, 77)
    path = str(tmp_path / "v.fpvd")
    fp.write_fpvd(path, video)
    pj = json.dumps(spec)
    seq, _ = oracle.ref_run_sequential(pj, video)
    tiled, traffic = oracle.ref_run_tiled(pj, dev_json, video, opts)
    diff = np.abs(seq - tiled)
    want_count = int((diff != 0).sum())
    if case != "exact":
        assert want_count > 0  # the case exercises erosion
    rep = json.loads(fp.simulate(fp.Pipeline(pj), fp.Device(dev_json), opts, video_path=path,
                                 fmt="json"))
    sim = rep["simulation"]
    assert sim["diff_count"] == want_count
    assert sim["max_abs_diff"] == pytest.approx(float(diff.max()) if want_count else 0.0)
    assert sim["interior_diffs"] + sim["boundary_diffs"] == want_count
    assert sim["outputs_identical"] == (want_count == 0)
    assert sim["measured_tiled_gmem"] == int(traffic[0] + traffic[1])
    assert sim["measured_serial_gmem"] == 2 * W * H * F * 5


@pytest.mark.parametrize("alpha", [0.3, 0.0, 1.0, 0.75])
def test_certified_pipeline_any_alpha(fp, cuda, oracle, alpha):
    """The frame pipeline takes any IIR alpha in [0, 1] (the reference's
    fl(fl(a x) + fl((1 - a) y)) update in the IIR warps), not only the folded
    alpha = 0.5 form: bit-exact, no drop to the FP64 kernel."""
    from paper_1509_04394_b200.fuseplan import hash_video_u8, spec_chain
    W, H, F = 256, 96, 30
    pipe = spec_chain(W, H, F, alpha=alpha, th=30.0)
    v = hash_video_u8(F, 4, H, W, 17)
    want = oracle.orc_chain(pipe, v)
    out, ex = run(fp, pipe, v, {"force_partition": "1-5"}, variant="fast", torch_dev=cuda)
    np.testing.assert_array_equal(out, want)
    assert "certified" in ex.describe()["last_chain_kernel"]


@pytest.mark.parametrize("shape,offset", [((204, 97, 12), 0), ((252, 64, 9), 0),
                                          ((256, 64, 9), 1), ((100, 40, 20), 3)])
def test_certified_pipeline_any_width_and_base(fp, cuda, oracle, shape, offset):
    """Widths that are not a multiple of 16 and video bases that are not
    16-byte aligned (a view at a byte offset) run the frame pipeline on a
    pitched copy of the R, G, B planes instead of the FP64 kernel."""
    import torch
    from paper_1509_04394_b200.fuseplan import hash_video_u8, spec_chain
    W, H, F = shape
    pipe = spec_chain(W, H, F, th=30.0)
    v = hash_video_u8(F, 4, H, W, 23)
    want = oracle.orc_chain(pipe, v)
    big = torch.empty(v.size + offset, dtype=torch.uint8, device=cuda)
    dv = big[offset:].view(F, 4, H, W)
    dv.copy_(torch.from_numpy(v))
    p = fp.Pipeline(json.dumps(pipe))
    ex = fp.Executor(p, fp.Plan(p, fp.Device.load("b200"), {"force_partition": "1-5"}),
                     variant="fast")
    out = ex.run(dv)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out.cpu().numpy().astype(np.float32), want)
    kern = ex.describe()["last_chain_kernel"]
    assert "certified" in kern
    assert ("pitched" in kern) == (W % 16 != 0 or offset != 0)


def _fuzz_cases(n, seed):
    rng = np.random.default_rng(seed)
    for i in range(n):
        big = i % 5 == 0
        W = int(rng.integers(4, 1100 if big else 520))
        H = int(rng.integers(6, 700 if big else 260))
        F = int(rng.integers(1, 12 if big else 48))
        alpha = float(rng.choice([0.5, 0.5, 0.25, 0.8125, 0.37]))
        sigma = float(rng.choice([1.0, 1.0, 0.7, 1.6]))
        th = float(rng.choice([8.0, 20.0, 45.0, 128.0]))
        yield i, (W, H, F, alpha, sigma, th, int(rng.integers(1 << 30)))


@pytest.mark.parametrize("part,variant", [("1-5", "auto"), ("1-5", "exact"),
                                          ("1-2,3-5", "auto"), ("1-2,3-5", "exact")])
@pytest.mark.parametrize("case", list(_fuzz_cases(40, 4242)), ids=lambda c: f"c{c[0]}")
def test_fuzz_shapes_every_pipeline(fp, cuda, oracle, part, variant, case):
    """Random frame sizes (any width / height, 1-47 frames), IIR alphas,
    gaussian sigmas and thresholds through every fused pipeline the executor
    routes to (certified / exact frame-pair, row-pair F345, exact F345 on
    planes, the FP64 tile fallbacks for shapes outside them): bit-exact."""
    from paper_1509_04394_b200.fuseplan import hash_video_u8, spec_chain
    _, (W, H, F, alpha, sigma, th, seed) = case
    pipe = spec_chain(W, H, F, alpha=alpha, sigma=sigma, th=th)
    v = hash_video_u8(F, 4, H, W, seed)
    want = oracle.orc_chain(pipe, v)
    out, ex = run(fp, pipe, v, {"force_partition": part}, variant=variant, torch_dev=cuda)
    np.testing.assert_array_equal(out, want, err_msg=ex.describe()["last_chain_kernel"])


@pytest.mark.parametrize("shape,part,variant", [((192, 432, 600), "1-5", "auto"),
                                                ((192, 432, 120), "1-5", "exact"),
                                                ((136, 61, 40), "1-5", "auto"),
                                                ((256, 96, 50), "1-2,3-5", "auto"),
                                                ((128, 64, 30), "1,2,3,4,5", "auto")])
def test_graph_capture_replay(fp, cuda, oracle, shape, part, variant):
    """A run captured as a CUDA graph (fp_exec_graph_create; config 1 takes
    three launches: time segments, seam check, fix-up) replays bit-exact, and
    a replay after refilling the video in place gives the new video's mask."""
    import torch
    from paper_1509_04394_b200.fuseplan import hash_video_u8, spec_chain
    W, H, F = shape
    pipe = spec_chain(W, H, F, th=30.0)
    p = fp.Pipeline(json.dumps(pipe))
    ex = fp.Executor(p, fp.Plan(p, fp.Device.load("b200"), {"force_partition": part}),
                     variant=variant)
    v1 = hash_video_u8(F, 4, H, W, 11)
    v2 = hash_video_u8(F, 4, H, W, 12)
    dv = torch.from_numpy(v1).to(cuda)
    g = ex.capture(dv)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(g.out.cpu().numpy().astype(np.float32),
                                  oracle.orc_chain(pipe, v1))
    g.out.zero_()
    dv.copy_(torch.from_numpy(v2))
    g.launch()
    g.launch()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(g.out.cpu().numpy().astype(np.float32),
                                  oracle.orc_chain(pipe, v2))
    g.close()


@pytest.mark.parametrize("part,variant", [("1-5", "exact"), ("1-5", "auto"),
                                          ("1-2,3-5", "exact"), ("1-2,3-5", "auto"),
                                          ("1,2,3,4,5", "auto")])
def test_threshold_at_exact_gradient_values(fp, cuda, oracle, part, variant):
    """Adversarial thresholds: th equal to gradient magnitudes the reference
    actually produces, so pixels sit exactly on the decision boundary and a
    one-ulp difference anywhere in the gaussian / Sobel / m arithmetic (e.g.
    a contracted multiply-add) flips them.  Every fused route stays exact."""
    from paper_1509_04394_b200.fuseplan import hash_video_u8, spec_chain
    W, H, F = 200, 120, 8
    v = hash_video_u8(F, 4, H, W, 2718)
    grad = oracle.orc_run_sequential(spec_chain(W, H, F), v)[3]
    vals = np.unique(grad[grad > 1.0])
    rng = np.random.default_rng(5)
    for th in rng.choice(vals, 48, replace=False):
        pipe = spec_chain(W, H, F, th=float(th))
        want = np.where(grad >= th, np.float32(255), np.float32(0))  # simulator.cpp:84-89
        out, ex = run(fp, pipe, v, {"force_partition": part}, variant=variant, torch_dev=cuda)
        np.testing.assert_array_equal(out, want, err_msg=f"th={float(th)!r} "
                                      f"{ex.describe()['last_chain_kernel']}")
