"""Multi-GPU through the C ABI (fp_shard_exec_*, fp_exec_converge): the video
T-sharded over several "devices" -- on the one-GPU test box they are the same
B200 named several times, which exercises the whole protocol (per-rank
executors and streams, carry copies, convergence check, rank-ordered repair)
-- bit-exact against the oracle, with warm-ups long enough to need no repair
and short enough to force repairs."""
import json
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("devices,warmup,expect_fix", [((0, 0), 48, False), ((0, 0), 1, True),
                                                       ((0, 0, 0), 2, True), ((0,) * 4, 0, True),
                                                       ((0,) * 5, 48, False)])
def test_sharded_executor_is_exact(fp, cuda, oracle, devices, warmup, expect_fix):
    from paper_1509_04394_b200.fuseplan import hash_video_u8, spec_chain
    W, H, F = 256, 96, 60
    pipe = spec_chain(W, H, F, th=40.0, kalman=True)
    v = hash_video_u8(F, 4, H, W, 91)
    want = oracle.orc_chain(pipe, v)
    p = fp.Pipeline(json.dumps(pipe))
    plan = fp.Plan(p, fp.Device.load("b200"))
    sx = fp.ShardedExecutor(p, plan, list(devices), warmup_frames=warmup)
    got = sx.run(v)
    np.testing.assert_array_equal(got.astype(np.float32), want)
    st = sx.stats()
    assert st["shards"] == len(devices)
    if expect_fix:
        assert st["fixups"] >= 1
        # the repair is sparse in time: fewer frames than whole shards
        assert st["fixed_frames"] <= st["fixups"] * (F // len(devices) + 1)
    else:
        assert st["fixups"] == 0


def test_converge_counts_the_frames_a_wrong_start_reaches(fp, cuda, oracle):
    """fp_exec_converge against a direct comparison of the two runs."""
    import torch
    from paper_1509_04394_b200.fuseplan import hash_video_u8, spec_chain
    W, H, F = 128, 64, 80
    pipe = spec_chain(W, H, F, th=40.0)
    v = torch.from_numpy(hash_video_u8(F, 4, H, W, 5)).to(cuda)
    p = fp.Pipeline(json.dumps(pipe))
    ex = fp.Executor(p, fp.Plan(p, fp.Device.load("b200"), {"force_partition": "1-5"}))
    s_true = torch.empty((1, H, W), device=cuda)
    s_warm = torch.empty((1, H, W), device=cuda)
    ex.run_range(v[:20], n_warm=20, state_out=s_true)   # true state before frame 20
    ex.run_range(v[17:20], n_warm=3, state_out=s_warm)  # a 3-frame warm-up
    a = ex.run_range(v[20:], state_in=s_true)
    b = ex.run_range(v[20:], state_in=s_warm)
    torch.cuda.synchronize()
    k = ex.converge(v[20:], s_true, s_warm)
    differ = (a != b).reshape(F - 20, -1).any(dim=1).cpu().numpy()
    assert 0 < k <= F - 20
    assert not differ[k:].any()  # every frame from k on is already exact
    assert ex.converge(v[20:], s_true, s_true) == 0


def test_plain_c_caller_shards_over_devices(fp, cuda, tmp_path):
    """tests/cpp/shard_capi.c, compiled here against include/fuseplan.h and
    the in-tree library: a C program drives 3 shards (one GPU) and gets the
    single-device output."""
    exe = tmp_path / "shard_capi"
    lib_dir = os.path.dirname(fp.LIB_PATH)
    subprocess.run(["gcc", "-O2", "-o", str(exe), os.path.join(ROOT, "tests", "cpp",
                                                               "shard_capi.c"),
                    "-I", os.path.join(ROOT, "include"), "-L", lib_dir, "-lfuseplan_b200",
                    f"-Wl,-rpath,{lib_dir}"], check=True)
    env = dict(os.environ, FUSEPLAN_DEVICE_DIR=fp.DATA_DIR)
    for warm in ("48", "1"):
        r = subprocess.run([str(exe), "200", "80", "45", warm, "0", "0", "0"],
                           capture_output=True, text=True, env=env, timeout=300)
        assert r.returncode == 0, r.stdout + r.stderr
        assert r.stdout.startswith("ok")
        stats = json.loads(r.stdout.split(" ", 1)[1])
        assert (stats["fixups"] > 0) == (warm == "1")


@pytest.mark.parametrize("halo_mode", ["cumulative", "paper-max"])
def test_cpp_api_run_sequential_and_run_tiled(fp, cuda, oracle, tmp_path, halo_mode):
    """include/fuseplan/simulator.hpp from C++ (tests/cpp/simulator_api.cpp):
    the GPU-backed run_sequential's every stage output and run_tiled's output
    equal the reference's own run_sequential / run_tiled (oracle/_ref), and
    the traffic tallies equal its counters."""
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    from paper_1509_04394_b200 import build as B
    from paper_1509_04394_b200.fuseplan import hash_video_u8, spec_chain
    exe = tmp_path / "simulator_api"
    lib_dir = os.path.dirname(fp.LIB_PATH)
    subprocess.run([B.CXX, "-std=c++20", "-O1", "-o", str(exe),
                    os.path.join(ROOT, "tests", "cpp", "simulator_api.cpp"),
                    "-I", os.path.join(ROOT, "include"), "-L", lib_dir, "-lfuseplan_b200",
                    f"-Wl,-rpath,{lib_dir}"], check=True)
    W, H, F = 160, 120, 10
    spec = spec_chain(W, H, F, th=24.0)
    video = hash_video_u8(F, 4, H, W, 3)
    (tmp_path / "p.json").write_text(json.dumps(spec))
    dev = open(os.path.join(fp.DATA_DIR, "k20_like.json")).read()
    (tmp_path / "d.json").write_text(dev)
    fp.write_fpvd(str(tmp_path / "v.fpvd"), video)
    r = subprocess.run([str(exe), str(tmp_path / "p.json"), str(tmp_path / "d.json"), halo_mode,
                        str(tmp_path / "v.fpvd"), str(tmp_path)], capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    rep = json.loads(r.stdout)
    final, stages = oracle.ref_run_sequential(json.dumps(spec), video, stages=True)
    for k in range(5):
        got = np.fromfile(tmp_path / f"stage{k}.f32", np.float32).reshape(F, H, W)
        np.testing.assert_array_equal(got, stages[k], err_msg=f"stage {k}")
    opts = {"halo_mode": halo_mode} if halo_mode == "paper-max" else None
    tiled, traffic = oracle.ref_run_tiled(json.dumps(spec), dev, video, opts)
    got = np.fromfile(tmp_path / "tiled.f32", np.float32).reshape(F, H, W)
    np.testing.assert_array_equal(got, tiled)
    assert rep["diff_count"] == int((final != tiled).sum())
    assert rep["interior"] + rep["boundary"] == rep["diff_count"]
    assert rep["tiled_gmem"] == int(traffic[0] + traffic[1])
    assert rep["seq_gmem"] == 2 * W * H * F * 5
