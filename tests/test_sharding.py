"""Multi-rank T-sharding protocol (paper_1509_04394_b200.sharding) on CPU:
world sizes 2 and 3 over the gloo backend, each rank computing its shard
with the oracle; the gathered result must equal the single-process run bit
for bit, with and without forced fix-ups (tiny warm-up)."""
import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _np_converge(video, lo, hi, s_true, s_warm):
    """fp_exec_converge restated in numpy (reference float32 order,
    simulator.cpp:51-62): leading frames of [lo, hi) whose IIR differs."""
    a, b = s_true.reshape(-1), s_warm.reshape(-1)
    idx = np.nonzero(a.view(np.uint32) != b.view(np.uint32))[0]
    if idx.size == 0:
        return 0
    a, b = a[idx].copy(), b[idx].copy()
    alpha = np.float32(0.5)
    beta = np.float32(1.0) - alpha
    wr, wg, wb = np.float32(0.299), np.float32(0.587), np.float32(0.114)
    first = np.full(idx.size, hi - lo)
    for t in range(hi - lo):
        f = video[lo + t].reshape(4, -1)[:, idx].astype(np.float32)
        x = (wr * f[0] + wg * f[1]) + wb * f[2]
        a = alpha * x + beta * a
        b = alpha * x + beta * b
        eq = (a.view(np.uint32) == b.view(np.uint32)) & (first == hi - lo)
        first[eq] = t
    return int(first.max())


def _worker(rank, world, port, frames, warmup, result_path, parallel=False, single=False,
            sparse=False):
    import sys
    sys.path.insert(0, ROOT)
    from oracle import oracle as O
    from paper_1509_04394_b200.fuseplan import hash_video_u8, spec_chain
    from paper_1509_04394_b200.sharding import run_sharded, shard_of

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    W, H = 48, 32
    pipe = spec_chain(W, H, frames, th=24.0)
    video = hash_video_u8(frames, 4, H, W, 777)
    sh = shard_of(rank, world, frames, warmup)

    def run_shard(first, n, n_warm, state_in):
        out, st = O.orc_chain(pipe, video[first:first + n], t_out=n_warm,
                              state_in=state_in, return_state=True, nthreads=1)
        return out, st

    def send(state, dst):
        dist.send(torch.from_numpy(np.ascontiguousarray(state)), dst)

    def recv(src):
        t = torch.empty((1, H, W), dtype=torch.float32)
        dist.recv(t, src)
        return t.numpy()

    def first_bad(k):
        t = torch.tensor([k], dtype=torch.int64)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return int(t.item())

    def warm_state(first, n):  # gray + IIR only over the warm-up frames
        p12 = dict(pipe, kernels=pipe["kernels"][:2])
        _, st = O.orc_chain(p12, video[first:first + n], t_out=n, return_state=True,
                            nthreads=1)
        return st

    def converge(s_true, s_warm):
        return _np_converge(video, sh.lo, sh.hi, s_true, s_warm)

    stats = {}
    out, _ = run_sharded(sh, run_shard, send, recv,
                         lambda a, b: np.array_equal(a.view(np.uint32), b.view(np.uint32)),
                         stats, first_bad if parallel else None,
                         warm_state if single else None,
                         converge=converge if sparse else None)
    if sparse and stats.get("fixups"):
        assert stats["fixed_frames"] <= stats["fixups"] * (sh.hi - sh.lo)
    # gather to rank 0
    full = [None] * world if rank == 0 else None
    dist.gather_object((sh.lo, out, stats["fixups"] if stats else 0), full, dst=0)
    if rank == 0:
        parts = sorted(full, key=lambda p: p[0])
        got = np.concatenate([p[1] for p in parts])
        want = O.orc_chain(pipe, video, nthreads=1)
        np.save(result_path, np.array([int(np.array_equal(got, want)),
                                       sum(p[2] for p in parts)]))
    dist.destroy_process_group()


@pytest.mark.parametrize("parallel,single,sparse", [(False, False, False), (True, False, False),
                                                    (True, True, False), (True, True, True),
                                                    (False, False, True)])
@pytest.mark.parametrize("world,frames,warmup,expect_fixups",
                         [(2, 40, 64, False), (2, 40, 3, True), (3, 45, 2, True),
                          (3, 45, 48, None), (4, 48, 1, True), (4, 48, 30, None)])
def test_sharded_run_is_exact(tmp_path, world, frames, warmup, expect_fixups, parallel, single,
                              sparse):
    """Sequential carry chain, the parallel verification (one exchange + one
    all-reduce, chain only from the first failing rank), the single-launch
    shard (warm-up inside, warm state from a gray+IIR side pass), and the
    time-sparse repair (only the frames a wrong warm start reaches)."""
    out = tmp_path / "r.npy"
    mp.spawn(_worker, args=(world, _free_port(), frames, warmup, str(out), parallel, single,
                            sparse),
             nprocs=world, join=True)
    ok, fixups = np.load(out)
    assert ok == 1
    if expect_fixups is True:
        assert fixups >= 1
    if expect_fixups is False:
        assert fixups == 0


def test_shard_bounds():
    from paper_1509_04394_b200.sharding import shard_of
    shards = [shard_of(r, 8, 1000) for r in range(8)]
    assert shards[0].lo == 0 and shards[-1].hi == 1000
    assert all(a.hi == b.lo for a, b in zip(shards, shards[1:]))
    assert shards[0].warm == 0 and all(s.warm == 48 for s in shards[1:])


def _halo_worker(rank, world, port, frames, warmup, t_radii, result_path, parallel):
    """Chain with temporal box_mean windows: rgba2gray, IIR, box_mean(rt=a),
    box_mean(rt=b), threshold.  The per-rank compute restates the stages with
    the oracle (temporal windows clamp at the range ends, as the device
    executor's range runs do) and numpy's float32 IIR (the reference's
    operation order, simulator.cpp:57-62)."""
    import sys
    sys.path.insert(0, ROOT)
    from oracle import oracle as O
    from paper_1509_04394_b200.fuseplan import hash_video_u8
    from paper_1509_04394_b200.sharding import run_sharded, shard_of

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    W, H, C = 24, 16, 4
    ks = [{"name": "g", "stencil_op": "rgba2gray"},
          {"name": "i", "stencil_op": "iir_temporal", "params": {"alpha": 0.5}}]
    ks += [{"name": f"b{j}", "stencil_op": "box_mean",
            "params": {"radius_x": 1, "radius_y": 1, "radius_t": rt}}
           for j, rt in enumerate(t_radii)]
    ks.append({"name": "t", "stencil_op": "threshold", "params": {"th": 120.0}})
    pipe = {"video": {"width": W, "height": H, "frames": frames, "channels": C},
            "kernels": ks}
    video = hash_video_u8(frames, C, H, W, 4242)
    alpha = np.float32(0.5)
    beta = np.float32(1.0) - alpha

    def gray(first, n):
        return O.orc_apply_stage(ks[0], video[first:first + n].astype(np.float32), 1)

    def iir(g, state_in):
        out = np.empty_like(g)
        prev = None if state_in is None else np.asarray(state_in, np.float32).reshape(H, W)
        for t in range(g.shape[0]):
            prev = g[t].copy() if prev is None else (alpha * g[t] + beta * prev).astype(
                np.float32)
            out[t] = prev
        return out

    def run_shard(first, n, n_warm, state_in):
        assert n_warm == 0
        cur = iir(gray(first, n), state_in)
        for k in ks[2:]:
            cur = O.orc_apply_stage(k, cur[:, None], 1)
        return cur, None

    def advance(first, n, state_in):
        return iir(gray(first, n), state_in)[-1][None].copy()

    def send(state, dst):
        dist.send(torch.from_numpy(np.ascontiguousarray(state)), dst)

    def recv(src):
        t = torch.empty((1, H, W), dtype=torch.float32)
        dist.recv(t, src)
        return t.numpy()

    def first_bad(k):
        t = torch.tensor([k], dtype=torch.int64)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return int(t.item())

    sh = shard_of(rank, world, frames, warmup, t_halo=sum(t_radii))
    stats = {}
    out, _ = run_sharded(sh, run_shard, send, recv,
                         lambda a, b: np.array_equal(a.view(np.uint32), b.view(np.uint32)),
                         stats, first_bad if parallel else None, advance=advance)
    full = [None] * world if rank == 0 else None
    dist.gather_object((sh.lo, out, stats.get("fixups", 0)), full, dst=0)
    if rank == 0:
        parts = sorted(full, key=lambda p: p[0])
        got = np.concatenate([p[1] for p in parts])
        want = O.orc_run_sequential(pipe, video, nthreads=1)[-1]
        np.save(result_path, np.array([int(np.array_equal(got, want)),
                                       sum(p[2] for p in parts)]))
    dist.destroy_process_group()


@pytest.mark.parametrize("parallel", [False, True])
@pytest.mark.parametrize("world,frames,warmup,t_radii,expect_fixups",
                         [(2, 30, 64, (2, 1), False), (3, 36, 2, (1, 2), True),
                          (4, 40, 40, (1, 1), False), (4, 40, 1, (3,), True)])
def test_sharded_temporal_halo_is_exact(tmp_path, world, frames, warmup, t_radii,
                                        expect_fixups, parallel):
    """T-shards of a chain with temporal windows: each
    rank computes R halo frames on both sides and keeps its own; the carry is
    taken before the next rank's context.  Equal to the single run bit for bit,
    with and without fix-ups."""
    out = tmp_path / "h.npy"
    mp.spawn(_halo_worker, args=(world, _free_port(), frames, warmup, t_radii, str(out),
                                 parallel), nprocs=world, join=True)
    ok, fixups = np.load(out)
    assert ok == 1
    if expect_fixups is True:
        assert fixups >= 1
    if expect_fixups is False:
        assert fixups == 0


def test_temporal_halo_bounds():
    from paper_1509_04394_b200.sharding import shard_of
    s = [shard_of(r, 4, 40, 8, t_halo=3) for r in range(4)]
    assert [(x.ctx_lo, x.ctx_hi) for x in s] == [(0, 13), (7, 23), (17, 33), (27, 40)]
    assert [x.first for x in s] == [0, 0, 9, 19]
    with pytest.raises(ValueError):
        shard_of(0, 8, 16, 8, t_halo=3)
