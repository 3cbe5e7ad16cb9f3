"""Frame (T) sharding of the fused chain across ranks, exact by construction.

The SPEC chain is frame-local except for the causal IIR:
rank g owns frames [lo_g, hi_g).  Its IIR state at lo_g depends on every
earlier frame, so each rank

  1. warms the recurrence up over the W frames before its shard (restarting
     it there, like the reference does at frame 0, simulator.cpp:136-147),
  2. runs its shard from that warm state, keeping the end state,
  3. sends its end state to rank g+1 and receives rank g-1's (all ranks at
     once: one send/recv of a W*H float plane per rank), compares it bit for
     bit with its warm state, and the ranks agree (one all-reduce MIN) on the
     first rank k whose warm state was wrong;
  4. if every warm state was right (k = world), every shard started from the
     exact state by induction (rank g's end state is exact when its start
     state was) -- done.  Otherwise ranks >= k walk the carry in order from
     k: each repairs its shard from the true state (the fix-up) and forwards
     its end state.  The repair is sparse in time: `converge(s_true,
     s_warm)` (fp_exec_converge) re-runs gray+IIR for only the pixels whose
     two states differ and returns how many leading frames of the shard they
     reach; the IIR is deterministic, so once both trajectories coincide at a
     pixel they stay equal, and only those frames are recomputed -- the end
     state changes (and the walk goes on) only when they reach the shard's
     end.

So the common case costs one exchange and one all-reduce whatever the rank
count, and the result is identical to a single-device run whatever W is;
W only decides how often the fix-up chain runs and how long it is
(W >= 48 gave no mismatch on 800x600 data).

`run_shard` is the compute: (frames, n_warm, state_in) -> (output, state_out)
on this rank.  In production it is the sm_100a executor (fp_exec_run_range
over NCCL-backed torch.distributed); tests plug in the CPU oracle over gloo.

Temporal windows (box_mean with radius_t): with R the
chain's cumulative temporal radius, rank g also computes the R frames on each
side of its shard (its "context"; the video itself is replicated or readable
by every rank, so these halo frames need no transfer) and keeps only its own
frames -- a range run clamps its temporal windows at the range ends, which is
exact at the video's ends and only disturbs the discarded halo frames
elsewhere.  The carried IIR state is then the one before rank g+1's context
start (hi - R), computed by a gray+IIR-only pass (`advance`), because the
full chain cannot be split there without clamping a temporal window.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional, Tuple

WARMUP_FRAMES = 48  # 48 frames -> 0 / 480 000 mismatching pixels


@dataclass
class Shard:
    rank: int
    world: int
    lo: int
    hi: int
    warm: int
    frames: int = 0   # video length (0: unknown, no temporal halo)
    t_halo: int = 0   # cumulative temporal radius R of the chain

    @property
    def ctx_lo(self) -> int:
        """First frame whose chain output this rank computes (halo included)."""
        return max(0, self.lo - self.t_halo)

    @property
    def ctx_hi(self) -> int:
        return min(self.frames, self.hi + self.t_halo) if self.t_halo else self.hi

    @property
    def first(self) -> int:
        """First frame this rank reads (warm-up included)."""
        return self.ctx_lo - self.warm


def shard_of(rank: int, world: int, frames: int, warmup: int = WARMUP_FRAMES,
             t_halo: int = 0) -> Shard:
    lo, hi = rank * frames // world, (rank + 1) * frames // world
    if t_halo and world > 1 and (frames // world) < t_halo:
        raise ValueError("shards must be at least as long as the temporal halo")
    ctx_lo = max(0, lo - t_halo)
    return Shard(rank, world, lo, hi, min(warmup, ctx_lo), frames, t_halo)


def run_sharded(shard: Shard, run_shard: Callable, send: Callable, recv: Callable,
                equal: Callable, stats: Optional[dict] = None,
                first_bad: Optional[Callable] = None,
                warm_state: Optional[Callable] = None,
                advance: Optional[Callable] = None,
                converge: Optional[Callable] = None) -> Tuple[object, object]:
    """Executes this rank's part of the protocol and returns (output, end_state).

    run_shard(first, n_frames, n_warm, state_in) -> (out, state_out): run
        frames [first, first + n_frames) of the video, the first n_warm only
        advancing the state; state_in None = restart at `first`.
    send(state, dst) / recv(src) -> state: point-to-point state exchange.
    equal(a, b) -> bool: bitwise comparison of two state planes.
    first_bad(k) -> int: all-reduce MIN over the ranks of k (None: the
        sequential chain of the original protocol is used for every rank).
    warm_state(first, n) -> state: the IIR state after n frames from a
        fresh start at `first` (a gray+IIR-only pass).  When given, the
        shard runs as ONE launch with its warm-up inside (n_warm = W) and the
        warm state used for verification comes from this side computation
        (it may run concurrently); the IIR arithmetic of both is the
        reference's, so the two warm states are identical.
    advance(first, n, state_in) -> state: gray+IIR state after n frames from
        state_in (None = fresh); required when shard.t_halo > 0.
    converge(s_true, s_warm) -> k: leading frames of this shard whose output
        a start from s_warm instead of s_true changes (fp_exec_converge); the
        fix-up then re-runs only those frames.  None: whole-shard re-runs.
    """
    if shard.t_halo:
        return _run_sharded_halo(shard, run_shard, send, recv, equal, stats, first_bad,
                                 advance)
    n_local = shard.hi - shard.lo
    if shard.warm and warm_state is not None:
        out, s_end = run_shard(shard.first, shard.warm + n_local, shard.warm, None)
        s_warm = warm_state(shard.first, shard.warm)
    elif shard.warm:
        _, s_warm = run_shard(shard.first, shard.warm, shard.warm, None)
        out, s_end = run_shard(shard.lo, n_local, 0, s_warm)
    else:
        s_warm = None
        out, s_end = run_shard(shard.lo, n_local, 0, None)
    fixups = 0
    fixed = [0]
    world, rank = shard.world, shard.rank
    start = 0  # first rank of the sequential fix-up chain

    def repair(s_true, out, s_end):
        # frames of this shard a start from s_warm (not s_true) got wrong
        k = n_local
        if converge is not None and s_warm is not None:
            k = min(int(converge(s_true, s_warm)), n_local)
        fixed[0] += k
        if k >= n_local:  # the whole shard, end state included
            return run_shard(shard.lo, n_local, 0, s_true)
        if k > 0:
            part, _ = run_shard(shard.lo, k, 0, s_true)
            if part is not None and out is not None:
                out[:k] = part
        return out, s_end
    if first_bad is not None and world > 1:
        # 3: every rank forwards its (tentative) end state at once; even /
        # odd ordering of send and recv keeps blocking point-to-point
        # backends deadlock-free
        s_true = None
        if rank % 2 == 0:
            if rank + 1 < world:
                send(s_end, rank + 1)
            if rank > 0:
                s_true = recv(rank - 1)
        else:
            s_true = recv(rank - 1)
            if rank + 1 < world:
                send(s_end, rank + 1)
        ok = rank == 0 or (s_warm is not None and equal(s_true, s_warm))
        start = first_bad(world if ok else rank)
        if start >= world:  # 4: all warm states were exact
            if stats is not None:
                stats["fixups"] = stats.get("fixups", 0)
            return out, s_end
        if rank == start:  # its received state is exact (all ranks < start verified)
            out, s_end = repair(s_true, out, s_end)
            fixups += 1
    # carry chain from `start`: rank r's end state is final once r verified
    for r in range(start, world - 1):
        if rank == r:
            send(s_end, r + 1)
        elif rank == r + 1:
            s_true = recv(r)
            if s_warm is None or not equal(s_true, s_warm):
                out, s_end = repair(s_true, out, s_end)
                fixups += 1
    if stats is not None:
        stats["fixups"] = stats.get("fixups", 0) + fixups
        stats["fixed_frames"] = stats.get("fixed_frames", 0) + fixed[0]
    return out, s_end


def _run_sharded_halo(shard: Shard, run_shard: Callable, send: Callable, recv: Callable,
                      equal: Callable, stats: Optional[dict], first_bad: Optional[Callable],
                      advance: Callable) -> Tuple[object, object]:
    """run_sharded for chains with temporal windows (module docstring).

    advance(first, n, state_in) -> the gray+IIR state after frames
    [first, first + n) from state_in (None: a fresh start at `first`)."""
    if advance is None:
        raise ValueError("temporal halos need the gray+IIR `advance` callback")
    world, rank = shard.world, shard.rank
    c_lo, c_hi = shard.ctx_lo, shard.ctx_hi
    keep = slice(shard.lo - c_lo, shard.hi - c_lo)
    # the carry point: the state before rank g+1's context start
    nxt = shard_of(rank + 1, world, shard.frames, shard.warm, shard.t_halo) \
        if rank + 1 < world else None
    c_next = nxt.ctx_lo if nxt is not None else None

    def compute(s_start):
        out, _ = run_shard(c_lo, c_hi - c_lo, 0, s_start)
        s_end = None
        if c_next is not None:
            s_end = advance(c_lo, c_next - c_lo, s_start) if c_next > c_lo else s_start
        return out[keep], s_end

    s_warm = advance(shard.first, shard.warm, None) if shard.warm else None
    out, s_end = compute(s_warm)
    fixups = 0
    start = 0
    if first_bad is not None and world > 1:
        s_true = None
        if rank % 2 == 0:
            if rank + 1 < world:
                send(s_end, rank + 1)
            if rank > 0:
                s_true = recv(rank - 1)
        else:
            s_true = recv(rank - 1)
            if rank + 1 < world:
                send(s_end, rank + 1)
        ok = rank == 0 or (s_warm is not None and equal(s_true, s_warm))
        start = first_bad(world if ok else rank)
        if start >= world:
            if stats is not None:
                stats["fixups"] = stats.get("fixups", 0)
            return out, s_end
        if rank == start:
            out, s_end = compute(s_true)
            fixups += 1
    for r in range(start, world - 1):
        if rank == r:
            send(s_end, r + 1)
        elif rank == r + 1:
            s_true = recv(r)
            if s_warm is None or not equal(s_true, s_warm):
                out, s_end = compute(s_true)
                fixups += 1
    if stats is not None:
        stats["fixups"] = stats.get("fixups", 0) + fixups
    return out, s_end
