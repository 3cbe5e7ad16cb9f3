"""Frame (T) sharding of the fused chain across ranks, exact by construction.

The SPEC chain is frame-local except for the causal IIR:
rank g owns frames [lo_g, hi_g).  Its IIR state at lo_g depends on every
earlier frame, so each rank

  1. warms the recurrence up over the W frames before its shard (restarting
     it there, like the reference does at frame 0, simulator.cpp:136-147),
  2. runs its shard from that warm state, keeping the end state,
  3. receives the TRUE end state of rank g-1 (send/recv of one W*H float
     plane -- the only collective of the path) and compares it bit for bit
     with its warm state; on any mismatch it re-runs its shard from the true
     state (the fix-up), which also corrects its own end state before it is
     forwarded to rank g+1.

Step 3 walks the ranks in order, so every shard ends up computed from the
exact state: the result is identical to a single-device run whatever W is;
W only decides how often a fix-up is needed (W >= 48 gave no
mismatch on 800x600 data).

`run_shard` is the compute: (frames, n_warm, state_in) -> (output, state_out)
on this rank.  In production it is the sm_100a executor (fp_exec_run_range
over NCCL-backed torch.distributed); tests plug in the CPU oracle over gloo.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional, Tuple

WARMUP_FRAMES = 64


@dataclass
class Shard:
    rank: int
    world: int
    lo: int
    hi: int
    warm: int

    @property
    def first(self) -> int:
        """First frame this rank reads (warm-up included)."""
        return self.lo - self.warm


def shard_of(rank: int, world: int, frames: int, warmup: int = WARMUP_FRAMES) -> Shard:
    lo, hi = rank * frames // world, (rank + 1) * frames // world
    return Shard(rank, world, lo, hi, min(warmup, lo))


def run_sharded(shard: Shard, run_shard: Callable, send: Callable, recv: Callable,
                equal: Callable, stats: Optional[dict] = None) -> Tuple[object, object]:
    """Executes this rank's part of the protocol and returns (output, end_state).

    run_shard(first, n_frames, n_warm, state_in) -> (out, state_out): run
        frames [first, first + n_frames) of the video, the first n_warm only
        advancing the state; state_in None = restart at `first`.
    send(state, dst) / recv(src) -> state: point-to-point state exchange.
    equal(a, b) -> bool: bitwise comparison of two state planes.
    """
    n_local = shard.hi - shard.lo
    if shard.warm:
        _, s_warm = run_shard(shard.first, shard.warm, shard.warm, None)
        out, s_end = run_shard(shard.lo, n_local, 0, s_warm)
    else:
        s_warm = None
        out, s_end = run_shard(shard.lo, n_local, 0, None)
    fixups = 0
    # carry chain: rank r's end state is final once rank r has verified
    for r in range(shard.world - 1):
        if shard.rank == r:
            send(s_end, r + 1)
        elif shard.rank == r + 1:
            s_true = recv(r)
            if s_warm is None or not equal(s_true, s_warm):
                out, s_end = run_shard(shard.lo, n_local, 0, s_true)
                fixups += 1
    if stats is not None:
        stats["fixups"] = stats.get("fixups", 0) + fixups
    return out, s_end
