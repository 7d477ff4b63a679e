"""Lockstep simulator of NCCL semantics for the plans' communication schedules
(fo_plan_export_calls).  TEST INFRASTRUCTURE: it executes every rank's
exported calls on numpy buffers exactly as NCCL defines them, and raises where
real NCCL would hang or misbehave:

  * collectives (AllReduce / ReduceScatter) are matched across ALL ranks in
    issue order: every rank's next collective must be of the same kind and
    count (NCCL requires identical call sequences on a communicator), else
    ScheduleError("collective mismatch");
  * a GROUP_START ... GROUP_END bracket is one grouped point-to-point call:
    every rank must be inside a group at the same step, and for every ordered
    pair (s, d) the sends s->d and the receives on d from s must match one to
    one in order with equal counts (ncclSend / ncclRecv pairing), else
    ScheduleError("p2p mismatch");
  * every offset range must lie inside its buffer.

Sums run in fp64 in ascending rank order (the oracle's collectives,
oracle/collectives.py); tests feed integer data so order does not matter.
"""
from __future__ import annotations

import numpy as np


class ScheduleError(AssertionError):
    pass


def _view(bufs, name, off, count, rank):
    if name not in bufs or bufs[name] is None:
        raise ScheduleError(f"rank {rank}: buffer {name!r} not provided")
    b = bufs[name]
    if off < 0 or count < 0 or off + count > b.size:
        raise ScheduleError(f"rank {rank}: range [{off}, {off + count}) outside {name!r} of {b.size} elements")
    return b[off:off + count]


def run(calls_per_rank, bufs_per_rank, log=None):
    """Execute the schedules in lockstep.  bufs_per_rank[r] maps buffer names
    ('send', 'recv', 'out', 'scratch') to flat float64 arrays (modified in
    place; 'recv' may be the same object as 'send').  Returns the number of
    collective steps executed."""
    W = len(calls_per_rank)
    pc = [0] * W
    steps = 0

    def local(r):
        """Run rank r's local copies up to its next communicator call."""
        cl = calls_per_rank[r]
        while pc[r] < len(cl) and cl[pc[r]]["kind"] == "local_copy":
            c = cl[pc[r]]
            src = _view(bufs_per_rank[r], c["src_buf"], c["src_off"], c["count"], r).copy()
            _view(bufs_per_rank[r], c["dst_buf"], c["dst_off"], c["count"], r)[:] = src
            pc[r] += 1

    while True:
        for r in range(W):
            local(r)
        done = [pc[r] >= len(calls_per_rank[r]) for r in range(W)]
        if all(done):
            return steps
        if any(done):
            raise ScheduleError(f"ranks {[r for r in range(W) if done[r]]} finished while others still have "
                                f"calls (collective mismatch / hang)")
        heads = [calls_per_rank[r][pc[r]] for r in range(W)]
        kinds = {h["kind"] for h in heads}
        if len(kinds) != 1:
            raise ScheduleError(f"collective mismatch at step {steps}: {[h['kind'] for h in heads]}")
        kind = kinds.pop()
        if log is not None:
            log.append((steps, kind, [h.get("group") for h in heads]))
        if kind in ("allreduce", "reducescatter"):
            counts = {h["count"] for h in heads}
            if len(counts) != 1:
                raise ScheduleError(f"collective mismatch at step {steps}: {kind} counts {[h['count'] for h in heads]}")
            cnt = counts.pop()
            if kind == "allreduce":
                srcs = [_view(bufs_per_rank[r], heads[r]["src_buf"], heads[r]["src_off"], cnt, r).copy()
                        for r in range(W)]
                acc = np.zeros(cnt)
                for x in srcs:
                    acc = acc + x
                for r in range(W):
                    _view(bufs_per_rank[r], heads[r]["dst_buf"], heads[r]["dst_off"], cnt, r)[:] = acc
            else:
                srcs = [_view(bufs_per_rank[r], heads[r]["src_buf"], heads[r]["src_off"], W * cnt, r).copy()
                        for r in range(W)]
                for k in range(W):
                    acc = np.zeros(cnt)
                    for r in range(W):
                        acc = acc + srcs[r][k * cnt:(k + 1) * cnt]
                    _view(bufs_per_rank[k], heads[k]["dst_buf"], heads[k]["dst_off"], cnt, k)[:] = acc
            for r in range(W):
                pc[r] += 1
        elif kind == "group_start":
            sends = {}   # (s, d) -> list of (count, data)
            recvs = {}   # (s, d) -> list of (count, view)
            for r in range(W):
                cl = calls_per_rank[r]
                i = pc[r] + 1
                while i < len(cl) and cl[i]["kind"] != "group_end":
                    c = cl[i]
                    if c["kind"] == "send":
                        if not 0 <= c["peer"] < W or c["peer"] == r:
                            raise ScheduleError(f"rank {r}: send to invalid peer {c['peer']}")
                        data = _view(bufs_per_rank[r], c["src_buf"], c["src_off"], c["count"], r).copy()
                        sends.setdefault((r, c["peer"]), []).append((c["count"], data))
                    elif c["kind"] == "recv":
                        if not 0 <= c["peer"] < W or c["peer"] == r:
                            raise ScheduleError(f"rank {r}: recv from invalid peer {c['peer']}")
                        view = _view(bufs_per_rank[r], c["dst_buf"], c["dst_off"], c["count"], r)
                        recvs.setdefault((c["peer"], r), []).append((c["count"], view))
                    else:
                        raise ScheduleError(f"rank {r}: {c['kind']} inside a p2p group")
                    i += 1
                if i >= len(cl):
                    raise ScheduleError(f"rank {r}: group_start without group_end")
                pc[r] = i + 1
            for pair in set(sends) | set(recvs):
                sl, rl = sends.get(pair, []), recvs.get(pair, [])
                if [c for c, _ in sl] != [c for c, _ in rl]:
                    raise ScheduleError(f"p2p mismatch {pair[0]}->{pair[1]}: sends {[c for c, _ in sl]} "
                                        f"recvs {[c for c, _ in rl]}")
                for (_, data), (_, view) in zip(sl, rl):
                    view[:] = data
        else:
            raise ScheduleError(f"unexpected call {kind} at step {steps}")
        steps += 1
