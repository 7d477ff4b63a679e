"""Oracle step O6: the collectives as explicit sums / scatters / permutations.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:245 (NCCL AllReduce / ReduceScatter / send-recv All-to-All),
PAPER.md:262-264 (which primitive follows the GEMM), PAPER.md:368 (one call per
wave group, on that group's contiguous range).

Sums run in fp64 in ascending rank order.  Pins: textbook identities
(tests/test_oracle_collectives.py): AR of x and -x is 0; RS followed by
AllGather equals AR; n = 1 is the identity; A2A with identity routing is a no-op.
"""
from __future__ import annotations

import numpy as np


def allreduce_groups(bufs, elem_ranges):
    """In-place AllReduce per group range; returns the (identical) per-rank buffers."""
    n = len(bufs)
    out = [b.copy() for b in bufs]
    for lo, hi in elem_ranges:
        acc = np.zeros(hi - lo, dtype=np.float64)
        for r in range(n):
            acc = acc + bufs[r][lo:hi]
        for r in range(n):
            out[r][lo:hi] = acc
    return out


def reduce_scatter_groups(bufs, elem_ranges):
    """ReduceScatter per group: group range split in n equal chunks; rank k
    receives the sum over ranks of chunk k.  Receive buffer of rank k = its
    chunks concatenated in group order."""
    n = len(bufs)
    recv = [[] for _ in range(n)]
    for lo, hi in elem_ranges:
        c = (hi - lo) // n
        for k in range(n):
            acc = np.zeros(c, dtype=np.float64)
            for r in range(n):
                acc = acc + bufs[r][lo + k * c:lo + (k + 1) * c]
            recv[k].append(acc)
    return [np.concatenate(x) if x else np.zeros(0) for x in recv]


def allgather(parts):
    """AllGather: every rank gets the concatenation of all ranks' parts."""
    full = np.concatenate(parts, axis=0)
    return [full.copy() for _ in parts]


def alltoall_groups(sends, P: int):
    """All-to-All per group: rank d receives, for group j and source s
    (ascending), pool_{s,d}[range_{s,d,j}].  Returns per receiver the list of
    (s, subtoken_array) in receive order [group][source]."""
    n = len(sends)
    recv = [[] for _ in range(n)]
    for j in range(P):
        for d in range(n):
            for s in range(n):
                a, b = sends[s].ranges[d][j]
                recv[d].append((s, sends[s].pools[d][a:b]))
    return recv
