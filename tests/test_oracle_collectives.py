"""Pins for oracle step O6 (collectives) by textbook identities."""
import numpy as np

from oracle import collectives as oc
from oracle import plan as op
from oracle import reorder as orr


def test_allreduce_x_minus_x_is_zero():
    rng = np.random.default_rng(0)
    x = rng.standard_normal(64)
    out = oc.allreduce_groups([x, -x], [(0, 32), (32, 64)])
    assert all(np.array_equal(o, np.zeros(64)) for o in out)


def test_allreduce_n1_identity():
    x = np.arange(10.0)
    assert np.array_equal(oc.allreduce_groups([x], [(0, 10)])[0], x)


def test_rs_then_allgather_equals_allreduce():
    rng = np.random.default_rng(1)
    for n in (1, 2, 3, 4):
        bufs = [rng.integers(-50, 50, size=24 * n).astype(float) for _ in range(n)]
        ranges = [(0, 12 * n), (12 * n, 24 * n)]
        rs = oc.reduce_scatter_groups(bufs, ranges)
        ar = oc.allreduce_groups(bufs, ranges)[0]
        # reassemble: group j chunk k lives in rank k's recv at offset sum_{j'<j}(len/n)
        full = np.zeros_like(ar)
        off = 0
        for lo, hi in ranges:
            c = (hi - lo) // n
            for k in range(n):
                full[lo + k * c:lo + (k + 1) * c] = rs[k][off:off + c]
            off += c
        assert np.array_equal(full, ar)
        gathered = oc.allgather([r[None, :] for r in rs])
        assert all(np.array_equal(g, gathered[0]) for g in gathered)


def test_alltoall_identity_routing_noop():
    pl = op.make_plan(4, 4, 2, 2, 2, [1, 1])
    Ys = [np.arange(16.0).reshape(4, 4) + 100 * r for r in range(2)]
    sends = [orr.a2a_pre(Ys[r], pl, np.full(4, r), 2) for r in range(2)]
    recv = oc.alltoall_groups(sends, 2)
    for d in range(2):
        assert all(s == d or len(c) == 0 for s, c in recv[d])
