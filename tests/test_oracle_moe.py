"""Pins for the MoE top-k combine oracle (R31):
the expert GEMM -> All-to-All -> combine chain of the oracle must equal the
direct definition of an MoE layer's combine, out[t] = sum_i w[t,i] x_t W_{e_i},
computed per token with no All-to-All machinery at all."""
import numpy as np
import pytest

import synthetic
from oracle import pipeline
from oracle import plan as op
from oracle import post


@pytest.mark.parametrize("n,k,skew", [(2, 1, 0.0), (2, 2, 0.0), (4, 2, 0.0), (4, 2, 1.5), (8, 2, 0.0)])
def test_a2a_combine_equals_direct_moe(n, k, skew):
    tokens, K, N, BM, BN = 32 * n, 64, 64, 16, 32
    rt = synthetic.moe_topk(tokens, n, k, seed=7 + n, skew=skew, pad=BM)
    rng = np.random.default_rng(n)
    X = rng.integers(-3, 4, size=(tokens, K)).astype(np.float64)
    W = [rng.integers(-2, 3, size=(N, K)).astype(np.float64) for _ in range(n)]   # Bt of expert e
    As, plans, rds = [], [], []
    for e in range(n):
        rows = rt["row_token"][e]
        A = np.where((rows >= 0)[:, None], X[np.maximum(rows, 0)], 0.0)
        rd = rt["row_dst"][e]
        tiles = (len(A) // BM) * (N // BN)
        S = max(1, tiles // 2)
        T = -(-tiles // S) if tiles else 1
        As.append(A)
        rds.append(rd)
        plans.append(op.make_plan(len(A), N, BM, BN, S, [T] if tiles else [1]))
    # every rank needs the same number of groups: one group each
    res = pipeline.run_alltoall(As, W, plans, rds)
    per = tokens // n
    for r in range(n):
        out = res["out"][r]
        got = post.topk_combine(out, rt["combine_idx"][r], rt["weight"][r * per:(r + 1) * per])
        want = np.zeros((per, N))
        for l in range(per):
            t = r * per + l
            for i in range(k):
                e = rt["top"][t, i]
                want[l] += rt["weight"][t, i] * (X[t] @ W[e].T)
        assert np.allclose(got, want, rtol=1e-12, atol=1e-9)


def test_routing_weights_and_skew():
    rt = synthetic.moe_topk(4096, 8, 2, seed=40000)
    assert np.allclose(rt["weight"].sum(axis=1), 1.0, atol=1e-6)
    assert all((np.diff(rt["row_token"][e]) > 0).all() for e in range(8))
    loads = np.array([len(x) for x in rt["row_token"]])
    assert loads.sum() == 4096 * 2
    sk = synthetic.moe_topk(4096, 8, 2, seed=40000, skew=2.0)
    sl = np.array([len(x) for x in sk["row_token"]])
    assert sl.sum() == 4096 * 2 and sl.max() / sl.min() > 2 * loads.max() / loads.min()


def test_combine_gather_and_dropped_slots():
    x = np.arange(12.0).reshape(4, 3)
    idx = np.array([[2, -1], [0, 3], [7, 1]])
    w = np.array([[1.0, 5.0], [0.25, 0.75], [9.0, 1.0]])
    out = post.topk_combine(x, idx, w, residual=np.ones((3, 3)))
    assert np.array_equal(out, np.array([x[2] + 1, 0.25 * x[0] + 0.75 * x[3] + 1, x[1] + 1]))
    # k = 1, w = 1: a pure row gather
    perm = np.array([[3], [1], [0], [2]])
    assert np.array_equal(post.topk_combine(x, perm, np.ones((4, 1))), x[perm[:, 0]])


def test_a2a_with_a_source_without_rows():
    """An expert rank no token was routed to (m = 0, R45): with P
    empty groups the overlapped A2A delivers exactly the plain all-to-all-v
    rows (the definition, oracle.pipeline.plain_alltoall) at every receiver;
    a partition of empty groups is only legal when there are no tiles."""
    n, N, K, BM, BN = 3, 256, 64, 128, 128
    Ms = [256, 0, 384]
    rng = np.random.default_rng(0)
    As, Bts, plans, rds = [], [], [], []
    for s in range(n):
        A, Bt = synthetic.exact_inputs(max(Ms[s], 1), N, K, seed=5 + s, nnz_per_row=32)
        A = A[:Ms[s]]
        rd = rng.integers(0, n, Ms[s]).astype(np.int32)
        tiles = (Ms[s] // BM) * (N // BN)
        part = [0, 0] if tiles == 0 else [1, op.num_waves(tiles, 2) - 1]
        plans.append(op.make_plan(Ms[s], N, BM, BN, 2, part))
        As.append(A), Bts.append(Bt), rds.append(rd)
    res = pipeline.run_alltoall(As, Bts, plans, rds)
    plain = pipeline.plain_alltoall(As, Bts, rds)
    for d in range(n):
        assert res["out"][d].shape[0] == sum(int((rd == d).sum()) for rd in rds)
        assert np.array_equal(res["out"][d], plain[d])
    assert res["send"][1].ranges == [[(0, 0), (0, 0)]] * n
    with pytest.raises(op.OracleError):
        op.group_ranges([0, 1], 2, 4)          # empty groups beside tiles
    with pytest.raises(op.OracleError):
        op.group_ranges([1, 0], 2, 0)          # waves without tiles
