"""Whole-pipeline pins: the overlapped method == the plain definition (O8),
bit-exactly on integer data (PAPER.md:834 claim C1; SPEC.md:392 acceptance)."""
import itertools

import numpy as np
import pytest

import synthetic
from oracle import pipeline as opl
from oracle import plan as op


def _int_inputs(rng, n, M, N, K):
    As = [rng.integers(-3, 4, size=(M, K)).astype(float) for _ in range(n)]
    Bts = [rng.integers(-3, 4, size=(N, K)).astype(float) for _ in range(n)]
    return As, Bts


def _parts(T):
    out = []
    for mask in range(1 << (T - 1)):
        cuts = [w + 1 for w in range(T - 1) if (mask >> w) & 1]
        b = [0] + cuts + [T]
        out.append([b[i + 1] - b[i] for i in range(len(b) - 1)])
    return out


def test_brute_force_all_orders_2x3_allreduce():
    """All 720 orders of a 2x3 tile grid x every partition x S in {1,2,3}, n=2."""
    rng = np.random.default_rng(0)
    BM, BN, K = 2, 2, 3
    As, Bts = _int_inputs(rng, 2, 2 * BM, 3 * BN, K)
    plain = opl.plain_allreduce(As, Bts)
    for order in itertools.permutations(range(6)):
        for S in (1, 2, 3):
            T = op.num_waves(6, S)
            for part in _parts(T):
                pl = op.make_plan(2 * BM, 3 * BN, BM, BN, S, part, order=list(order))
                res = opl.run_allreduce(As, Bts, pl)
                for r in range(2):
                    assert np.array_equal(res["out"][r], plain[r])


@pytest.mark.parametrize("n", [1, 2, 3])
def test_brute_force_orders_rs_a2a(n):
    """Every 6th order of the 2x3 grid x every partition x S, for RS and A2A."""
    rng = np.random.default_rng(n)
    BM, BN, K = 6, 1, 2
    M, N = 2 * BM, 3 * BN
    As, Bts = _int_inputs(rng, n, M, N, K)
    plain_rs = opl.plain_reducescatter(As, Bts, BM)
    row_dsts = [rng.integers(0, n, size=M) for _ in range(n)]
    plain_a2a = opl.plain_alltoall(As, Bts, row_dsts)
    for oi, order in enumerate(itertools.permutations(range(6))):
        if oi % 6:
            continue
        for S in (1, 2, 3):
            for part in _parts(op.num_waves(6, S)):
                pl = op.make_plan(M, N, BM, BN, S, part, order=list(order))
                rs = opl.run_reducescatter(As, Bts, pl)
                for k in range(n):
                    assert np.array_equal(rs["out"][k], plain_rs[k])
                a2a = opl.run_alltoall(As, Bts, [pl] * n, row_dsts)
                for d in range(n):
                    assert np.array_equal(a2a["out"][d], plain_a2a[d])


@pytest.mark.parametrize("n", [2, 4, 8])
@pytest.mark.parametrize("swz", [1, 2, 4])
def test_seeded_acceptance_sweep(n, swz):
    """n in {2,4,8} x swizzle in {1,2,4} x 20 seeded cases per primitive."""
    rng = np.random.default_rng(100 * n + swz)
    for case in range(20):
        BM, BN = 2 * n, int(rng.choice([1, 2, 4]))
        Mt, Nt = int(rng.integers(1, 5)), int(rng.integers(1, 5))
        M, N, K = Mt * BM, Nt * BN, int(rng.integers(1, 5))
        ntiles = Mt * Nt
        S = int(rng.integers(1, ntiles + 1))
        part = synthetic.random_partition(op.num_waves(ntiles, S), case)
        pl = op.make_plan(M, N, BM, BN, S, part, swizzle=swz)
        As, Bts = _int_inputs(rng, n, M, N, K)
        ar = opl.run_allreduce(As, Bts, pl)
        assert all(np.array_equal(o, p) for o, p in zip(ar["out"], opl.plain_allreduce(As, Bts)))
        rs = opl.run_reducescatter(As, Bts, pl)
        assert all(np.array_equal(o, p) for o, p in zip(rs["out"], opl.plain_reducescatter(As, Bts, BM)))
        # RS -> AllGather -> row exchange == AllReduce
        gathered = np.concatenate(rs["out"], axis=0)
        assert np.array_equal(opl.row_exchange(gathered, BM, n), opl.plain_allreduce(As, Bts)[0])
        # A2A with per-rank M (imbalance)
        plans, row_dsts, As2, Bts2 = [], [], [], []
        for s in range(n):
            Mts = int(rng.integers(1, 4))
            Ms = Mts * BM
            ntl = Mts * Nt
            Ss = int(rng.integers(1, ntl + 1))
            Ts = op.num_waves(ntl, Ss)
            plans.append((Ms, Ss, Ts))
        P = min(t for _, _, t in plans)
        pls = []
        for s, (Ms, Ss, Ts) in enumerate(plans):
            # same number of groups P on every rank
            part_s = [1] * (P - 1) + [Ts - (P - 1)]
            pls.append(op.make_plan(Ms, N, BM, BN, Ss, part_s, swizzle=swz))
            row_dsts.append(rng.integers(0, n, size=Ms))
            As2.append(rng.integers(-3, 4, size=(Ms, K)).astype(float))
            Bts2.append(rng.integers(-3, 4, size=(N, K)).astype(float))
        a2a = opl.run_alltoall(As2, Bts2, pls, row_dsts)
        for o, p in zip(a2a["out"], opl.plain_alltoall(As2, Bts2, row_dsts)):
            assert np.array_equal(o, p)


def test_float_regime_equivalence_model_bf16():
    """With bf16 rounding of each rank's GEMM output the pipeline still equals
    the plain definition computed from the same rounded values."""
    rng = np.random.default_rng(7)
    n, M, N, K = 2, 8, 8, 16
    As = [rng.standard_normal((M, K)) for _ in range(n)]
    Bts = [rng.standard_normal((N, K)) for _ in range(n)]
    pl = op.make_plan(M, N, 4, 4, 2, [1, 1], swizzle=2)
    res = opl.run_allreduce(As, Bts, pl, model_bf16=True)
    plain = opl.plain_allreduce(As, Bts, model_bf16=True)
    assert np.array_equal(res["out"][0], plain[0])
