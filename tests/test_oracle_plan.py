"""Pins for oracle steps O1-O3 (tile grid, execution order, waves, groups)."""
import itertools
import json
import os

import numpy as np
import pytest

from oracle import plan as op
from oracle import reorder as orr

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "orders.json")))


@pytest.mark.parametrize("case", GOLD["grid"], ids=lambda c: c["id"])
def test_grid_and_waves(case):
    Mt, Nt = op.tile_grid(case["M"], case["N"], case["BM"], case["BN"])
    assert Mt * Nt == case["tiles"]
    assert op.num_waves(Mt * Nt, case["S"]) == case["T"]


@pytest.mark.parametrize("case", GOLD["orders"], ids=lambda c: c["id"])
def test_default_order_examples(case):
    o = op.default_order(case["Mt"], case["Nt"], case["s"])
    assert o.tolist() == case["order"]
    if "wave1" in case:
        # wave W1 = the first S positions (PAPER.md:235 wave definition)
        assert sorted(o[: case["S"]].tolist()) == case["wave1"]


def test_paper_slot_statement_g2():
    """tiles 0 and 3 get reordered indices 0 and 1, checked through
    the actual AR pre-reorder of a tile-id-coded matrix (not the order table)."""
    case = [c for c in GOLD["orders"] if c["id"] == "g2"][0]
    BM = BN = 2
    M, N = case["Mt"] * BM, case["Nt"] * BN
    pl = op.make_plan(M, N, BM, BN, case["S"], None, swizzle=case["s"])
    Y = np.zeros((M, N))
    for t in range(pl.ntiles):
        i, j = op.tile_coords(t, pl.Nt)
        Y[i * BM:(i + 1) * BM, j * BN:(j + 1) * BN] = t
    buf = orr.ar_pre(Y, pl)
    slot_tile = [int(buf[s * BM * BN]) for s in range(pl.ntiles)]
    for t, s in case["slot_of_tile"].items():
        assert slot_tile[s] == int(t)


def test_order_special_cases_and_permutation():
    rng = np.random.default_rng(0)
    for _ in range(200):
        Mt, Nt = int(rng.integers(1, 9)), int(rng.integers(1, 9))
        s = int(rng.integers(1, 10))
        o = op.default_order(Mt, Nt, s)
        assert sorted(o.tolist()) == list(range(Mt * Nt))
        if s == 1:
            assert o.tolist() == list(range(Mt * Nt))
        if s >= Mt:
            assert o.tolist() == [i * Nt + j for j in range(Nt) for i in range(Mt)]


def test_order_validation():
    with pytest.raises(op.OracleError):
        op.validate_order([0, 0, 1], 3)
    with pytest.raises(op.OracleError):
        op.validate_order([0, 1], 3)
    with pytest.raises(op.OracleError):
        op.tile_grid(100, 64, 64, 64)


@pytest.mark.parametrize("case", GOLD["groups"], ids=lambda c: c["id"])
def test_group_examples(case):
    if "tiles" in case:
        ntiles = case["tiles"]
    else:
        ntiles = case["Mt"] * case["Nt"]
    assert op.group_thresholds(case["partition"], case["S"], ntiles) == case["thresholds"]
    if "ranges" in case:
        assert [list(r) for r in op.group_ranges(case["partition"], case["S"], ntiles)] == case["ranges"]
    if "slot_of_tile" in case:
        o = op.default_order(case["Mt"], case["Nt"], case["s"])
        slot = {int(t): p for p, t in enumerate(o)}
        assert {str(k): v for k, v in slot.items()} == case["slot_of_tile"]


def test_every_tile_in_exactly_one_group():
    """SURVEY §8(c) O3 invariant, over every partition of small T."""
    for ntiles in range(1, 13):
        for S in range(1, ntiles + 1):
            T = op.num_waves(ntiles, S)
            for part in itertools.product(range(1, T + 1), repeat=min(T, 4)):
                if sum(part) != T:
                    continue
                seen = np.zeros(ntiles, int)
                for lo, hi in op.group_ranges(part, S, ntiles):
                    seen[lo:hi] += 1
                assert (seen == 1).all()
                assert sum(op.group_thresholds(part, S, ntiles)) == ntiles
                gp = op.group_of_position(part, S, ntiles)
                assert (np.diff(gp) >= 0).all()


def test_partition_errors():
    with pytest.raises(op.OracleError):
        op.group_ranges([1, 1], 2, 8)         # sums to 2, T = 4
    with pytest.raises(op.OracleError):
        op.group_ranges([0, 4], 2, 8)         # zero-size group
