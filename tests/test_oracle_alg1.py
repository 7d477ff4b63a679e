"""Pins for the Alg. 1 oracle and the design space."""
import json
import os

import pytest

from oracle import alg1

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "alg1.json")))


def _compositions(T):
    """Independent enumeration: all tuples of positive ints summing to T."""
    if T == 0:
        return [()]
    return [(first,) + rest for first in range(1, T + 1) for rest in _compositions(T - first)]


@pytest.mark.parametrize("T", range(1, 11))
def test_space_is_all_compositions(T):
    c = alg1.candidates(T)
    assert len(c) == 2 ** (T - 1) == len(set(c))
    assert sorted(c) == sorted(_compositions(T))


def test_space_paper_examples():
    for case in GOLD["space"]:
        space = alg1.candidates(case["T"])
        if "unpruned" in case:
            assert len(space) == case["unpruned"]
        for m in case.get("members", []):
            assert tuple(m) in space


@pytest.mark.parametrize("T", range(1, 12))
def test_pruned_space(T):
    got = alg1.pruned_candidates(T, 2, 4)
    want = [c for c in _compositions(T) if (T == 1 or (c[0] <= 2 and c[-1] <= 4))]
    assert sorted(got) == sorted(want)
    # O(2^(T-2)) bound of PAPER.md:446
    assert len(got) <= max(1, 2 ** (T - 2)) * 2 * 4


@pytest.mark.parametrize("case", GOLD["traces"], ids=lambda c: c["id"])
def test_hand_traces(case):
    T, dur, S, tiles = case["T"], case["duration_us"], case["S"], case["tiles"]
    per = case["per_wave_comm_us"]

    def lat(nbytes):  # 1 byte per tile, linear comm
        return per * nbytes / S

    for k, want in case["expect"].items():
        part = tuple(int(x) for x in k.split(","))
        sizes = alg1.group_bytes(part, S, tiles, 1)
        assert alg1.predict(part, dur, T, sizes, lat) == pytest.approx(want)


def test_single_group_is_gemm_plus_full_comm():
    curve = [(2 ** 16, 10.0), (2 ** 20, 100.0), (2 ** 26, 400.0)]
    for T in range(1, 9):
        sizes = alg1.group_bytes((T,), 64, 64 * T, 65536)
        full = alg1.interp_latency_us(curve, 64 * T * 65536)
        assert alg1.predict((T,), 100.0, T, sizes, lambda b: alg1.interp_latency_us(curve, b)) == pytest.approx(100.0 + full)


def test_comm_bound_finest_meets_bound():
    """Linear comm, comm-bound: the all-ones partition attains the PAPER.md:622 bound."""
    T, dur, per = 6, 30.0, 20.0
    sizes = alg1.group_bytes((1,) * T, 1, T, 1)
    t = alg1.predict((1,) * T, dur, T, sizes, lambda b: per * b)
    assert t == pytest.approx(alg1.perfect_overlap_bound(dur, T, per * T, per))


def test_interp_log_linear():
    curve = [(1024, 10.0), (4096, 30.0)]
    assert alg1.interp_bandwidth(curve, 1024) == 10.0
    assert alg1.interp_bandwidth(curve, 2048) == pytest.approx(20.0)   # geometric midpoint
    assert alg1.interp_bandwidth(curve, 100) == 10.0                   # clamp
    assert alg1.interp_bandwidth(curve, 1 << 30) == 30.0


def test_search_tie_break_and_knee():
    # infinite bandwidth -> every partition predicts dur; tie -> single group
    best, t = alg1.search(5, 50.0, lambda G: alg1.group_bytes(G, 1, 5, 1), lambda b: 0.0, prune=False)
    assert best == (5,) and t == pytest.approx(50.0)
    # pruned (|G1| <= 2): fewest groups, then lexicographically smallest
    best, t = alg1.search(5, 50.0, lambda G: alg1.group_bytes(G, 1, 5, 1), lambda b: 0.0)
    assert best == (1, 4) and t == pytest.approx(50.0)
    # a curve with a knee: tiny messages are slow -> not the all-ones partition
    curve = [(2 ** 10, 1.0), (2 ** 22, 1.0), (2 ** 24, 200.0), (2 ** 28, 400.0)]
    lat = lambda b: alg1.interp_latency_us(curve, b)
    best, _ = alg1.search(8, 400.0, lambda G: alg1.group_bytes(G, 64, 512, 65536), lat)
    assert best != (1,) * 8


def test_multi_balanced_equals_scalar():
    """balanced A2A routing -> the per-GPU-max prediction equals
    the scalar prediction."""
    curve = [(2 ** 12, 5.0), (2 ** 20, 100.0), (2 ** 26, 400.0)]
    lat = lambda b: alg1.interp_latency_us(curve, b)
    for T in range(1, 7):
        wb = [3 * 2 ** 19] * T
        for G in alg1.candidates(T):
            single = alg1.predict(G, 120.0, T, [sum(wb[:g]) for g in G], lat)
            multi = alg1.predict_multi(G, [120.0] * 4, [wb] * 4, lat)
            assert multi == pytest.approx(single)


def test_multi_hand_trace_and_monotone():
    # two ranks, T = 2, partition (1, 1); linear comm 1 us per byte unit
    lat = lambda b: float(b)
    # rank 0: dur 10, bytes per wave (4, 4); rank 1: dur 20, bytes (1, 9)
    # i=1: t_acc_m = 0; t_acc_p = (5, 10)
    # i=2: p_max = 10; t_acc_m = max(10, 0) + max(4, 1) = 14; t_acc_p = (10, 20)
    # end: max(20, 14) + max(4, 9) = 29
    assert alg1.predict_multi((1, 1), [10.0, 20.0], [[4, 4], [1, 9]], lat) == pytest.approx(29.0)
    # a slower rank never lowers the prediction
    base = alg1.predict_multi((1, 1), [10.0, 10.0], [[4, 4], [4, 4]], lat)
    assert alg1.predict_multi((1, 1), [10.0, 30.0], [[4, 4], [4, 4]], lat) >= base


def test_interp_latency_units_by_hand():
    """Alg. 1 line 14's bytes -> latency conversion, by hand (VERDICT r1 pin):
    bandwidth in GB/s = 1e9 bytes/s, latency in microseconds."""
    flat1 = [(1, 1.0), (1 << 40, 1.0)]                        # 1 GB/s everywhere
    assert alg1.interp_latency_us(flat1, 1e6) == pytest.approx(1000.0, rel=1e-15)      # 1 MB at 1 GB/s = 1 ms
    assert alg1.interp_latency_us(flat1, 2 ** 20) == pytest.approx(1048.576, rel=1e-15)
    flat400 = [(1024, 400.0), (1 << 30, 400.0)]
    assert alg1.interp_latency_us(flat400, 4e6) == pytest.approx(10.0, rel=1e-15)      # 4 MB at 400 GB/s = 10 us
    assert alg1.interp_latency_us(flat400, 0) == 0.0
    # on the log-linear curve: 2 KiB sits halfway between 1 KiB @ 10 and 4 KiB @ 30 GB/s -> 20 GB/s
    assert alg1.interp_latency_us([(1024, 10.0), (4096, 30.0)], 2048) == pytest.approx(2048 / 20e9 * 1e6, rel=1e-15)


def test_perfect_overlap_bound_both_branches_by_hand():
    """"summing up the original GEMM latency and the
    communication latency of the final wave (if GEMM takes more time), or the
    GEMM latency of the first wave and the original communication latency (if
    communication takes more time)" — hand values for both branches."""
    # GEMM-bound: 100 us GEMM in 4 waves, 40 us of communication, 10 us for the last wave
    assert alg1.perfect_overlap_bound(100.0, 4, 40.0, 10.0) == 110.0
    # communication-bound: 40 us GEMM in 4 waves (10 us first wave), 100 us of communication
    assert alg1.perfect_overlap_bound(40.0, 4, 100.0, 25.0) == 110.0
    # the GEMM-bound branch is attained by Alg. 1's finest partition when a
    # wave's communication (10 us) hides under the next wave (25 us)
    T, dur, per = 4, 100.0, 10.0
    sizes = alg1.group_bytes((1,) * T, 1, T, 1)
    assert alg1.predict((1,) * T, dur, T, sizes, lambda b: per * b) == pytest.approx(
        alg1.perfect_overlap_bound(dur, T, per * T, per))
