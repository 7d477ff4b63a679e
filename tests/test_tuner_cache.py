"""Plan cache with nearest-neighbour reuse (SPEC.md:339-341
examples) — host logic, CPU only (the tuner itself is injected)."""
import pytest

from paper_2504_19519_b200 import tuner


def fake_tuner(calls):
    def t(M, N, K, coll="allreduce", world=1, **kw):
        calls.append((M, N, K))
        tiles = (M // 256) * (N // 256)
        S = tuner.default_workers(tiles, 148)
        T = -(-tiles // S)
        groups = [1] * (T - 1) + [1] if T > 1 else [1]
        return tuner.TunedPlan(M, N, K, coll, world, 256, 256, S, 0, groups, 1.0, 1.0, [], "tuned")
    return t


def test_empty_cache_tunes_and_stores(tmp_path):
    calls = []
    c = tuner.PlanCache(str(tmp_path / "plans.json"))
    tp = c.lookup_or_tune(4096, 4096, 1792, tuner=fake_tuner(calls))
    assert tp.source == "tuned" and calls == [(4096, 4096, 1792)]
    c2 = tuner.PlanCache(str(tmp_path / "plans.json"))   # persisted
    assert tuner.key_of(4096, 4096, 1792, "allreduce", 1) in c2.entries


def test_exact_hit(tmp_path):
    calls = []
    c = tuner.PlanCache(str(tmp_path / "p.json"))
    c.lookup_or_tune(4096, 4096, 1792, tuner=fake_tuner(calls))
    tp = c.lookup_or_tune(4096, 4096, 1792, tuner=fake_tuner(calls))
    assert len(calls) == 1 and tp.source == "tuned"


def test_neighbour_within_threshold_reused():
    calls = []
    c = tuner.PlanCache(None)
    c.lookup_or_tune(4096, 4096, 1792, tuner=fake_tuner(calls))
    # (4096, 4096, 3584): distance 1 -> reuse (same tile grid, same T)
    tp = c.lookup_or_tune(4096, 4096, 3584, tuner=fake_tuner(calls))
    assert len(calls) == 1 and tp.source.startswith("neighbour:")
    # far away (distance 4): tune
    c.lookup_or_tune(16384, 16384, 7168, tuner=fake_tuner(calls))
    assert len(calls) == 2


def test_neighbour_with_incompatible_waves_is_retuned():
    calls = []
    c = tuner.PlanCache(None)
    c.lookup_or_tune(4096, 4096, 1792, tuner=fake_tuner(calls))
    # M doubled (distance 1) -> twice the tiles, different T -> cannot reuse the partition
    tp = c.lookup_or_tune(8192, 4096, 1792, tuner=fake_tuner(calls))
    assert len(calls) == 2 and tp.source == "tuned"


def test_distance():
    assert tuner.distance((4096, 4096, 4096), (8192, 4096, 2048)) == pytest.approx(2.0)


def test_tune_alltoall_imbalanced_census():
    """A2A imbalance extension: per-wave send bytes come from the plan census;
    a rank with more off-rank traffic / a slower GEMM dominates the prediction."""
    import numpy as np

    from oracle import alg1
    from paper_2504_19519_b200 import build

    build.build()
    n, N = 2, 256
    rng = np.random.default_rng(0)
    specs = []
    for r in range(n):
        rd = rng.integers(0, n, size=512).astype(np.int32)
        specs.append(dict(coll="alltoall", m=512, n=N, k=64, tile_m=128, tile_n=128, workers=2, row_dst=rd))
    wb = tuner.a2a_wave_bytes(specs)
    assert len(wb) == n and len(wb[0]) == 4
    # rank r's total off-rank bytes = rows routed elsewhere x N x 2
    for r in range(n):
        off = int((specs[r]["row_dst"] != r).sum())
        assert sum(wb[r]) == off * N * 2
    curve = [(2 ** 12, 5.0), (2 ** 20, 100.0), (2 ** 26, 400.0)]
    G, t = tuner.tune_alltoall(specs, [50.0, 80.0], curve)
    lat = lambda b: alg1.interp_latency_us(curve, b)
    assert t == pytest.approx(alg1.search_multi(4, [50.0, 80.0], wb, lat)[1], rel=1e-12)
    assert sum(G) == 4


def test_effective_curve_adds_post_cost():
    curve = [(1 << 20, 100.0), (1 << 24, 400.0)]
    eff = tuner.effective_curve(curve, post_us_per_byte=1e-5, post_fixed_us=2.0)
    for (b, bw), (_, ebw) in zip(curve, eff):
        t = b / (bw * 1e9) * 1e6
        te = b / (ebw * 1e9) * 1e6
        assert te == pytest.approx(t + 2.0 + 1e-5 * b)


def test_tune_alltoall_with_an_expert_without_rows():
    """An expert with no rows (m = 0, R45) sends nothing in every
    wave and takes duration 0; the common partition is the search over the
    other experts' waves, equal to the oracle's multi-rank Alg. 1."""
    import numpy as np

    from oracle import alg1
    from paper_2504_19519_b200 import build

    build.build()
    n, N = 3, 256
    rng = np.random.default_rng(1)
    specs = []
    for r in range(n):
        m = 0 if r == 1 else 512
        specs.append(dict(coll="alltoall", m=m, n=N, k=64, tile_m=128, tile_n=128, workers=2,
                          row_dst=rng.integers(0, n, size=m).astype(np.int32)))
    wb = tuner.a2a_wave_bytes(specs)
    assert [len(w) for w in wb] == [4, 4, 4] and sum(wb[1]) == 0
    for r in (0, 2):
        assert sum(wb[r]) == int((specs[r]["row_dst"] != r).sum()) * N * 2
    curve = [(2 ** 12, 5.0), (2 ** 20, 100.0), (2 ** 26, 400.0)]
    durs = [50.0, 0.0, 80.0]
    G, t = tuner.tune_alltoall(specs, durs, curve)
    lat = lambda b: alg1.interp_latency_us(curve, b)
    assert t == pytest.approx(alg1.search_multi(4, durs, wb, lat)[1], rel=1e-12)
