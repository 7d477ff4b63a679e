"""R42: Alg. 1 with the in-situ curve for the groups whose comm-stream work
overlaps the GEMM and the standalone curve for the last group (CPU only; the
library's tune_predict through the C ABI, no GPU)."""
import numpy as np
import pytest

from oracle import alg1 as oa

fo = pytest.importorskip("paper_2504_19519_b200")
from paper_2504_19519_b200 import tuner  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2504_19519_b200 import build

    build.build()


def _curve(rng, knee):
    """A bandwidth curve with a knee (small messages are slow)."""
    sizes = [1 << s for s in range(16, 29)]
    return [(b, float(800.0 * b / (b + knee) + rng.uniform(0, 5))) for b in sizes]


def test_last_group_swap_equals_two_curve_recurrence():
    """predict_insitu == Alg. 1 lines 10-22 restated with latency lat_i for
    every group but the last and lat_b for the last (the recurrence adds the
    last group's latency as its final term, so the swap is exact)."""
    rng = np.random.default_rng(42)
    for _ in range(200):
        S = int(rng.integers(1, 80))
        tiles = int(rng.integers(1, 12 * S + 1))
        T = -(-tiles // S)
        tile_bytes = int(rng.choice([32768, 65536, 131072]))
        dur = float(rng.uniform(10, 500))
        base = _curve(rng, float(rng.choice([1 << 20, 1 << 22])))
        icur = [(b, bw * float(rng.uniform(0.5, 1.0))) for b, bw in base]   # contended: slower
        cuts = sorted(set(int(c) for c in rng.integers(1, T, size=int(rng.integers(0, T)))) if T > 1 else [])
        b_ = [0] + cuts + [T]
        G = [y - x for x, y in zip(b_[:-1], b_[1:])]
        sizes = oa.group_bytes(G, S, tiles, tile_bytes)
        t_acc_p = t_acc_m = 0.0
        for i, g in enumerate(G):
            t_m = oa.interp_latency_us(icur, sizes[i - 1]) if i > 0 else 0.0
            t_acc_m = max(t_acc_p, t_acc_m) + t_m
            t_acc_p += dur / T * g
        want = max(t_acc_p, t_acc_m) + oa.interp_latency_us(base, sizes[-1])
        got = tuner.predict_insitu(G, dur, tiles, S, tile_bytes, icur, base)
        assert got == pytest.approx(want, rel=1e-9, abs=1e-9), (G, S, tiles)
        # one curve for both: the plain Alg. 1 prediction (the oracle's)
        same = tuner.predict_insitu(G, dur, tiles, S, tile_bytes, base, base)
        assert same == pytest.approx(oa.predict(G, dur, T, sizes, lambda x: oa.interp_latency_us(base, x)),
                                     rel=1e-9, abs=1e-9)


def test_single_group_is_gemm_plus_standalone_collective():
    """One group: the whole GEMM, then the collective after it — the
    standalone curve, whatever the in-situ one says (SPEC.md:307 closed form)."""
    base = [(1 << 20, 100.0), (1 << 26, 500.0)]
    icur = [(1 << 20, 10.0), (1 << 26, 50.0)]
    tiles, S, tb, dur = 256, 64, 131072, 300.0
    got = tuner.predict_insitu([4], dur, tiles, S, tb, icur, base)
    assert got == pytest.approx(dur + oa.interp_latency_us(base, tiles * tb), rel=1e-12)
