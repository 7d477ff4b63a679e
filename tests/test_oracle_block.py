"""Pins of oracle/block.py (the TP block oracle): SwiGLU closed forms and
layout by hand, the n = 1 reduction to the plain block, and the TP identity
(the AllReduce over n K-shards equals one rank holding all of K)."""
import numpy as np
import pytest

from oracle import block as ob
from oracle import numerics as onum


def test_silu_closed_forms():
    assert ob.silu(0.0) == 0.0
    x = np.linspace(-3, 3, 13)
    # silu(x) - silu(-x) = x (x sigma(x) - (-x) sigma(-x) = x (sigma(x) + sigma(-x)) = x)
    np.testing.assert_allclose(ob.silu(x) - ob.silu(-x), x, rtol=0, atol=1e-15)
    assert ob.silu(50.0) == pytest.approx(50.0, rel=1e-15)
    assert abs(ob.silu(-50.0)) < 1e-19
    assert ob.silu(1.0) == pytest.approx(1.0 / (1.0 + np.exp(-1.0)), rel=1e-15)


def test_swiglu_interleave_by_hand():
    """block = 2: columns [g0 g1 u0 u1 g2 g3 u2 u3] -> [silu(g0) u0, silu(g1) u1, silu(g2) u2, silu(g3) u3]."""
    g = np.array([0.5, -1.0, 2.0, 0.0])
    u = np.array([3.0, 4.0, -1.0, 7.0])
    gu = np.array([[g[0], g[1], u[0], u[1], g[2], g[3], u[2], u[3]]])
    want = [[ob.silu(g[i]) * u[i] for i in range(4)]]
    np.testing.assert_allclose(ob.swiglu_interleaved(gu, block=2), want, rtol=1e-15)
    with pytest.raises(ValueError):
        ob.swiglu_interleaved(np.zeros((1, 6)), block=2)


def _ints(rng, shape, lo=-2, hi=3):
    return rng.integers(lo, hi, size=shape).astype(np.float64)


def test_one_rank_is_the_plain_block():
    """n = 1: the block written out by hand with the same bf16 storage points."""
    rng = np.random.default_rng(1)
    T, H, I = 8, 256, 256
    attn, x = rng.standard_normal((T, H)), rng.standard_normal((T, H))
    Wo, Wgu, Wd = (rng.standard_normal(s) * 0.05 for s in ((H, H), (2 * I, H), (H, I)))
    gamma = rng.standard_normal(H)
    rb = onum.round_bf16
    c = rb(attn @ Wo.T)
    hh = c + x
    nn = rb(hh / np.sqrt(np.mean(hh * hh, axis=1, keepdims=True) + 1e-5) * gamma)
    gu = nn @ Wgu.T
    a = np.empty((T, I))
    for b in range(I // 128):
        gcol, ucol = gu[:, 256 * b:256 * b + 128], gu[:, 256 * b + 128:256 * b + 256]
        a[:, 128 * b:128 * b + 128] = gcol / (1 + np.exp(-gcol)) * ucol
    y = rb(rb(rb(rb(a) @ Wd.T)) + rb(hh))
    got_y, got_h = ob.tp_block([attn], x, [Wo], [Wgu], [Wd], gamma)
    np.testing.assert_array_equal(got_h, rb(hh))
    np.testing.assert_allclose(got_y, y, rtol=0, atol=0)


def test_tp_identity_on_integers():
    """With integer data small enough that nothing rounds, n ranks each holding
    a K-shard of o_proj / down-proj and an I-shard of gate/up give the n = 1
    result (the TP decomposition of PAPER.md:262)."""
    rng = np.random.default_rng(2)
    T, H, I, n = 4, 256, 512, 2
    attn = _ints(rng, (T, H))
    Wo = _ints(rng, (H, H), -1, 2)
    x = _ints(rng, (T, H))
    gamma = np.ones(H)
    Wd = _ints(rng, (H, I), -1, 2) * 0
    Wgu = _ints(rng, (2 * I, H), -1, 2) * 0          # zero MLP: y = bf16(h)
    y1, h1 = ob.tp_block([attn], x, [Wo], [Wgu], [Wd], gamma)
    Hs = H // n
    y2, h2 = ob.tp_block([attn[:, r * Hs:(r + 1) * Hs] for r in range(n)], x,
                         [Wo[:, r * Hs:(r + 1) * Hs] for r in range(n)],
                         [Wgu[r * (2 * I // n):(r + 1) * (2 * I // n)] for r in range(n)],
                         [Wd[:, r * (I // n):(r + 1) * (I // n)] for r in range(n)], gamma)
    np.testing.assert_array_equal(h1, h2)
    np.testing.assert_array_equal(y1, y2)
    np.testing.assert_array_equal(y1, onum.round_bf16(attn @ Wo.T + x))
