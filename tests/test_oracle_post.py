"""Pins for the fused elementwise oracle (residual add + RMSNorm, reading R12)."""
import numpy as np

from oracle import post


def test_constant_rows():
    c, eps = 3.0, 1e-5
    y = np.full((4, 16), c)
    g = np.linspace(0.5, 2.0, 16)
    out = post.rmsnorm(y, g, eps)
    assert np.allclose(out, c / np.sqrt(c * c + eps) * g[None, :], rtol=0, atol=1e-15)


def test_unit_rms_rows_unchanged():
    rng = np.random.default_rng(0)
    y = rng.standard_normal((8, 32))
    y /= np.sqrt(np.mean(y * y, axis=1, keepdims=True))
    assert np.allclose(post.rmsnorm(y, np.ones(32), 0.0), y, rtol=1e-14, atol=1e-14)


def test_scale_invariance_and_add():
    rng = np.random.default_rng(1)
    x, r = rng.standard_normal((8, 32)), rng.standard_normal((8, 32))
    g = rng.standard_normal(32)
    a = post.add_rmsnorm(x, r, g, 0.0)
    b = post.add_rmsnorm(7 * x, 7 * r, g, 0.0)
    assert np.allclose(a, b, rtol=1e-12, atol=1e-12)
    assert np.array_equal(post.add(x, r), x + r)
