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


def test_add_rmsnorm_residual_keeps_the_rounded_sum():
    """The residual-writing variant: out equals add_rmsnorm, and the new
    residual is the bf16 rounding of x + residual — exact for sums that are
    bf16-representable (small integers), rounded to nearest even otherwise."""
    x = np.array([[1.0, 2.0, -3.0, 4.0], [256.0, 1.0, 0.5, -0.25]])
    r = np.array([[1.0, 1.0, 1.0, 1.0], [1.0, 0.0, 0.0, 0.0]])
    g = np.ones(4)
    out, res = post.add_rmsnorm_residual(x, r, g, 1e-5)
    assert np.array_equal(out, post.add_rmsnorm(x, r, g, 1e-5))
    assert np.array_equal(res[0], [2.0, 3.0, -2.0, 5.0])
    # 257 is not representable in bf16 (8 significant bits): ties to even -> 256
    assert res[1, 0] == 256.0 and np.array_equal(res[1, 1:], [1.0, 0.5, -0.25])
