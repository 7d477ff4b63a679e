"""Oracle for the elementwise op fused after the post-communication reorder.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:394 ("can be seamlessly fused into the subsequent element-wise kernel")
and PAPER.md:671 (an RMSNorm kernel fused with the post-reorder).  The paper
does not define its RMSNorm; reading R12:

    y   = x + residual                    (FO_POST_ADD)
    out = y / sqrt(mean_j(y_j^2) + eps) * gamma   (FO_POST_ADD_RMSNORM, per row)

Pins (tests/test_oracle_post.py): rows of a constant c give c/sqrt(c^2+eps)*gamma;
scaling invariance out(a*y) ~= out(y) for eps -> 0; unit-norm rows unchanged
when gamma = 1 and eps = 0.
"""
from __future__ import annotations

import numpy as np


def add(x, residual):
    return np.asarray(x, np.float64) + np.asarray(residual, np.float64)


def rmsnorm(y, gamma, eps: float):
    y = np.asarray(y, np.float64)
    ms = np.mean(y * y, axis=1, keepdims=True)
    return y / np.sqrt(ms + eps) * np.asarray(gamma, np.float64)[None, :]


def add_rmsnorm(x, residual, gamma, eps: float):
    return rmsnorm(add(x, residual), gamma, eps)
