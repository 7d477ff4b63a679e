"""Oracle for the elementwise op fused after the post-communication reorder.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:394 ("can be seamlessly fused into the subsequent element-wise kernel")
and PAPER.md:671 (an RMSNorm kernel fused with the post-reorder).  The paper
does not define its RMSNorm; reading R12:

    y   = x + residual                    (FO_POST_ADD)
    out = y / sqrt(mean_j(y_j^2) + eps) * gamma   (FO_POST_ADD_RMSNORM, per row)
    FO_POST_ADD_RMSNORM_RESIDUAL: the same out, and the residual buffer
    becomes bf16(y) — the residual stream of a pre-norm transformer block
    (NEXT f4's TP block; the fused add + RMSNorm of inference engines).

MoE combine after the expert GEMM + All-to-All (the A2A
"transfer[s] the processed data back to the original GPUs after expert
computation"; fused into the post-reorder per PAPER.md:394; R31):

    out[t] = sum_i [idx[t,i] valid] * w[t,i] * x[idx[t,i]]   (+ residual[t])

where x is the rank's A2A output (standard order) and idx[t,i] the row of
token t's i-th expert result; an index < 0 or >= rows is a dropped slot.

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


def add_rmsnorm_residual(x, residual, gamma, eps: float):
    """(out, new_residual): out = add_rmsnorm(x, residual); new_residual =
    round-to-nearest-even bf16 of y = x + residual (the buffer is bf16)."""
    from .numerics import round_bf16

    y = add(x, residual)
    return rmsnorm(y, gamma, eps), round_bf16(y)


def topk_combine(x, idx, w, residual=None):
    """MoE top-k weighted combine (module header), fp64, one token at a time."""
    x = np.asarray(x, np.float64)
    idx = np.asarray(idx)
    w = np.asarray(w, np.float64)
    T, k = idx.shape
    out = np.zeros((T, x.shape[1]))
    for t in range(T):
        for i in range(k):
            r = int(idx[t, i])
            if 0 <= r < x.shape[0]:
                out[t] += w[t, i] * x[r]
    if residual is not None:
        out += np.asarray(residual, np.float64)
    return out
