"""Oracle step O4: the per-rank GEMM in fp64, and bf16 round-to-nearest-even.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:224: "A^{MxK} x B^{KxN} = C^{MxN}".  The GEMM is the plain definition
C[i, j] = sum_k A[i, k] * Bt[j, k], evaluated by numpy's fp64 matmul (a library
primitive standing for one step).  bf16 inputs are widened exactly to fp64.

`round_bf16` models the GPU epilogue's fp32 -> bf16 conversion (RNE; DESIGN.md
reading R10); it is written out from the bf16 definition (8 significant bits,
round half to even) rather than calling a library conversion.

Pins (tests/test_oracle_numerics.py): gemm vs a brute-force triple loop on tiny
inputs; exact-integer regime closed form; round_bf16 vs torch's fp32->bf16
conversion on fp32-representable values (a library routine), and on the
hand-checkable tie cases 1 + 2^-8 -> 1, 1 + 3*2^-8 -> 1 + 2^-6.
"""
from __future__ import annotations

import numpy as np


def to_f64(x) -> np.ndarray:
    """bf16 (torch tensor or array) -> exact fp64 numpy array."""
    try:
        import torch

        if isinstance(x, torch.Tensor):
            return x.detach().to(torch.float64).cpu().numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(x, dtype=np.float64)


def gemm(A, Bt) -> np.ndarray:
    """C = A @ Bt^T in fp64 (A: [M, K], Bt: [N, K])."""
    A64 = to_f64(A)
    B64 = to_f64(Bt)
    if A64.shape[1] != B64.shape[1]:
        raise ValueError("K mismatch")
    return A64 @ B64.T


def round_bf16(x) -> np.ndarray:
    """Round fp64 values to the nearest bf16 value, ties to even.

    bf16 keeps 8 significant bits.  Write |x| = m * 2^e with 0.5 <= m < 1
    (np.frexp); the bf16 value is rint(m * 2^8) * 2^(e-8) where rint rounds
    half to even.  (Normal range only; the workloads never reach bf16
    subnormals or overflow, and zero maps to zero.)"""
    x = np.asarray(x, dtype=np.float64)
    m, e = np.frexp(x)
    q = np.rint(m * 256.0)
    return np.ldexp(q, e - 8)
