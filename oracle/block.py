"""Oracle of the tensor-parallel transformer block (NEXT f4, second workload):
the communication-bearing half of a pre-norm decoder block, composed from the
oracle's own steps, on `n` simulated TP ranks.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:262 (TP row-parallel linear followed by AllReduce), PAPER.md:394 and
671 (the post-communication reorder fused into the following RMSNorm),
PAPER.md:559-578 (the Llama end-to-end setting).  Per rank r:

    c   = bf16(sum_r bf16(attn_r @ Wo_r^T))        o_proj + AllReduce (O4, O6, O8)
    h   = x + c
    n   = bf16(RMSNorm(h) * gamma); x <- bf16(h)   fused add + RMSNorm, residual stream
    gu  = n @ Wgu_r^T                              gate/up (column-parallel), fp64
    a_r = bf16(silu(g) * u)                        SwiGLU on the interleaved layout below
    y   = bf16(bf16(h) + bf16(sum_r bf16(a_r @ Wd_r^T)))   down-proj + AllReduce + residual add

bf16 roundings sit exactly where the library stores bf16 (R10: the
GEMM epilogue's output, the AllReduce's bf16 buffer, the fused op's outputs);
the AllReduce sums the bf16 partials in fp64 and rounds the sum once (R11).  The fused op's sum y = x + c is rounded once, when it
is stored.

SwiGLU weight layout (FO_OPT_GEMM_SWIGLU, include/flashoverlap.h): the gate
and up weight rows are interleaved in blocks of 128 — rows [256b, 256b+128)
are gate rows 128b..128b+127 and rows [256b+128, 256b+256) the matching up
rows — so output column 128b + i = silu(gu[:, 256b + i]) * gu[:, 256b + 128 + i].

Pins (tests/test_oracle_block.py): silu closed forms (silu(0) = 0, odd part
x/2, silu(x) -> x and -> 0 at +-large x); the interleave on a hand-built
case; n = 1 reduces to the plain single-device block; the AllReduce of n
ranks equals one rank holding the concatenated K shards (TP identity).
"""
from __future__ import annotations

import numpy as np

from . import numerics
from . import post


def silu(x):
    x = np.asarray(x, np.float64)
    return x / (1.0 + np.exp(-x))


def swiglu_interleaved(gu, block: int = 128):
    """gu [T, 2I] with gate / up rows interleaved in blocks of `block` -> [T, I]."""
    gu = np.asarray(gu, np.float64)
    T, two_i = gu.shape
    if two_i % (2 * block):
        raise ValueError("gate/up width must be a multiple of 2*block")
    v = gu.reshape(T, two_i // (2 * block), 2, block)
    return (silu(v[:, :, 0, :]) * v[:, :, 1, :]).reshape(T, two_i // 2)


def tp_block(attn, x, Wo, Wgu, Wd, gamma, eps: float = 1e-5):
    """attn[r] [T, H/n], Wo[r] [H, H/n], Wgu[r] [2I/n, H], Wd[r] [H, I/n] per
    rank; x [T, H] the residual stream; gamma [H].  Returns (y, h_bf16) with y
    the block output [T, H] (identical on every rank) and h_bf16 the updated
    residual stream."""
    n = len(attn)
    rb = numerics.round_bf16
    # o_proj, row-parallel: each rank's bf16 partial, AllReduce (sum)
    c = rb(sum(rb(numerics.gemm(attn[r], Wo[r])) for r in range(n)))
    # fused add + RMSNorm that also writes the residual stream back
    n_out, h_bf16 = post.add_rmsnorm_residual(c, x, gamma, eps)
    n_bf16 = rb(n_out)
    # gate/up + SwiGLU (column-parallel: every rank its own I/n columns), down-proj partials
    parts = []
    for r in range(n):
        a_r = rb(swiglu_interleaved(numerics.gemm(n_bf16, Wgu[r])))
        parts.append(rb(numerics.gemm(a_r, Wd[r])))
    y = rb(post.add(rb(sum(parts)), h_bf16))
    return y, h_bf16
