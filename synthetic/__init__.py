"""Seeded synthetic input generators shared by the tests, the bench and smoke().

This module holds NONE of the method's arithmetic (no tiling, no reordering, no
GEMM, no collective).  It only draws seeded random inputs with the shapes and
value distributions of the paper's workloads ("we use randomly
generated inputs").  Both the CPU oracle (`oracle/`)
and the CUDA path consume what it returns; neither imports the other.

All matrices are returned as CPU `torch.bfloat16` tensors (row-major,
contiguous).  A is [M, K_loc] (activations, K-major); Bt is [N, K_loc] (the
nn.Linear weight layout, K-major), so C = A @ Bt^T.
"""
from __future__ import annotations

import hashlib

import numpy as np
import torch

__all__ = [
    "rank_seed",
    "cell_seed",
    "normal_bf16",
    "exact_int_A",
    "exact_int_B",
    "float_inputs",
    "exact_inputs",
    "random_order",
    "random_partition",
    "moe_routing",
    "balanced_moe_row_dst",
    "random_row_dst",
]


def rank_seed(base: int, tp: int, rank: int) -> int:
    """Seed recipe of SURVEY.md §8(d): seed = base + 100*TP + rank."""
    return int(base) + 100 * int(tp) + int(rank)


def cell_seed(*parts) -> int:
    """Deterministic seed from a tuple of cell parameters (sweep cells)."""
    h = hashlib.sha256(repr(tuple(parts)).encode()).digest()
    return int.from_bytes(h[:4], "little")


def _gen(seed: int, device="cpu") -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed) & 0x7FFFFFFFFFFFFFFF)
    return g


def normal_bf16(shape, std: float, seed: int, device="cpu") -> torch.Tensor:
    """N(0, std^2) draws rounded to bf16 (torch's own fp32->bf16 conversion).
    device="cuda" draws with the CUDA generator (a different, equally seeded
    stream) for full-size inputs; callers copy what the oracle needs to CPU."""
    x = torch.randn(*shape, generator=_gen(seed, device), dtype=torch.float32, device=device)
    if std != 1.0:
        x = x * std
    return x.to(torch.bfloat16).contiguous()


def exact_int_A(M: int, K: int, seed: int, nnz_per_row: int) -> torch.Tensor:
    """Exact-integer regime: entries in {-1,0,1}, at most
    `nnz_per_row` nonzeros per row.  The caller picks nnz_per_row so that the
    nonzeros per output row summed over all ranks stay <= 256, which keeps
    every partial sum an integer of magnitude <= 256 (exact in bf16 and fp32)."""
    g = _gen(seed)
    nnz = max(0, min(int(nnz_per_row), K))
    A = torch.zeros(M, K, dtype=torch.float32)
    if nnz > 0 and M > 0:
        # random column subset per row + random signs
        keys = torch.rand(M, K, generator=g)
        cols = keys.argsort(dim=1)[:, :nnz]
        signs = torch.randint(0, 2, (M, nnz), generator=g).float() * 2 - 1
        # allow some zeros inside the support too
        keep = (torch.rand(M, nnz, generator=g) < 0.9).float()
        A.scatter_(1, cols, signs * keep)
    return A.to(torch.bfloat16).contiguous()


def exact_int_B(N: int, K: int, seed: int) -> torch.Tensor:
    """Dense {-1,0,1} weights for the exact-integer regime."""
    g = _gen(seed)
    B = torch.randint(-1, 2, (N, K), generator=g).float()
    return B.to(torch.bfloat16).contiguous()


def float_inputs(M: int, N: int, K: int, seed: int, device="cpu"):
    """Float regime of SURVEY.md §8(d): A ~ N(0,1) (activations), Bt ~ N(0,0.02^2)
    (weights), both bf16."""
    A = normal_bf16((M, K), 1.0, seed * 2 + 1, device)
    Bt = normal_bf16((N, K), 0.02, seed * 2 + 2, device)
    return A, Bt


def balanced_moe_row_dst(rows_per_src: int, n_ranks: int) -> np.ndarray:
    """Exact-balanced EP routing (SURVEY.md §8(d) C4 variant): an expert rank
    holds rows_per_src rows from every source rank, sorted by source."""
    return np.repeat(np.arange(n_ranks, dtype=np.int32), rows_per_src)


def exact_inputs(M: int, N: int, K: int, seed: int, nnz_per_row: int):
    A = exact_int_A(M, K, seed * 2 + 1, nnz_per_row)
    Bt = exact_int_B(N, K, seed * 2 + 2)
    return A, Bt


def random_order(ntiles: int, seed: int) -> np.ndarray:
    """A random explicit tile execution order (a permutation), int32."""
    rng = np.random.default_rng(seed)
    return rng.permutation(ntiles).astype(np.int32)


def random_partition(T: int, seed: int) -> list[int]:
    """A random composition of T (random communicate/not decision after each
    wave but the last)."""
    rng = np.random.default_rng(seed)
    cuts = [w for w in range(1, T) if rng.random() < 0.5]
    bounds = [0] + cuts + [T]
    return [bounds[i + 1] - bounds[i] for i in range(len(bounds) - 1)]


def random_row_dst(M: int, n: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.integers(0, n, size=M).astype(np.int32)


def moe_topk(tokens: int, n_ranks: int, topk: int, seed: int, skew: float = 0.0, pad: int = 1) -> dict:
    """Mixtral-style top-k routing with one expert per rank (expert e on rank
    e; BASELINE.json configs[3], EP = number of experts) — the inputs of the
    MoE combine that follows the expert GEMM + All-to-All (R31).

    Tokens are spread evenly over the ranks (token t lives on rank t // (tokens
    // n_ranks)).  Router logits ~ N(0,1) from `seed`, plus `skew` * (-log(e+1))
    for expert e (skew > 0: a Zipf-like preference for low experts -> expert
    load imbalance).  Each token picks its top-k experts; its
    combine weights are the softmax over those k logits (fp32).

    Returns dict:
      top     [tokens, k] int   expert ids (descending logit)
      weight  [tokens, k] f32   combine weights
      row_token[e]  int64 [M_e] global token of each row expert e computes,
                                rows sorted by (source rank, token id) as the
                                dispatch All-to-All delivers them; with pad > 1
                                M_e is rounded up to a multiple of pad by rows
                                of token -1 (zero activations, kept on rank e)
      row_dst[e]    int32 [M_e] source rank of each row (= the A2A destination)
      combine_idx[r] int32 [tokens/n, k]: for rank r's local token l and slot i,
                                the row of r's A2A output holding expert
                                top[t, i]'s result (A2A output order: source
                                expert ascending, then source row ascending)"""
    g = _gen(seed)
    logits = torch.randn(tokens, n_ranks, generator=g, dtype=torch.float64)
    if skew:
        logits = logits - skew * torch.log(torch.arange(1, n_ranks + 1, dtype=torch.float64))[None, :]
    top_l, top = logits.topk(topk, dim=1)
    weight = torch.softmax(top_l, dim=1).to(torch.float32).numpy()
    top = top.numpy()
    per_rank = tokens // n_ranks
    row_token, row_dst = [], []
    for e in range(n_ranks):
        toks = np.flatnonzero((top == e).any(axis=1))          # ascending token id = (source, token) order
        npad = (-len(toks)) % pad
        row_token.append(np.concatenate([toks, np.full(npad, -1)]).astype(np.int64))
        row_dst.append(np.concatenate([toks // per_rank, np.full(npad, e)]).astype(np.int32))
    combine_idx = []
    for r in range(n_ranks):
        # rank r's A2A output: for each expert e ascending, the rows of e whose
        # destination is r, in e's row order
        base, pos = 0, {}
        for e in range(n_ranks):
            mine = row_token[e][row_dst[e] == r]
            for q, t in enumerate(mine):
                if t >= 0:
                    pos[(int(t), e)] = base + q
            base += len(mine)
        idx = np.empty((per_rank, topk), np.int32)
        for l in range(per_rank):
            t = r * per_rank + l
            for i in range(topk):
                idx[l, i] = pos[(t, int(top[t, i]))]
        combine_idx.append(idx)
    return {"top": top, "weight": weight, "row_token": row_token, "row_dst": row_dst,
            "combine_idx": combine_idx}


def moe_routing(tokens: int, n_experts: int, topk: int, n_ranks: int, seed: int):
    """Mixtral-style top-k routing (BASELINE.json configs[3]; SURVEY.md ambiguity 20).

    `tokens` tokens are spread evenly over `n_ranks` source ranks (token t lives
    on rank t // (tokens // n_ranks)).  Router logits ~ N(0,1) from `seed`;
    each token picks its top-k experts.  Experts are placed one per rank
    (expert e on rank e % n_ranks).

    Returns a list, per expert rank e, of the int32 array `row_dst` giving the
    source rank of each row that expert computes; rows are sorted by source
    rank (then token id), as the dispatch All-to-All would deliver them."""
    g = _gen(seed)
    logits = torch.randn(tokens, n_experts, generator=g)
    top = logits.topk(topk, dim=1).indices.numpy()
    per_rank = tokens // n_ranks
    out = []
    for r in range(n_ranks):
        experts_here = [e for e in range(n_experts) if e % n_ranks == r]
        rows = []
        for t in range(tokens):
            for e in experts_here:
                if e in top[t]:
                    rows.append((t // per_rank, t))
        rows.sort()
        out.append(np.array([s for s, _ in rows], dtype=np.int32))
    return out


def pad_row_dst(row_dst, multiple: int, own_rank: int) -> np.ndarray:
    """Pad an expert's routed rows to a multiple of the GEMM tile height, as MoE
    expert kernels pad token counts; padding rows (zero activations) stay on the
    expert's own rank and are appended after the routed rows."""
    row_dst = np.asarray(row_dst, np.int32)
    pad = (-len(row_dst)) % multiple
    return np.concatenate([row_dst, np.full(pad, own_rank, np.int32)])
