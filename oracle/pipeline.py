"""Oracle steps O4-O9 composed: the overlapped pipeline on n simulated ranks,
and the plain definition it must equal.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

run_*  : GEMM (O4) -> pre-reorder (O5) -> per-group collective (O6) ->
         post-reorder (O7), in the paper's order (PAPER.md:297 fig:framework
         caption: "when each group ... finishes, it first reorders the tiles in
         the group to contiguous addresses, and then signals to trigger the
         corresponding inter-GPU communication ... the tiles are reordered back
         when communication finishes").
plain_*: O8, the sequential GEMM -> collective result by its definition
         (PAPER.md:834 claim C1 "mathematical equivalence with the non-overlap
         implementation"):  AR: sum_r Y_r;  RS: rows R_k of sum_r Y_r;
         A2A: concat_s Y_s[rows with destination me].

Pins (tests/test_oracle_pipeline.py): run_* == plain_* bit-exactly on
integer data for every order of a 2x3 tile grid x every partition x
S in {1,2,3} x n in {1,2,3} (brute force on tiny inputs), and on seeded random
cases for n in {2,4,8} x swizzle in {1,2,4}.
"""
from __future__ import annotations

import numpy as np

from . import collectives, numerics, reorder
from .plan import Plan


def _Y(A, Bt, model_bf16: bool):
    Y = numerics.gemm(A, Bt)
    return numerics.round_bf16(Y) if model_bf16 else Y


# ------------------------------------------------------------------ AllReduce
def run_allreduce(As, Bts, plan: Plan, layout="slot", model_bf16=False):
    n = len(As)
    Ys = [_Y(As[r], Bts[r], model_bf16) for r in range(n)]
    bufs = [reorder.ar_pre(Ys[r], plan, layout) for r in range(n)]
    red = collectives.allreduce_groups(bufs, reorder.group_elem_ranges(plan, layout))
    outs = [reorder.ar_post(red[r], plan, layout) for r in range(n)]
    return {"Y": Ys, "send": bufs, "recv": red, "out": outs}


def plain_allreduce(As, Bts, model_bf16=False):
    n = len(As)
    C = None
    for r in range(n):
        Y = _Y(As[r], Bts[r], model_bf16)
        C = Y if C is None else C + Y
    return [C.copy() for _ in range(n)]


# ------------------------------------------------------------------ ReduceScatter
def run_reducescatter(As, Bts, plan: Plan, layout="slot", model_bf16=False):
    n = len(As)
    Ys = [_Y(As[r], Bts[r], model_bf16) for r in range(n)]
    bufs = [reorder.rs_pre(Ys[r], plan, n, layout) for r in range(n)]
    recv = collectives.reduce_scatter_groups(bufs, reorder.group_elem_ranges(plan, layout))
    outs = [reorder.rs_post(recv[k], plan, n, layout) for k in range(n)]
    return {"Y": Ys, "send": bufs, "recv": recv, "out": outs}


def rs_rows_of_rank(M: int, BM: int, n: int, k: int) -> np.ndarray:
    """R_k = { g : floor((g mod BM) / (BM/n)) == k }, ascending."""
    h = BM // n
    g = np.arange(M)
    return g[((g % BM) // h) == k]


def plain_reducescatter(As, Bts, BM: int, model_bf16=False):
    n = len(As)
    C = plain_allreduce(As, Bts, model_bf16)[0]
    return [C[rs_rows_of_rank(C.shape[0], BM, n, k)] for k in range(n)]


def row_exchange(gathered: np.ndarray, BM: int, n: int) -> np.ndarray:
    """RS follow-on: after AllGather of the block-cyclic local
    outputs (rank order), restore standard row order.  Gathered row
    k*(M/n) + l is global row rs_local_to_global_row(l, BM, h, k)."""
    M = gathered.shape[0]
    h = BM // n
    out = np.empty_like(gathered)
    for k in range(n):
        for l in range(M // n):
            out[reorder.rs_local_to_global_row(l, BM, h, k)] = gathered[k * (M // n) + l]
    return out


# ------------------------------------------------------------------ All-to-All
def run_alltoall(As, Bts, plans, row_dsts, model_bf16=False, layout="slot"):
    """plans[s], row_dsts[s]: source rank s's own plan (its M may differ from
    the others', PAPER.md:264 imbalance) and row destinations."""
    n = len(As)
    P = len(plans[0].ranges)
    if any(len(p.ranges) != P for p in plans):
        raise reorder.OracleError("all ranks need the same number of wave groups")
    Ys = [_Y(As[s], Bts[s], model_bf16) for s in range(n)]
    sends = [reorder.a2a_pre(Ys[s], plans[s], row_dsts[s], n, layout) for s in range(n)]
    recv = collectives.alltoall_groups(sends, P)
    N, BN = plans[0].N, plans[0].BN
    outs = [reorder.a2a_post(recv[d], [sends[s].meta[d] for s in range(n)], row_dsts, d, N, BN)
            for d in range(n)]
    return {"Y": Ys, "send": sends, "recv": recv, "out": outs}


def plain_alltoall(As, Bts, row_dsts, model_bf16=False):
    n = len(As)
    Ys = [_Y(As[s], Bts[s], model_bf16) for s in range(n)]
    outs = []
    for d in range(n):
        parts = [Ys[s][np.asarray(row_dsts[s]) == d] for s in range(n)]
        outs.append(np.concatenate(parts, axis=0))
    return outs
