"""GPU parity at BASELINE.json's full sizes (configs[1..3]) in the launch
configuration bench.py uses (256x256 CTA-pair tiles, S = 64 pairs), on the
FULL output matrices against the fp64 oracle (float regime, tolerance 1e-2).

Multi-rank configurations run every rank's GEMM + pre-reorder epilogue on the
one GPU through fo_gemm_stage; the collective between them is emulated on the
GPU by this test in two ways: as NCCL's ring computes a bf16 sum (the bf16
partials added one rank at a time, rounded to bf16 after every hop) and as a
reduction that accumulates in fp32 and rounds once (NVLS-style); each
receiver's post-reorder runs through fo_post_stage.  The ring result is held
to (a) the first-order rounding bound of the whole computation
against the unrounded fp64 definition, |g - o| <= u (sum_r |p_r| + sum_k |s_k|)
+ K 2^-23 sum_r |A_r||B_r|^T (u = 2^-8, p_r the fp64 partials, s_k the
computed running sums of the ring, the last term each rank's fp32
accumulation over its K products); the fp32-reduction result to (b) the
north_star 1e-2 against the oracle in its bf16 model (bf16 partials summed,
bf16 output; R11).  The ring's error against that model (and both against the
plain fp64 definition) is printed, not asserted: a bf16 ring sum of 8 partials
exceeds 1e-2 at the tails by itself (R11).
The single-rank bench configuration runs through fo_run with the real NCCL.
"""
import numpy as np
import pytest
import torch

import synthetic
from oracle import numerics as onum
from oracle import reorder as orr

pytestmark = pytest.mark.gpu
fo = pytest.importorskip("paper_2504_19519_b200")
TOL = 1e-2
BM = BN = 256
S = 64


@pytest.fixture(scope="module", autouse=True)
def _dev():
    from paper_2504_19519_b200 import build

    build.build()
    torch.cuda.set_device(0)


U = 2.0 ** -8  # bf16 unit roundoff: 8 significand bits, round to nearest -> |fl(x) - x| <= 2^-8 |x|


def _check_rows(got_rows, want_rows, partials=None, running=None, absprod=None, K=0, tol=True):
    """Tolerance check (R10/R11).

    want_rows: the oracle value (fp64).  With `partials` (per-rank fp64 values)
    the oracle is taken in its bf16 model (each rank's partial rounded to bf16,
    R10: the send buffer is bf16 by construction; their sum rounded to the bf16
    output) for the 1e-2 metric,
    and the unrounded fp64 definition is held to the elementwise first-order
    bound of the emulated bf16 ring sum: |g - o| <= u (sum_r |p_r| + sum_k
    |s_k|), `running` = sum_k |s_k| over the computed running sums (without it,
    one rounding of the total: u (sum_r |p_r| + |o|)), plus the fp32
    accumulation of each rank's K products, K 2^-23 sum_r (|A_r| |B_r|^T)
    (`absprod`; 2^-23 allows a truncating accumulator)."""
    g = got_rows.double().cpu().numpy() if isinstance(got_rows, torch.Tensor) else got_rows
    o = np.asarray(want_rows, np.float64)
    if partials is not None:
        absum = np.zeros_like(o)
        model = None
        for p in partials:
            absum += np.abs(p)
            q = onum.round_bf16(p)
            model = q if model is None else model + q
        bound = 1.01 * U * (absum + (running if running is not None else np.abs(o)))
        if absprod is not None:
            bound += 1.01 * K * 2.0 ** -23 * absprod
        ratio = np.max(np.abs(g - o) / bound)
        print(f"  |g - o| / rounding bound: max {ratio:.3f}")
        assert ratio <= 1.0, "outside the bf16 rounding bound of the plain definition"
        rms0 = np.sqrt(np.mean(o * o))
        print(f"  max rel err vs the plain fp64 definition (no tolerance; DESIGN.md R11): "
              f"{np.max(np.abs(g - o) / np.maximum(np.abs(o), rms0)):.3e}")
        del absum, bound
        o = onum.round_bf16(model)           # the output is bf16: the model's too
    rms = np.sqrt(np.mean(o * o))
    err = np.max(np.abs(g - o) / np.maximum(np.abs(o), rms))
    if tol:
        assert err <= TOL, f"max rel err {err}"
    return err


def _ring_sum(sends):
    """NCCL-style bf16 ring reduction of the ranks' bf16 send buffers: added
    one rank at a time in fp32, rounded to bf16 after every hop.  Returns the
    bf16 sum and sum_k |s_k| (fp64, on the CPU) for the rounding bound."""
    acc = sends[0].clone()
    run = torch.zeros(acc.numel(), dtype=torch.float64)
    for x in sends[1:]:
        acc = (acc.float() + x.float()).to(torch.bfloat16)
        run += acc.double().abs().cpu()
    return acc, run.numpy()


def _fp32_sum(sends):
    """A reduction that accumulates in fp32 and rounds once (NVLS in-switch
    reduction with an fp32 accumulator, or a tree that widens)."""
    acc = torch.zeros(sends[0].numel(), dtype=torch.float32, device="cuda")
    for x in sends:
        acc += x.float()
    return acc.to(torch.bfloat16)


def _gemm_full(A, Bt):
    """fp64 oracle GEMM of a whole (CPU) operand pair."""
    return onum.gemm(A.cpu() if isinstance(A, torch.Tensor) else A, Bt.cpu() if isinstance(Bt, torch.Tensor) else Bt)


def _absprod(As, Bts):
    """sum_r |A_r| |B_r|^T in fp64 (the scale of the fp32 accumulation error)."""
    out = None
    for A, Bt in zip(As, Bts):
        x = _gemm_full(A.abs(), Bt.abs())
        out = x if out is None else out + x
    return out


def test_c2_bench_config_tp1_fo_run():
    """configs[1] at TP=1 exactly as bench.py runs it (fo_run, NCCL world 1)."""
    M, N, K = 4096, 4096, 14336
    A, Bt = synthetic.float_inputs(M, N, K, seed=synthetic.rank_seed(20000, 1, 0))
    plan = fo.Plan(coll="allreduce", m=M, n=N, k=K, tile_m=BM, tile_n=BN, workers=S, group_waves=[1, 2, 1])
    assert plan.info["ar_layout"] == 1  # ROWBAND at S=64, Nt=16
    ctx = fo.Context.create(0, 0, 1, fo.unique_id())
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    fo.run(ctx, plan, A.cuda(), Bt.cuda(), out)
    torch.cuda.synchronize()
    _check_rows(out, _gemm_full(A, Bt))
    ctx.close()


@pytest.mark.parametrize("layout", ["slot", "rowband"])
def test_c2_tp8_allreduce(layout):
    """configs[1] at TP=8: M=N=4096, K_loc=1792, 8 ranks."""
    n, M, N, K = 8, 4096, 4096, 14336 // 8
    groups = [1, 2, 1]
    As, Bts, plans, sends = [], [], [], []
    for r in range(n):
        A, Bt = synthetic.float_inputs(M, N, K, seed=synthetic.rank_seed(20000, n, r), device="cuda")
        plan = fo.Plan(coll="allreduce", m=M, n=N, k=K, tile_m=BM, tile_n=BN, workers=S, group_waves=groups,
                       ar_layout=layout, rank=r, world=n)
        send = torch.empty(M * N, dtype=torch.bfloat16, device="cuda")
        fo.gemm_stage(plan, A, Bt, send)
        sends.append(send)
        As.append(A)
        Bts.append(Bt)
        plans.append(plan)
    # every group's AllReduce reduces the same positions on all ranks, so the
    # ring sum of the whole buffers is the per-group sums side by side
    ring, running = _ring_sum(sends)
    flat = _fp32_sum(sends)
    del sends
    parts = [_gemm_full(As[r], Bts[r]) for r in range(n)]
    want = sum(parts)
    absprod = _absprod(As, Bts)
    for r in (0, n - 1):
        out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        # (a) ring, bf16 after every hop: the rounding bound against the plain definition
        fo.post_stage(plans[r], ring, out)
        torch.cuda.synchronize()
        # the running sums live in send-buffer order: bring them to C's order
        run_c = running[plans[r].export_send_map()].reshape(M, N)
        err_ring = _check_rows(out, want, parts, run_c, absprod, K, tol=False)
        # (b) fp32-accumulating reduction: 1e-2 against the bf16-epilogue model
        fo.post_stage(plans[r], flat, out)
        torch.cuda.synchronize()
        err = _check_rows(out, want, parts, None, absprod, K)
        print(f"TP=8 AllReduce ({layout}), rank {r}: max rel err vs the bf16-epilogue model {err:.3e} "
              f"(fp32 reduction), {err_ring:.3e} (bf16 ring, bound-checked)")


def test_c3_tp8_reducescatter():
    """configs[2]: Llama-3-70B o_proj, M=N=8192, K_loc=1024, RS at TP=8."""
    n, M, N, K = 8, 8192, 8192, 8192 // 8
    groups = [2, 4, 6, 4]  # T = 1024 tiles / 64 = 16
    plans = [fo.Plan(coll="reducescatter", m=M, n=N, k=K, tile_m=BM, tile_n=BN, workers=S, group_waves=groups,
                     rank=r, world=n) for r in range(n)]
    As, Bts, sends = [], [], []
    for r in range(n):
        A, Bt = synthetic.float_inputs(M, N, K, seed=synthetic.rank_seed(30000, n, r), device="cuda")
        send = torch.empty(M * N, dtype=torch.bfloat16, device="cuda")
        fo.gemm_stage(plans[r], A, Bt, send)
        sends.append(send)
        As.append(A)
        Bts.append(Bt)
    ring, running = _ring_sum(sends)
    flat = _fp32_sum(sends)
    del sends
    h = BM // n
    for k in (0, 5):
        # every local row of rank k: global row floor(l/h)*BM + k*h + l%h (R8)
        grows = [orr.rs_local_to_global_row(l, BM, h, k) for l in range(M // n)]
        parts_o = [_gemm_full(As[r][grows], Bts[r]) for r in range(n)]
        absprod = _absprod([A[grows] for A in As], Bts)
        run_c = running[plans[k].export_send_map()].reshape(M, N)[grows]
        errs = []
        for summed, run in ((ring, run_c), (flat, None)):
            # ReduceScatter of every group range: rank k keeps chunk k
            parts = []
            for j in range(len(groups)):
                _, _, b, e = plans[k].group(j)
                c = (e - b) // n
                parts.append(summed[b + k * c:b + (k + 1) * c])
            recv = torch.cat(parts)
            out = torch.empty(M // n, N, dtype=torch.bfloat16, device="cuda")
            fo.post_stage(plans[k], recv, out)
            torch.cuda.synchronize()
            errs.append(_check_rows(out, sum(parts_o), parts_o, run, absprod, K, tol=run is None))
        print(f"TP=8 ReduceScatter, rank {k}: max rel err vs the bf16-epilogue model {errs[1]:.3e} "
              f"(fp32 reduction), {errs[0]:.3e} (bf16 ring, bound-checked)")


@pytest.mark.parametrize("routing", ["balanced", "router"])
@pytest.mark.parametrize("layout", ["slot", "auto"])
def test_c4_ep8_alltoall(routing, layout):
    """configs[3]: Mixtral-8x7B w2 (hidden 4096, ffn 14336), 8 experts one per
    rank, 4096 tokens top-2 -> ~1024 rows per expert, A2A back to the token
    owners."""
    n, N, K = 8, 4096, 14336
    if routing == "balanced":
        rds = [synthetic.balanced_moe_row_dst(128, n) for _ in range(n)]
    else:
        rds = [synthetic.pad_row_dst(rd, BM, e) for e, rd in enumerate(synthetic.moe_routing(4096, 8, 2, n, 40000))]
    P = 2
    BNe = 128  # 1024 rows x 4096 cols -> 128 tiles of 256x128 -> T = 2 at S = 64
    specs = []
    for e in range(n):
        M = len(rds[e])
        tiles = (M // BM) * (N // BNe)
        Se = min(S, tiles)
        T = -(-tiles // Se)
        specs.append(dict(coll="alltoall", m=M, n=N, k=K, tile_m=BM, tile_n=BNe, workers=Se,
                          group_waves=[1, T - 1] if T > 1 else [1], row_dst=rds[e], ar_layout=layout))
    if any(len(s["group_waves"]) != P for s in specs):
        pytest.skip("an expert got a single wave")
    plans = [fo.Plan(rank=e, world=n, peers=specs, **specs[e]) for e in range(n)]
    sends, As, Bts = [], [], []
    for e in range(n):
        M = specs[e]["m"]
        A, Bt = synthetic.float_inputs(M, N, K, seed=synthetic.rank_seed(40000, n, e), device="cuda")
        send = torch.empty(plans[e].info["send_elems"], dtype=torch.bfloat16, device="cuda")
        fo.gemm_stage(plans[e], A, Bt, send)
        sends.append(send)
        As.append(A)
        Bts.append(Bt)
    # the exchange emulated from the plans' own communication schedules
    # (fo_plan_export_calls): every receive on rank d is paired, in order, with
    # the matching send of its source (NCCL's send/recv pairing); the self part
    # is the local copy.  Layout-agnostic: the paper's [group][source] receive
    # buffer, or R41's output rows (every source's groups are bands here when
    # the routing pads the experts to whole waves of tile-rows)
    calls = [p.export_calls(0) for p in plans]
    sends_to = [{d: [c for c in calls[s_] if c["kind"] == "send" and c["peer"] == d] for d in range(n)}
                for s_ in range(n)]
    for d in (0, n - 1):
        recv = torch.full((plans[d].info["recv_elems"],), float("nan"), dtype=torch.bfloat16, device="cuda")
        cursor = [0] * n
        for c in calls[d]:
            if c["kind"] == "recv":
                m = sends_to[c["peer"]][d][cursor[c["peer"]]]
                cursor[c["peer"]] += 1
                assert m["count"] == c["count"] and m["group"] == c["group"]
                recv[c["dst_off"]:c["dst_off"] + c["count"]] = sends[c["peer"]][m["src_off"]:m["src_off"] + m["count"]]
            elif c["kind"] == "local_copy":
                recv[c["dst_off"]:c["dst_off"] + c["count"]] = sends[d][c["src_off"]:c["src_off"] + c["count"]]
        assert all(cursor[s_] == len(sends_to[s_][d]) for s_ in range(n))
        out = torch.empty(plans[d].info["out_rows"], N, dtype=torch.bfloat16, device="cuda")
        fo.post_stage(plans[d], recv, out)
        torch.cuda.synchronize()
        # output row -> (source, source row) in all-to-all-v order
        want = np.concatenate([_gemm_full(As[s][torch.from_numpy(np.flatnonzero(rds[s] == d)).cuda()], Bts[s])
                               for s in range(n)], axis=0)
        _check_rows(out, want)
    print(f"C4 EP=8 A2A ({routing}): layout {'rowband' if plans[0].info['ar_layout'] == 1 else 'slot'}")


def test_c2_bench_config_tp1_tail_split():
    """configs[1] at TP=1 with all 74 CTA pairs and the last partial wave split
    along K (the N=1 bench launch configuration)."""
    M, N, K = 4096, 4096, 14336
    A, Bt = synthetic.float_inputs(M, N, K, seed=synthetic.rank_seed(20000, 1, 0))
    plan = fo.Plan(coll="allreduce", m=M, n=N, k=K, tile_m=BM, tile_n=BN, workers=74, group_waves=[1, 2, 1],
                   swizzle=0)
    plan.set_option("tail_split", -1)
    ctx = fo.Context.create(0, 0, 1, fo.unique_id())
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    fo.run(ctx, plan, A.cuda(), Bt.cuda(), out)
    torch.cuda.synchronize()
    _check_rows(out, _gemm_full(A, Bt))          # every element, the split tail tiles included
    # 34 tail tiles in f = 2 slices: the distributed fold (default) adds the
    # same two fp32 terms per element as the owner-only fold (a + b == b + a)
    alt = fo.Plan(coll="allreduce", m=M, n=N, k=K, tile_m=BM, tile_n=BN, workers=74, group_waves=[1, 2, 1],
                  swizzle=0, options={"tail_split": -1, "dist_fold": 0})
    out2 = torch.empty_like(out)
    fo.run(ctx, alt, A.cuda(), Bt.cuda(), out2)
    torch.cuda.synchronize()
    assert torch.equal(out, out2)
    ctx.close()


def test_c2_bench_plan_exact():
    """The plan bench.py's tuner picks at N=1 (profiles/r02_final_bench_n1.json:
    256x256 CTA pairs, S=74, the auto order, one ROWBAND group — the AllReduce
    in place in C — and the split tail), through fo_run: every element vs the
    fp64 oracle product."""
    M, N, K = 4096, 4096, 14336
    A, Bt = synthetic.float_inputs(M, N, K, seed=synthetic.rank_seed(20000, 1, 0))
    plan = fo.Plan(coll="allreduce", m=M, n=N, k=K, tile_m=BM, tile_n=BN, workers=74, group_waves=[4],
                   swizzle=0, ar_layout="rowband", options={"tail_split": -1})
    assert plan.info["ar_layout"] == 1
    ctx = fo.Context.create(0, 0, 1, fo.unique_id())
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    fo.run(ctx, plan, A.cuda(), Bt.cuda(), out)
    torch.cuda.synchronize()
    _check_rows(out, _gemm_full(A, Bt))
    ctx.close()


def test_c0_two_ranks_four_groups():
    """configs[0] exactly as BASELINE.json states it: M=N=256, K=512 split over
    2 simulated ranks (K_loc=256), AllReduce, 64x64 tiles (tcgen05.mma M=64),
    4 signal groups: 16 tiles, S=4, T=4, groups (1,1,1,1) of 4 tiles each.
    Exact-integer regime, bit-exact send buffers, counters and outputs for both
    ranks."""
    from oracle import pipeline as opl
    from oracle import plan as op

    n, M, N, K = 2, 256, 256, 256
    groups = [1, 1, 1, 1]
    As, Bts = [], []
    for r in range(n):
        A, Bt = synthetic.exact_inputs(M, N, K, seed=synthetic.rank_seed(0, n, r), nnz_per_row=128)
        As.append(A)
        Bts.append(Bt)
    oplan = op.make_plan(M, N, 64, 64, 4, groups, swizzle=2)
    assert oplan.ntiles == 16 and oplan.T == 4
    ores = opl.run_allreduce(As, Bts, oplan)
    for r in range(n):
        plan = fo.Plan(coll="allreduce", m=M, n=N, k=K, tile_m=64, tile_n=64, workers=4, swizzle=2,
                       group_waves=groups, ar_layout="slot", rank=r, world=n)
        assert plan.info["tiles"] == 16 and plan.info["waves"] == 4
        send = torch.empty(M * N, dtype=torch.bfloat16, device="cuda")
        fo.gemm_stage(plan, As[r].cuda(), Bts[r].cuda(), send)
        torch.cuda.synchronize()
        assert np.array_equal(send.double().cpu().numpy(), ores["send"][r])
        assert plan.read_counters().tolist() == [4, 4, 4, 4]
        out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        fo.post_stage(plan, torch.from_numpy(ores["recv"][r]).to(torch.bfloat16).cuda(), out)
        torch.cuda.synchronize()
        assert np.array_equal(out.double().cpu().numpy(), opl.plain_allreduce(As, Bts)[r])
