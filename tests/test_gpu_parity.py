"""GPU parity: the sm_100a kernels through the C ABI vs the CPU oracle.

Exact-integer regime -> bit-exact buffers and outputs;
float regime -> max |g - o| / max(|o|, rms(o)) <= 1e-2 (north_star tolerance).
Multi-rank plans are exercised on ONE GPU through the stage entry points:
fo_gemm_stage (GEMM + pre-reorder epilogue + counters) is compared with the
oracle's send buffer, and fo_post_stage is fed the oracle's receive buffer (what
NCCL delivers) and compared with the oracle's output.  fo_run itself (streams,
stream waits, NCCL) is exercised at world = 1.
"""
import numpy as np
import pytest
import torch

import synthetic
from oracle import collectives as oc
from oracle import numerics as onum
from oracle import pipeline as opl
from oracle import plan as op
from oracle import post as opost
from oracle import reorder as orr

pytestmark = pytest.mark.gpu

fo = pytest.importorskip("paper_2504_19519_b200")
TOL = 1e-2


@pytest.fixture(scope="module", autouse=True)
def _dev():
    from paper_2504_19519_b200 import build

    build.build()
    fo.load()
    torch.cuda.set_device(0)
    yield


@pytest.fixture(scope="module")
def ctx1():
    c = fo.Context.create(0, 0, 1, fo.unique_id())
    yield c
    c.close()


def _dev_bf16(x):
    if isinstance(x, torch.Tensor):
        return x.to(torch.bfloat16).cuda().contiguous()
    return torch.from_numpy(np.ascontiguousarray(x)).to(torch.bfloat16).cuda()


def _host(t):
    return t.double().cpu().numpy()


def _rel_err(g, o):
    g, o = np.asarray(g, np.float64), np.asarray(o, np.float64)
    rms = np.sqrt(np.mean(o * o)) if o.size else 1.0
    return float(np.max(np.abs(g - o) / np.maximum(np.abs(o), rms))) if o.size else 0.0


def _counters_ok(plan, oplan):
    # each CTA signals once per tile it finishes; a 256-row tile is finished by a CTA pair
    mult = max(1, oplan.BM // 128)
    want = [mult * t for t in op.group_thresholds(oplan.partition, oplan.S, oplan.ntiles)]
    assert plan.read_counters().tolist() == want


# ------------------------------------------------------------------ plain GEMM
@pytest.mark.parametrize("BM", [64, 128, 256])
@pytest.mark.parametrize("BN", [64, 128, 256])
@pytest.mark.parametrize("shape", [(256, 256, 64), (768, 512, 320), (512, 768, 1024)])
def test_gemm_rowmajor_exact(BM, BN, shape):
    M, N, K = shape
    if N % BN or M % BM:
        pytest.skip("shape not divisible")
    A, Bt = synthetic.exact_inputs(M, N, K, seed=M + N + K, nnz_per_row=256)
    tiles = (M // BM) * (N // BN)
    S = max(1, min(tiles, 7))
    plan = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=BM, tile_n=BN, workers=S, swizzle=2)
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    fo.gemm_stage(plan, _dev_bf16(A), _dev_bf16(Bt), out)
    torch.cuda.synchronize()
    assert np.array_equal(_host(out), onum.gemm(A, Bt))
    _counters_ok(plan, op.make_plan(M, N, BM, BN, S, None, swizzle=2))


@pytest.mark.parametrize("BM", [64, 128, 256])
@pytest.mark.parametrize("BN", [128, 256])
def test_gemm_float_regime(BM, BN):
    M, N, K = 512, 512, 2048
    A, Bt = synthetic.float_inputs(M, N, K, seed=11)
    plan = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=BM, tile_n=BN, workers=3)
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    fo.gemm_stage(plan, _dev_bf16(A), _dev_bf16(Bt), out)
    torch.cuda.synchronize()
    assert _rel_err(_host(out), onum.gemm(A, Bt)) <= TOL


# ------------------------------------------------------------------ multi-rank stages on one GPU
def _rank_inputs(n, M, N, K, seed, exact=True):
    As, Bts = [], []
    for r in range(n):
        if exact:
            A, Bt = synthetic.exact_inputs(M, N, K, seed=synthetic.rank_seed(seed, n, r), nnz_per_row=max(1, 256 // n))
        else:
            A, Bt = synthetic.float_inputs(M, N, K, seed=synthetic.rank_seed(seed, n, r))
        As.append(A)
        Bts.append(Bt)
    return As, Bts


CASES = [
    # M, N, K, BN, S, BM, swizzle
    (512, 512, 128, 128, 3, 128, 2),
    (384, 768, 192, 256, 2, 128, 1),
    (640, 256, 64, 64, 4, 128, 3),
    (768, 512, 128, 256, 2, 256, 2),
    (512, 768, 192, 128, 3, 256, 1),
]


def _groups(tiles, S, seed):
    return synthetic.random_partition(op.num_waves(tiles, S), seed)


@pytest.mark.parametrize("n", [1, 2, 4, 8])
@pytest.mark.parametrize("case", range(len(CASES)))
@pytest.mark.parametrize("layout", ["slot", "auto"])
def test_allreduce_stages_exact(n, case, layout):
    M, N, K, BN, S, BM, swz = CASES[case]
    tiles = (M // BM) * (N // BN)
    groups = _groups(tiles, S, case + 10 * n)
    order = synthetic.random_order(tiles, case) if (case in (1, 4) and layout == "slot") else None
    As, Bts = _rank_inputs(n, M, N, K, 100 + case)
    oplan = op.make_plan(M, N, BM, BN, S, groups, order=order, swizzle=swz)
    plans = [fo.Plan(coll="allreduce", m=M, n=N, k=K, tile_m=BM, tile_n=BN, workers=S, tile_order=order, swizzle=swz,
                     group_waves=groups, ar_layout=layout, rank=r, world=n) for r in range(n)]
    lay = "rowband" if plans[0].info["ar_layout"] == 1 else "slot"
    ores = opl.run_allreduce(As, Bts, oplan, layout=lay)
    for r in range(n):
        send = torch.empty(M * N, dtype=torch.bfloat16, device="cuda")
        fo.gemm_stage(plans[r], _dev_bf16(As[r]), _dev_bf16(Bts[r]), send)
        torch.cuda.synchronize()
        assert np.array_equal(_host(send), ores["send"][r]), f"rank {r} send buffer"
        _counters_ok(plans[r], oplan)
        out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        fo.post_stage(plans[r], _dev_bf16(ores["recv"][r]), out)
        torch.cuda.synchronize()
        assert np.array_equal(_host(out), opl.plain_allreduce(As, Bts)[r])


@pytest.mark.parametrize("n", [1, 2, 4, 8])
@pytest.mark.parametrize("case", range(len(CASES)))
def test_reducescatter_stages_exact(n, case):
    M, N, K, BN, S, BM, swz = CASES[case]
    tiles = (M // BM) * (N // BN)
    groups = _groups(tiles, S, case + 20 * n)
    As, Bts = _rank_inputs(n, M, N, K, 200 + case)
    oplan = op.make_plan(M, N, BM, BN, S, groups, swizzle=swz)
    ores = opl.run_reducescatter(As, Bts, oplan)
    plain = opl.plain_reducescatter(As, Bts, BM)
    for r in range(n):
        plan = fo.Plan(coll="reducescatter", m=M, n=N, k=K, tile_m=BM, tile_n=BN, workers=S, swizzle=swz, group_waves=groups,
                       ar_layout="slot", rank=r, world=n)
        send = torch.empty(M * N, dtype=torch.bfloat16, device="cuda")
        fo.gemm_stage(plan, _dev_bf16(As[r]), _dev_bf16(Bts[r]), send)
        torch.cuda.synchronize()
        assert np.array_equal(_host(send), ores["send"][r]), f"rank {r} send buffer"
        _counters_ok(plan, oplan)
        out = torch.empty(M // n, N, dtype=torch.bfloat16, device="cuda")
        fo.post_stage(plan, _dev_bf16(ores["recv"][r]), out)
        torch.cuda.synchronize()
        assert np.array_equal(_host(out), plain[r])


@pytest.mark.parametrize("n", [1, 2, 4, 8])
@pytest.mark.parametrize("BM,BN,Mt,Nt,rows_per_wave,K", [(256, 256, 6, 3, 1, 256), (256, 128, 8, 2, 2, 128),
                                                         (128, 256, 5, 4, 1, 192), (64, 128, 6, 2, 2, 128)])
def test_reducescatter_rowband_stages_exact(n, BM, BN, Mt, Nt, rows_per_wave, K):
    """RS ROWBAND (R40): raster order, waves of whole tile-rows, random
    partitions -> ascending bands; every rank's send buffer (EPI_RS_BAND: TMA
    stores when h >= a warp's rows, st.global below), counters, and the
    received chunks (the output itself) bit-exact vs the oracle."""
    if BM % n:
        pytest.skip("tile_m not divisible by world")
    M, N = Mt * BM, Nt * BN
    S = rows_per_wave * Nt
    tiles = Mt * Nt
    groups = _groups(tiles, S, 7 * n + BM)
    As, Bts = _rank_inputs(n, M, N, K, 260 + n)
    oplan = op.make_plan(M, N, BM, BN, S, groups, swizzle=1)
    assert orr.rs_rowband_ok(oplan)
    ores = opl.run_reducescatter(As, Bts, oplan, layout="rowband")
    plain = opl.plain_reducescatter(As, Bts, BM)
    for r in range(n):
        plan = fo.Plan(coll="reducescatter", m=M, n=N, k=K, tile_m=BM, tile_n=BN, workers=S, swizzle=1,
                       group_waves=groups, rank=r, world=n)
        assert plan.info["ar_layout"] == 1
        for tma in (1, 0):
            plan.set_option("tma_store", tma)
            send = torch.empty(M * N, dtype=torch.bfloat16, device="cuda")
            fo.gemm_stage(plan, _dev_bf16(As[r]), _dev_bf16(Bts[r]), send)
            torch.cuda.synchronize()
            assert np.array_equal(_host(send), ores["send"][r]), f"rank {r} send buffer (tma_store={tma})"
            _counters_ok(plan, oplan)
        assert np.array_equal(ores["recv"][r].reshape(M // n, N), plain[r])
        out = torch.empty(M // n, N, dtype=torch.bfloat16, device="cuda")
        fo.post_stage(plan, _dev_bf16(ores["recv"][r]), out)   # identity map
        torch.cuda.synchronize()
        assert np.array_equal(_host(out), plain[r])


@pytest.mark.parametrize("BM", [64, 128, 256])
@pytest.mark.parametrize("n", [1, 2, 4, 8])
@pytest.mark.parametrize("layout", ["slot", "rowband"])
def test_alltoall_stages_exact(n, BM, layout):
    """Every rank's pools (the paper's subtoken order, or R41's complete rows),
    counters and post pass bit-exact vs the oracle."""
    rng = np.random.default_rng(n)
    N, K, BN, P = 512, 128, 128, 2
    Nt = N // BN
    specs, oplans, As, Bts, rds = [], [], [], [], []
    for s in range(n):
        Mt = int(rng.integers(2, 5))
        M = Mt * BM
        tiles = Mt * Nt
        S = int(rng.integers(1, tiles // P + 1))
        swz = 2
        if layout == "rowband":   # raster, waves of whole tile-rows
            S, swz = Nt * int(rng.integers(1, Mt // P + 1)), 1
        T = op.num_waves(tiles, S)
        part = [1] * (P - 1) + [T - (P - 1)]
        rd = synthetic.random_row_dst(M, n, 1000 + s)
        A, Bt = synthetic.exact_inputs(M, N, K, seed=300 + s, nnz_per_row=64)
        specs.append(dict(coll="alltoall", m=M, n=N, k=K, tile_m=BM, tile_n=BN, workers=S, swizzle=swz,
                          group_waves=part, row_dst=rd, ar_layout=layout))
        oplans.append(op.make_plan(M, N, BM, BN, S, part, swizzle=swz))
        As.append(A), Bts.append(Bt), rds.append(rd)
    ores = opl.run_alltoall(As, Bts, oplans, rds, layout=layout)
    plain = opl.plain_alltoall(As, Bts, rds)
    for me in range(n):
        plan = fo.Plan(rank=me, world=n, peers=specs, **specs[me])
        assert plan.info["ar_layout"] == (1 if layout == "rowband" else 0)
        send = torch.empty(plan.info["send_elems"], dtype=torch.bfloat16, device="cuda")
        fo.gemm_stage(plan, _dev_bf16(As[me]), _dev_bf16(Bts[me]), send)
        torch.cuda.synchronize()
        flat = np.concatenate([ores["send"][me].pools[d].reshape(-1) for d in range(n)])
        assert np.array_equal(_host(send), flat)
        _counters_ok(plan, oplans[me])
        if layout == "rowband":   # the receive layout is the output itself
            recv = ores["out"][me].reshape(-1)
        else:
            recv = np.concatenate([c.reshape(-1) for _, c in ores["recv"][me]]) if ores["recv"][me] else np.zeros(0)
        out = torch.empty(plan.info["out_rows"], N, dtype=torch.bfloat16, device="cuda")
        fo.post_stage(plan, _dev_bf16(recv), out)
        torch.cuda.synchronize()
        assert np.array_equal(_host(out), plain[me])


# ------------------------------------------------------------------ fused elementwise (float regime)
@pytest.mark.parametrize("post", ["add", "add_rmsnorm"])
def test_post_fused_ops(post):
    M, N, K, BN, S = 512, 1024, 256, 256, 3
    tiles = (M // 128) * (N // BN)
    groups = _groups(tiles, S, 7)
    A, Bt = synthetic.float_inputs(M, N, K, seed=3)
    res = synthetic.normal_bf16((M, N), 1.0, 99)
    gamma = synthetic.normal_bf16((N,), 1.0, 98)
    plan = fo.Plan(coll="allreduce", m=M, n=N, k=K, tile_n=BN, workers=S, swizzle=2, group_waves=groups,
                   ar_layout="slot", post=post, eps=1e-5)
    oplan = op.make_plan(M, N, 128, BN, S, groups, swizzle=2)
    ores = opl.run_allreduce([A], [Bt], oplan, model_bf16=True)
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    fo.post_stage(plan, _dev_bf16(ores["recv"][0]), out, _dev_bf16(res), _dev_bf16(gamma))
    torch.cuda.synchronize()
    x = ores["out"][0]
    want = opost.add(x, onum.to_f64(res)) if post == "add" else opost.add_rmsnorm(x, onum.to_f64(res), onum.to_f64(gamma), 1e-5)
    assert _rel_err(_host(out), want) <= TOL


# ------------------------------------------------------------------ full path with NCCL (world = 1)
@pytest.mark.parametrize("BM", [128, 256])
@pytest.mark.parametrize("coll", ["allreduce", "reducescatter", "alltoall", "nocomm"])
@pytest.mark.parametrize("post", ["none", "add_rmsnorm"])
def test_fo_run_world1(ctx1, coll, post, BM):
    M, N, K, BN, S = 1024, 512, 256, 128, 5
    tiles = (M // BM) * (N // BN)
    groups = _groups(tiles, S, 3)
    A, Bt = synthetic.exact_inputs(M, N, K, seed=5, nnz_per_row=200)
    kw = dict(coll=coll, m=M, n=N, k=K, tile_m=BM, tile_n=BN, workers=S, swizzle=2, group_waves=groups, post=post)
    if coll == "alltoall":
        kw["row_dst"] = np.zeros(M, np.int32)
        plan = fo.Plan(rank=0, world=1, peers=[kw], **kw)
    else:
        plan = fo.Plan(**kw)
    res = synthetic.normal_bf16((M, N), 1.0, 1)
    gamma = synthetic.normal_bf16((N,), 1.0, 2)
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    args = (_dev_bf16(res), _dev_bf16(gamma)) if post != "none" else (None, None)
    Ad, Bd = _dev_bf16(A), _dev_bf16(Bt)
    for _ in range(3):  # repeated runs: counters reset each time
        fo.run(ctx1, plan, Ad, Bd, out, *args)
    torch.cuda.synchronize()
    C = onum.gemm(A, Bt)
    if post == "none":
        assert np.array_equal(_host(out), C)
    else:
        want = opost.add_rmsnorm(C, onum.to_f64(res), onum.to_f64(gamma), 1e-5)
        assert _rel_err(_host(out), want) <= TOL
    out2 = torch.empty_like(out)
    if coll != "alltoall" or True:
        fo.run_sequential(ctx1, plan, Ad, Bd, out2, *args)
        torch.cuda.synchronize()
        if post == "none":
            assert np.array_equal(_host(out2), C)


@pytest.mark.parametrize("BM", [128, 256])
def test_tile_timestamps_follow_waves(BM):
    """Per-tile %globaltimer: every tile of wave w+1 signals after the first
    tile of wave w (wave pattern; X1 analogue)."""
    M, N, K, BN = 2048, 2048, 4096, 256
    S = 16
    A, Bt = synthetic.float_inputs(M, N, K, seed=1)
    plan = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=BM, tile_n=BN, workers=S)
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    ts = torch.zeros(plan.info["tiles"], dtype=torch.int64, device="cuda")
    fo.gemm_stage_timed(plan, _dev_bf16(A), _dev_bf16(Bt), out, ts)
    torch.cuda.synchronize()
    t = ts.cpu().numpy().astype(np.int64)
    waves = t.reshape(-1, S)
    assert (waves[1:].min(axis=1) > waves[:-1].min(axis=1)).all()


# ------------------------------------------------------------------ tail split (split-K of the last wave)
@pytest.mark.parametrize("BM,BN,M,N,K,S,split", [
    (256, 256, 1024, 1024, 512, 12, -1),    # 16 tiles, T=2, R=4 -> f=3
    (256, 128, 768, 1024, 256, 10, 2),      # 24 tiles, T=3, R=4 -> f=2
    (128, 256, 512, 1024, 1024, 14, 4),     # 16 tiles, T=2, R=2 -> f=4
    (256, 256, 2048, 2048, 2048, 28, -1),   # 64 tiles, T=3, R=8 -> f=3
    (256, 256, 1024, 1024, 512, 12, -2),    # stream-K: 4 tail tiles x 8 k-blocks over 12 workers
    (256, 256, 1024, 2048, 1024, 10, -2),   # stream-K, 1 wave: 32 tiles... T=4, R=2 over 10 workers
    (256, 128, 768, 1024, 576, 20, -2),     # stream-K: 24 tiles, T=2, R=4, 9 k-blocks (uneven ranges)
    (128, 256, 512, 1024, 1024, 14, -2),    # stream-K with single-CTA tiles
    (256, 64, 512, 512, 256, 12, 2),        # 16 tiles, R=4, f=2, one 64-col chunk: slice 1 owns none
    (256, 128, 512, 1024, 512, 14, 3),      # 16 tiles, R=2, f=3, two chunks: slice 2 owns none
    (256, 256, 1024, 4096, 2048, 74, -3),   # DP + suffix (R43): one wave of 64 tiles on 74 pairs, x = 28 of 32
    (128, 256, 1024, 2048, 1024, 100, -3),  # DP + suffix, single-CTA tiles: 64 tiles, 36 helpers, 2 each
    (256, 128, 768, 1024, 576, 14, -3),     # DP + suffix: 24 tiles, T=2, R=10 > S/2, 9 k-blocks (uneven)
])
@pytest.mark.parametrize("dist_fold", [1, 0])
def test_tail_split_exact(ctx1, BM, BN, M, N, K, S, split, dist_fold):
    """Split tail (R34), both folds of an f-slice split (FO_OPT_DIST_FOLD: the
    slices reduce the tile together / the k-block-0 slice folds everything)."""
    if split in (-2, -3) and dist_fold == 0:
        pytest.skip("stream-K / DP + suffix always fold in the owner")
    A, Bt = synthetic.exact_inputs(M, N, K, seed=77, nnz_per_row=256)
    C = onum.gemm(A, Bt)
    for coll in ("nocomm", "allreduce"):
        plan = fo.Plan(coll=coll, m=M, n=N, k=K, tile_m=BM, tile_n=BN, workers=S, swizzle=2, ar_layout="slot")
        plan.set_option("tail_split", split)
        plan.set_option("dist_fold", dist_fold)
        # one group: keep it counter-triggered so the counting table is exercised (R32)
        plan.set_option("last_group_in_order", 0)
        out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        Ad, Bd = _dev_bf16(A), _dev_bf16(Bt)
        for _ in range(3):  # flags must reset between runs
            out.zero_()
            if coll == "nocomm":
                fo.gemm_stage(plan, Ad, Bd, out)
            else:
                fo.run(ctx1, plan, Ad, Bd, out)
            torch.cuda.synchronize()
            assert np.array_equal(_host(out), C)
        _counters_ok(plan, op.make_plan(M, N, BM, BN, S, None, swizzle=2))
        for _ in range(2):
            out.zero_()
            fo.run_sequential(ctx1, plan, Ad, Bd, out)
            torch.cuda.synchronize()
            assert np.array_equal(_host(out), C)


@pytest.mark.parametrize("post", ["none", "add_rmsnorm"])
def test_tail_split_rowband_single_group(ctx1, post):
    """The tuner's bench plan shape (R34): ROWBAND, one group, auto tail split,
    through fo_run — the exact-integer output equals the plain GEMM, and the
    fused add + RMSNorm equals the split-free plan's bit for bit."""
    M, N, K, S = 1024, 1024, 512, 7           # 16 tiles of 256x256, T = 3, R = 2 -> f = 3
    A, Bt = synthetic.exact_inputs(M, N, K, seed=78, nnz_per_row=256)
    C = onum.gemm(A, Bt)
    kw = dict(coll="allreduce", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, swizzle=0,
              group_waves=[3], ar_layout="rowband", post=post)
    on = fo.Plan(options={"tail_split": -1}, **kw)
    off = fo.Plan(**kw)
    assert on.info["ar_layout"] == 1
    Ad, Bd = _dev_bf16(A), _dev_bf16(Bt)
    res = synthetic.normal_bf16((M, N), 1.0, 79, device="cuda") if post != "none" else None
    gam = synthetic.normal_bf16((N,), 1.0, 80, device="cuda") if post != "none" else None
    o1 = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    o2 = torch.empty_like(o1)
    for _ in range(3):
        o1.fill_(float("nan"))
        fo.run(ctx1, on, Ad, Bd, o1, res, gam)
        fo.run(ctx1, off, Ad, Bd, o2, res, gam)
        torch.cuda.synchronize()
        assert torch.equal(o1, o2)
    if post == "none":
        assert np.array_equal(_host(o1), C)


def test_tail_split_rejects_oversubscription():
    plan = fo.Plan(coll="nocomm", m=1024, n=1024, k=128, tile_m=256, tile_n=256, workers=4)  # T=4, R=4
    plan.set_option("tail_split", 2)   # 4 tail tiles x 2 > S = 4
    A = torch.zeros(1024, 128, dtype=torch.bfloat16, device="cuda")
    out = torch.empty(1024, 1024, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(fo.FOError, match="INVALID_ARG"):
        fo.gemm_stage(plan, A, A[:1024], out)


# ------------------------------------------------------------------ RS follow-on: AllGather + row exchange (f2)
@pytest.mark.parametrize("n", [1, 2, 4, 8])
@pytest.mark.parametrize("post", ["none", "add_rmsnorm"])
def test_rs_allgather_rowexchange(n, post):
    """RS -> (elementwise) -> AllGather -> row exchange == AllReduce
    (PAPER.md:390); the rank-major gather is emulated, the row exchange (fused
    with the elementwise op) runs on the GPU."""
    M, N, K, BN, S, BM = 1024, 512, 128, 128, 5, 256
    tiles = (M // BM) * (N // BN)
    groups = _groups(tiles, S, 31 + n)
    As, Bts = _rank_inputs(n, M, N, K, 500)
    oplan = op.make_plan(M, N, BM, BN, S, groups, swizzle=2)
    rs = opl.run_reducescatter(As, Bts, oplan)
    gathered = np.concatenate(rs["out"], axis=0)          # rank-major AllGather
    plan = fo.Plan(coll="reducescatter", m=M, n=N, k=K, tile_m=BM, tile_n=BN, workers=S, swizzle=2,
                   group_waves=groups, rank=0, world=n, post=post)
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    res = synthetic.normal_bf16((M, N), 1.0, 8)
    gam = synthetic.normal_bf16((N,), 1.0, 9)
    extra = (_dev_bf16(res), _dev_bf16(gam)) if post != "none" else (None, None)
    fo.rowexchange_stage(plan, _dev_bf16(gathered), out, *extra)
    torch.cuda.synchronize()
    C = opl.plain_allreduce(As, Bts)[0]
    assert np.array_equal(opl.row_exchange(gathered, BM, n), C)
    if post == "none":
        assert np.array_equal(_host(out), C)
    else:
        want = opost.add_rmsnorm(C, onum.to_f64(res), onum.to_f64(gam), 1e-5)
        assert _rel_err(_host(out), want) <= TOL


def test_run_allgather_world1(ctx1):
    M, N, K = 512, 512, 128
    A, Bt = synthetic.exact_inputs(M, N, K, seed=3, nnz_per_row=100)
    plan = fo.Plan(coll="reducescatter", m=M, n=N, k=K, tile_m=256, tile_n=128, workers=3, swizzle=2)
    local = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    fo.run(ctx1, plan, _dev_bf16(A), _dev_bf16(Bt), local)
    full = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    for rx in (True, False):
        fo.run_allgather(ctx1, plan, local, full, row_exchange=rx)
        torch.cuda.synchronize()
        assert np.array_equal(_host(full), onum.gemm(A, Bt))


# ------------------------------------------------------------------ tag runs
def _tag_inputs(M, N, code, on_rows):
    """K=64 GEMM with one nonzero k-column: C[r, c] = code[r] (on_rows) or code[c]."""
    A = torch.zeros(M, 64)
    Bt = torch.zeros(N, 64)
    if on_rows:
        A[:, 0] = torch.as_tensor(code, dtype=torch.float32)
        Bt[:, 0] = 1.0
    else:
        A[:, 0] = 1.0
        Bt[:, 0] = torch.as_tensor(code, dtype=torch.float32)
    return A.to(torch.bfloat16), Bt.to(torch.bfloat16)


@pytest.mark.parametrize("coll,n", [("allreduce", 1), ("reducescatter", 4), ("alltoall", 3)])
def test_tag_runs_decode_every_element(coll, n):
    """Four K=64 GEMMs whose outputs are (row mod 256, row div 256, col mod 256,
    col div 256) - all integers <= 255, exact in bf16 - decode the source
    coordinate of every send-buffer element through the real epilogue; it must
    equal the plan's (oracle-verified) send map."""
    M, N, BM, BN, S = 1024, 768, 256, 128, 5
    tiles = (M // BM) * (N // BN)
    groups = _groups(tiles, S, 3)
    kw = dict(coll=coll, m=M, n=N, k=64, tile_m=BM, tile_n=BN, workers=S, swizzle=2, group_waves=groups,
              ar_layout="slot")
    if coll == "alltoall":
        kw["row_dst"] = synthetic.random_row_dst(M, n, 5)
        plan = fo.Plan(rank=0, world=n, peers=[kw] * n, **kw)
    else:
        plan = fo.Plan(rank=0, world=n, **kw)
    send_elems = plan.info["send_elems"]
    rows = np.arange(M)
    cols = np.arange(N)
    codes = []
    for vec, on_rows in ((rows % 256, True), (rows // 256, True), (cols % 256, False), (cols // 256, False)):
        A, Bt = _tag_inputs(M, N, vec, on_rows)
        send = torch.empty(send_elems, dtype=torch.bfloat16, device="cuda")
        fo.gemm_stage(plan, A.cuda(), Bt.cuda(), send)
        torch.cuda.synchronize()
        codes.append(send.float().cpu().numpy().astype(np.int64))
    r = codes[0] + 256 * codes[1]
    c = codes[2] + 256 * codes[3]
    decoded = r * N + c                          # flat source index of every send element
    want = np.empty(send_elems, np.int64)
    want[plan.export_send_map()] = np.arange(M * N)
    assert np.array_equal(decoded, want)


# ------------------------------------------------------------------ MN-major operands (weight-gradient GEMMs, NEXT f4)
@pytest.mark.parametrize("mj", [1, 2, 3])
@pytest.mark.parametrize("BM,BN", [(128, 128), (128, 256), (256, 128), (256, 256)])
def test_gemm_mn_major_exact(mj, BM, BN):
    M, N, K = 768, 768, 320
    if M % BM or N % BN:
        pytest.skip("shape")
    A, Bt = synthetic.exact_inputs(M, N, K, seed=40 + mj, nnz_per_row=256)
    a_st = A.t().contiguous() if mj & 1 else A       # [K, M] when M-major
    b_st = Bt.t().contiguous() if mj & 2 else Bt     # [K, N] when N-major
    plan = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=BM, tile_n=BN, workers=5, swizzle=2,
                   a_mn_major=mj & 1, b_mn_major=(mj >> 1) & 1)
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    fo.gemm_stage(plan, _dev_bf16(a_st), _dev_bf16(b_st), out)
    torch.cuda.synchronize()
    assert np.array_equal(_host(out), onum.gemm(A, Bt))


@pytest.mark.parametrize("coll", ["allreduce", "reducescatter"])
@pytest.mark.parametrize("n", [2, 4])
def test_weight_gradient_dp_fsdp(coll, n):
    """NEXT f4: data-parallel gradient AllReduce / FSDP
    ReduceScatter after the weight-gradient GEMM dW_r = dY_r^T X_r, with dY_r
    [tokens, out] and X_r [tokens, in] used in place (M- / N-major operands).
    Every rank's GEMM + pre-reorder runs on the GPU; the collective is emulated;
    the result is compared with sum_r dY_r^T X_r (exact-integer regime)."""
    T_tok, OUT, IN, BM, BN, S = 512, 512, 768, 256, 128, 4
    tiles = (OUT // BM) * (IN // BN)
    groups = _groups(tiles, S, 9)
    dYs, Xs = [], []
    for r in range(n):
        # dY_r^T plays A ([out, tokens] logical), X_r^T plays Bt ([in, tokens] logical)
        A_log, Bt_log = synthetic.exact_inputs(OUT, IN, T_tok, seed=600 + r, nnz_per_row=max(1, 256 // n))
        dYs.append(A_log.t().contiguous())    # dY_r stored [tokens, out]
        Xs.append(Bt_log.t().contiguous())    # X_r stored [tokens, in]
    oplan = op.make_plan(OUT, IN, BM, BN, S, groups, swizzle=2)
    logical_A = [d.t() for d in dYs]
    logical_Bt = [x.t() for x in Xs]
    if coll == "allreduce":
        ores = opl.run_allreduce(logical_A, logical_Bt, oplan)
        plain = opl.plain_allreduce(logical_A, logical_Bt)
    else:
        ores = opl.run_reducescatter(logical_A, logical_Bt, oplan)
        plain = opl.plain_reducescatter(logical_A, logical_Bt, BM)
    for r in range(n):
        plan = fo.Plan(coll=coll, m=OUT, n=IN, k=T_tok, tile_m=BM, tile_n=BN, workers=S, swizzle=2,
                       group_waves=groups, ar_layout="slot", rank=r, world=n, a_mn_major=1, b_mn_major=1)
        send = torch.empty(plan.info["send_elems"], dtype=torch.bfloat16, device="cuda")
        fo.gemm_stage(plan, _dev_bf16(dYs[r]), _dev_bf16(Xs[r]), send)
        torch.cuda.synchronize()
        assert np.array_equal(_host(send), ores["send"][r])
        out = torch.empty(plan.info["out_rows"], IN, dtype=torch.bfloat16, device="cuda")
        fo.post_stage(plan, _dev_bf16(ores["recv"][r]), out)
        torch.cuda.synchronize()
        assert np.array_equal(_host(out), plain[r])


# ------------------------------------------------------------------ edge cases
@pytest.mark.parametrize("BM,BN,M,N,K,S", [
    (128, 64, 128, 64, 64, 1),      # one tile, one k-block, one worker
    (256, 256, 256, 256, 64, 1),    # one pair tile
    (128, 128, 512, 256, 64, 16),   # more workers than tiles (idle workers)
    (256, 128, 512, 512, 128, 1),   # a single worker runs every position (T = tiles)
])
def test_gemm_edge_shapes(ctx1, BM, BN, M, N, K, S):
    A, Bt = synthetic.exact_inputs(M, N, K, seed=M + K, nnz_per_row=64)
    plan = fo.Plan(coll="allreduce", m=M, n=N, k=K, tile_m=BM, tile_n=BN, workers=S, ar_layout="slot")
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    fo.run(ctx1, plan, _dev_bf16(A), _dev_bf16(Bt), out)
    torch.cuda.synchronize()
    assert np.array_equal(_host(out), onum.gemm(A, Bt))


def test_rs_one_row_subtiles():
    """RS with world == tile_m: subtiles of a single row (h = 1)."""
    n, M, N, K, BM, BN, S = 128, 256, 128, 64, 128, 128, 1
    As, Bts = _rank_inputs(1, M, N, K, 77)
    oplan = op.make_plan(M, N, BM, BN, S, None)
    Y = onum.gemm(As[0], Bts[0])
    for lay in ("slot", "rowband"):   # S = 1, one tile-row per wave: both layouts are legal
        plan = fo.Plan(coll="reducescatter", m=M, n=N, k=K, tile_m=BM, tile_n=BN, workers=S, rank=5, world=n,
                       ar_layout=lay)
        send = torch.empty(M * N, dtype=torch.bfloat16, device="cuda")
        fo.gemm_stage(plan, _dev_bf16(As[0]), _dev_bf16(Bts[0]), send)
        torch.cuda.synchronize()
        assert np.array_equal(_host(send), orr.rs_pre(Y, oplan, n, lay)), lay


def test_alltoall_rank_receiving_nothing():
    """Rank 1 gets no rows from anyone; rank 0 gets everything (zero counts are legal)."""
    n, N, K, BM, BN = 2, 256, 64, 128, 128
    specs, As, Bts, oplans, rds = [], [], [], [], []
    for s in range(n):
        M = 256 * (s + 1)
        rd = np.zeros(M, np.int32)
        A, Bt = synthetic.exact_inputs(M, N, K, seed=90 + s, nnz_per_row=64)
        specs.append(dict(coll="alltoall", m=M, n=N, k=K, tile_m=BM, tile_n=BN, workers=2, group_waves=[1, (M // BM * 2 + 1) // 2 - 1], row_dst=rd,
                          ar_layout="slot"))
        oplans.append(op.make_plan(M, N, BM, BN, 2, specs[-1]["group_waves"]))
        As.append(A), Bts.append(Bt), rds.append(rd)
    ores = opl.run_alltoall(As, Bts, oplans, rds)
    for me in range(n):
        plan = fo.Plan(rank=me, world=n, peers=specs, **specs[me])
        assert plan.info["out_rows"] == (sum(s["m"] for s in specs) if me == 0 else 0)
        recv = np.concatenate([c.reshape(-1) for _, c in ores["recv"][me]])
        if me == 1:
            assert recv.size == 0 and plan.info["recv_elems"] == 0
            continue
        out = torch.empty(plan.info["out_rows"], N, dtype=torch.bfloat16, device="cuda")
        fo.post_stage(plan, _dev_bf16(recv), out)
        torch.cuda.synchronize()
        assert np.array_equal(_host(out), opl.plain_alltoall(As, Bts, rds)[me])


@pytest.mark.parametrize("n", [1, 4])
def test_rowband_with_swizzled_panels(ctx1, n):
    """ROWBAND layout with a non-raster order: panels of 2 tile-rows visited
    column-major, one panel per wave, so every group is a band of whole
    tile-rows and the epilogue writes row-major C in place (H11a)."""
    M, N, K, BM, BN, S = 1024, 512, 128, 128, 128, 8    # Mt=8, Nt=4, panel = 2 rows = 8 tiles = S
    groups = [1, 2, 1]
    plan = fo.Plan(coll="allreduce", m=M, n=N, k=K, tile_m=BM, tile_n=BN, workers=S, swizzle=2,
                   group_waves=groups, ar_layout="rowband", rank=0, world=n)
    assert plan.info["ar_layout"] == 1
    assert plan.export_order()[:4].tolist() == [0, 4, 1, 5]
    As, Bts = _rank_inputs(n, M, N, K, 123)
    oplan = op.make_plan(M, N, BM, BN, S, groups, swizzle=2)
    ores = opl.run_allreduce(As, Bts, oplan, layout="rowband")
    send = torch.empty(M * N, dtype=torch.bfloat16, device="cuda")
    fo.gemm_stage(plan, _dev_bf16(As[0]), _dev_bf16(Bts[0]), send)
    torch.cuda.synchronize()
    assert np.array_equal(_host(send), ores["send"][0])
    for j in range(len(groups)):
        assert plan.group(j)[2:] == orr.group_elem_ranges(oplan, "rowband")[j]
    if n == 1:
        out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        fo.run(ctx1, plan, _dev_bf16(As[0]), _dev_bf16(Bts[0]), out)
        torch.cuda.synchronize()
        assert np.array_equal(_host(out), opl.plain_allreduce(As, Bts)[0])


# ------------------------------------------------------------------ MoE top-k combine (R31, NEXT f3)
def _combine_close(g, o):
    # fp32 accumulation of k bf16 rows, one bf16 rounding: <= 2^-8 relative
    g, o = np.asarray(g, np.float64), np.asarray(o, np.float64)
    return bool(np.all(np.abs(g - o) <= 2.0 ** -8 * np.abs(o) + 1e-6))


@pytest.mark.parametrize("n,k,skew", [(2, 2, 0.0), (4, 2, 1.0), (8, 2, 0.0), (8, 2, 2.0), (4, 1, 0.0)])
def test_moe_combine_stages(n, k, skew):
    """Expert GEMM stage per rank (A2A plan), the oracle's exchange, then the
    fused combine on each token rank vs the oracle's combine of its A2A output."""
    BM, BN, N, K = 128, 128, 512, 256
    tokens = 192 * n
    rt = synthetic.moe_topk(tokens, n, k, seed=40000 + n, skew=skew, pad=BM)
    X = synthetic.exact_int_A(tokens, K, 77, 64)
    specs, oplans, As, Bts = [], [], [], []
    for e in range(n):
        rows = torch.from_numpy(rt["row_token"][e])
        A = torch.where((rows >= 0)[:, None], X[rows.clamp(min=0)], torch.zeros((), dtype=X.dtype))
        Bt = synthetic.exact_int_B(N, K, 500 + e)
        M = A.shape[0]
        tiles = (M // BM) * (N // BN)
        S = max(1, tiles // 3)
        T = op.num_waves(tiles, S)
        part = [1, T - 1] if T > 1 else None
        if part is None:
            S = max(1, tiles // 2)
            T = op.num_waves(tiles, S)
            part = [1, T - 1]
        specs.append(dict(coll="alltoall", m=M, n=N, k=K, tile_m=BM, tile_n=BN, workers=S, swizzle=1,
                          group_waves=part, row_dst=rt["row_dst"][e], ar_layout="slot"))
        oplans.append(op.make_plan(M, N, BM, BN, S, part, swizzle=1))
        As.append(A), Bts.append(Bt)
    ores = opl.run_alltoall(As, Bts, oplans, rt["row_dst"])
    per = tokens // n
    for r in range(n):
        plan = fo.Plan(rank=r, world=n, peers=specs, **specs[r])
        recv = np.concatenate([c.reshape(-1) for _, c in ores["recv"][r]]) if ores["recv"][r] else np.zeros(0)
        idx = torch.from_numpy(rt["combine_idx"][r]).cuda()
        w = torch.from_numpy(np.ascontiguousarray(rt["weight"][r * per:(r + 1) * per])).cuda()
        res = synthetic.normal_bf16((per, N), 1.0, 900 + r)
        out = torch.empty(per, N, dtype=torch.bfloat16, device="cuda")
        fo.combine_stage(plan, _dev_bf16(recv), out, idx, w, _dev_bf16(res))
        torch.cuda.synchronize()
        want = opost.topk_combine(ores["out"][r], rt["combine_idx"][r], rt["weight"][r * per:(r + 1) * per],
                                  residual=onum.to_f64(res))
        assert _combine_close(_host(out), want), r
        # dropped slots: every second token loses its last slot
        idx2 = idx.clone()
        idx2[::2, -1] = -1
        fo.combine_stage(plan, _dev_bf16(recv), out, idx2, w)
        torch.cuda.synchronize()
        want2 = opost.topk_combine(ores["out"][r], idx2.cpu().numpy(), rt["weight"][r * per:(r + 1) * per])
        assert _combine_close(_host(out), want2), r


@pytest.mark.parametrize("BN,N,k", [(64, 1600, 2), (128, 1536, 3), (64, 1536, 1), (256, 4096, 2), (64, 512, 2), (128, 640, 8), (128, 640, 36)])
def test_moe_combine_table_broadcast(BN, N, k):
    """The combine's async-copy kernel (R31b) loads the unit's topk x
    tiles-per-unit table entries once and broadcasts them: exercise the most
    entries (BN=64: 16 tile columns per 1024-column unit, k=4 -> 64), a ragged
    last unit (N % 1024), dropped slots, a residual, and k > 4 (the register
    kernel) — each vs the oracle's combine of the A2A output at world 1."""
    BM, K = 64, 64
    tokens = 96
    M = tokens * k
    M += (-M) % BM
    rd = np.zeros(M, np.int32)
    A = synthetic.exact_int_A(M, K, 31, 16)
    Bt = synthetic.exact_int_B(N, K, 32)
    tiles = (M // BM) * (N // BN)
    S = max(1, tiles // 3)
    T = op.num_waves(tiles, S)
    spec = dict(coll="alltoall", m=M, n=N, k=K, tile_m=BM, tile_n=BN, workers=S, swizzle=1,
                group_waves=[1, T - 1], row_dst=rd, ar_layout="slot")
    plan = fo.Plan(peers=[spec], **spec)
    ores = opl.run_alltoall([A], [Bt], [op.make_plan(M, N, BM, BN, S, [1, T - 1], swizzle=1)], [rd])
    recv = np.concatenate([c.reshape(-1) for _, c in ores["recv"][0]])
    rng = np.random.default_rng(BN + k)
    idx = rng.permutation(M)[:tokens * k].astype(np.int32).reshape(tokens, k)
    idx[::3, -1] = -1                      # dropped slots
    idx[1::5, 0] = M + 7                   # out of range -> dropped
    w = rng.random((tokens, k)).astype(np.float32)
    res = synthetic.normal_bf16((tokens, N), 1.0, 11)
    out = torch.empty(tokens, N, dtype=torch.bfloat16, device="cuda")
    for r in (None, res):
        args = (_dev_bf16(r),) if r is not None else ()
        fo.combine_stage(plan, _dev_bf16(recv), out, torch.from_numpy(idx).cuda(), torch.from_numpy(w).cuda(), *args)
        torch.cuda.synchronize()
        want = opost.topk_combine(ores["out"][0], idx, w, residual=None if r is None else onum.to_f64(r))
        assert _combine_close(_host(out), want), (BN, N, k, r is None)


@pytest.mark.parametrize("layout", ["slot", "rowband"])
def test_moe_combine_full_path_world1(ctx1, layout):
    """fo_run_combine at one rank (one expert, top-1): GEMM + A2A (local) +
    fused combine through the streams, vs the oracle; ROWBAND (R41): the rows
    land in the library's receive buffer in the output layout and the combine
    reads them through the identity map."""
    BM, BN, N, K = 256, 256, 1024, 512
    tokens = 1024
    rt = synthetic.moe_topk(tokens, 1, 1, seed=5, pad=BM)
    A, Bt = synthetic.float_inputs(tokens, N, K, seed=8)
    M = A.shape[0]
    tiles = (M // BM) * (N // BN)
    spec = dict(coll="alltoall", m=M, n=N, k=K, tile_m=BM, tile_n=BN, workers=tiles // 4,
                group_waves=[1, 1, 2], row_dst=rt["row_dst"][0], ar_layout=layout)
    if layout == "rowband":   # raster, one tile-row per wave
        spec.update(workers=N // BN, swizzle=1, group_waves=[1, 1, M // BM - 2])
    plan = fo.Plan(peers=[spec], **spec)
    assert plan.info["ar_layout"] == (1 if layout == "rowband" else 0)
    # permute the slots: token t reads row perm[t] (a gather through the map)
    perm = np.random.default_rng(3).permutation(tokens).astype(np.int32)[:, None]
    w = torch.full((tokens, 1), 0.5, dtype=torch.float32, device="cuda")
    out = torch.empty(tokens, N, dtype=torch.bfloat16, device="cuda")
    fo.run_combine(ctx1, plan, _dev_bf16(A), _dev_bf16(Bt), out, torch.from_numpy(perm).cuda(), w)
    torch.cuda.synchronize()
    Y = opl.run_alltoall([A], [Bt], [op.make_plan(M, N, BM, BN, spec["workers"], spec["group_waves"],
                                                  swizzle=spec.get("swizzle", 1))], rt["row_dst"],
                         model_bf16=True, layout=layout)["out"][0]
    want = opost.topk_combine(Y, perm, np.full((tokens, 1), 0.5))
    # float regime: the GEMM's own bf16 rounding (fp32 accumulation) may differ
    # from the model's by an ulp -> the north_star tolerance
    assert _rel_err(_host(out), want) <= TOL
    with pytest.raises(fo.FOError):
        bad = fo.Plan(coll="allreduce", m=M, n=N, k=K, tile_m=BM, tile_n=BN, workers=4)
        fo.run_combine(ctx1, bad, _dev_bf16(A), _dev_bf16(Bt), out, torch.from_numpy(perm).cuda(), w)


@pytest.mark.parametrize("coll,layout,groups,N", [("allreduce", "rowband", [1, 2, 1], 1024),
                                                  ("allreduce", "slot", [2, 2], 1024),
                                                  ("reducescatter", "auto", [1, 3], 1024),
                                                  # 4096 columns: resident row-looping grid with next-row prefetch
                                                  ("allreduce", "rowband", [4, 8, 4], 4096),
                                                  ("allreduce", "slot", [8, 8], 4096)])
def test_add_rmsnorm_residual_in_place(ctx1, coll, layout, groups, N):
    """FO_POST_ADD_RMSNORM_RESIDUAL (the residual stream of a pre-norm block,
    NEXT f4): out equals the ADD_RMSNORM output bit for bit, and the residual
    buffer is overwritten with bf16(x + residual) — bit-exact vs the oracle in
    the exact-integer regime (per row band for ROWBAND, once at the end else)."""
    M, K, S = 2048, 512, 8
    A, Bt = synthetic.exact_inputs(M, N, K, seed=91, nnz_per_row=200)
    rows = M
    kw = dict(coll=coll, m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, swizzle=1, group_waves=groups,
              ar_layout=layout)
    p_res = fo.Plan(post="add_rmsnorm_res", **kw)
    p_norm = fo.Plan(post="add_rmsnorm", **kw)
    rng = np.random.default_rng(92)
    res0 = torch.from_numpy(rng.integers(-8, 9, size=(rows, N)).astype(np.float32)).to(torch.bfloat16)
    gam = synthetic.normal_bf16((N,), 1.0, 93, device="cuda")
    Ad, Bd = _dev_bf16(A), _dev_bf16(Bt)
    o_norm = torch.empty(rows, N, dtype=torch.bfloat16, device="cuda")
    fo.run(ctx1, p_norm, Ad, Bd, o_norm, res0.cuda(), gam)
    res = res0.cuda()
    o_res = torch.empty_like(o_norm)
    fo.run(ctx1, p_res, Ad, Bd, o_res, res, gam)
    torch.cuda.synchronize()
    assert torch.equal(o_res, o_norm)
    C = onum.gemm(A, Bt)                                  # exact integers, bf16-representable
    want_out, want_res = opost.add_rmsnorm_residual(C, _host(res0.cuda()), _host(gam), 1e-5)
    assert np.array_equal(_host(res), want_res)
    assert _rel_err(_host(o_res), want_out) <= TOL


@pytest.mark.parametrize("S,swz,split", [(8, 0, 0), (3, 2, 0), (7, 0, -1), (10, 0, -2)])
def test_gemm_swiglu_epilogue(S, swz, split):
    """FO_OPT_GEMM_SWIGLU: the fused MLP activation in the GEMM epilogue
    equals silu(gate) * up of the fp64 product within one bf16 rounding
    (interleaved weight rows: blocks of 128 gate / 128 up)."""
    M, N2, K = 1024, 512, 768                     # output [M, 512] from a [M, 1024] GEMM
    A, Wg = synthetic.float_inputs(M, N2, K, seed=61)
    Wu = synthetic.float_inputs(M, N2, K, seed=62)[1]
    Wi = torch.empty(2 * N2, K, dtype=torch.bfloat16)
    for j in range(N2 // 128):
        Wi[256 * j:256 * j + 128] = Wg[128 * j:128 * (j + 1)]
        Wi[256 * j + 128:256 * (j + 1)] = Wu[128 * j:128 * (j + 1)]
    plan = fo.Plan(coll="nocomm", m=M, n=2 * N2, k=K, tile_m=256, tile_n=256, workers=S, swizzle=swz)
    plan.set_option("gemm_swiglu", 1)
    plan.set_option("tail_split", split)      # the owner folds the parts' partials in before the activation
    out = torch.full((M, N2), float("nan"), dtype=torch.bfloat16, device="cuda")
    fo.gemm_stage(plan, _dev_bf16(A), _dev_bf16(Wi), out)
    torch.cuda.synchronize()
    g = onum.gemm(A, Wg)
    u = onum.gemm(A, Wu)
    want = g / (1.0 + np.exp(-g)) * u
    assert _rel_err(_host(out), want) <= TOL
    with pytest.raises(fo.FOError, match="UNSUPPORTED"):
        fo.Plan(coll="allreduce", m=M, n=2 * N2, k=K, tile_m=256, tile_n=256, workers=S).set_option("gemm_swiglu", 1)
