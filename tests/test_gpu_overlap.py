"""Evidence that the signaling chain is correct and overlapped (world = 1,
real fo_run with stream waits + NCCL):

* causality: the comm stream's wait for group j is released only after every
  tile of group j signalled (%globaltimer of the release >= the last tile of
  the group) — PAPER.md:368 "Once the j-th number reaches |G_j|, the
  communication of G_j starts";
* overlap: group 0's wait is released (and its per-group post-reorder done)
  while the GEMM still computes later waves;
* memory ordering under stress: the library's send/receive
  buffers are poisoned with NaN before every run and inputs alternate between
  two data sets; any collective or post-reorder reading a group before its
  tiles' stores are visible would leak NaN or stale values into the output;
* per-group post-reorder (H11b) == one post-reorder after the last group.
"""
import numpy as np
import pytest
import torch

import synthetic

pytestmark = pytest.mark.gpu
fo = pytest.importorskip("paper_2504_19519_b200")


@pytest.fixture(scope="module")
def ctx():
    from paper_2504_19519_b200 import build

    build.build()
    torch.cuda.set_device(0)
    c = fo.Context.create(0, 0, 1, fo.unique_id())
    yield c
    c.close()


@pytest.mark.parametrize("wait_kernel", [0, 1])
@pytest.mark.parametrize("coll", ["allreduce", "reducescatter"])
def test_causality_and_overlap(ctx, coll, wait_kernel):
    M, N, K, S = 4096, 4096, 7168, 64
    groups = [1, 1, 1, 1]
    A, Bt = synthetic.float_inputs(M, N, K, seed=3, device="cuda")
    plan = fo.Plan(coll=coll, m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, swizzle=2, group_waves=groups,
                   ar_layout="slot")
    plan.set_option("wait_kernel", wait_kernel)
    tiles = plan.info["tiles"]
    tile_ts = torch.zeros(tiles, dtype=torch.int64, device="cuda")
    group_ts = torch.zeros(2 * len(groups), dtype=torch.int64, device="cuda")
    plan.set_debug(tile_ts, group_ts)
    out = torch.empty(plan.info["out_rows"], N, dtype=torch.bfloat16, device="cuda")
    for _ in range(3):
        fo.run(ctx, plan, A, Bt, out)
    torch.cuda.synchronize()
    t = tile_ts.cpu().numpy()
    g = group_ts.cpu().numpy()
    gemm_end = t.max()
    for j in range(len(groups)):
        lo, hi, _, _ = plan.group(j)
        assert g[2 * j] >= t[lo:hi].max(), f"group {j} released before its last tile signalled"
        assert g[2 * j + 1] >= g[2 * j]
    assert g[0] < gemm_end, "group 0's communication did not start before the GEMM finished"
    assert g[1] < gemm_end, "group 0's collective + post-reorder did not finish inside the GEMM"


@pytest.mark.parametrize("wait_kernel", [0, 1])
@pytest.mark.parametrize("coll", ["allreduce", "reducescatter", "alltoall"])
def test_memory_ordering_stress(ctx, coll, wait_kernel):
    M, N, K, S = 2048, 2048, 1024, 16
    groups = [1, 1, 1, 1]  # 64 tiles of 256x256, 16 pairs -> 4 waves
    kw = dict(coll=coll, m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, swizzle=2, group_waves=groups,
              ar_layout="slot")
    if coll == "alltoall":
        kw["row_dst"] = np.zeros(M, np.int32)
        plan = fo.Plan(rank=0, world=1, peers=[kw], **kw)
    else:
        plan = fo.Plan(**kw)
    plan.set_option("wait_kernel", wait_kernel)
    inputs = [synthetic.float_inputs(M, N, K, seed=s, device="cuda") for s in (11, 12)]
    want = []
    for A, Bt in inputs:
        o = torch.empty(plan.info["out_rows"], N, dtype=torch.bfloat16, device="cuda")
        fo.run_sequential(ctx, plan, A, Bt, o)
        want.append(o)
    torch.cuda.synchronize()
    out = torch.empty_like(want[0])
    bad = 0
    for it in range(300):
        A, Bt = inputs[it % 2]
        plan.fill_buffers(0x7FC0)  # bf16 NaN
        out.fill_(float("nan"))
        fo.run(ctx, plan, A, Bt, out)
        if not torch.equal(out, want[it % 2]):
            bad += 1
    torch.cuda.synchronize()
    assert bad == 0, f"{bad} of 300 overlapped runs read data before it was complete"


@pytest.mark.parametrize("coll,post", [("allreduce", "none"), ("allreduce", "add"), ("reducescatter", "add"),
                                       ("alltoall", "none")])
def test_group_post_equals_single_post(ctx, coll, post):
    M, N, K, S = 2048, 1024, 512, 8
    tiles = (M // 256) * (N // 128)
    T = -(-tiles // S)
    groups = synthetic.random_partition(T, 4)
    kw = dict(coll=coll, m=M, n=N, k=K, tile_m=256, tile_n=128, workers=S, swizzle=3, group_waves=groups,
              ar_layout="slot", post=post)
    if coll == "alltoall":
        kw["row_dst"] = np.zeros(M, np.int32)
        mk = lambda: fo.Plan(rank=0, world=1, peers=[kw], **kw)
    else:
        mk = lambda: fo.Plan(**kw)
    p_on, p_off = mk(), mk()
    p_off.set_debug(group_post=0)
    A, Bt = synthetic.float_inputs(M, N, K, seed=9, device="cuda")
    res = synthetic.normal_bf16((p_on.info["out_rows"], N), 1.0, 5, device="cuda")
    o1 = torch.empty(p_on.info["out_rows"], N, dtype=torch.bfloat16, device="cuda")
    o2 = torch.empty_like(o1)
    fo.run(ctx, p_on, A, Bt, o1, res if post != "none" else None)
    fo.run(ctx, p_off, A, Bt, o2, res if post != "none" else None)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2)


@pytest.mark.parametrize("post", ["add", "add_rmsnorm"])
def test_rowband_band_post_equals_single_post(ctx, post):
    """ROWBAND: the fused add / RMSNorm runs per band right after the band's
    AllReduce; it must equal the single post after the last group, and the
    oracle within tolerance."""
    from oracle import numerics as onum
    from oracle import post as opost

    M, N, K, S = 2048, 1024, 512, 8          # 256x256 pairs: 8x4 tiles, S=8 -> waves of 2 tile-rows
    kw = dict(coll="allreduce", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, swizzle=1,
              group_waves=[1, 2, 1], ar_layout="rowband", post=post)
    p_on, p_off = fo.Plan(**kw), fo.Plan(**kw)
    p_off.set_debug(group_post=0)
    assert p_on.info["ar_layout"] == 1
    A, Bt = synthetic.float_inputs(M, N, K, seed=21)
    res = synthetic.normal_bf16((M, N), 1.0, 22)
    gam = synthetic.normal_bf16((N,), 1.0, 23)
    o1 = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    o2 = torch.empty_like(o1)
    args = (A.cuda(), Bt.cuda())
    fo.run(ctx, p_on, *args, o1, res.cuda(), gam.cuda())
    fo.run(ctx, p_off, *args, o2, res.cuda(), gam.cuda())
    torch.cuda.synchronize()
    assert torch.equal(o1, o2)
    x = onum.round_bf16(onum.gemm(A, Bt))
    want = opost.add(x, onum.to_f64(res)) if post == "add" else opost.add_rmsnorm(x, onum.to_f64(res), onum.to_f64(gam), 1e-5)
    g = o1.double().cpu().numpy()
    rms = np.sqrt(np.mean(want * want))
    assert np.max(np.abs(g - want) / np.maximum(np.abs(want), rms)) <= 1e-2


def test_post_sm_partition_option_equal_results(ctx):
    M, N, K, S = 2048, 1024, 512, 8
    kw = dict(coll="allreduce", m=M, n=N, k=K, tile_m=256, tile_n=128, workers=S, swizzle=3, group_waves=[2, 3, 3],
              ar_layout="slot", post="add")
    p_on, p_off = fo.Plan(**kw), fo.Plan(**kw)
    p_on.set_option("post_sm_partition", 1)
    A, Bt = synthetic.float_inputs(M, N, K, seed=31, device="cuda")
    res = synthetic.normal_bf16((M, N), 1.0, 32, device="cuda")
    o1 = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    o2 = torch.empty_like(o1)
    fo.run(ctx, p_on, A, Bt, o1, res)
    fo.run(ctx, p_off, A, Bt, o2, res)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2)


@pytest.mark.parametrize("coll,post,layout", [("allreduce", "none", "slot"), ("allreduce", "add_rmsnorm", "slot"),
                                              ("allreduce", "add_rmsnorm", "rowband"),
                                              ("reducescatter", "add", "slot"), ("reducescatter", "add", "auto"),
                                              ("reducescatter", "add_rmsnorm", "rowband"),
                                              ("alltoall", "none", "auto")])
def test_last_group_in_order_equals_counter_trigger(ctx, coll, post, layout):
    """FO_OPT_LAST_GROUP_IN_ORDER: the last group's collective issued on the
    caller stream after the GEMM gives bit-identical results to triggering it
    by its counter on the comm stream, over repeated runs."""
    M, N, K, S = 2048, 1024, 512, 8
    kw = dict(coll=coll, m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, swizzle=1,
              group_waves=[1, 2, 1], ar_layout=layout, post=post)
    if coll == "alltoall":
        kw["row_dst"] = np.zeros(M, np.int32)
        mk = lambda: fo.Plan(rank=0, world=1, peers=[kw], **kw)
    else:
        mk = lambda: fo.Plan(**kw)
    p_on, p_off = mk(), mk()
    p_off.set_option("last_group_in_order", 0)
    A, Bt = synthetic.float_inputs(M, N, K, seed=31, device="cuda")
    rows = p_on.info["out_rows"]
    res = synthetic.normal_bf16((rows, N), 1.0, 32, device="cuda") if post != "none" else None
    gam = synthetic.normal_bf16((N,), 1.0, 33, device="cuda") if post == "add_rmsnorm" else None
    o1 = torch.empty(rows, N, dtype=torch.bfloat16, device="cuda")
    o2 = torch.empty_like(o1)
    for _ in range(20):
        p_on.fill_buffers(0x7FC0)
        o1.fill_(float("nan"))
        fo.run(ctx, p_on, A, Bt, o1, res, gam)
        fo.run(ctx, p_off, A, Bt, o2, res, gam)
        torch.cuda.synchronize()
        assert torch.equal(o1, o2)


@pytest.mark.parametrize("coll,post,layout", [("allreduce", "none", "rowband"), ("allreduce", "add", "slot"),
                                              ("allreduce", "add_rmsnorm", "rowband"),
                                              ("reducescatter", "add", "slot"), ("reducescatter", "add", "auto"),
                                              ("alltoall", "none", "auto")])
def test_single_group_in_order_equals_sequential(ctx, coll, post, layout):
    """One group issued in stream order (R32): no counters, no fork — the
    overlapped op must equal fo_run_sequential bit for bit, repeatedly."""
    M, N, K, S = 2048, 1024, 512, 8
    kw = dict(coll=coll, m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, swizzle=1,
              group_waves=[4], ar_layout=layout, post=post)
    if coll == "alltoall":
        kw["row_dst"] = np.zeros(M, np.int32)
        plan = fo.Plan(rank=0, world=1, peers=[kw], **kw)
    else:
        plan = fo.Plan(**kw)
    A, Bt = synthetic.float_inputs(M, N, K, seed=35, device="cuda")
    rows = plan.info["out_rows"]
    res = synthetic.normal_bf16((rows, N), 1.0, 36, device="cuda") if post != "none" else None
    gam = synthetic.normal_bf16((N,), 1.0, 37, device="cuda") if post == "add_rmsnorm" else None
    want = torch.empty(rows, N, dtype=torch.bfloat16, device="cuda")
    fo.run_sequential(ctx, plan, A, Bt, want, res, gam)
    got = torch.empty_like(want)
    for _ in range(10):
        plan.fill_buffers(0x7FC0)
        got.fill_(float("nan"))
        fo.run(ctx, plan, A, Bt, got, res, gam)
        torch.cuda.synchronize()
        assert torch.equal(got, want)


def test_watchdog_times_out_and_releases():
    """fo_plan_sync (the debug watchdog, SURVEY §8(b) FO_ERR_TIMEOUT): a run
    whose group 0 can never fire (FO_OPT_DEBUG_STALL_GROUP) is detected, the
    communicator aborted, the waits released (the streams drain), and the
    context refuses further runs; a healthy run syncs OK."""
    c = fo.Context.create(0, 0, 1, fo.unique_id())
    M, N, K, S = 2048, 1024, 512, 8
    kw = dict(coll="allreduce", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, swizzle=2,
              group_waves=[1, 2, 1], ar_layout="slot")
    A, Bt = synthetic.float_inputs(M, N, K, seed=41, device="cuda")
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    good = fo.Plan(**kw)
    fo.run(c, good, A, Bt, out)
    fo.plan_sync(c, good, timeout_ms=5000)
    for wait_kernel in (0, 1):
        c2 = fo.Context.create(0, 0, 1, fo.unique_id())
        bad = fo.Plan(**kw)
        bad.set_option("wait_kernel", wait_kernel)
        bad.set_option("debug_stall_group", 0)
        fo.run(c2, bad, A, Bt, out)
        with pytest.raises(fo.FOError, match="TIMEOUT"):
            fo.plan_sync(c2, bad, timeout_ms=300)
        torch.cuda.synchronize()          # everything drained after the release
        with pytest.raises(fo.FOError, match="STATE"):
            fo.run(c2, bad, A, Bt, out)
        c2.close()
    fo.run(c, good, A, Bt, out)           # other contexts are unaffected
    fo.plan_sync(c, good, timeout_ms=5000)
    c.close()
