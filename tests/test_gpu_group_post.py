"""Per-group post-communication reorder: running every wave group's pass
(fo_group_post_stage, the pass fo_run issues right after each group's
collective) over a receive buffer must write exactly what the one-shot
post-reorder writes (fo_post_stage, itself pinned to the oracle by
test_gpu_parity), bit for bit, for the AR slot (256- and 128-row tiles), RS
(n = 2, 8) and A2A layouts with post none and residual add (
DESIGN.md H11b)."""
import numpy as np
import pytest
import torch

import synthetic

pytestmark = pytest.mark.gpu
fo = pytest.importorskip("paper_2504_19519_b200")


@pytest.fixture(scope="module", autouse=True)
def _dev():
    from paper_2504_19519_b200 import build

    build.build()
    torch.cuda.set_device(0)


def _plans(kind, post):
    if kind == "slot":
        sp = dict(coll="allreduce", m=1024, n=1536, k=64, tile_m=256, tile_n=256, workers=5, swizzle=2,
                  group_waves=[1, 2, 2], ar_layout="slot", post=post)
        return fo.Plan(**sp)
    if kind == "slot128":
        sp = dict(coll="allreduce", m=768, n=640, k=64, tile_m=128, tile_n=128, workers=7, swizzle=3,
                  group_waves=[1, 2, 2], ar_layout="slot", post=post)
        return fo.Plan(**sp)
    if kind.startswith("rs"):
        n = int(kind[2:])
        sp = dict(coll="reducescatter", m=2048, n=1024, k=64, tile_m=256, tile_n=128, workers=11, swizzle=2,
                  group_waves=[1, 2, 3], post=post)
        return fo.Plan(rank=1 % n, world=n, **sp)
    # A2A: three sources with random routing, seen from rank 1
    n = 3
    specs = []
    for s in range(n):
        M = 256 * (s + 1)
        rd = synthetic.random_row_dst(M, n, 50 + s)
        specs.append(dict(coll="alltoall", m=M, n=512, k=64, tile_m=256, tile_n=128, workers=2, swizzle=1,
                          group_waves=[1, -(-(M // 256) * 4 // 2) - 1], row_dst=rd, post=post, ar_layout="slot"))
    return fo.Plan(rank=1, world=n, peers=specs, **specs[1])


@pytest.mark.parametrize("kind", ["slot", "slot128", "rs2", "rs8", "a2a"])
@pytest.mark.parametrize("post", ["none", "add"])
def test_group_post_equals_full_post(kind, post):
    plan = _plans(kind, post)
    rows, N = plan.info["out_rows"], plan.info["out_cols"]
    g = torch.Generator(device="cuda").manual_seed(3)
    recv = torch.randn(plan.info["recv_elems"], generator=g, device="cuda").to(torch.bfloat16)
    res = torch.randn(rows, N, generator=g, device="cuda").to(torch.bfloat16) if post == "add" else None
    want = torch.empty(rows, N, dtype=torch.bfloat16, device="cuda")
    fo.post_stage(plan, recv, want, res)
    got = torch.full((rows, N), float("nan"), dtype=torch.bfloat16, device="cuda")
    for j in range(plan.info["num_groups"]):
        fo.group_post_stage(plan, j, recv, got, res)
    torch.cuda.synchronize()
    assert torch.equal(got, want)


def test_group_post_inside_fo_run():
    """fo_run with the per-group post (RS and AR slot at world 1, groups
    beside the GEMM) == fo_run_sequential, repeatedly."""
    ctx = fo.Context.create(0, 0, 1, fo.unique_id())
    M, N, K = 2048, 2048, 512
    A, Bt = synthetic.exact_inputs(M, N, K, seed=5, nnz_per_row=64)
    A, Bt = A.cuda(), Bt.cuda()
    # RS "auto" here is the rowband layout (R40: waves of 2 whole tile-rows,
    # panels of 2): no post pass at all
    for coll, lay in (("allreduce", "slot"), ("reducescatter", "slot"), ("reducescatter", "auto")):
        plan = fo.Plan(coll=coll, m=M, n=N, k=K, tile_m=256, tile_n=256, workers=16, swizzle=2,
                       group_waves=[1, 2, 1], ar_layout=lay)
        assert plan.info["ar_layout"] == (1 if lay == "auto" else 0)
        plan.set_option("group_post", 1)
        want = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        fo.run_sequential(ctx, plan, A, Bt, want)
        for _ in range(3):
            out = torch.full((M, N), float("nan"), dtype=torch.bfloat16, device="cuda")
            fo.run(ctx, plan, A, Bt, out)
            torch.cuda.synchronize()
            assert torch.equal(out, want), coll
    ctx.close()


@pytest.mark.parametrize("kind", ["ar_slot", "ar_rowband", "rs_slot", "a2a_slot", "rowx"])
@pytest.mark.parametrize("post", ["add_rmsnorm", "add_rmsnorm_res"])
def test_bulk_rmsnorm_equals_register_kernel(kind, post):
    """The bulk-staged add + RMSNorm (rows in shared memory by cp.async.bulk,
    outputs >= 64 MB) gives the register kernel's bits through every map (same
    chunk -> thread map and fp32 sum order), and matches the oracle's
    add + RMSNorm within the north_star tolerance."""
    from oracle import numerics as onum
    from oracle import post as opost
    M, N = 8192, 4096
    base = dict(m=M, n=N, k=64, tile_m=256, tile_n=256, workers=64, post=post)
    if kind == "ar_slot":
        plan = fo.Plan(coll="allreduce", swizzle=2, group_waves=[2, 2, 4], ar_layout="slot", **base)
    elif kind == "ar_rowband":
        plan = fo.Plan(coll="allreduce", swizzle=1, group_waves=[2, 2, 4], ar_layout="rowband", **base)
    elif kind in ("rs_slot", "rowx"):
        base["m"] = 2 * M                     # 2 ranks: 8192 output rows each
        plan = fo.Plan(coll="reducescatter", swizzle=2, group_waves=[4, 12], ar_layout="slot", rank=1, world=2, **base)
    else:
        spec = dict(coll="alltoall", swizzle=2, group_waves=[2, 6], row_dst=np.zeros(M, np.int32), ar_layout="slot",
                    **base)
        plan = fo.Plan(rank=0, world=1, peers=[spec], **spec)
    rows = plan.info["out_rows"] if kind != "rowx" else base["m"]
    g = torch.Generator(device="cuda").manual_seed(11)
    n_in = plan.info["recv_elems"] if kind != "rowx" else rows * N
    recv = torch.randn(n_in, generator=g, device="cuda").to(torch.bfloat16)
    res0 = torch.randn(rows, N, generator=g, device="cuda").to(torch.bfloat16)
    gam = torch.randn(N, generator=g, device="cuda").to(torch.bfloat16)
    outs, ress = [], []
    for bulk in (1, 0):
        plan.set_option("post_bulk", bulk)
        out = torch.full((rows, N), float("nan"), dtype=torch.bfloat16, device="cuda")
        res = res0.clone()
        if kind == "rowx":
            fo.rowexchange_stage(plan, recv, out, res, gam)
        else:
            fo.post_stage(plan, recv, out, res, gam)
        torch.cuda.synchronize()
        outs.append(out)
        ress.append(res)
    assert rows * N * 2 >= 64 << 20                   # the bulk kernel's size class
    assert torch.equal(outs[0], outs[1])
    assert torch.equal(ress[0], ress[1])
    # against the oracle: x = the reordered received data, read back from the
    # no-op pass (post none on the same map)
    if kind == "ar_rowband":
        x = recv.view(rows, N).double().cpu().numpy()
        want = opost.add_rmsnorm(x, onum.to_f64(res0.cpu()), onum.to_f64(gam.cpu()), 1e-5)
        got = outs[0].double().cpu().numpy()
        rms = np.sqrt(np.mean(want * want))
        assert float(np.max(np.abs(got - want) / np.maximum(np.abs(want), rms))) <= 1e-2
