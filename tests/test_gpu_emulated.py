"""The emulated-link evaluation backend (fo_ctx_create_emulated): its
collectives take the modelled NVLink time and leave the documented data
(timing only), and fo_run runs its whole schedule through it."""
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
    fo.load()
    torch.cuda.set_device(0)
    yield


@pytest.mark.parametrize("coll,n", [("allreduce", 2), ("allreduce", 8), ("reducescatter", 8)])
def test_collective_time_follows_the_link_model(coll, n):
    gbps, lat = 770.0, 6.0
    ctx = fo.Context.emulated(0, 0, n, gbps, lat, 16)
    for nbytes in (1 << 22, 1 << 25):
        t = ctx.time_collective(coll, nbytes, 5)
        bus = (2.0 * (n - 1) / n if coll == "allreduce" else (n - 1) / n) * nbytes
        model = lat + bus / (gbps * 1e3)
        # lower bound: the link model; upper: the call's own HBM traffic on 16
        # CTAs may take longer than the wire time when n is small (2 ranks:
        # 64 MB moved for a 32 MB AllReduce), so the bound is loose there
        assert model <= t <= 1.5 * model + 15.0, (coll, n, nbytes, t, model)
    ctx.close()


@pytest.mark.parametrize("coll,layout", [("allreduce", "rowband"), ("allreduce", "slot"),
                                         ("reducescatter", "rowband"), ("reducescatter", "slot")])
def test_fo_run_through_the_emulated_link(coll, layout):
    """At emulated world 4 the AllReduce leaves each rank's own partial and the
    ReduceScatter its own chunk, so fo_run must return rank 0's GEMM (AR) or
    its block-cyclic rows R_0 of it (RS), bit for bit, through the whole
    overlapped schedule (counters, stream waits, per-group calls, post pass)."""
    n, M, N, K, S = 4, 2048, 1024, 512, 8
    ctx = fo.Context.emulated(0, 0, n, 770.0, 6.0, 16)
    A, Bt = synthetic.float_inputs(M, N, K, seed=3, device="cuda")
    plan = fo.Plan(coll=coll, m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, swizzle=1 if layout == "rowband" else 2,
                   group_waves=[1, 2, 1], ar_layout=layout, rank=0, world=n)
    assert plan.info["ar_layout"] == (1 if layout == "rowband" else 0)
    gp = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, tile_order=plan.export_order())
    C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    fo.gemm_stage(gp, A, Bt, C)
    out = torch.full((plan.info["out_rows"], N), float("nan"), dtype=torch.bfloat16, device="cuda")
    for _ in range(2):
        fo.run(ctx, plan, A, Bt, out)
    torch.cuda.synchronize()
    if coll == "allreduce":
        want = C
    else:
        h = 256 // n
        rows = np.array([(l // h) * 256 + l % h for l in range(M // n)])     # R_0 (rank 0's subtile rows)
        want = C[torch.from_numpy(rows).cuda()]
    assert torch.equal(out, want)
    ctx.close()
