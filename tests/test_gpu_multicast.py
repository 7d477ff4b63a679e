"""FO_OPT_MULTICAST: clusters of two CTA pairs with TMA multicast of a shared
operand panel must give bit-identical GEMM / epilogue output to independent
pairs (the multicast changes only which CTA loads which rows), and the exact
oracle values in the exact-integer regime.  Covers orders whose consecutive
positions share the A tile-row, the B tile-column or neither, an odd tile
count (the last cluster round runs one pair alone) and every epilogue mode."""
import numpy as np
import pytest
import torch

import paper_2504_19519_b200 as fo
import synthetic

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _dev():
    from paper_2504_19519_b200 import build

    build.build()
    torch.cuda.set_device(0)


def _pair(kw, order=None):
    plans = []
    for mc in (1, 0):
        pl = fo.Plan(tile_order=order, **kw)
        pl.set_option("multicast", mc)
        plans.append(pl)
    return plans


@pytest.mark.parametrize("swizzle", [1, 2, 4, 0])
@pytest.mark.parametrize("bn", [128, 256])
def test_multicast_bit_identical_default_orders(swizzle, bn):
    M, N, K = 2048, 2048, 1024
    S = 8
    kw = dict(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=bn, workers=S, swizzle=swizzle)
    A, Bt = synthetic.float_inputs(M, N, K, seed=41, device="cuda")
    on, off = _pair(kw)
    assert on.multicast_used() and not off.multicast_used()
    assert fo.Plan(**kw).gemm_cluster() == 2  # default: independent pairs
    c1 = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    c2 = torch.empty_like(c1)
    for _ in range(3):
        c1.fill_(float("nan"))
        fo.gemm_stage(on, A, Bt, c1)
        fo.gemm_stage(off, A, Bt, c2)
        torch.cuda.synchronize()
        assert torch.equal(c1, c2)
    ref = (A.float() @ Bt.float().t())
    assert ((c1.float() - ref).abs().max() / ref.abs().max()).item() < 1e-2


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_multicast_random_orders_and_odd_tile_count(seed):
    """Random explicit orders (consecutive positions share A, B or nothing) and
    an odd number of tiles (a solo final round)."""
    rng = np.random.default_rng(seed)
    M, N, K = 256 * 5, 256 * 3, 512   # 15 tiles, S = 4 -> rounds of 2 + a solo pair at the end
    order = rng.permutation(15).astype(np.int32)
    kw = dict(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=4)
    A, Bt = synthetic.exact_inputs(M, N, K, seed=seed, nnz_per_row=64)
    A, Bt = A.cuda(), Bt.cuda()
    on, off = _pair(kw, order)
    assert on.multicast_used()
    c1 = torch.full((M, N), float("nan"), dtype=torch.bfloat16, device="cuda")
    c2 = torch.empty_like(c1)
    fo.gemm_stage(on, A, Bt, c1)
    fo.gemm_stage(off, A, Bt, c2)
    torch.cuda.synchronize()
    assert torch.equal(c1, c2)
    # exact-integer regime: the plain product is exact in bf16
    ref = (A.double() @ Bt.double().t()).to(torch.bfloat16)
    assert torch.equal(c1, ref)


@pytest.mark.parametrize("coll,layout", [("allreduce", "slot"), ("allreduce", "rowband"), ("reducescatter", "auto"),
                                         ("alltoall", "auto")])
def test_multicast_through_fo_run(coll, layout):
    """The overlapped op with multicast clusters equals the one with
    independent pairs (send/receive layouts, signals, groups), world 1."""
    ctx = fo.Context.create(0, 0, 1, fo.unique_id())
    try:
        M, N, K, S = 2048, 2048, 1024, 8
        kw = dict(coll=coll, m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, swizzle=0,
                  group_waves=[2, 4, 2], ar_layout=layout)
        if coll == "alltoall":
            kw["row_dst"] = np.zeros(M, np.int32)
            mk = lambda: fo.Plan(rank=0, world=1, peers=[kw], **kw)
        else:
            mk = lambda: fo.Plan(**kw)
        on, off = mk(), mk()
        on.set_option("multicast", 1)
        off.set_option("multicast", 0)
        A, Bt = synthetic.float_inputs(M, N, K, seed=43, device="cuda")
        o1 = torch.empty(on.info["out_rows"], N, dtype=torch.bfloat16, device="cuda")
        o2 = torch.empty_like(o1)
        for _ in range(5):
            o1.fill_(float("nan"))
            fo.run(ctx, on, A, Bt, o1)
            fo.run(ctx, off, A, Bt, o2)
            torch.cuda.synchronize()
            assert torch.equal(o1, o2)
    finally:
        ctx.close()


def test_multicast_full_size_bench_config():
    """configs[1] at TP=1 (4096x4096x14336, S=64 pairs = 32 clusters): identical
    to independent pairs."""
    M, N, K = 4096, 4096, 14336
    kw = dict(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=64, swizzle=0)
    A, Bt = synthetic.float_inputs(M, N, K, seed=44, device="cuda")
    on, off = _pair(kw)
    assert on.multicast_used()
    c1 = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    c2 = torch.empty_like(c1)
    fo.gemm_stage(on, A, Bt, c1)
    fo.gemm_stage(off, A, Bt, c2)
    torch.cuda.synchronize()
    assert torch.equal(c1, c2)
