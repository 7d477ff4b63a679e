"""Small runs of every device path for compute-sanitizer (memcheck / racecheck
/ synccheck): GEMM (CTA and CTA-pair, tail split), every epilogue mode,
fo_run at world 1 for AR/RS/A2A (+ fused RMSNorm), per-group post, row
exchange.  Dev tool; exits non-zero on a numerical mismatch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402
import synthetic  # noqa: E402


def main():
    torch.cuda.set_device(0)
    ctx = fo.Context.create(0, 0, 1, fo.unique_id())
    M, N, K = 512, 512, 256
    A, Bt = synthetic.exact_inputs(M, N, K, seed=1, nnz_per_row=100)
    Ad, Bd = A.cuda(), Bt.cuda()
    C = (A.double() @ Bt.double().t()).to(torch.bfloat16).cuda()
    res = torch.zeros(M, N, dtype=torch.bfloat16, device="cuda")
    gam = torch.ones(N, dtype=torch.bfloat16, device="cuda")
    bad = 0
    # the MoE combine (R31 / R31b): async-copy kernel (k <= 2 [+ residual]) and
    # register kernel (k = 3 + residual, k = 5), dropped slots, ragged last unit
    Mc, Nc = 768, 1600
    kwc = dict(coll="alltoall", m=Mc, n=Nc, k=64, tile_m=128, tile_n=64, workers=8, swizzle=1,
               ar_layout="slot", row_dst=np.zeros(Mc, np.int32))
    pc = fo.Plan(rank=0, world=1, peers=[kwc], **kwc)
    recv_c = torch.randn(Mc * Nc, device="cuda").to(torch.bfloat16)
    for kc, with_res in ((1, False), (2, True), (2, False), (3, True), (5, False)):
        tok = Mc // kc
        idx_c = torch.randperm(Mc, device="cuda")[:tok * kc].to(torch.int32).view(tok, kc).contiguous()
        idx_c[::3, -1] = -1
        w_c = torch.rand(tok, kc, device="cuda")
        out_c = torch.empty(tok, Nc, dtype=torch.bfloat16, device="cuda")
        args_c = (torch.randn(tok, Nc, device="cuda").to(torch.bfloat16),) if with_res else ()
        fo.combine_stage(pc, recv_c, out_c, idx_c, w_c, *args_c)
    torch.cuda.synchronize()
    if os.environ.get("SANITIZE_ONLY") == "combine":
        print("sanitize cases done, mismatches:", bad)
        return
    for BM in (128, 256):
        for coll in ("nocomm", "allreduce", "reducescatter", "alltoall"):
            for post in ("none", "add"):
                kw = dict(coll=coll, m=M, n=N, k=K, tile_m=BM, tile_n=128, workers=3, swizzle=2,
                          ar_layout="slot", post=post)
                if coll == "alltoall":
                    kw["row_dst"] = np.zeros(M, np.int32)
                    plan = fo.Plan(rank=0, world=1, peers=[kw], **kw)
                else:
                    plan = fo.Plan(**kw)
                out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
                fo.run(ctx, plan, Ad, Bd, out, res if post != "none" else None)
                torch.cuda.synchronize()
                if not torch.equal(out, C):
                    print("mismatch", BM, coll, post)
                    bad += 1
    # tail split
    plan = fo.Plan(coll="nocomm", m=1024, n=1024, k=256, tile_m=256, tile_n=256, workers=12, swizzle=2)
    plan.set_option("tail_split", -1)
    A2, B2 = synthetic.exact_inputs(1024, 1024, 256, seed=2, nnz_per_row=100)
    out = torch.empty(1024, 1024, dtype=torch.bfloat16, device="cuda")
    fo.gemm_stage(plan, A2.cuda(), B2.cuda(), out)
    torch.cuda.synchronize()
    if not torch.equal(out.cpu(), (A2.double() @ B2.double().t()).to(torch.bfloat16)):
        print("mismatch tail split")
        bad += 1
    # TMA multicast across clusters of two pairs (FO_OPT_MULTICAST), an odd
    # tile count (solo final round), and multi-group runs with the last group
    # in stream order vs counter-triggered (R32), single in-order group
    for bn in (128, 256):
        Mm, Nm = 256 * 3, 256 * 3
        A3, B3 = synthetic.exact_inputs(Mm, Nm, 256, seed=3, nnz_per_row=100)
        plan = fo.Plan(coll="nocomm", m=Mm, n=Nm, k=256, tile_m=256, tile_n=bn, workers=4, swizzle=2)
        plan.set_option("multicast", 1)
        out = torch.empty(Mm, Nm, dtype=torch.bfloat16, device="cuda")
        fo.gemm_stage(plan, A3.cuda(), B3.cuda(), out)
        torch.cuda.synchronize()
        if not torch.equal(out.cpu(), (A3.double() @ B3.double().t()).to(torch.bfloat16)):
            print("mismatch multicast", bn)
            bad += 1
    for lio in (0, 1):
        for groups in ([1, 1, 1], [3]):
            plan = fo.Plan(coll="allreduce", m=M, n=N, k=K, tile_m=256, tile_n=128, workers=3, swizzle=2,
                           group_waves=groups, ar_layout="slot")
            plan.set_option("last_group_in_order", lio)
            out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
            fo.run(ctx, plan, Ad, Bd, out)
            torch.cuda.synchronize()
            if not torch.equal(out, C):
                print("mismatch last_group_in_order", lio, groups)
                bad += 1
    # SwiGLU epilogue with a split tail, and the residual-writing RMSNorm
    Ms, Ks = 256 * 3, 256
    A4, W4 = synthetic.exact_inputs(Ms, 512, Ks, seed=4, nnz_per_row=50)
    plan = fo.Plan(coll="nocomm", m=Ms, n=512, k=Ks, tile_m=256, tile_n=256, workers=5, swizzle=0)
    plan.set_option("gemm_swiglu", 1)
    plan.set_option("tail_split", -1)
    sw = torch.empty(Ms, 256, dtype=torch.bfloat16, device="cuda")
    fo.gemm_stage(plan, A4.cuda(), W4.cuda(), sw)
    plan = fo.Plan(coll="allreduce", m=M, n=N, k=K, tile_m=256, tile_n=128, workers=4, swizzle=1,
                   group_waves=[1, 1], ar_layout="rowband", post="add_rmsnorm_res")
    res2 = torch.zeros(M, N, dtype=torch.bfloat16, device="cuda")
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    fo.run(ctx, plan, Ad, Bd, out, res2, gam)
    torch.cuda.synchronize()
    if not torch.equal(res2, C):
        print("mismatch residual stream")
        bad += 1
    # fused RMSNorm + row exchange
    plan = fo.Plan(coll="reducescatter", m=M, n=N, k=K, tile_m=256, tile_n=128, workers=3, post="add_rmsnorm")
    local = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    fo.run(ctx, plan, Ad, Bd, local, res, gam)
    full = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    fo.run_allgather(ctx, plan, local, full, res, gam)
    torch.cuda.synchronize()
    # round 2: ROWBAND layouts of RS (EPI_RS_BAND, TMA-stored and 16-B
    # subtile rows) and A2A, at world 1 (NCCL) and as world-4 stages
    for coll in ("reducescatter", "alltoall"):
        for post in ("none", "add"):
            kw = dict(coll=coll, m=M, n=N, k=K, tile_m=256, tile_n=128, workers=4, swizzle=1, group_waves=[1, 1],
                      ar_layout="rowband", post=post)
            if coll == "alltoall":
                kw["row_dst"] = np.zeros(M, np.int32)
                plan = fo.Plan(rank=0, world=1, peers=[kw], **kw)
            else:
                plan = fo.Plan(**kw)
            out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
            fo.run(ctx, plan, Ad, Bd, out, res if post != "none" else None)
            torch.cuda.synchronize()
            if not torch.equal(out, C):
                print(f"mismatch {coll} rowband post={post}")
                bad += 1
    for n, bn in ((4, 128), (8, 256)):   # h = 64 (TMA stores) / h = 32 with 256-column tiles
        plan = fo.Plan(coll="reducescatter", m=M, n=N, k=K, tile_m=256, tile_n=bn, workers=N // bn, swizzle=1,
                       group_waves=[1, 1], ar_layout="rowband", rank=1, world=n)
        send = torch.empty(M * N, dtype=torch.bfloat16, device="cuda")
        fo.gemm_stage(plan, Ad, Bd, send)
    specs = []
    for s_ in range(4):
        specs.append(dict(coll="alltoall", m=M, n=N, k=K, tile_m=256, tile_n=128, workers=4, swizzle=1,
                          group_waves=[1, 1], ar_layout="rowband", row_dst=(np.arange(M) % 4).astype(np.int32)))
    plan = fo.Plan(rank=2, world=4, peers=specs, **specs[2])
    send = torch.empty(plan.info["send_elems"], dtype=torch.bfloat16, device="cuda")
    fo.gemm_stage(plan, Ad, Bd, send)
    # the bulk-staged add + RMSNorm (>= 64 MB outputs) through the slot map, residual written back
    Mb, Nb = 8192, 4096
    plan = fo.Plan(coll="allreduce", m=Mb, n=Nb, k=64, tile_m=256, tile_n=256, workers=64, swizzle=2,
                   group_waves=[2, 2, 4], ar_layout="slot", post="add_rmsnorm_res")
    recv = torch.randn(Mb * Nb, device="cuda").to(torch.bfloat16)
    rb = torch.randn(Mb, Nb, device="cuda").to(torch.bfloat16)
    ob = torch.empty(Mb, Nb, dtype=torch.bfloat16, device="cuda")
    fo.post_stage(plan, recv, ob, rb, torch.ones(Nb, dtype=torch.bfloat16, device="cuda"))
    # the emulated-link evaluation backend: fo_run at emulated world 4
    ectx = fo.Context.emulated(0, 0, 4, 770.0, 6.0, 16)
    plan = fo.Plan(coll="allreduce", m=M, n=N, k=K, tile_m=256, tile_n=128, workers=4, swizzle=1,
                   group_waves=[1, 1], ar_layout="rowband", rank=0, world=4)
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    fo.run(ectx, plan, Ad, Bd, out)
    torch.cuda.synchronize()
    if not torch.equal(out, C):
        print("mismatch emulated-link fo_run")
        bad += 1
    ectx.close()
    ctx.close()
    print("sanitize cases done, mismatches:", bad)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
