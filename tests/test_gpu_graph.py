"""fo_run is host-asynchronous and CUDA-graph capturable (memset, fork/join
events, the persistent GEMM, cuStreamWaitValue32 nodes, NCCL calls, per-group
post-reorder): capture once, replay with new inputs copied into the static
buffers, compare with eager runs bit-exactly."""
import os

import numpy as np
import pytest
import torch

import synthetic

pytestmark = pytest.mark.gpu
fo = pytest.importorskip("paper_2504_19519_b200")


@pytest.mark.parametrize("coll,layout", [("allreduce", "slot"), ("allreduce", "rowband"), ("reducescatter", "auto"),
                                         ("alltoall", "auto")])
def test_graph_capture_replay(coll, layout):
    from paper_2504_19519_b200 import build

    build.build()
    torch.cuda.set_device(0)
    ctx = fo.Context.create(0, 0, 1, fo.unique_id())
    M, N, K, S = 2048, 2048, 1024, 16
    kw = dict(coll=coll, m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, group_waves=[1, 2, 1], ar_layout=layout,
              swizzle=1 if layout == "rowband" else 2)
    if coll == "alltoall":
        kw["row_dst"] = np.zeros(M, np.int32)
        plan = fo.Plan(rank=0, world=1, peers=[kw], **kw)
    else:
        plan = fo.Plan(**kw)
    inputs = [synthetic.float_inputs(M, N, K, seed=s, device="cuda") for s in (1, 2, 3)]
    A = torch.empty_like(inputs[0][0])
    Bt = torch.empty_like(inputs[0][1])
    out = torch.empty(plan.info["out_rows"], N, dtype=torch.bfloat16, device="cuda")
    # eager reference outputs
    want = []
    for a, b in inputs:
        o = torch.empty_like(out)
        fo.run(ctx, plan, a, b, o)
        want.append(o)
    torch.cuda.synchronize()
    A.copy_(inputs[0][0])
    Bt.copy_(inputs[0][1])
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fo.run(ctx, plan, A, Bt, out)  # warm-up on the capture stream
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fo.run(ctx, plan, A, Bt, out)
    for it in range(6):
        a, b = inputs[it % 3]
        A.copy_(a)
        Bt.copy_(b)
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, want[it % 3])
    ctx.close()


def test_run_host_matches_device_run():
    """fo_run_host (host buffers, copies inside the call) == fo_run."""
    from paper_2504_19519_b200 import build

    build.build()
    torch.cuda.set_device(0)
    ctx = fo.Context.create(0, 0, 1, fo.unique_id())
    M, N, K = 1024, 1024, 512
    plan = fo.Plan(coll="allreduce", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=8, group_waves=[1, 1],
                   ar_layout="slot", swizzle=2, post="add_rmsnorm")
    A, Bt = synthetic.float_inputs(M, N, K, seed=4)
    res = synthetic.normal_bf16((M, N), 1.0, 6)
    gam = synthetic.normal_bf16((N,), 1.0, 7)
    out_h = torch.empty(M, N, dtype=torch.bfloat16).pin_memory()
    fo.run_host(ctx, plan, A.pin_memory(), Bt.pin_memory(), out_h, res.pin_memory(), gam.pin_memory())
    torch.cuda.synchronize()
    out_d = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    fo.run(ctx, plan, A.cuda(), Bt.cuda(), out_d, res.cuda(), gam.cuda())
    torch.cuda.synchronize()
    assert torch.equal(out_h, out_d.cpu())
    # mixed: device-resident weights and gamma, host activations / residual / output
    out_h2 = torch.empty(M, N, dtype=torch.bfloat16).pin_memory()
    fo.run_host(ctx, plan, A.pin_memory(), Bt.cuda(), out_h2, res, gam.cuda())
    torch.cuda.synchronize()
    assert torch.equal(out_h2, out_d.cpu())
    ctx.close()


def test_run_host_swiglu_and_residual_writeback():
    """fo_run_host sizes its output by what the GEMM writes (SwiGLU: [m, n/2])
    and, for FO_POST_ADD_RMSNORM_RESIDUAL with a host residual, copies the
    updated residual stream back to the caller."""
    from paper_2504_19519_b200 import build

    build.build()
    torch.cuda.set_device(0)
    ctx = fo.Context.create(0, 0, 1, fo.unique_id())
    M, N, K = 512, 1024, 256
    A, Bt = synthetic.float_inputs(M, N, K, seed=14)
    plan = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=4)
    plan.set_option("gemm_swiglu", 1)
    guard = 64                                   # host output with a guard band past [m, n/2]
    buf = torch.full((M * N // 2 + guard,), 7.0, dtype=torch.bfloat16).pin_memory()
    fo.run_host(ctx, plan, A.pin_memory(), Bt.cuda(), buf[:M * N // 2].view(M, N // 2))
    torch.cuda.synchronize()
    dev = torch.empty(M, N // 2, dtype=torch.bfloat16, device="cuda")
    fo.run(ctx, plan, A.cuda(), Bt.cuda(), dev)
    torch.cuda.synchronize()
    assert torch.equal(buf[:M * N // 2].view(M, N // 2), dev.cpu())
    assert torch.all(buf[M * N // 2:] == 7.0)     # nothing written past the output
    with pytest.raises(fo.FOError):
        p2 = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=4, post="add")
        p2.set_option("gemm_swiglu", 1)
    # residual stream write-back
    plan = fo.Plan(coll="allreduce", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=4, group_waves=[2],
                   post="add_rmsnorm_res")
    res = synthetic.normal_bf16((M, N), 1.0, 16)
    gam = synthetic.normal_bf16((N,), 1.0, 17)
    res_h = res.clone().pin_memory()
    out_h = torch.empty(M, N, dtype=torch.bfloat16).pin_memory()
    fo.run_host(ctx, plan, A.pin_memory(), Bt.cuda(), out_h, res_h, gam.cuda())
    torch.cuda.synchronize()
    res_d = res.cuda()
    out_d = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    fo.run(ctx, plan, A.cuda(), Bt.cuda(), out_d, res_d, gam.cuda())
    torch.cuda.synchronize()
    assert torch.equal(out_h, out_d.cpu())
    assert not torch.equal(res_d.cpu(), res)      # the residual stream was updated ...
    assert torch.equal(res_h, res_d.cpu())        # ... and the host copy with it
    ctx.close()


@pytest.mark.parametrize("buffers", ["registered", "window"])
def test_registered_buffers_world1(buffers):
    """fo_ctx_config.buffers: plans' send / receive buffers from ncclMemAlloc,
    registered with the communicator (ncclCommRegister / symmetric windows),
    and a caller `out` from fo_mem_alloc: every layout stays bit-identical to
    fo_run_sequential; time_collective reports the bus bandwidth."""
    from paper_2504_19519_b200 import build

    build.build()
    torch.cuda.set_device(0)
    ctx = fo.Context.create(0, 0, 1, fo.unique_id(), nccl_max_ctas=16, cta_policy="efficiency", buffers=buffers)
    M, N, K = 1024, 1024, 256
    A, Bt = synthetic.exact_inputs(M, N, K, seed=21, nnz_per_row=64)
    A, Bt = A.cuda(), Bt.cuda()
    for coll, lay, groups in (("allreduce", "slot", [1, 1, 2]), ("allreduce", "rowband", [2, 2]),
                              ("reducescatter", "auto", [1, 3])):
        plan = fo.Plan(coll=coll, m=M, n=N, k=K, tile_m=256, tile_n=256, workers=4, swizzle=1 if lay == "rowband" else 2,
                       group_waves=groups, ar_layout=lay)
        plan.prepare(ctx=ctx)
        want = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        fo.run_sequential(ctx, plan, A, Bt, want)
        out = ctx.mem_alloc((M, N))
        for _ in range(2):
            out.fill_(float("nan"))
            fo.run(ctx, plan, A, Bt, out)
            torch.cuda.synchronize()
            assert torch.equal(out, want), (buffers, coll, lay)
        del out
        plan.close()
    rd = synthetic.random_row_dst(M, 1, 3)
    spec = dict(coll="alltoall", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=4, group_waves=[1, 3], row_dst=rd)
    plan = fo.Plan(rank=0, world=1, peers=[spec], **spec)
    want = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    fo.run_sequential(ctx, plan, A, Bt, want)
    out = torch.full((M, N), float("nan"), dtype=torch.bfloat16, device="cuda")
    fo.run(ctx, plan, A, Bt, out)
    torch.cuda.synchronize()
    assert torch.equal(out, want)
    us, bus = ctx.time_collective_bw("allreduce", 1 << 22, 3)
    assert us > 0 and bus == 0.0               # one rank: 2(n-1)/n = 0 bus bytes
    ctx2 = fo.Context.create(0, 0, 1, fo.unique_id())
    with pytest.raises(fo.FOError):            # registered with ctx, not ctx2
        fo.run(ctx2, plan, A, Bt, out)
    plan.close()
    ctx2.close()
    ctx.close()


def test_time_collective_world1():
    from paper_2504_19519_b200 import build

    build.build()
    torch.cuda.set_device(0)
    ctx = fo.Context.create(0, 0, 1, fo.unique_id())
    for coll in ("allreduce", "reducescatter", "alltoall"):
        us = ctx.time_collective(coll, 1 << 20, iters=3)
        assert 0.0 < us < 1e4
    curve = ctx.sample_curve("allreduce", [1 << 16, 1 << 20], iters=2)
    assert len(curve) == 2 and all(b > 0 for _, b in curve)
    ctx.close()


def test_tune_layer_world1_returns_a_valid_plan():
    from paper_2504_19519_b200 import build
    from paper_2504_19519_b200 import tuner

    build.build()
    torch.cuda.set_device(0)
    ctx = fo.Context.create(0, 0, 1, fo.unique_id())
    M, N, K = 2048, 2048, 1024
    for post in ("none", "add_rmsnorm"):
        ch = tuner.tune_layer(M, N, K, ctx, "allreduce", post, iters=3, sizes=[1 << 18, 1 << 22])
        tiles = (M // 256) * (N // 256)
        assert sum(ch.groups) == -(-tiles // ch.workers)
        assert len(ch.candidates) >= 2 and all(len(c) >= 5 for c in ch.candidates)
        plan = fo.Plan(**ch.spec(M, N, K, "allreduce", post))
        A, Bt = synthetic.float_inputs(M, N, K, seed=3, device="cuda")
        out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        res = synthetic.normal_bf16((M, N), 1.0, 4, device="cuda")
        gam = synthetic.normal_bf16((N,), 1.0, 5, device="cuda")
        fo.run(ctx, plan, A, Bt, out, *((res, gam) if post != "none" else ()))
        torch.cuda.synchronize()
    ch = tuner.tune_layer(M, N, K, ctx, "reducescatter", "none", iters=3, sizes=[1 << 18, 1 << 22])
    assert ch.layout in ("rowband", "slot")            # both RS layouts are searched (R40)
    assert any(":rowband" in c[1] for c in ch.candidates) and any(":slot" in c[1] for c in ch.candidates)
    plan = fo.Plan(**ch.spec(M, N, K, "reducescatter"))
    assert plan.info["ar_layout"] == (1 if ch.layout == "rowband" else 0)
    fo.run(ctx, plan, A, Bt, out)
    want = torch.empty_like(out)
    fo.run_sequential(ctx, plan, A, Bt, want)    # one rank: the RS output is every row, in order
    torch.cuda.synchronize()
    assert torch.equal(out, want)
    # two communicators (CTA caps): the SM split is searched across both and
    # the chosen context's index comes back
    ctx2 = fo.Context.create(0, 0, 1, fo.unique_id(), nccl_max_ctas=32)
    ch = tuner.tune_layer(M, N, K, [ctx, ctx2], "allreduce", "none", iters=3, sizes=[1 << 18, 1 << 22])
    assert ch.ctx_index in (0, 1)
    assert any("+ctas32" in c[1] for c in ch.candidates) and any("+ctas0" in c[1] for c in ch.candidates)
    plan = fo.Plan(**ch.spec(M, N, K, "allreduce"))
    fo.run([ctx, ctx2][ch.ctx_index], plan, A, Bt, out)
    torch.cuda.synchronize()
    ctx2.close()
    ctx.close()


@pytest.mark.parametrize("case", ["rowband", "rowband_norm", "slot", "rs", "nocomm", "ragged"])
def test_run_host_pipelined_matches_device_run(case):
    """FO_OPT_HOST_PIPELINE: A copied in tile-row chunks the GEMM producer
    waits on, per-group D2H of ROWBAND output — bit-identical to fo_run on
    device operands, over repeated calls with fresh A each time (a stale chunk
    or a missed release shows up as a mismatch), pinned and pageable."""
    from paper_2504_19519_b200 import build

    build.build()
    torch.cuda.set_device(0)
    ctx = fo.Context.create(0, 0, 1, fo.unique_id())
    M, N, K = (2304, 1024, 1024) if case == "ragged" else (4096, 1024, 1024)
    coll = {"rs": "reducescatter", "nocomm": "nocomm"}.get(case, "allreduce")
    post = "add_rmsnorm" if case == "rowband_norm" else "none"
    layout = "slot" if case == "slot" else ("rowband" if coll == "allreduce" else "auto")
    Nt = N // 256
    S = 8 if case != "ragged" else 12
    tiles = (M // 256) * Nt
    T = -(-tiles // S)
    plan = fo.Plan(coll=coll, m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S,
                   group_waves=[1] * T if T <= 8 else [2] * (T // 2) + [1] * (T % 2),
                   ar_layout=layout if coll == "allreduce" else "auto", swizzle=1, post=post)
    res = synthetic.normal_bf16((M, N), 1.0, 6)
    gam = synthetic.normal_bf16((N,), 1.0, 7)
    Bt_d = synthetic.float_inputs(M, N, K, seed=9)[1].cuda()
    extra_d = (res.cuda(), gam.cuda()) if post != "none" else ()
    extra_h = (res.pin_memory(), gam.cuda()) if post != "none" else ()
    for it, pinned in enumerate([True, True, False]):
        A = synthetic.float_inputs(M, N, K, seed=20 + it)[0]
        out_d = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        fo.run(ctx, plan, A.cuda(), Bt_d, out_d, *extra_d)
        torch.cuda.synchronize()
        for pipe in (7, 3, 1, 2, 0):
            plan.set_option("host_pipeline", pipe)
            out_h = torch.full((M, N), float("nan"), dtype=torch.bfloat16)
            A_h = A.clone()
            if pinned:
                out_h, A_h = out_h.pin_memory(), A_h.pin_memory()
            fo.run_host(ctx, plan, A_h, Bt_d, out_h, *extra_h)
            torch.cuda.synchronize()
            assert torch.equal(out_h, out_d.cpu()), (case, it, pipe)
    ctx.close()


@pytest.mark.parametrize("layout", ["rowband", "slot"])
def test_run_host_back_to_back_two_staging_sets(layout):
    """FO_OPT_HOST_PIPELINE bit 2: consecutive fo_run_host calls alternate two
    staging sets, so call i+1's H2D overlaps call i — issued back to back
    without a host sync, each call with fresh activations and its own host
    output, every output must equal the device run of its own inputs."""
    from paper_2504_19519_b200 import build

    build.build()
    torch.cuda.set_device(0)
    ctx = fo.Context.create(0, 0, 1, fo.unique_id())
    M, N, K, S = 4096, 1024, 1024, 8
    tiles = (M // 256) * (N // 256)
    T = -(-tiles // S)
    plan = fo.Plan(coll="allreduce", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, group_waves=[1] * T,
                   ar_layout=layout, swizzle=1)
    assert plan.info["ar_layout"] == (1 if layout == "rowband" else 0)
    Bt_d = synthetic.float_inputs(M, N, K, seed=9)[1].cuda()
    As = [synthetic.float_inputs(M, N, K, seed=40 + i)[0].pin_memory() for i in range(5)]
    outs = [torch.full((M, N), float("nan"), dtype=torch.bfloat16).pin_memory() for _ in range(5)]
    for A_h, o in zip(As, outs):
        fo.run_host(ctx, plan, A_h, Bt_d, o)
    torch.cuda.synchronize()
    for i, (A_h, o) in enumerate(zip(As, outs)):
        want = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        fo.run(ctx, plan, A_h.cuda(), Bt_d, want)
        torch.cuda.synchronize()
        assert torch.equal(o, want.cpu()), (layout, i)
    ctx.close()


@pytest.mark.parametrize("world", [1, 2])
def test_tp_block_matches_oracle(world):
    """NEXT f4 second workload: the TP block (o_proj + AllReduce + fused add +
    RMSNorm updating the residual stream, gate/up GEMM with the fused SwiGLU,
    down-proj + AllReduce + residual add) through the library, overlapped and
    sequential, at TP = 1 (NCCL) and TP = 2 (loopback, one GPU), against the
    oracle's TP block (oracle/block.py) within 2^-6, two bf16 ulps
    (tests/tp_block_worker.py derives it)."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, CUDA_DEVICE_MAX_CONNECTIONS="32", CUDA_MODULE_LOADING="EAGER")
    r = subprocess.run([sys.executable, os.path.join(root, "tests", "tp_block_worker.py"), str(world)], cwd=root,
                       env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and f"tp block W={world}: OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]