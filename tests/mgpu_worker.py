"""One rank of the real multi-GPU parity check (launched by
tests/test_gpu_multi.py through torch.distributed.run, one process per GPU).

Each rank builds its plans through paper_2504_19519_b200.dist (library NCCL
communicator, A2A census), runs fo_run (overlapped: counter-triggered groups,
NCCL over NVLink, per-group post-reorder) and fo_run_sequential on
exact-integer inputs, and compares both with the plain definition computed by
this script with torch.distributed in fp32 (exact for these integers):
AllReduce = sum_r C_r; ReduceScatter = rows R_k of the sum (block-cyclic,
DESIGN.md R8) for fo_run and contiguous rows for fo_run_sequential (NCCL's
standard ReduceScatter of row-major C), and the AllGather + row exchange = the
AllReduce result;
All-to-All = concat over sources of the rows routed here (R9).  One AllReduce
also runs on a context built on torch's own communicator (fo_ctx_create_from_comm).  Exit status 0 = every comparison bit-exact.  Test infrastructure.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402
import synthetic  # noqa: E402
from paper_2504_19519_b200 import dist as fodist  # noqa: E402


def exact_inputs(M, N, K, rank, world, seed):
    A, Bt = synthetic.exact_inputs(M, N, K, seed=synthetic.rank_seed(seed, world, rank),
                                   nnz_per_row=max(1, 256 // world))
    return A.cuda(), Bt.cuda()


def check(name, got, want, bad):
    if not torch.equal(got, want):
        diff = (got.float() - want.float()).abs().max().item()
        print(f"[rank {dist.get_rank()}] MISMATCH {name}: max |diff| {diff}", flush=True)
        bad.append(name)


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    ctx = fodist.make_context(local, nccl_max_ctas=16)
    bad = []
    M, N, K = 2048, 1024, 512                   # 256x256 pairs: 8x4 tiles; S = 8 -> 4 waves
    for coll, layout, groups in (("allreduce", "slot", [1, 2, 1]), ("allreduce", "rowband", [1, 1, 2]),
                                 ("allreduce", "rowband", [4]), ("reducescatter", "slot", [2, 1, 1]),
                                 ("reducescatter", "rowband", [1, 1, 2])):
        A, Bt = exact_inputs(M, N, K, rank, world, 11)
        spec = dict(coll=coll, m=M, n=N, k=K, tile_m=256, tile_n=256, workers=8,
                    swizzle=1 if layout == "rowband" else 2, group_waves=groups, ar_layout=layout)
        plan = fodist.make_plan(**spec)
        C = (A.float() @ Bt.float().t())
        full = C.clone()
        dist.all_reduce(full)
        if coll == "allreduce":
            want = full.to(torch.bfloat16)
        else:
            h = 256 // world
            g = torch.arange(M, device="cuda")
            mine = ((g % 256) // h) == rank        # R_k, ascending global row
            want = full[mine].to(torch.bfloat16)
        for trig in (0, 1):
            plan.set_option("last_group_in_order", trig)
            out = torch.full((plan.info["out_rows"], N), float("nan"), dtype=torch.bfloat16, device="cuda")
            for _ in range(3):
                fo.run(ctx, plan, A, Bt, out)
            torch.cuda.synchronize()
            check(f"{coll}/{layout}/{groups}/in_order={trig}", out, want, bad)
        seq = torch.empty_like(out)
        fo.run_sequential(ctx, plan, A, Bt, seq)
        torch.cuda.synchronize()
        # the sequential ReduceScatter is NCCL's standard one on row-major C:
        # contiguous rows [rank*M/n, (rank+1)*M/n) (include/flashoverlap.h)
        want_seq = want if coll == "allreduce" else \
            full[rank * (M // world):(rank + 1) * (M // world)].to(torch.bfloat16)
        check(f"{coll}/{layout}/{groups}/sequential", seq, want_seq, bad)
        # host buffers (chunked H2D the GEMM waits on, per-band D2H, two staging
        # sets): back-to-back calls, each must equal the device result
        outs = [torch.full((plan.info["out_rows"], N), float("nan"), dtype=torch.bfloat16).pin_memory()
                for _ in range(3)]
        A_h = A.cpu().pin_memory()
        for o in outs:
            fo.run_host(ctx, plan, A_h, Bt, o)
        torch.cuda.synchronize()
        for i, o in enumerate(outs):
            check(f"{coll}/{layout}/{groups}/run_host[{i}]", o.cuda(), want, bad)
        if coll == "reducescatter":
            # RS follow-on (NEXT f2): AllGather + row exchange restores the
            # standard row order, i.e. the AllReduce result
            gathered = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
            fo.run_allgather(ctx, plan, out, gathered)
            torch.cuda.synchronize()
            check("reducescatter/allgather+rowexchange", gathered, full.to(torch.bfloat16), bad)
    # a context on torch's own communicator (fo_ctx_create_from_comm: borrowed,
    # the process group stays usable after the context is destroyed)
    tctx = fodist.context_from_process_group(local)
    A, Bt = exact_inputs(M, N, K, rank, world, 31)
    plan = fodist.make_plan(coll="allreduce", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=8,
                            swizzle=2, group_waves=[1, 2, 1], ar_layout="slot")
    full = A.float() @ Bt.float().t()
    dist.all_reduce(full)
    out = torch.full((M, N), float("nan"), dtype=torch.bfloat16, device="cuda")
    fo.run(tctx, plan, A, Bt, out)
    torch.cuda.synchronize()
    check("allreduce/torch-comm", out, full.to(torch.bfloat16), bad)
    tctx.close()
    probe = torch.ones(1, device="cuda")
    dist.all_reduce(probe)
    if probe.item() != world:
        bad.append("process group after borrowed-context destroy")
    # All-to-All (EP combine): imbalanced experts, random routing; the paper's
    # subtoken pools and the ROWBAND rows received straight into `out` (R41)
    rng = np.random.default_rng(7)
    Ms = [256 * int(rng.integers(2, 5)) for _ in range(world)]    # >= 2 tile-rows: two one-row waves
    rds = [np.random.default_rng(100 + s).integers(0, world, size=Ms[s]).astype(np.int32) for s in range(world)]
    Me = Ms[rank]
    A, Bt = exact_inputs(Me, N, K, rank, world, 23)
    C = (A.float() @ Bt.float().t()).to(torch.bfloat16)
    # plain A2A: rows with dst d go to rank d, source-major then row-major
    send = [C[torch.from_numpy(rds[rank] == d).cuda()] for d in range(world)]
    counts = [torch.tensor([s.shape[0]], device="cuda") for s in send]
    recv_counts = [torch.zeros(1, dtype=torch.int64, device="cuda") for _ in range(world)]
    dist.all_to_all(recv_counts, [c.to(torch.int64) for c in counts])
    recv = [torch.empty(int(c.item()), N, dtype=torch.bfloat16, device="cuda") for c in recv_counts]
    dist.all_to_all(recv, send)
    want = torch.cat(recv, 0)
    tiles = (Me // 256) * (N // 256)
    for layout in ("slot", "rowband"):
        S = 2 if layout == "slot" else N // 256
        T = -(-tiles // S)
        spec = dict(coll="alltoall", m=Me, n=N, k=K, tile_m=256, tile_n=256, workers=S,
                    swizzle=2 if layout == "slot" else 1, group_waves=[1, T - 1], row_dst=rds[rank],
                    ar_layout=layout)   # T >= 2 on every rank: the same P = 2
        plan = fodist.make_plan(**spec)
        out = torch.full((plan.info["out_rows"], N), float("nan"), dtype=torch.bfloat16, device="cuda")
        for _ in range(3):
            fo.run(ctx, plan, A, Bt, out)
        torch.cuda.synchronize()
        check(f"alltoall/{layout}", out, want, bad)
        seq = torch.full_like(out, float("nan"))
        fo.run_sequential(ctx, plan, A, Bt, seq)     # unsorted row_dst: one message per run of a destination
        torch.cuda.synchronize()
        check(f"alltoall/{layout}/sequential", seq, want, bad)
    ok = torch.tensor([0 if not bad else 1], device="cuda")
    dist.all_reduce(ok)
    ctx.close()
    dist.destroy_process_group()
    if rank == 0:
        print("multi-GPU parity:", "OK" if ok.item() == 0 else f"{ok.item()} rank(s) failed", flush=True)
    sys.exit(0 if ok.item() == 0 else 1)


if __name__ == "__main__":
    main()
