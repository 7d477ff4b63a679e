"""Per-rank cost of the RS / A2A layouts on one GPU (dev tool, R40/R41).

For the BASELINE configs whose exchange needs the other ranks (C3: RS at TP=8,
C4: A2A at EP=8) and the AR TP shards, one rank's side of the overlapped layer
is timed in both layouts, L2 flushed, round-robin medians:
  gemm      the plain GEMM (row-major C) in the plan's execution order
  epi       the GEMM with the layout's pre-communication epilogue
  post      the post-communication pass the layout needs after the collective
            (slot: the reorder kernel over the whole output; rowband: none —
            the collective lands the rows in the output)
The collective itself is the same bytes in both layouts.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402
import synthetic  # noqa: E402


def timeit_many(fns, iters=20, warm=3, flush=None):
    for _ in range(warm):
        for f in fns:
            f()
    torch.cuda.synchronize()
    ts = [[] for _ in fns]
    for _ in range(iters):
        for i, f in enumerate(fns):
            if flush is not None:
                flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(100_000)
            s.record()
            f()
            e.record()
            torch.cuda.synchronize()
            ts[i].append(s.elapsed_time(e) * 1e3)
    return [sorted(t)[len(t) // 2] for t in ts]


def case(name, coll, M, N, K, BM, BN, S, groups, world, rank, row_dst=None, peers=None):
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    A, Bt = synthetic.float_inputs(M, N, K, seed=synthetic.cell_seed(M, N, K), device="cuda")
    res = {}
    for layout in ("slot", "rowband"):
        kw = dict(coll=coll, m=M, n=N, k=K, tile_m=BM, tile_n=BN, workers=S, group_waves=groups,
                  ar_layout=layout, swizzle=0)
        if coll == "alltoall":
            specs = [dict(kw, row_dst=rd) for rd in peers]
            plan = fo.Plan(rank=rank, world=world, peers=specs, **specs[rank])
        else:
            plan = fo.Plan(rank=rank, world=world, **kw)
        gp = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=BM, tile_n=BN, workers=S, tile_order=plan.export_order())
        C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        send = torch.empty(max(1, plan.info["send_elems"]), dtype=torch.bfloat16, device="cuda")
        recv = torch.randn(max(1, plan.info["recv_elems"]), device="cuda").to(torch.bfloat16)
        out = torch.empty(plan.info["out_rows"], N, dtype=torch.bfloat16, device="cuda")
        fns = [lambda: fo.gemm_stage(gp, A, Bt, C), lambda: fo.gemm_stage(plan, A, Bt, send)]
        if layout == "slot":
            fns.append(lambda: fo.post_stage(plan, recv, out))
        t = timeit_many(fns, flush=flush)
        res[layout] = (t[0], t[1], t[2] if layout == "slot" else 0.0, plan.info["ar_layout"])
    for layout, (g, e, p, lay) in res.items():
        print(f"{name:38s} {layout:8s} (resolved {'rowband' if lay == 1 else 'slot':7s}) gemm {g:8.2f} us  "
              f"epi {e:8.2f} us ({100 * (e / g - 1):+5.1f}%)  post {p:6.2f} us  epi+post {e + p:8.2f} us", flush=True)


def main():
    torch.cuda.set_device(0)
    # C3: Llama-3-70B o_proj, RS at TP=8 (rank 0's GEMM; h = 32 rows per subtile)
    case("C3 8192x8192x1024 RS n=8 [2,4,6,4]", "reducescatter", 8192, 8192, 1024, 256, 256, 64, [2, 4, 6, 4], 8, 0)
    case("C3 8192x8192x1024 RS n=8 [1]*16", "reducescatter", 8192, 8192, 1024, 256, 256, 64, [1] * 16, 8, 0)
    # C4: Mixtral w2 expert, EP=8, balanced routing (rows sorted by source)
    rds = [synthetic.balanced_moe_row_dst(128, 8) for _ in range(8)]
    case("C4 1024x4096x14336 A2A n=8 [1,1]", "alltoall", 1024, 4096, 14336, 256, 128, 64, [1, 1], 8, 0,
         row_dst=rds[0], peers=rds)
    # AR TP shards
    case("C2c 4096x4096x1792 AR n=8 [1,1,2]", "allreduce", 4096, 4096, 1792, 256, 256, 64, [1, 1, 2], 8, 0)


if __name__ == "__main__":
    main()
