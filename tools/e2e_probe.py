"""End-to-end fo_run_host at the bench shape (host A and out, resident Bt):
whole-buffer staging vs the pipelined staging (FO_OPT_HOST_PIPELINE) —
chunked H2D the GEMM waits on, per-group D2H."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402
import synthetic  # noqa: E402


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="64:1x4:8:rowband;64:1x4:16:rowband;32:1x8:8:rowband;32:1x8:16:rowband;"
                    "16:1x16:16:rowband;64:1,3:8:rowband;64:1,1,2:8:slot",
                    help="';'-separated S:groups:chunks:layout entries; groups '1x4' = [1]*4")
    ap.add_argument("--pipes", default="0,3")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    ctx = fo.Context.create(0, 0, 1, fo.unique_id())
    M, N, K = 4096, 4096, 14336
    A, Bt = synthetic.float_inputs(M, N, K, seed=1)
    A = A.pin_memory()
    Bt = Bt.cuda()
    out = torch.empty(M, N, dtype=torch.bfloat16).pin_memory()
    h2d = M * K * 2 / 1e9
    for cfg in args.configs.split(";"):
        S, g, chunks, layout = cfg.split(":")
        S, chunks = int(S), int(chunks)
        groups = [int(g.split("x")[0])] * int(g.split("x")[1]) if "x" in g else [int(x) for x in g.split(",")]
        plan = fo.Plan(coll="allreduce", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, swizzle=1,
                       group_waves=groups, ar_layout=layout)
        plan.set_option("host_chunks", chunks)
        for pipe in map(int, args.pipes.split(",")):
            plan.set_option("host_pipeline", pipe)
            for _ in range(3):
                fo.run_host(ctx, plan, A, Bt, out)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ts = []
            for _ in range(10):
                s.record()
                fo.run_host(ctx, plan, A, Bt, out)
                e.record()
                torch.cuda.synchronize()
                ts.append(s.elapsed_time(e) * 1e3)
            ts.sort()
            print(f"S={S:3d} {layout:8s} groups={groups} chunks={chunks} pipeline={pipe}: e2e median {ts[5]:.1f} us "
                  f"(min {ts[0]:.1f}); H2D of A alone at 55 GB/s would be {h2d / 55e-6:.0f} us", flush=True)
    # the copies alone, and H2D concurrent with D2H
    o_d = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    side = torch.cuda.Stream()
    dA0 = torch.empty(M, K, dtype=torch.bfloat16, device="cuda")
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        dA0.copy_(A, non_blocking=True)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(3):
                out.copy_(o_d, non_blocking=True)
    torch.cuda.current_stream().wait_stream(side)
    e.record()
    torch.cuda.synchronize()
    print(f"H2D of A with 3x D2H of out beside it: {s.elapsed_time(e) * 1e3 / 5:.1f} us per A")
    t0 = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        out.copy_(o_d, non_blocking=True)
    e.record()
    torch.cuda.synchronize()
    print(f"D2H of out alone: {s.elapsed_time(e) * 1e3 / 5:.1f} us")
    # the copy alone
    dA = torch.empty(M, K, dtype=torch.bfloat16, device="cuda")
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        dA.copy_(A, non_blocking=True)
    e.record()
    torch.cuda.synchronize()
    print(f"H2D of A alone: {s.elapsed_time(e) * 1e3 / 5:.1f} us ({h2d / (s.elapsed_time(e) / 5e3):.1f} GB/s)")
    ctx.close()


if __name__ == "__main__":
    main()
