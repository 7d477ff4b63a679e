"""Epilogue write-pattern probe (dev tool): the same GEMM (same order, same
S) with the row-major epilogue vs the AR-slot, RS-subtile and A2A-pool
reorder epilogues, interleaved, device time (stream pre-loaded), medians."""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402
import synthetic  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="8192x8192x1024,4096x4096x1792,4096x4096x14336")
    ap.add_argument("--s", type=int, default=74)
    ap.add_argument("--iters", type=int, default=15)
    ap.add_argument("--reverse", action="store_true", help="time the variants in reverse order")
    args = ap.parse_args()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for sh in args.shapes.split(","):
        M, N, K = map(int, sh.split("x"))
        A, Bt = synthetic.float_inputs(M, N, K, seed=3, device="cuda")
        tiles = (M // 256) * (N // 256)
        S = min(args.s, tiles)
        T = -(-tiles // S)
        base = dict(m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, swizzle=0, group_waves=[1] * T)
        plans = {"slot": fo.Plan(coll="allreduce", ar_layout="slot", **base),
                 "rs n=1": fo.Plan(coll="reducescatter", **base),
                 "rs n=8": fo.Plan(coll="reducescatter", rank=0, world=8, **base)}
        kw = dict(coll="alltoall", row_dst=np.zeros(M, np.int32), **base)
        plans["a2a"] = fo.Plan(rank=0, world=1, peers=[kw], **kw)
        order = plans["slot"].export_order()
        plans["rowmajor"] = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, tile_order=order)
        bufs = {k: torch.empty(max(pl.info["send_elems"], M * N), dtype=torch.bfloat16, device="cuda")
                for k, pl in plans.items()}
        keys = list(plans)[::-1] if args.reverse else list(plans)
        fns = {k: (lambda pl=plans[k], b=bufs[k]: fo.gemm_stage(pl, A, Bt, b)) for k in keys}
        for f in fns.values():
            f()
        torch.cuda.synchronize()
        ts = {k: [] for k in fns}
        for _ in range(args.iters):
            for k, f in fns.items():
                flush.zero_()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda._sleep(200_000)
                s.record()
                f()
                e.record()
                torch.cuda.synchronize()
                ts[k].append(s.elapsed_time(e) * 1e3)
        ref = statistics.median(ts["rowmajor"])
        for k, v in ts.items():
            m = statistics.median(v)
            print(f"{sh:18s} S={S:3d} {k:9s} {m:8.2f} us  {100 * (m / ref - 1):+6.2f}% vs row-major", flush=True)


if __name__ == "__main__":
    main()
