"""A/B of a GEMM plan option (FO_OPT_WAVE_SYNC, FO_OPT_MULTICAST, FO_OPT_DIST_FOLD, ...; dev tool): the two plans (and cuBLAS)
run interleaved, L2 flushed before each, so clock / power drift hits all
alike; medians."""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="4096x4096x14336,4096x16384x16384,8192x16384x16384,16384x16384x16384")
    ap.add_argument("--s", default="64,74")
    ap.add_argument("--iters", type=int, default=15)
    ap.add_argument("--opt", default="wave_sync")
    ap.add_argument("--vals", default="0,1")
    ap.add_argument("--base", default="", help="options set on every plan, e.g. tail_split=-1")
    args = ap.parse_args()
    base = {kv.split("=")[0]: int(kv.split("=")[1]) for kv in args.base.split(",") if kv}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for sh in args.shapes.split(","):
        M, N, K = map(int, sh.split("x"))
        A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        B = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
        C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        fns = {"cublas": lambda: torch.matmul(A, B.t(), out=C)}
        for S in map(int, args.s.split(",")):
            for wv in map(int, args.vals.split(",")):
                if args.opt == "swizzle":
                    pl = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, swizzle=wv)
                else:
                    pl = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, swizzle=0,
                                 options=base)
                    pl.set_option(args.opt, wv)
                fns[f"S={S} {args.opt}={wv}"] = (lambda pl=pl: fo.gemm_stage(pl, A, B, C))
        for f in fns.values():
            f()
        torch.cuda.synchronize()
        ts = {k: [] for k in fns}
        for _ in range(args.iters):
            for k, f in fns.items():
                flush.zero_()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda._sleep(200_000)  # pre-load: device time only
                s.record()
                f()
                e.record()
                torch.cuda.synchronize()
                ts[k].append(s.elapsed_time(e) * 1e3)
        fl = 2.0 * M * N * K
        for k, v in ts.items():
            med = statistics.median(v)
            print(f"{sh:20s} {k:18s} median {med:9.1f} us {fl / med / 1e6:7.1f} TF", flush=True)
        del A, B, C


if __name__ == "__main__":
    main()
