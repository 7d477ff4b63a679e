"""Run the headline GEMM once with cuBLAS (torch.matmul) and once with our
tcgen05 kernel, a few times each, for ncu captures of both (dev tool).

    ncu --set full -k regex:'nvjet|gemm|fo_gemm' python tools/gemm_pair.py
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="4096x4096x14336")
    ap.add_argument("--workers", type=int, default=64)
    ap.add_argument("--iters", type=int, default=2)
    ap.add_argument("--wave", type=int, default=1)
    ap.add_argument("--no-cublas", action="store_true")
    ap.add_argument("--multicast", type=int, default=0)
    ap.add_argument("--tail-split", type=int, default=0)
    ap.add_argument("--tile", default="256x256", help="tile_m x tile_n")
    args = ap.parse_args()
    M, N, K = map(int, args.shape.split("x"))
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    plan = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=int(args.tile.split("x")[0]),
                   tile_n=int(args.tile.split("x")[1]), workers=args.workers, swizzle=0)
    plan.set_option("wave_sync", args.wave)
    plan.set_option("multicast", args.multicast)
    plan.set_option("tail_split", args.tail_split)
    for _ in range(args.iters):
        if not args.no_cublas:
            torch.matmul(A, B.t(), out=C)
        fo.gemm_stage(plan, A, B, C)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
