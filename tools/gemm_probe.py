"""Quick GEMM timing probe (our tcgen05 kernel vs torch.matmul/cuBLAS) on one GPU.
Dev tool; prints one line per (shape, BN, S)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402


def timeit(fn, iters=20, warm=5, flush=None):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(iters):
        if flush is not None:
            flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        tot += s.elapsed_time(e)
    return tot / iters * 1e3  # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="4096x4096x14336,4096x4096x7168,4096x4096x3584,4096x4096x1792,8192x8192x1024")
    ap.add_argument("--bn", default="128,256")
    ap.add_argument("--s", default="148,144,132")
    ap.add_argument("--bm", default="128,256")
    ap.add_argument("--swizzle", type=int, default=0)
    ap.add_argument("--split", default="0")
    ap.add_argument("--wave", default="1", help="FO_OPT_WAVE_SYNC values to try")
    args = ap.parse_args()
    sms = fo.device_sm_count(0)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for sh in args.shapes.split(","):
        M, N, K = map(int, sh.split("x"))
        A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        B = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
        C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        fl = 2.0 * M * N * K
        t = timeit(lambda: torch.matmul(A, B.t(), out=C), flush=flush)
        print(f"{sh} cublas {t:8.1f} us {fl / t / 1e6:7.1f} TF", flush=True)
        ref = C.float().clone()
        for bm in map(int, args.bm.split(",")):
            for bn in map(int, args.bn.split(",")):
                for S in map(int, args.s.split(",")):
                  Sw = min(S, sms) // (bm // 128)
                  for split in map(int, args.split.split(",")):
                   for wv in map(int, args.wave.split(",")):
                    plan = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=bm, tile_n=bn, workers=Sw,
                                   swizzle=args.swizzle)
                    try:
                        plan.set_option("tail_split", split)
                        plan.set_option("wave_sync", wv)
                        t = timeit(lambda: fo.gemm_stage(plan, A, B, C), flush=flush)
                    except fo.FOError as e:
                        print(f"{sh} BM={bm} BN={bn} S={Sw} split={split}: {e}")
                        continue
                    err = (C.float() - ref).abs().max().item()
                    print(f"{sh} fo BM={bm} BN={bn} S={Sw} split={split} wave={wv} {t:8.1f} us {fl / t / 1e6:7.1f} TF  "
                          f"maxdiff {err:.3g}", flush=True)


if __name__ == "__main__":
    main()
