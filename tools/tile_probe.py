"""Tile-shape probe (dev tool): for each GEMM shape, our kernel at every
supported 2-CTA / 1-CTA tile shape x wave width S x tail split, against
cuBLAS, timed interleaved (device time, stream pre-loaded, L2 flushed,
medians).  Decides which tile shapes the tuner should search.

    python tools/tile_probe.py [--shapes 1024x4096x4096,...] [--iters 9]
"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402
import synthetic  # noqa: E402



def widths(tiles, cg):
    """Candidate wave widths: one full wave of pairs/CTAs, and the widths that
    make every wave full with the fewest waves."""
    full = 74 if cg == 2 else 148
    out = {min(tiles, full)}
    for T in range(1, 9):
        S = -(-tiles // T)
        if S <= full:
            out.add(S)
    out = sorted(out, reverse=True)[:4]
    if cg == 2 and full not in out:
        out.append(full)          # stream-K candidates use every pair
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="1024x4096x4096,2048x4096x4096,4096x4096x4096,1024x8192x8192,"
                                        "4096x4096x1792,4096x4096x3584,8192x8192x2048")
    ap.add_argument("--iters", type=int, default=9)
    ap.add_argument("--tiles", default="256x256,256x128,128x256,128x128")
    args = ap.parse_args()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for sh in args.shapes.split(","):
        M, N, K = map(int, sh.split("x"))
        A, Bt = synthetic.float_inputs(M, N, K, seed=3, device="cuda")
        C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        fns = {"cublas": lambda: torch.matmul(A, Bt.t(), out=C)}
        for tm, tn in [tuple(map(int, t.split("x"))) for t in args.tiles.split(",")]:
            if M % tm or N % tn:
                continue
            tiles = (M // tm) * (N // tn)
            for S in widths(tiles, 2 if tm == 256 else 1):
                for ts in ((0, -1, -2) if tm == 256 and tn == 256 else (0, -1)):
                    pl = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=tm, tile_n=tn, workers=S, swizzle=0,
                                 options={"tail_split": ts})
                    fns[f"{tm}x{tn} S={S} ts={ts}"] = (lambda pl=pl: fo.gemm_stage(pl, A, Bt, C))
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
        med = {k: statistics.median(v) for k, v in ts.items()}
        cb = med.pop("cublas")
        ranked = sorted(med.items(), key=lambda kv: kv[1])
        tf = lambda us: 2.0 * M * N * K / (us * 1e-6) / 1e12  # noqa: E731
        print(f"{sh}: cublas {cb:.1f} us ({tf(cb):.0f} TF/s)", flush=True)
        for k, v in ranked[:6]:
            print(f"   {k:24s} {v:8.1f} us {tf(v):6.0f} TF/s  {cb / v:5.3f}x cublas", flush=True)
        best256 = min(v for k, v in med.items() if k.startswith("256x256"))
        print(f"   best 256x256: {best256:.1f} us ({cb / best256:.3f}x cublas)", flush=True)


if __name__ == "__main__":
    main()
