"""DP + suffix-helper tail (FO_OPT_TAIL_SPLIT -3, R43) vs the plain
last wave, the f-slice split and cuBLAS on shapes whose last wave holds more
than half the workers (dev probe; interleaved, L2 flushed, medians)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import torch  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402
import synthetic  # noqa: E402


def timeit_many(fns, flush, iters=15):
    for f in fns:
        f()
    torch.cuda.synchronize()
    ts = [[] for _ in fns]
    for _ in range(iters):
        for i, f in enumerate(fns):
            flush.zero_()
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(200_000)
            s.record()
            f()
            e.record()
            torch.cuda.synchronize()
            ts[i].append(s.elapsed_time(e) * 1e3)
    return [sorted(t)[len(t) // 2] for t in ts]


def main():
    torch.cuda.set_device(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for (M, N, K) in [(1024, 4096, 14336), (1024, 4096, 4096), (2048, 4096, 4096), (1024, 8192, 8192),
                      (4096, 4096, 1792), (1024, 4096, 7168)]:
        A, Bt = synthetic.float_inputs(M, N, K, seed=1, device="cuda")
        C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        tiles = (M // 256) * (N // 256)
        variants = {}
        for S in (64, 74):
            for ts in (0, -1, -3):
                T = -(-tiles // S)
                R = tiles - (T - 1) * S
                if ts == -1 and not (2 * R <= S):
                    continue
                if ts == -3 and not (2 * R > S and R < S):
                    continue
                p = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, swizzle=0,
                            options={"tail_split": ts} if ts else None)
                variants[f"S{S}{'' if ts == 0 else ('+fslice' if ts == -1 else '+suffix')}"] = \
                    (lambda p=p: fo.gemm_stage(p, A, Bt, C))
        variants["cuBLAS"] = lambda: torch.matmul(A, Bt.t(), out=C)
        t = timeit_many(list(variants.values()), flush)
        fl = 2.0 * M * N * K
        print(f"{M}x{N}x{K} ({tiles} tiles): " + "  ".join(
            f"{k} {v:.1f} us ({fl / v / 1e6:.0f} TF/s)" for k, v in zip(variants, t)), flush=True)
        del A, Bt, C
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
