"""GEMM plan-option A/B (dev tool): the same GEMM with option OPT = 0 and 1
(env AB_OPT, default k_snake), interleaved with cuBLAS, L2 flushed, device
time medians; one line per (shape, S, tail split)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402


def main():
    torch.cuda.set_device(0)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    cases = [(4096, 4096, 14336, 74, -1), (4096, 4096, 14336, 64, 0), (4096, 4096, 7168, 74, -1),
             (4096, 4096, 1792, 64, 0), (8192, 8192, 1024, 74, 0), (8192, 8192, 8192, 74, 0),
             (16384, 16384, 16384, 74, 0), (8192, 16384, 16384, 74, 0)]
    only = os.environ.get("KSNAKE_CASES")
    if only:
        cases = [cases[int(i)] for i in only.split(",")]
    for M, N, K, S, ts in cases:
        A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        Bt = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
        C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        plans = []
        opt = os.environ.get("AB_OPT", "k_snake")
        for v in (0, 1):
            p = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, swizzle=0,
                        options={"tail_split": ts, opt: v} if ts else {opt: v})
            plans.append(p)
        fns = [lambda p=p: fo.gemm_stage(p, A, Bt, C) for p in plans] + [lambda: torch.matmul(A, Bt.t(), out=C)]
        for f in fns:
            for _ in range(3):
                f()
        torch.cuda.synchronize()
        ts_ = [[] for _ in fns]
        for _ in range(15):
            for i, f in enumerate(fns):
                flush.zero_()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda._sleep(100_000)
                s.record()
                f()
                e.record()
                torch.cuda.synchronize()
                ts_[i].append(s.elapsed_time(e) * 1e3)
        med = [statistics.median(v) for v in ts_]
        fl = 2.0 * M * N * K
        print(f"{M}x{N}x{K} S={S} ts={ts}: {opt}=0 {med[0]:8.2f} us ({fl / med[0] / 1e6:6.0f} TF/s)  "
              f"{opt}=1 {med[1]:8.2f} us ({fl / med[1] / 1e6:6.0f} TF/s)  cuBLAS {med[2]:8.2f} us  "
              f"ratio 1/0 {med[1] / med[0]:.4f}", flush=True)


if __name__ == "__main__":
    main()
