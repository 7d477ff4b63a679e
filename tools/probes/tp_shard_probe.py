"""GEMM time of the TP-shard layers at the wave widths the N>1 tuner can pick
(S = 66 / 64 / 58 / 56 pairs, i.e. 16 / 20 / 32 / 36 SMs left to NCCL), with and
without the split tail; interleaved, L2 flushed, device-time medians."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402

torch.cuda.set_device(0)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for K in (7168, 3584, 1792):
    M = N = 4096
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    Bt = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
    C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    cfgs = [(74, -1), (66, 0), (66, -1), (64, 0), (58, 0), (58, -1), (56, 0), (56, -1)]
    plans = []
    for S, ts in cfgs:
        try:
            plans.append(fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, swizzle=0,
                                 options={"tail_split": ts} if ts else None))
        except Exception as e:
            plans.append(None)
    fns = [(lambda p=p: fo.gemm_stage(p, A, Bt, C)) if p else None for p in plans] + \
          [lambda: torch.matmul(A, Bt.t(), out=C)]
    live = [f for f in fns if f]
    for f in live:
        for _ in range(3):
            f()
    torch.cuda.synchronize()
    ts_ = {i: [] for i, f in enumerate(fns) if f}
    for _ in range(15):
        for i, f in enumerate(fns):
            if not f:
                continue
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(100_000)
            s.record()
            f()
            e.record()
            torch.cuda.synchronize()
            ts_[i].append(s.elapsed_time(e) * 1e3)
    med = {i: statistics.median(v) for i, v in ts_.items()}
    line = "  ".join(f"S{S}{'+ts' if t else ''} {med[i]:.1f}" for i, (S, t) in enumerate(cfgs) if i in med)
    print(f"4096x4096x{K}: {line}  cuBLAS {med[len(cfgs)]:.1f} us", flush=True)
