"""Per-wave tile-completion windows of the bench GEMM (dev probe): %globaltimer
at each execution position's signal (fo_gemm_stage_timed), for the bench plan
(S=74 + split tail) and S=64 (4 full waves), best span of 7 runs, L2 flushed.
Wave w's window is reported relative to the earliest signal of the run minus
one tile time (~ the kernel's first MMA)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402
import synthetic  # noqa: E402

M, N, K = 4096, 4096, 14336
A, Bt = synthetic.float_inputs(M, N, K, seed=1, device="cuda")
out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for S, ts_opt in ((74, -1), (74, 0), (64, 0)):
    plan = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S,
                   options={"tail_split": ts_opt} if ts_opt else None)
    tiles = plan.info["tiles"]
    ts = torch.zeros(tiles, dtype=torch.int64, device="cuda")
    best = None
    for _ in range(7):
        flush.zero_()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(200_000)
        s.record()
        fo.gemm_stage_timed(plan, A, Bt, out, ts)
        e.record()
        torch.cuda.synchronize()
        t = ts.cpu().numpy().astype(np.int64)
        if best is None or t.max() - t.min() < best[0].max() - best[0].min():
            best = (t, s.elapsed_time(e) * 1e3)
    t, ev = best
    T = -(-tiles // S)
    w0 = np.sort(t[:S])
    tile_us = None
    print(f"S={S} tail_split={ts_opt}: event time {ev:.1f} us, signal span {(t.max() - t.min()) / 1e3:.1f} us")
    base = t.min()
    prev_end = None
    for w in range(T):
        q = t[w * S:min(tiles, (w + 1) * S)]
        q = (q - base) / 1e3
        print(f"   wave {w}: {len(q):3d} tiles  first {q.min():7.1f}  median {np.median(q):7.1f}  last {q.max():7.1f} us"
              + (f"  (median - prev median {np.median(q) - prev_end:6.1f})" if prev_end is not None else ""))
        prev_end = np.median(q)
