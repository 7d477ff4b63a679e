"""Calibration (dev probe): split-tail slice + fold time vs the slice count f.
4096x4096x14336 on S=62 pairs (4 full waves + 8 tail tiles): tail tiles in f =
2 or 4 K-slices; per tile, signal time - the later of its slices' workers'
previous (wave-3) signal, median over tiles and runs."""
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
S = 62
for f in (2, 4):
    plan = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, options={"tail_split": f})
    ts = torch.zeros(256, dtype=torch.int64, device="cuda")
    vals, tile_us = [], []
    for _ in range(7):
        flush.zero_()
        torch.cuda.synchronize()
        fo.gemm_stage_timed(plan, A, Bt, out, ts)
        torch.cuda.synchronize()
        t = ts.cpu().numpy().astype(np.int64) / 1e3
        prev = t[3 * S:4 * S]                     # wave-3 signal per worker
        tail = t[4 * S:]
        R = len(tail)
        start = np.array([prev[r * f:(r + 1) * f].max() for r in range(R)])
        vals.append(np.median(tail - start))
        tile_us.append(np.median(np.diff([np.median(t[w * S:(w + 1) * S]) for w in range(4)])))
    tt = float(np.median(tile_us))
    v = float(np.median(vals))
    print(f"f={f}: tile {tt:.1f} us, slice work {tt / f:.1f} us, signal - later slice start {v:.1f} us "
          f"-> overhead {v - tt / f:.1f} us")
