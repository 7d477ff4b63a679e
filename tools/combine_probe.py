"""MoE combine kernel (fo_combine_stage, R31) bandwidth: the token
rank's gather of k expert rows through the A2A map + weighted sum (+ residual).
Algorithmic bytes = tokens * N * 2 * (k + 1 [+ 1 residual])."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import json  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402
import synthetic  # noqa: E402


def main():
    torch.cuda.set_device(0)
    peaks = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))
    hbm = peaks.get("hbm_gbs") or peaks.get("hbm_copy_gbs") or 7700.0
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for tokens, N, k in ((4096, 4096, 2), (8192, 4096, 2), (16384, 4096, 2), (8192, 7168, 8)):
        BM = 256
        rows = tokens * k                                  # one rank holding every slot's row
        rd = np.zeros(rows, np.int32)
        spec = dict(coll="alltoall", m=rows, n=N, k=64, tile_m=BM, tile_n=256, workers=16, row_dst=rd)
        plan = fo.Plan(peers=[spec], **spec)
        recv = synthetic.normal_bf16((rows, N), 1.0, 1, device="cuda")
        idx = torch.from_numpy(np.random.default_rng(0).permutation(rows).astype(np.int32).reshape(tokens, k)).cuda()
        w = torch.rand(tokens, k, device="cuda")
        res = synthetic.normal_bf16((tokens, N), 1.0, 2, device="cuda")
        out = torch.empty(tokens, N, dtype=torch.bfloat16, device="cuda")
        for with_res in (False, True):
            args = (res,) if with_res else ()
            for _ in range(3):
                fo.combine_stage(plan, recv, out, idx, w, *args)
            ts = []
            for _ in range(20):
                flush.zero_()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                fo.combine_stage(plan, recv, out, idx, w, *args)
                e.record()
                torch.cuda.synchronize()
                ts.append(s.elapsed_time(e) * 1e3)
            us = sorted(ts)[10]
            byts = tokens * N * 2 * (k + 1 + (1 if with_res else 0))
            print(f"tokens={tokens} N={N} k={k} residual={with_res}: {us:.1f} us, {byts / us / 1e3:.0f} GB/s "
                  f"algorithmic ({byts / us / 1e3 / hbm:.2f} of {hbm:.0f} GB/s)", flush=True)
        # achievable gather bandwidth at this size: torch.index_select of the same rows
        flat = idx.flatten().long()
        g = torch.empty(rows, N, dtype=torch.bfloat16, device="cuda")
        ts = []
        for _ in range(20):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            torch.index_select(recv, 0, flat, out=g)
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e) * 1e3)
        us = sorted(ts)[10]
        byts = 2 * rows * N * 2
        print(f"    torch.index_select of the same {rows} rows: {us:.1f} us, {byts / us / 1e3:.0f} GB/s "
              f"({byts / us / 1e3 / hbm:.2f})", flush=True)


if __name__ == "__main__":
    main()
