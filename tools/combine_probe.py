"""MoE combine kernel (fo_combine_stage, R31) bandwidth: the token
rank's gather of k expert rows through the A2A map + weighted sum (+ residual).
Algorithmic bytes = tokens * N * 2 * (k + 1 [+ 1 residual]).

Both A2A layouts: the paper's (rows arrive as 512-byte subtokens scattered in
execution order) and ROWBAND (R41: whole rows in output order, identity map).
Timing as tools/post_probe.py: stream pre-loaded by a sleep kernel, L2
evicted by a 512 MiB read (clean lines), medians of 20."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1:   # A/B: import the package from another build's root
    sys.path.insert(0, sys.argv[1])

import json  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402
import synthetic  # noqa: E402


def timeit(fn, flush_fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        flush_fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(100_000)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    return sorted(ts)[len(ts) // 2]


def main():
    torch.cuda.set_device(0)
    peaks = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))
    hbm = peaks.get("hbm_gbs") or 6550.0
    buf = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    fbuf = buf.view(torch.float32)
    flush_fn = lambda: fbuf.amax()  # noqa: E731
    print(f"# HBM peak {hbm:.0f} GB/s (MEASURED_PEAKS.json)", flush=True)
    for tokens, N, k in ((4096, 4096, 2), (8192, 4096, 2), (16384, 4096, 2), (8192, 4096, 4), (8192, 7168, 8)):
        BM, BN = 256, 256
        rows = tokens * k                                  # one rank holding every slot's row
        rd = np.zeros(rows, np.int32)
        recv = synthetic.normal_bf16((rows, N), 1.0, 1, device="cuda")
        idx = torch.from_numpy(np.random.default_rng(0).permutation(rows).astype(np.int32).reshape(tokens, k)).cuda()
        w = torch.rand(tokens, k, device="cuda")
        res = synthetic.normal_bf16((tokens, N), 1.0, 2, device="cuda")
        out = torch.empty(tokens, N, dtype=torch.bfloat16, device="cuda")
        for layout in ("slot", "rowband"):
            spec = dict(coll="alltoall", m=rows, n=N, k=64, tile_m=BM, tile_n=BN, row_dst=rd, ar_layout=layout,
                        workers=16 if layout == "slot" else N // BN, swizzle=0 if layout == "slot" else 1)
            plan = fo.Plan(peers=[spec], **spec)
            for with_res in (False, True):
                args = (res,) if with_res else ()
                us = timeit(lambda: fo.combine_stage(plan, recv, out, idx, w, *args), flush_fn)
                byts = tokens * N * 2 * (k + 1 + (1 if with_res else 0))
                print(f"tokens={tokens} N={N} k={k} {layout:7s} residual={with_res!s:5s}: {us:7.1f} us, "
                      f"{byts / us / 1e3:5.0f} GB/s algorithmic ({byts / us / 1e3 / hbm:.2f} of peak)", flush=True)
        # achievable gather bandwidth at this size: torch.index_select of the same rows
        flat = idx.flatten().long()
        g = torch.empty(rows, N, dtype=torch.bfloat16, device="cuda")
        us = timeit(lambda: torch.index_select(recv, 0, flat, out=g), flush_fn)
        byts = 2 * rows * N * 2
        print(f"    torch.index_select of the same {rows} rows: {us:.1f} us, {byts / us / 1e3:.0f} GB/s "
              f"({byts / us / 1e3 / hbm:.2f})", flush=True)
        del recv, res, out, g
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
