"""FO_OPT_L2_HINTS A/B (dev probe; needs the REVERTED hint build — the option no longer exists,
profiles/r02_l2hint_probe.txt): device time of the GEMM with the operand
loads' L2 policy off (0), next-wave panels evict_last (1), + the rest
evict_first (2); interleaved, stream pre-loaded, L2 flushed, means and
medians of 30.  `ncu` mode: one launch per mode for dram__bytes."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import torch  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402
import synthetic  # noqa: E402

CASES = [(4096, 4096, 14336, 74, -1), (4096, 4096, 14336, 64, 0), (8192, 8192, 8192, 74, -1),
         (4096, 4096, 7168, 64, 0), (8192, 8192, 1024, 74, 0), (16384, 16384, 4096, 74, -1),
         (16384, 8192, 8192, 74, -1), (4096, 16384, 16384, 74, -1), (16384, 4096, 4096, 74, -1)]


def main():
    ncu = len(sys.argv) > 1 and sys.argv[1] == "ncu"
    torch.cuda.set_device(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    fns = []
    for (M, N, K, S, ts) in CASES:
        A, Bt = synthetic.float_inputs(M, N, K, seed=1, device="cuda")
        C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        for mode in (0, 1, 2):
            opts = {"l2_hints": mode}
            if ts:
                opts["tail_split"] = ts
            p = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, swizzle=0, options=opts)
            fns.append(((M, N, K, S, mode), lambda p=p, A=A, Bt=Bt, C=C: fo.gemm_stage(p, A, Bt, C)))
    if ncu:
        for _, f in fns:
            flush.zero_()
            f()
        torch.cuda.synchronize()
        return
    for _, f in fns:
        for _ in range(3):
            f()
    torch.cuda.synchronize()
    ts_ = {k: [] for k, _ in fns}
    for _ in range(30):
        for k, f in fns:
            flush.zero_()
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(200_000)
            s.record()
            f()
            e.record()
            torch.cuda.synchronize()
            ts_[k].append(s.elapsed_time(e) * 1e3)
    for k, v in ts_.items():
        M, N, K, S, mode = k
        print(f"{M}x{N}x{K} S={S} l2_hints={mode}: mean {statistics.mean(v):7.2f} us  median {statistics.median(v):7.2f} us "
              f"({2 * M * N * K / statistics.mean(v) / 1e6:.0f} TF/s)", flush=True)


if __name__ == "__main__":
    main()
