"""A/B of two builds of the GEMM (dev probe): `python ab_gemm.py <package root>`
imports paper_2504_19519_b200 from that root and prints device-time means
(stream pre-loaded, L2 flushed; the CUDA event clock ticks in ~2 us steps on
these boxes, so the MEAN of 40 samples is reported) for the bench plan and
one-wave / short-K shapes."""
import os
import sys

root = sys.argv[1]
sys.path.insert(0, root)
sys.path.insert(1, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import torch  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402
import synthetic  # noqa: E402


def main():
    torch.cuda.set_device(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    cases = [(4096, 4096, 14336, 74, -1), (1024, 4096, 4096, 64, 0), (1024, 4096, 14336, 64, 0),
             (4096, 4096, 1792, 64, 0), (8192, 8192, 1024, 64, 0), (2048, 4096, 4096, 64, 0)]
    fns = []
    for (M, N, K, S, ts) in cases:
        A, Bt = synthetic.float_inputs(M, N, K, seed=1, device="cuda")
        C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        p = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, swizzle=0,
                    options={"tail_split": ts} if ts else None)
        fns.append(((M, N, K, S, ts), lambda p=p, A=A, Bt=Bt, C=C: fo.gemm_stage(p, A, Bt, C)))
    for _, f in fns:
        for _ in range(3):
            f()
    torch.cuda.synchronize()
    ts_ = {k: [] for k, _ in fns}
    for _ in range(40):
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
    print(root, " ".join(f"{k[0]}x{k[1]}x{k[2]}/S{k[3]}: {sum(v) / len(v):.2f}" for k, v in ts_.items()), flush=True)


if __name__ == "__main__":
    main()
