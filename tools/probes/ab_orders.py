"""A/B of two builds' default (swizzle 0) tile orders on several GEMM shapes
(dev probe): `python ab_orders.py <package root>`; device-time means of 20."""
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
    cases = [(4096, 4096, 14336, 74, -1), (4096, 4096, 14336, 64, 0), (8192, 8192, 1024, 64, 0),
             (8192, 8192, 4096, 74, 0), (4096, 4096, 1792, 64, 0), (4096, 16384, 16384, 74, 0),
             (2048, 8192, 8192, 74, 0), (16384, 16384, 4096, 74, 0)]
    fns = []
    for (M, N, K, S, ts) in cases:
        A, Bt = synthetic.float_inputs(M, N, K, seed=1, device="cuda")
        C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        p = fo.Plan(coll="allreduce", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, swizzle=0,
                    options={"tail_split": ts} if ts else None)
        gp = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, tile_order=p.export_order(),
                     options={"tail_split": ts} if ts else None)
        fns.append(((M, N, K, S), lambda gp=gp, A=A, Bt=Bt, C=C: fo.gemm_stage(gp, A, Bt, C)))
    for _, f in fns:
        f()
    torch.cuda.synchronize()
    ts_ = {k: [] for k, _ in fns}
    for _ in range(20):
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
    print(root, " ".join(f"{k[0]}x{k[1]}x{k[2]}/S{k[3]}: {sum(v) / len(v):.1f}" for k, v in ts_.items()), flush=True)


if __name__ == "__main__":
    main()
