"""Tile order experiment (dev probe): the bench GEMM (4096x4096x14336, 256x256
pair tiles, 16x16 grid) at S=74 + split tail / S=64 in the R25 panel order vs a
Hilbert-curve order (consecutive positions stay spatially compact for any S,
so a 74-wide wave does not straddle panel boundaries).  Device-time means of
20, stream pre-loaded, L2 flushed."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import torch  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402
import synthetic  # noqa: E402


def hilbert_d2xy(n, d):
    x = y = 0
    s, t = 1, d
    while s < n:
        rx = 1 & (t // 2)
        ry = 1 & (t ^ rx)
        if ry == 0:
            if rx == 1:
                x, y = s - 1 - x, s - 1 - y
            x, y = y, x
        x += s * rx
        y += s * ry
        t //= 4
        s *= 2
    return x, y


def hilbert_order(Mt, Nt):
    n = 1
    while n < max(Mt, Nt):
        n *= 2
    out = []
    for d in range(n * n):
        x, y = hilbert_d2xy(n, d)
        if x < Mt and y < Nt:
            out.append(x * Nt + y)
    return out


def footprint(order, S, Nt):
    fps = []
    for w0 in range(0, len(order), S):
        ts = order[w0:w0 + S]
        fps.append(len({t // Nt for t in ts}) + len({t % Nt for t in ts}))
    return sum(fps)


def main():
    M, N, K = [int(x) for x in (sys.argv[1:4] or (4096, 4096, 14336))]
    torch.cuda.set_device(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    A, Bt = synthetic.float_inputs(M, N, K, seed=1, device="cuda")
    C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    Mt, Nt = M // 256, N // 256
    hil = hilbert_order(Mt, Nt)
    v = {}
    for S, ts in ((74, -1), (64, 0)):
        opts = {"tail_split": ts} if ts else None
        p0 = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, swizzle=0, options=opts)
        p1 = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, tile_order=hil, options=opts)
        print(f"S={S}: panel-order footprint (panels touched, summed over waves) "
              f"{footprint(list(p0.export_order()), S, Nt)}, Hilbert {footprint(hil, S, Nt)}", flush=True)
        v[f"S{S} R25"] = (lambda p=p0: fo.gemm_stage(p, A, Bt, C))
        v[f"S{S} Hilbert"] = (lambda p=p1: fo.gemm_stage(p, A, Bt, C))
    v["cuBLAS"] = lambda: torch.matmul(A, Bt.t(), out=C)
    for f in v.values():
        f()
    torch.cuda.synchronize()
    ts_ = {k: [] for k in v}
    for _ in range(20):
        for k, f in v.items():
            flush.zero_()
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(200_000)
            s.record()
            f()
            e.record()
            torch.cuda.synchronize()
            ts_[k].append(s.elapsed_time(e) * 1e3)
    fl = 2.0 * M * N * K
    for k, x in ts_.items():
        m = sum(x) / len(x)
        print(f"{M}x{N}x{K} {k:12s} {m:8.1f} us {fl / m / 1e6:6.0f} TF/s", flush=True)


if __name__ == "__main__":
    main()
