"""GEMM time vs wave width S and order for one shape (dev probe; device-time
means of 20, stream pre-loaded, L2 flushed)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import torch  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402
import synthetic  # noqa: E402

M, N, K = [int(x) for x in sys.argv[1:4]]
torch.cuda.set_device(0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
A, Bt = synthetic.float_inputs(M, N, K, seed=1, device="cuda")
C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
variants = {}
for S in (64, 66, 74):
    for swz in (0, 1, 2, 4, 8):
        for ks in (-1, 0):
            p = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, swizzle=swz)
            p.set_option("k_snake", ks)
            variants[f"S{S} swz{swz} snake{ks}"] = (lambda p=p: fo.gemm_stage(p, A, Bt, C))
variants["cuBLAS"] = lambda: torch.matmul(A, Bt.t(), out=C)
for f in variants.values():
    f()
torch.cuda.synchronize()
ts = {k: [] for k in variants}
for _ in range(8):
    for k, f in variants.items():
        flush.zero_()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(200_000)
        s.record()
        f()
        e.record()
        torch.cuda.synchronize()
        ts[k].append(s.elapsed_time(e) * 1e3)
fl = 2.0 * M * N * K
for k, v in ts.items():
    m = sum(v) / len(v)
    print(f"{M}x{N}x{K} {k:22s} {m:9.1f} us {fl / m / 1e6:6.0f} TF/s", flush=True)
