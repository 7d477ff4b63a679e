"""Loopback communicator speed (dev probe): W in-process ranks, each fo_run of
a K=64 AllReduce plan (GEMM negligible) of M x N bf16, device time per call."""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 2
torch.cuda.set_device(0)
grp = fo.LoopbackGroup(0, W)
ctxs = grp.contexts()
M = N = 4096
plans = [fo.Plan(coll="allreduce", m=M, n=N, k=64, tile_m=256, tile_n=256, workers=64, swizzle=1, group_waves=[4],
                 rank=r, world=W) for r in range(W)]
for p in plans:
    p.prepare()
A = [torch.zeros(M, 64, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
B = [torch.zeros(N, 64, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
out = [torch.empty(M, N, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
streams = [torch.cuda.Stream() for _ in range(W)]
pool = ThreadPoolExecutor(W)
res = {}


def one(r, iters):
    torch.cuda.set_device(0)
    with torch.cuda.stream(streams[r]):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(iters):
            fo.run(ctxs[r], plans[r], A[r], B[r], out[r], stream=streams[r])
        e.record()
    streams[r].synchronize()
    res[r] = s.elapsed_time(e) * 1e3 / iters


for iters in (2, 10):
    t0 = time.time()
    for f in [pool.submit(one, r, iters) for r in range(W)]:
        f.result()
    print(f"W={W} iters={iters}: per call {[round(res[r], 1) for r in range(W)]} us "
          f"({2 * M * N / (max(res.values()) * 1e-6) / 1e9:.0f} GB/s of {2 * M * N / 1e6:.0f} MB), wall {time.time() - t0:.3f} s",
          flush=True)
for c in ctxs:
    c.close()
grp.close()
