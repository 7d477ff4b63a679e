"""Head-to-head GEMM timing of execution orders (swizzle panel heights) in one
process (dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402
from tools.gemm_probe import timeit  # noqa: E402

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for sh in sys.argv[1].split(","):
    M, N, K = map(int, sh.split("x"))
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    fl = 2.0 * M * N * K
    tiles = (M // 256) * (N // 256)
    S = -(-tiles // -(-tiles // 74))
    t = timeit(lambda: torch.matmul(A, B.t(), out=C), iters=10, flush=flush)
    res = [f"cublas {fl / t / 1e6:6.0f}"]
    for swz in (1, 0, 2, 4, 8, 16):
        plan = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, swizzle=swz)
        t = timeit(lambda: fo.gemm_stage(plan, A, B, C), iters=10, flush=flush)
        res.append(f"s{swz}:{fl / t / 1e6:6.0f}")
    print(sh, f"S={S}", " ".join(res), flush=True)
