"""Weight-gradient GEMM dW = dY^T X with dY [tokens, out], X [tokens, in] used
in place (M-/N-major operands) vs cuBLAS on the same layout (dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402
from tools.gemm_probe import timeit  # noqa: E402

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for T, OUT, IN in [(8192, 4096, 14336), (8192, 14336, 4096), (16384, 4096, 4096), (4096, 8192, 8192)]:
    dY = torch.randn(T, OUT, device="cuda").to(torch.bfloat16)
    X = torch.randn(T, IN, device="cuda").to(torch.bfloat16)
    C = torch.empty(OUT, IN, dtype=torch.bfloat16, device="cuda")
    fl = 2.0 * OUT * IN * T
    t_cb = timeit(lambda: torch.matmul(dY.t(), X, out=C), iters=10, flush=flush)
    ref = C.float().clone()
    tiles = (OUT // 256) * (IN // 256)
    S = -(-tiles // -(-tiles // 74))
    plan = fo.Plan(coll="nocomm", m=OUT, n=IN, k=T, tile_m=256, tile_n=256, workers=S, swizzle=0,
                   a_mn_major=1, b_mn_major=1)
    t = timeit(lambda: fo.gemm_stage(plan, dY, X, C), iters=10, flush=flush)
    err = ((C.float() - ref).abs().max() / ref.abs().max()).item()
    print(f"dW {OUT}x{IN} tokens={T}: cublas {fl / t_cb / 1e6:7.1f} TF  fo(MN-major) {fl / t / 1e6:7.1f} TF  "
          f"rel diff {err:.2e}", flush=True)
