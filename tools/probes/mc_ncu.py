"""Plain pairs vs TMA-multicast clusters (FO_OPT_MULTICAST) at S=64 (dev probe,
run under ncu): `python tools/probes/mc_ncu.py M N K [swizzle]` launches the
plain GEMM then the multicast one, 3 times each, then cuBLAS 3 times."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2504_19519_b200 as fo  # noqa: E402
import synthetic  # noqa: E402

M, N, K = (int(v) for v in sys.argv[1:4])
swz = int(sys.argv[4]) if len(sys.argv) > 4 else 0
A, Bt = synthetic.float_inputs(M, N, K, seed=1, device="cuda")
C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
plans = [fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=64, swizzle=swz,
                 options={"multicast": mc}) for mc in (0, 1)]
for p in plans:
    for _ in range(3):
        fo.gemm_stage(p, A, Bt, C)
for _ in range(3):
    torch.matmul(A, Bt.t(), out=C)
torch.cuda.synchronize()
