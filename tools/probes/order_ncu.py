"""DRAM bytes and time of the bench GEMM (S=74 + split tail) under several tile
orders (dev probe, run under ncu --metrics dram__bytes_read.sum,...)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2504_19519_b200 as fo  # noqa: E402
import synthetic  # noqa: E402
M, N, K = 4096, 4096, 14336
A, Bt = synthetic.float_inputs(M, N, K, seed=1, device="cuda")
C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
plans = []
for swz in (7, 8, 9, -1):
    plans.append(fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=74, swizzle=swz,
                         options={"tail_split": -1}))
for _ in range(2):
    for p in plans:
        fo.gemm_stage(p, A, Bt, C)
torch.cuda.synchronize()
