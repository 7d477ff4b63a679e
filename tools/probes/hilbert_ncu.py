import sys, torch
sys.path.insert(0, "."); sys.path.insert(0, "tools/probes")
import paper_2504_19519_b200 as fo
import synthetic
from hilbert_probe import hilbert_order
M, N, K = 4096, 4096, 14336
A, Bt = synthetic.float_inputs(M, N, K, seed=1, device="cuda")
C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
p0 = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=74, swizzle=0, options={"tail_split": -1})
p1 = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=74, tile_order=hilbert_order(16, 16), options={"tail_split": -1})
for _ in range(2):
    fo.gemm_stage(p0, A, Bt, C); fo.gemm_stage(p1, A, Bt, C)
torch.cuda.synchronize()
