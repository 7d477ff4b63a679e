import sys, torch
sys.path.insert(0, ".")
import paper_2504_19519_b200 as fo
import synthetic
M, N, K = 1024, 4096, 4096
A, Bt = synthetic.float_inputs(M, N, K, seed=1, device="cuda")
C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
p = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=64, swizzle=0)
for _ in range(3):
    fo.gemm_stage(p, A, Bt, C)
    torch.matmul(A, Bt.t(), out=C)
torch.cuda.synchronize()
