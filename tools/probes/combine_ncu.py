"""One MoE combine launch for ncu (dev probe): 8192 tokens x 4096, top-2,
residual, the A2A ROWBAND receive layout (the async-copy kernel, R31b)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402
import synthetic  # noqa: E402

tokens, N, k, BM, BN = 8192, 4096, 2, 256, 256
rows = tokens * k
spec = dict(coll="alltoall", m=rows, n=N, k=64, tile_m=BM, tile_n=BN, row_dst=np.zeros(rows, np.int32),
            ar_layout="rowband", workers=N // BN, swizzle=1)
plan = fo.Plan(peers=[spec], **spec)
recv = synthetic.normal_bf16((rows, N), 1.0, 1, device="cuda")
idx = torch.from_numpy(np.random.default_rng(0).permutation(rows).astype(np.int32).reshape(tokens, k)).cuda()
w = torch.rand(tokens, k, device="cuda")
res = synthetic.normal_bf16((tokens, N), 1.0, 2, device="cuda")
out = torch.empty(tokens, N, dtype=torch.bfloat16, device="cuda")
for _ in range(3):
    fo.combine_stage(plan, recv, out, idx, w, res)
torch.cuda.synchronize()
