"""Print tune_layer's candidates (prediction, GEMM time, measured) for one
cell on the emulated link (dev probe)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import torch  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402
from paper_2504_19519_b200 import tuner  # noqa: E402

M, N, K, n, coll = [int(x) for x in sys.argv[1:5]] + [sys.argv[5]]
torch.cuda.set_device(0)
ctx = fo.Context.emulated(0, 0, n, 770.0, 6.0, 16)
ctx.nccl_max_ctas = 16
ctx_u = fo.Context.emulated(0, 0, n, 770.0, 6.0, 32)
ctx_u.nccl_max_ctas = 0
ch = tuner.tune_layer(M, N, K, [ctx, ctx_u], coll, "none", device=0, iters=3, verify=4,
                      tile_shapes=[(256, 256), (128, 256)])
print("picked", ch.tile_m, ch.tile_n, ch.workers, ch.layout, ch.groups, ch.tail_split, "ctx", ch.ctx_index)
for c in ch.candidates[:30]:
    print(c)
