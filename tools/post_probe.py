"""Post-communication reorder kernel timing (dev tool): achieved HBM GB/s per map/op."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402
from tools.gemm_probe import timeit  # noqa: E402


def main():
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    cases = [
        ("AR slot 4096x4096 256x256 S64", dict(coll="allreduce", m=4096, n=4096, k=64, tile_m=256, tile_n=256,
                                                workers=64, swizzle=2, group_waves=[1, 2, 1], ar_layout="slot"), 1, 0),
        ("RS n=8 8192x8192 256x256 S64", dict(coll="reducescatter", m=8192, n=8192, k=64, tile_m=256, tile_n=256,
                                               workers=64, group_waves=[2, 4, 6, 4]), 8, 0),
        ("A2A n=8 1024x4096 256x256", None, 8, 0),
    ]
    for name, spec, world, rank in cases:
        if spec is None:
            rng = np.random.default_rng(0)
            specs = []
            for s in range(world):
                rd = np.sort(rng.integers(0, world, size=1024)).astype(np.int32)
                specs.append(dict(coll="alltoall", m=1024, n=4096, k=64, tile_m=256, tile_n=256, workers=32,
                                  group_waves=[1, 1], row_dst=rd))
            plan_args = [(dict(specs[rank], post=op), dict(rank=rank, world=world, peers=specs))
                         for op in ("none", "add", "add_rmsnorm")]
        else:
            plan_args = [(dict(spec, post=op), dict(rank=rank, world=world)) for op in ("none", "add", "add_rmsnorm")]
        for sp, kw in plan_args:
            plan = fo.Plan(**kw, **sp)
            rows, N = plan.info["out_rows"], plan.info["out_cols"]
            recv = torch.randn(plan.info["recv_elems"], device="cuda").to(torch.bfloat16)
            out = torch.empty(rows, N, dtype=torch.bfloat16, device="cuda")
            res = torch.randn(rows, N, device="cuda").to(torch.bfloat16)
            gam = torch.randn(N, device="cuda").to(torch.bfloat16)
            t = timeit(lambda: fo.post_stage(plan, recv, out, res, gam), iters=30, flush=flush)
            nb = 2 * rows * N * 2 + (rows * N * 2 if sp["post"] != "none" else 0)
            print(f"{name:32s} post={sp['post']:12s} {t:8.2f} us  {nb / t / 1e3:8.1f} GB/s  ({nb / 1e6:.1f} MB)",
                  flush=True)
            # achievable at this size: torch's own copy / add over the same bytes
            src = recv[:rows * N].view(rows, N)
            if sp["post"] == "none":
                tr = timeit(lambda: out.copy_(src), iters=30, flush=flush)
                ref = "torch copy_"
            else:
                tr = timeit(lambda: torch.add(src, res, out=out), iters=30, flush=flush)
                ref = "torch add"
            print(f"{'':32s} {ref:17s} {tr:8.2f} us  {nb / tr / 1e3:8.1f} GB/s  (same bytes, no reorder)", flush=True)


if __name__ == "__main__":
    main()
