"""Text timeline of one overlapped run (the nsys-timeline substitute; nsys is
not installed): per-tile signal times of the persistent GEMM (%globaltimer in
the epilogue) and, on the comm stream, when each group's stream wait released
and when its collective + per-group post-reorder finished.  Also times fo_run
vs fo_run_sequential for the same plan."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402
import synthetic  # noqa: E402
from tools.gemm_probe import timeit  # noqa: E402


def one(ctx, coll, M, N, K, BN, S, groups, layout="slot", flush=None, wait_kernel=0):
    kw = dict(coll=coll, m=M, n=N, k=K, tile_m=256, tile_n=BN, workers=S, swizzle=1 if layout == "rowband" else 2,
              group_waves=groups, ar_layout=layout)
    if coll == "alltoall":
        kw["row_dst"] = np.zeros(M, np.int32)
        plan = fo.Plan(rank=0, world=1, peers=[kw], **kw)
    else:
        plan = fo.Plan(**kw)
    plan.set_option("wait_kernel", wait_kernel)
    A, Bt = synthetic.float_inputs(M, N, K, seed=1, device="cuda")
    out = torch.empty(plan.info["out_rows"], N, dtype=torch.bfloat16, device="cuda")
    t_ov = timeit(lambda: fo.run(ctx, plan, A, Bt, out), flush=flush)
    t_seq = timeit(lambda: fo.run_sequential(ctx, plan, A, Bt, out), flush=flush)
    tile_ts = torch.zeros(plan.info["tiles"], dtype=torch.int64, device="cuda")
    group_ts = torch.zeros(2 * len(groups), dtype=torch.int64, device="cuda")
    plan.set_debug(tile_ts, group_ts)
    for _ in range(3):
        fo.run(ctx, plan, A, Bt, out)
    torch.cuda.synchronize()
    t, g = tile_ts.cpu().numpy(), group_ts.cpu().numpy()
    t0 = t.min()
    print(f"\n{coll} {M}x{N}x{K} tile 256x{BN} S={S} groups={groups} layout={plan.info['ar_layout']} "
          f"trigger={'spin-kernel' if wait_kernel else 'stream-wait'}: "
          f"fo_run {t_ov:.1f} us, sequential {t_seq:.1f} us, speedup {t_seq / t_ov:.3f}")
    print(f"  GEMM: first tile signal 0.0 us, last tile signal {(t.max() - t0) / 1e3:.1f} us")
    for j in range(len(groups)):
        lo, hi, _, _ = plan.group(j)
        print(f"  group {j}: tiles [{lo:4d},{hi:4d}) last signal {(t[lo:hi].max() - t0) / 1e3:8.1f} us | "
              f"wait released {(g[2 * j] - t0) / 1e3:8.1f} us | collective+post done {(g[2 * j + 1] - t0) / 1e3:8.1f} us")


def main():
    ap = argparse.ArgumentParser()
    ap.parse_args()
    torch.cuda.set_device(0)
    ctx = fo.Context.create(0, 0, 1, fo.unique_id())
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for wk in (0, 1):
        one(ctx, "allreduce", 4096, 4096, 14336, 256, 64, [1, 1, 1, 1], "slot", flush, wk)
        one(ctx, "allreduce", 4096, 4096, 14336, 256, 64, [1, 2, 1], "rowband", flush, wk)
        one(ctx, "reducescatter", 8192, 8192, 1024, 256, 64, [2, 4, 6, 4], "auto", flush, wk)
        one(ctx, "alltoall", 1024, 4096, 14336, 128, 64, [1, 1], "auto", flush, wk)
    ctx.close()


if __name__ == "__main__":
    main()
