"""Orchestration overhead of fo_run at one rank (dev tool): the bench layer's
GEMM alone, fo_run_sequential, and fo_run with the last group triggered by
its counter vs issued in stream order (FO_OPT_LAST_GROUP_IN_ORDER), for a
few partitions and layouts.  Interleaved, L2 flushed, medians."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402
import synthetic  # noqa: E402


def main():
    torch.cuda.set_device(0)
    ctx = fo.Context.create(0, 0, 1, fo.unique_id())
    M, N, K = 4096, 4096, 14336
    A, Bt = synthetic.float_inputs(M, N, K, seed=1, device="cuda")
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    res = synthetic.normal_bf16((M, N), 1.0, 2, device="cuda")
    gam = synthetic.normal_bf16((N,), 1.0, 3, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    fns = {}
    gp = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=64, swizzle=1)
    fns["gemm alone"] = lambda: fo.gemm_stage(gp, A, Bt, out)
    for layout, groups, post in (("rowband", [4], "none"), ("rowband", [1, 3], "none"),
                                 ("rowband", [1, 1, 1, 1], "none"), ("slot", [1, 2, 1], "none"),
                                 ("rowband", [1, 1, 1, 1], "add_rmsnorm")):
        for lio in (0, 1):
            pl = fo.Plan(coll="allreduce", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=64, swizzle=1,
                         group_waves=groups, ar_layout=layout, post=post)
            pl.set_option("last_group_in_order", lio)
            args = (res, gam) if post != "none" else (None, None)
            fns[f"run {layout} {groups} {post} in_order={lio}"] = (lambda pl=pl, a=args: fo.run(ctx, pl, A, Bt, out, *a))
            if lio == 0:
                fns[f"seq {layout} {groups} {post}"] = (lambda pl=pl, a=args: fo.run_sequential(ctx, pl, A, Bt, out, *a))
    for f in fns.values():
        for _ in range(3):
            f()
    torch.cuda.synchronize()
    ts = {k: [] for k in fns}
    for _ in range(30):
        for k, f in fns.items():
            flush.zero_()
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            f()
            e.record()
            torch.cuda.synchronize()
            ts[k].append(s.elapsed_time(e) * 1e3)
    for k, v in ts.items():
        print(f"{k:55s} median {statistics.median(v):8.1f} us  p10 {sorted(v)[3]:8.1f}", flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
