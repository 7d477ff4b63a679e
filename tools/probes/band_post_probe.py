"""Band post beside the GEMM (dev probe): the fused add + RMSNorm of each row
band runs on the post stream while the persistent GEMM holds S CTA pairs; A/B
of the bulk-staged vs the register kernel, with the per-band spans from the
comm-stream timestamps (wait released -> band post done)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import torch  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402
import synthetic  # noqa: E402
from tools.predictor_check import timeit_pre  # noqa: E402


def main():
    torch.cuda.set_device(0)
    ctx = fo.Context.create(0, 0, 1, fo.unique_id())
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for (M, N, K) in [(4096, 4096, 3584), (4096, 4096, 14336), (8192, 8192, 1024)]:
        S = 64
        tiles = (M // 256) * (N // 256)
        T = -(-tiles // S)
        A, Bt = synthetic.float_inputs(M, N, K, seed=1, device="cuda")
        res = synthetic.normal_bf16((M, N), 1.0, 1, device="cuda")
        gam = synthetic.normal_bf16((N,), 1.0, 2, device="cuda")
        out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        gp = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, swizzle=1)
        g_us = timeit_pre(lambda: fo.gemm_stage(gp, A, Bt, out), flush)
        print(f"{M}x{N}x{K} S={S} T={T}: GEMM {g_us:.1f} us", flush=True)
        for G in ([T], [1] * T, [1, T - 2, 1] if T > 2 else [1, 1]):
            for bulk in (0, 1):
                plan = fo.Plan(coll="allreduce", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, swizzle=1,
                               group_waves=G, ar_layout="rowband", post="add_rmsnorm")
                plan.set_option("post_bulk", bulk)
                t = timeit_pre(lambda: fo.run(ctx, plan, A, Bt, out, res, gam), flush)
                seq = timeit_pre(lambda: fo.run_sequential(ctx, plan, A, Bt, out, res, gam), flush)
                ts = torch.zeros(2 * len(G), dtype=torch.int64, device="cuda")
                plan.set_debug(None, ts)
                fo.run(ctx, plan, A, Bt, out, res, gam)
                torch.cuda.synchronize()
                g = ts.cpu().tolist()
                spans = [(g[2 * j + 1] - g[2 * j]) / 1e3 for j in range(len(G))]
                rel = [(g[2 * j] - g[0]) / 1e3 for j in range(len(G))]
                print(f"  groups {str(G):22s} bulk={bulk}: fo_run {t:7.1f} us, sequential {seq:7.1f} us; band posts "
                      + ", ".join(f"[start +{r:.1f}: {sp:.1f} us]" for r, sp in zip(rel, spans)), flush=True)
                plan.close()
        del A, Bt, res, gam, out
        torch.cuda.empty_cache()
    ctx.close()


if __name__ == "__main__":
    main()
