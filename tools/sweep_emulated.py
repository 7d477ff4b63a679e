"""configs[4] shape sweep at n = 2/4/8 on the EMULATED link (R42; one GPU,
rank 0 of an emulated TP group whose collectives last latency + bus bytes /
link bandwidth — a timing model, not NVLink): M in {1k,2k,4k,8k,16k} x
N = K in {4k,8k,16k} (per-rank GEMM sizes, R21) x {AllReduce,
ReduceScatter}.  Per cell: the tuned overlapped layer (tune_layer: tile shape,
S, layout, tail split, partition, in-situ curve, measured verification) vs the
sequential GEMM (all 74 pairs, split tail) -> one collective, and the layer
roofline max(GEMM at the measured peak, collective on the link model).  The
north_star asks the overlapped layer to beat the sequential one on every
shape; this checks the schedule against that bar under the link model.
Dev tool; prints one line per cell and a summary.

    python tools/sweep_emulated.py [--ms 1024,2048,...] [--nk 4096,...] [--n 2,4,8] [--colls allreduce,reducescatter] [--tiles 256x256,128x256]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402
import synthetic  # noqa: E402
from paper_2504_19519_b200 import tuner  # noqa: E402
from tools.sweep import interleaved  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ms", default="1024,2048,4096,8192,16384")
    ap.add_argument("--nk", default="4096,8192,16384")
    ap.add_argument("--n", default="2,4,8")
    ap.add_argument("--colls", default="allreduce,reducescatter")
    ap.add_argument("--gbps", type=float, default=770.0)
    ap.add_argument("--lat", type=float, default=6.0)
    ap.add_argument("--tiles", default="256x256,128x256", help="tile shapes the tuner searches")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    sms = fo.device_sm_count(0)
    print(f"# EMULATED link {args.gbps} GB/s per direction, {args.lat} us latency, 16 CTAs per call (R42); "
          f"GEMM peak {peak} TF/s (MEASURED_PEAKS.json)", flush=True)
    shapes = [tuple(int(v) for v in t.split("x")) for t in args.tiles.split(",")]
    wins, ties, cells = 0, 0, 0
    fracs = []
    for n in [int(x) for x in args.n.split(",")]:
        ctx = fo.Context.emulated(0, 0, n, args.gbps, args.lat, 16)
        ctx.nccl_max_ctas = 16
        ctx_u = fo.Context.emulated(0, 0, n, args.gbps, args.lat, 32)   # "uncapped": NCCL's default CTAs
        ctx_u.nccl_max_ctas = 0
        ctxs = [ctx, ctx_u]
        for coll in args.colls.split(","):
            for nk in [int(x) for x in args.nk.split(",")]:
                for M in [int(x) for x in args.ms.split(",")]:
                    N = K = nk
                    A, Bt = synthetic.float_inputs(M, N, K, seed=synthetic.cell_seed(M, N, K), device="cuda")
                    ch = tuner.tune_layer(M, N, K, ctxs, coll, "none", device=0, iters=3, verify=4,
                                          tile_shapes=shapes)
                    plan = fo.Plan(rank=0, world=n, **ch.spec(M, N, K, coll))
                    out = torch.empty(plan.info["out_rows"], N, dtype=torch.bfloat16, device="cuda")
                    tiles = (M // 256) * (N // 256)
                    S_seq = min(sms // 2, tiles)
                    T_seq = -(-tiles // S_seq)
                    R = tiles - (T_seq - 1) * S_seq
                    seq = fo.Plan(rank=0, world=n, coll=coll, m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S_seq,
                                  swizzle=0, group_waves=[T_seq], ar_layout="auto",
                                  options={"tail_split": -1} if 0 < R and 2 * R <= S_seq else None)
                    t_ov, t_seq = interleaved([lambda: fo.run(ctxs[ch.ctx_index], plan, A, Bt, out),
                                               lambda: fo.run_sequential(ctx_u, seq, A, Bt, out)], flush, iters=5)
                    fac = 2.0 * (n - 1) / n if coll == "allreduce" else (n - 1) / n
                    roof = max(2.0 * M * N * K / (peak * 1e6), args.lat + fac * M * N * 2 / (args.gbps * 1e3))
                    cells += 1
                    wins += t_ov < 0.99 * t_seq
                    ties += 0.99 * t_seq <= t_ov <= 1.01 * t_seq
                    fracs.append(roof / t_ov)
                    print(f"{coll:13s} n={n} {M:5d}x{N:5d}x{K:5d}: overlapped {t_ov:9.1f} us ({ch.tile_m}x{ch.tile_n} "
                          f"S={ch.workers} {ch.layout} groups {ch.groups} ts={ch.tail_split} ctx{ch.ctx_index}), sequential {t_seq:9.1f} us, "
                          f"speedup {t_seq / t_ov:.3f}, roofline {roof:8.1f} us = {roof / t_ov:.2f}", flush=True)
                    del A, Bt, out
                    torch.cuda.empty_cache()
        ctx.close()
        ctx_u.close()
    fracs.sort()
    print(f"# {cells} cells: overlapped faster than sequential (by > 1%) in {wins}, within 1% in {ties}, slower in "
          f"{cells - wins - ties}; fraction of the layer roofline: "
          f"median {fracs[len(fracs) // 2]:.2f}, min {fracs[0]:.2f}, max {fracs[-1]:.2f}", flush=True)


if __name__ == "__main__":
    main()
