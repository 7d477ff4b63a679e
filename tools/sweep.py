"""configs[4] shape sweep at N=1 (the heatmap analogue):
M in {1k,2k,4k,8k,16k} x N=K in {4k,8k,16k}.  Per cell: our GEMM kernel
(CTA-pair 256x256, wave-quantisation-aware S) vs cuBLAS (torch.matmul), the
overlapped fo_run (AllReduce, world 1) vs fo_run_sequential, and the GEMM's
fraction of the measured bf16 peak.  Dev tool; prints a table."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402
import synthetic  # noqa: E402
from paper_2504_19519_b200 import tuner  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def interleaved(fns, flush, iters=10):
    import statistics

    for f in fns:
        f()
    torch.cuda.synchronize()
    ts = [[] for _ in fns]
    for _ in range(iters):
        for i, f in enumerate(fns):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(200_000)  # pre-load the stream: device time, host enqueue excluded
            s.record()
            f()
            e.record()
            torch.cuda.synchronize()
            ts[i].append(s.elapsed_time(e) * 1e3)
    return [statistics.median(t) for t in ts]


def main():
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"]
    torch.cuda.set_device(0)
    sms = fo.device_sm_count(0)
    ctx = fo.Context.create(0, 0, 1, fo.unique_id())
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    print(f"{'M':>6} {'N=K':>6} {'tiles':>5} {'S':>3} {'T':>3} {'cublas_TF':>9} {'fo_TF':>7} {'frac':>5} "
          f"{'fo_run_us':>9} {'seq_us':>8} {'speedup':>7} layout groups")
    for M in (1024, 2048, 4096, 8192, 16384):
        for NK in (4096, 8192, 16384):
            N = K = NK
            A, Bt = synthetic.float_inputs(M, N, K, seed=synthetic.cell_seed(M, N, K), device="cuda")
            C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
            fl = 2.0 * M * N * K
            ch = tuner.tune_layer(M, N, K, ctx, "allreduce", "none", tile_shapes=[(256, 256), (128, 256)])
            tiles = (M // ch.tile_m) * (N // ch.tile_n)
            S, T, groups = ch.workers, -(-tiles // ch.workers), ch.groups
            plan = fo.Plan(**ch.spec(M, N, K, "allreduce"))
            gplan = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=ch.tile_m, tile_n=ch.tile_n, workers=S,
                            tile_order=plan.export_order(), options=ch.spec(M, N, K, "allreduce").get("options"))
            # interleaved (one flushed run of each per round, medians) so clock /
            # power drift hits the four alike
            t_cb, t_fo, t_ov, t_sq = interleaved([lambda: torch.matmul(A, Bt.t(), out=C),
                                                  lambda: fo.gemm_stage(gplan, A, Bt, C),
                                                  lambda: fo.run(ctx, plan, A, Bt, C),
                                                  lambda: fo.run_sequential(ctx, plan, A, Bt, C)], flush)
            tf = fl / t_fo / 1e6
            print(f"{M:6d} {NK:6d} {tiles:5d} {S:3d} {T:3d} {fl / t_cb / 1e6:9.1f} {tf:7.1f} {tf / peak:5.2f} "
                  f"{t_ov:9.1f} {t_sq:8.1f} {t_sq / t_ov:7.3f} "
                  f"{('rowband' if plan.info['ar_layout'] == 1 else 'slot') + ('+ts' if ch.tail_split else ''):10s} "
                  f"{ch.tile_m}x{ch.tile_n} "
                  f"{list(groups)}", flush=True)
            del A, Bt, C
            torch.cuda.empty_cache()
    ctx.close()


if __name__ == "__main__":
    main()
