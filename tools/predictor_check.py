"""Alg. 1 predictor validation on one B200 (NEXT f1; the paper's E2 / fig:prediction
analogue: mean prediction error 3.41% / 3.44%, searched
partition >99% of the optimum).

At one rank the collective moves no bytes, so each group's comm-stream work is
the fused residual-add + RMSNorm of its row band (ROWBAND layout), whose cost
is measured offline and folded into the curve (tuner.effective_curve, DESIGN.md
R28).  For every candidate partition (all 2^(T-1) for T <= 8, a seeded sample
otherwise) the predicted latency is compared with the measured fo_run latency;
the predictive search's pick is compared with the measured optimum."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402
import synthetic  # noqa: E402
from paper_2504_19519_b200 import tuner  # noqa: E402
from tools.gemm_probe import timeit  # noqa: E402


def candidates(T, limit, seed):
    allc = []
    for mask in range(1 << (T - 1)):
        part, run = [], 0
        for w in range(T):
            run += 1
            if w == T - 1 or (mask >> w) & 1:
                part.append(run)
                run = 0
        allc.append(part)
    if len(allc) <= limit:
        return allc
    rng = np.random.default_rng(seed)
    pick = rng.choice(len(allc), size=limit, replace=False)
    return [allc[i] for i in sorted(pick)] + [[1] * T, [T]]


MODE = sys.argv[1] if len(sys.argv) > 1 else "standalone"   # "standalone" | "insitu" | "emulate" (see notes)
# note: "insitu" divides each group's [wait released, post done] span by its
# bytes; the span includes queueing behind earlier groups' posts, so it
# overestimates the cost — kept only as a diagnostic


def main():
    torch.cuda.set_device(0)
    ctx = fo.Context.create(0, 0, 1, fo.unique_id())
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    errs, ratios, ierrs, iratios = [], [], [], []
    for (M, N, K) in [(4096, 4096, 14336), (4096, 4096, 3584), (4096, 4096, 1792), (8192, 4096, 1024),
                      (8192, 8192, 1024)]:
        S = 64
        tiles = (M // 256) * (N // 256)
        T = -(-tiles // S)
        A, Bt = synthetic.float_inputs(M, N, K, seed=synthetic.cell_seed(M, N, K), device="cuda")
        res = synthetic.normal_bf16((M, N), 1.0, 1, device="cuda")
        gam = synthetic.normal_bf16((N,), 1.0, 2, device="cuda")
        out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        out2 = torch.empty_like(out)
        gplan = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, swizzle=1)
        dur = timeit_pre(lambda: fo.gemm_stage(gplan, A, Bt, out), flush, iters=10)
        probe = fo.Plan(coll="allreduce", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, swizzle=1,
                        ar_layout="rowband", post="add_rmsnorm")
        norm_us = timeit_pre(lambda: fo.post_stage(probe, out, out2, res, gam), flush, iters=10)
        # in-situ offline stage (PAPER.md:498 (3), resource contention): the
        # comm-stream work of a group measured inside an overlapped run, on the
        # SMs the GEMM leaves free (group timestamps of the groups that overlap it)
        insitu = fo.Plan(coll="allreduce", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, swizzle=1,
                         group_waves=[1] * T, ar_layout="rowband", post="add_rmsnorm")
        gts = torch.zeros(2 * T, dtype=torch.int64, device="cuda")
        insitu.set_debug(None, gts)
        costs = []
        for _ in range(3):
            fo.run(ctx, insitu, A, Bt, out, res, gam)
            torch.cuda.synchronize()
            g = gts.cpu().numpy()
            costs += [(g[2 * j + 1] - g[2 * j]) / 1e3 for j in range(T - 1)]
        band_bytes = (M // T) * N * 2
        per_byte = statistics.median(costs) / band_bytes
        curve = tuner.effective_curve(ctx.sample_curve("allreduce", [1 << s for s in range(18, 28)], iters=3),
                                      per_byte if MODE == "insitu" else norm_us / (M * N * 2))
        # R42: group 0's band post measured beside the GEMM (groups (g, T-g))
        icurve = tuner.insitu_curve(ctx, dict(coll="allreduce", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S,
                                              swizzle=1, ar_layout="rowband", post="add_rmsnorm"),
                                    A, Bt, out, T, S, 256 * 256 * 2, curve, run_args=(res, gam))
        rows = []
        for G in candidates(T, 24, M + K):
            plan = fo.Plan(coll="allreduce", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, swizzle=1,
                           group_waves=G, ar_layout="rowband", post="add_rmsnorm")
            pred = fo.tune_predict(G, dur, tiles, S, 256 * 256 * 2, curve)
            ipred = tuner.predict_insitu(G, dur, tiles, S, 256 * 256 * 2, icurve, curve)
            meas = timeit_pre(lambda: fo.run(ctx, plan, A, Bt, out, res, gam), flush)
            rows.append((G, pred, meas, ipred))
            errs.append(abs(meas - pred) / meas)
            ierrs.append(abs(meas - ipred) / meas)
        ipick = min(rows, key=lambda r: r[3])[0]   # argmin of the in-situ prediction over the candidates
        iplan = fo.Plan(coll="allreduce", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, swizzle=1,
                        group_waves=list(ipick), ar_layout="rowband", post="add_rmsnorm")
        ipick_meas = timeit_pre(lambda: fo.run(ctx, iplan, A, Bt, out, res, gam), flush)
        best_meas = min(r[2] for r in rows)
        pick, pick_pred = fo.tune_search(dur, tiles, S, 256 * 256 * 2, curve)
        pplan = fo.Plan(coll="allreduce", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, swizzle=1,
                        group_waves=list(pick), ar_layout="rowband", post="add_rmsnorm")
        pick_meas = timeit_pre(lambda: fo.run(ctx, pplan, A, Bt, out, res, gam), flush)
        ratios.append(best_meas / pick_meas)
        iratios.append(best_meas / ipick_meas)
        one = [r for r in rows if r[0] == [1] * T]
        print(f"[{MODE}] {M}x{N}x{K} T={T} gemm {dur:.1f} us, norm pass {norm_us:.1f} us standalone / "
              f"{per_byte * M * N * 2:.1f} us in situ, {len(rows)} partitions: "
              f"mean |err| {100 * statistics.mean(abs(m - p) / m for _, p, m, _ in rows):.2f}%, "
              f"search picks {list(pick)} -> {pick_meas:.1f} us vs measured optimum {best_meas:.1f} us "
              f"({100 * best_meas / pick_meas:.1f}%)"
              + (f"; one-wave groups {one[0][2]:.1f} us" if one else "")
              + f"; in-situ curve: error mean {100 * statistics.mean(ierrs[-len(rows):]):.2f}%, picks {list(ipick)} -> "
              f"{ipick_meas:.1f} us ({100 * best_meas / ipick_meas:.1f}%)", flush=True)
        del A, Bt, res, out, out2
        torch.cuda.empty_cache()
    e = sorted(errs)
    print(f"[{MODE}] ALL: {len(errs)} (shape, partition) cases, prediction error mean {100 * statistics.mean(e):.2f}%, "
          f"median {100 * e[len(e) // 2]:.2f}%, p90 {100 * e[int(0.9 * len(e))]:.2f}%, max {100 * e[-1]:.2f}%; "
          f"searched / optimum: min {100 * min(ratios):.1f}%, mean {100 * statistics.mean(ratios):.1f}%")
    e = sorted(ierrs)
    print(f"[{MODE}] ALL with the in-situ curve (R42): prediction error mean {100 * statistics.mean(e):.2f}%, "
          f"median {100 * e[len(e) // 2]:.2f}%, p90 {100 * e[int(0.9 * len(e))]:.2f}%, max {100 * e[-1]:.2f}%; "
          f"searched / optimum: min {100 * min(iratios):.1f}%, mean {100 * statistics.mean(iratios):.1f}%")
    ctx.close()


def timeit_pre(fn, flush, iters=8, warm=2):
    """Device time of fn on a stream pre-loaded by a sleep kernel (host launch
    cost outside the events), L2 flushed, median."""
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        flush.zero_()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(200_000)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    return sorted(ts)[len(ts) // 2]


def main_emulate(link_gbps=770.0, latency_us=6.0, ctas=16):
    """Emulated NVLink (fo_ctx_create_emulated; timing only): the TP shards of
    BASELINE configs[1..2] at their real world sizes, each collective taking
    latency + bus bytes / link bandwidth on 16 CTAs of the SMs the GEMM
    leaves free.  Per shape: the offline stages (GEMM duration at S, the
    curve sampled on the emulated communicator), Alg. 1's prediction of every
    partition (all 2^(T-1) for T <= 8, a seeded sample of 24 otherwise) vs
    the measured fo_run, the predictive search's pick vs the measured optimum
    (PAPER.md:638-647), and the overlapped layer vs GEMM -> one collective."""
    torch.cuda.set_device(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    errs, ratios, ierrs, iratios = [], [], [], []
    print(f"[emulate] link {link_gbps} GB/s per direction, latency {latency_us} us, {ctas} CTAs per call", flush=True)
    for (M, N, K, n, coll) in [(4096, 4096, 7168, 2, "allreduce"), (4096, 4096, 3584, 4, "allreduce"),
                               (4096, 4096, 1792, 8, "allreduce"), (8192, 8192, 1024, 8, "reducescatter")]:
        ctx = fo.Context.emulated(0, 0, n, link_gbps, latency_us, ctas)
        S = 64
        tiles = (M // 256) * (N // 256)
        T = -(-tiles // S)
        A, Bt = synthetic.float_inputs(M, N, K, seed=synthetic.cell_seed(M, N, K), device="cuda")
        rows = M if coll == "allreduce" else M // n
        out = torch.empty(rows, N, dtype=torch.bfloat16, device="cuda")
        C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        spec = dict(coll=coll, m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, swizzle=0, ar_layout="rowband")
        probe = fo.Plan(rank=0, world=n, group_waves=[1] * T, **spec)
        gplan = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S,
                        tile_order=probe.export_order())
        dur = timeit_pre(lambda: fo.gemm_stage(gplan, A, Bt, C), flush, iters=10)
        sizes = [1 << s for s in range(18, 28)]
        curve = ctx.sample_curve(coll, sizes, iters=5)
        fac = 2.0 * (n - 1) / n if coll == "allreduce" else (n - 1) / n
        print(f"[emulate] {coll} n={n} curve (bytes: measured us / link model us): " + ", ".join(
            f"{b_ >> 20} MB: {b_ / (g_ * 1e3):.1f}/{latency_us + fac * b_ / (link_gbps * 1e3):.1f}"
            for b_, g_ in curve if b_ >= 1 << 21), flush=True)
        # the contended curve (offline stage (3) measured in situ, tuner.insitu_curve, R42)
        icurve = tuner.insitu_curve(ctx, dict(spec, rank=0, world=n), A, Bt, out, T, S, 256 * 256 * 2, curve)
        print(f"[emulate] {coll} n={n} in-situ curve points (bytes: us): " + ", ".join(
            f"{b_ >> 20} MB: {b_ / (g_ * 1e3):.1f}" for b_, g_ in icurve if b_ >= 1 << 21), flush=True)
        rows_ = []
        for G in candidates(T, 24, M + K + n):
            plan = fo.Plan(rank=0, world=n, group_waves=G, **spec)
            pred = fo.tune_predict(G, dur, tiles, S, 256 * 256 * 2, curve)
            ipred = tuner.predict_insitu(G, dur, tiles, S, 256 * 256 * 2, icurve, curve)
            meas = timeit_pre(lambda: fo.run(ctx, plan, A, Bt, out), flush)
            rows_.append((G, pred, meas, ipred))
            errs.append(abs(meas - pred) / meas)
            ierrs.append(abs(meas - ipred) / meas)
        ipick = min(rows_, key=lambda r: r[3])[0]   # argmin of the in-situ prediction over the candidates
        iplan = fo.Plan(rank=0, world=n, group_waves=list(ipick), **spec)
        ipick_meas = timeit_pre(lambda: fo.run(ctx, iplan, A, Bt, out), flush)
        best = min(rows_, key=lambda r: r[2])
        pick, _ = fo.tune_search(dur, tiles, S, 256 * 256 * 2, curve)
        pplan = fo.Plan(rank=0, world=n, group_waves=list(pick), **spec)
        pick_meas = timeit_pre(lambda: fo.run(ctx, pplan, A, Bt, out), flush)
        ratios.append(best[2] / pick_meas)
        iratios.append(best[2] / ipick_meas)
        # sequential: the GEMM on every SM (all 74 CTA pairs, split tail), then one collective
        seq = fo.Plan(rank=0, world=n, group_waves=[-(-tiles // 74)], options={"tail_split": -1},
                      **dict(spec, workers=74, ar_layout="auto"))
        seq_us = timeit_pre(lambda: fo.run_sequential(ctx, seq, A, Bt, out), flush)
        comm_full = ctx.time_collective(coll, M * N * 2, 5)
        e = [abs(m - p) / m for _, p, m, _ in rows_]
        ie = [abs(m - p) / m for _, _, m, p in rows_]
        print(f"[emulate] {coll} n={n} {M}x{N}x{K}: T={T}, GEMM {dur:.1f} us at S={S}, full collective "
              f"{comm_full:.1f} us; {len(rows_)} partitions: prediction error mean {100 * statistics.mean(e):.2f}% "
              f"max {100 * max(e):.2f}%; search picks {list(pick)} -> {pick_meas:.1f} us, measured optimum "
              f"{best[0]} {best[2]:.1f} us ({100 * best[2] / pick_meas:.1f}%); sequential {seq_us:.1f} us -> "
              f"speedup {seq_us / pick_meas:.3f}x (best {seq_us / best[2]:.3f}x); with the in-situ curve: error mean "
              f"{100 * statistics.mean(ie):.2f}% max {100 * max(ie):.2f}%, search picks {list(ipick)} -> "
              f"{ipick_meas:.1f} us ({100 * best[2] / ipick_meas:.1f}%), speedup {seq_us / ipick_meas:.3f}x", flush=True)
        # the whole tuner (tile shape, S, layout, tail split, partition; in-situ
        # curve; measured verification of the best predictions)
        ch = tuner.tune_layer(M, N, K, ctx, coll, "none", device=0, tile_shapes=[(256, 256), (128, 256)])
        tplan = fo.Plan(rank=0, world=n, **ch.spec(M, N, K, coll))
        tout = torch.empty(tplan.info["out_rows"], N, dtype=torch.bfloat16, device="cuda")
        t_us = timeit_pre(lambda: fo.run(ctx, tplan, A, Bt, tout), flush)
        print(f"[emulate] {coll} n={n}: tune_layer -> {ch.tile_m}x{ch.tile_n} S={ch.workers} {ch.layout} "
              f"groups {ch.groups} tail_split {ch.tail_split}: {t_us:.1f} us = {seq_us / t_us:.3f}x sequential; "
              f"layer roofline max(GEMM at peak, collective on the link) "
              f"{max(2.0 * M * N * K / 1631.4e6, latency_us + fac * M * N * 2 / (link_gbps * 1e3)):.1f} us", flush=True)
        for G, p_, m_, ip_ in sorted(rows_, key=lambda r: r[2])[:4]:
            print(f"           {str(G):28s} predicted {p_:7.1f} us (in-situ curve {ip_:7.1f})  measured {m_:7.1f} us",
                  flush=True)
        del A, Bt, out, C
        torch.cuda.empty_cache()
        ctx.close()
    e = sorted(errs)
    print(f"[emulate] ALL: {len(errs)} (shape, partition) cases, prediction error mean {100 * statistics.mean(e):.2f}%, "
          f"median {100 * e[len(e) // 2]:.2f}%, p90 {100 * e[int(0.9 * len(e))]:.2f}%, max {100 * e[-1]:.2f}%; "
          f"searched / optimum: min {100 * min(ratios):.1f}%, mean {100 * statistics.mean(ratios):.1f}%", flush=True)
    e = sorted(ierrs)
    print(f"[emulate] ALL with the in-situ curve: prediction error mean {100 * statistics.mean(e):.2f}%, "
          f"median {100 * e[len(e) // 2]:.2f}%, p90 {100 * e[int(0.9 * len(e))]:.2f}%, max {100 * e[-1]:.2f}%; "
          f"searched / optimum: min {100 * min(iratios):.1f}%, mean {100 * statistics.mean(iratios):.1f}%", flush=True)


if __name__ == "__main__":
    if MODE == "emulate":
        main_emulate()
    else:
        main()
