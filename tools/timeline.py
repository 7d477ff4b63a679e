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


def one(ctx, coll, M, N, K, BN, S, groups, layout="slot", flush=None, wait_kernel=0, world=1):
    kw = dict(coll=coll, m=M, n=N, k=K, tile_m=256, tile_n=BN, workers=S, swizzle=1 if layout == "rowband" else 2,
              group_waves=groups, ar_layout=layout)
    if coll == "alltoall":
        kw["row_dst"] = np.zeros(M, np.int32)
        plan = fo.Plan(rank=0, world=1, peers=[kw], **kw)
    else:
        plan = fo.Plan(rank=0, world=world, **kw)
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
    print(f"\n{coll} n={world} {M}x{N}x{K} tile 256x{BN} S={S} groups={groups} layout={plan.info['ar_layout']} "
          f"trigger={'spin-kernel' if wait_kernel else 'stream-wait'}: "
          f"fo_run {t_ov:.1f} us, sequential {t_seq:.1f} us, speedup {t_seq / t_ov:.3f}")
    print(f"  GEMM: first tile signal 0.0 us, last tile signal {(t.max() - t0) / 1e3:.1f} us")
    for j in range(len(groups)):
        lo, hi, _, _ = plan.group(j)
        print(f"  group {j}: tiles [{lo:4d},{hi:4d}) last signal {(t[lo:hi].max() - t0) / 1e3:8.1f} us | "
              f"wait released {(g[2 * j] - t0) / 1e3:8.1f} us | collective+post done {(g[2 * j + 1] - t0) / 1e3:8.1f} us")
    return plan, t, g


def chrome_trace(name, plan, t, g, S, pid):
    """Chrome trace events (chrome://tracing / Perfetto) from the %globaltimer
    stamps: one track per GEMM worker (tile p spans from the worker's previous
    signal, or one median tile time before its first, to its own signal) and a
    track for the communication stream (wait released -> collective + post
    done), so the overlap of each group's collective with the GEMM's later
    waves is visible as in an nsys timeline."""
    ev = [{"name": "process_name", "ph": "M", "pid": pid, "args": {"name": name}}]
    tiles = len(t)
    per = {}
    for p in range(tiles):
        per.setdefault(p % S, []).append(p)
    durs = [int(t[b] - t[a]) for ps in per.values() for a, b in zip(ps, ps[1:])]
    med = int(np.median(durs)) if durs else 0
    t0 = int(t.min()) - med  # ~ the GEMM's start
    for w, ps in per.items():
        prev = None
        for p in ps:
            end = int(t[p])
            start = end - med if prev is None else prev
            ev.append({"name": f"tile pos {p} (group {int(np.searchsorted([plan.group(j)[1] for j in range(plan.info['num_groups'])], p, side='right'))})",
                       "ph": "X", "pid": pid, "tid": f"GEMM worker {w:02d}", "ts": (start - t0) / 1e3,
                       "dur": max(end - start, 1) / 1e3})
            prev = end
    for j in range(len(g) // 2):
        ev.append({"name": f"group {j}: collective + post", "ph": "X", "pid": pid, "tid": "comm stream",
                   "ts": (int(g[2 * j]) - t0) / 1e3, "dur": max(int(g[2 * j + 1]) - int(g[2 * j]), 1) / 1e3})
    return ev


def loopback(W, coll, M, N, K, S, groups, layout, trace_events=None):
    """World-W run on one GPU through the loopback communicator (R37): every
    rank's tile signals and, on its comm stream, each group's wait release and
    exchange + post completion, on one clock (%globaltimer).  The exchange is
    real (rank r's group j data reaches the other ranks while the GEMMs run)
    but not NVLink: the loopback's kernels share the one GPU's SMs and HBM."""
    from concurrent.futures import ThreadPoolExecutor

    grp = fo.LoopbackGroup(0, W)
    ctxs = grp.contexts()
    plans, As, Bts, outs, tts, gts = [], [], [], [], [], []
    for r in range(W):
        kw = dict(coll=coll, m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, swizzle=1 if layout == "rowband" else 2,
                  group_waves=groups, ar_layout=layout)
        pl = fo.Plan(rank=r, world=W, **kw)
        pl.prepare(sequential=True)
        A, Bt = synthetic.float_inputs(M, N, K, seed=100 + r, device="cuda")
        plans.append(pl), As.append(A), Bts.append(Bt)
        outs.append(torch.empty(pl.info["out_rows"], N, dtype=torch.bfloat16, device="cuda"))
        tts.append(torch.zeros(pl.info["tiles"], dtype=torch.int64, device="cuda"))
        gts.append(torch.zeros(2 * len(groups), dtype=torch.int64, device="cuda"))
        pl.set_debug(tts[r], gts[r])
    streams = [torch.cuda.Stream() for _ in range(W)]
    pool = ThreadPoolExecutor(W)

    def each(fn):
        def one_(r):
            torch.cuda.set_device(0)
            with torch.cuda.stream(streams[r]):
                fn(r)
            streams[r].synchronize()
        for f in [pool.submit(one_, r) for r in range(W)]:
            f.result()
    for _ in range(3):
        each(lambda r: fo.run(ctxs[r], plans[r], As[r], Bts[r], outs[r], stream=streams[r]))
    torch.cuda.synchronize()
    ts = [x.cpu().numpy() for x in tts]
    gs = [x.cpu().numpy() for x in gts]
    t0 = min(t.min() for t in ts)
    print(f"\nloopback world {W}: {coll} {M}x{N}x{K} S={S} groups={groups} layout={layout} (one GPU, all ranks)")
    for r in range(W):
        t, g = ts[r], gs[r]
        print(f"  rank {r}: GEMM last tile signal {(t.max() - t0) / 1e3:8.1f} us")
        for j in range(len(groups)):
            lo, hi, _, _ = plans[r].group(j)
            print(f"    group {j}: tiles [{lo:4d},{hi:4d}) last signal {(t[lo:hi].max() - t0) / 1e3:8.1f} us | "
                  f"wait released {(g[2 * j] - t0) / 1e3:8.1f} us | exchange+post done {(g[2 * j + 1] - t0) / 1e3:8.1f} us")
        if trace_events is not None:
            trace_events += chrome_trace(f"loopback rank {r}: {coll} groups {groups}", plans[r], t, g, S, 10 + r)
    for p in plans:
        p.close()
    for c in ctxs:
        c.close()
    grp.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trace", default=None, help="also write a Chrome trace JSON of the first AR plans")
    ap.add_argument("--loopback", type=int, default=0,
                    help="world size of a one-GPU loopback run (needs CUDA_MODULE_LOADING=EAGER) instead")
    ap.add_argument("--emulate", type=int, default=0,
                    help="rank 0 of this world size on the emulated-link evaluation backend (R42; timing model)")
    args = ap.parse_args()
    if args.emulate:
        torch.cuda.set_device(0)
        n = args.emulate
        ctx = fo.Context.emulated(0, 0, n, 770.0, 6.0, 16)
        flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        events = []
        print(f"EMULATED NVLink (fo_ctx_create_emulated: 770 GB/s per direction, 6 us latency, 16 CTAs per call): "
              f"rank 0 of {n}; a timing model, not a measurement of NVLink")
        K = 14336 // n
        r1 = one(ctx, "allreduce", 4096, 4096, K, 256, 64, [1, 1, 1, 1], "rowband", flush, 0, n)
        r2 = one(ctx, "allreduce", 4096, 4096, K, 256, 64, [1, 3], "rowband", flush, 0, n)
        r3 = one(ctx, "reducescatter", 8192, 8192, 1024, 256, 64, [1, 4, 8, 3], "rowband", flush, 0, n)
        events += chrome_trace(f"emulated TP={n} AR rowband S=64 groups [1,1,1,1]", *r1, 64, 1)
        events += chrome_trace(f"emulated TP={n} AR rowband S=64 groups [1,3]", *r2, 64, 2)
        events += chrome_trace(f"emulated TP={n} RS rowband S=64 groups [1,4,8,3]", *r3, 64, 3)
        ctx.close()
        if args.trace:
            import json
            with open(args.trace, "w") as f:
                json.dump({"traceEvents": events, "displayTimeUnit": "ns"}, f)
        return
    if args.loopback:
        torch.cuda.set_device(0)
        events = []
        loopback(args.loopback, "allreduce", 4096, 4096, 3584, 32, [2, 2, 4], "rowband", events)
        loopback(args.loopback, "reducescatter", 4096, 4096, 2048, 32, [2, 2, 4], "auto", events)
        if args.trace:
            import json
            with open(args.trace, "w") as f:
                json.dump({"traceEvents": events, "displayTimeUnit": "ns"}, f)
        return
    torch.cuda.set_device(0)
    ctx = fo.Context.create(0, 0, 1, fo.unique_id())
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    events = []
    for wk in (0, 1):
        r1 = one(ctx, "allreduce", 4096, 4096, 14336, 256, 64, [1, 1, 1, 1], "slot", flush, wk)
        r2 = one(ctx, "allreduce", 4096, 4096, 14336, 256, 64, [1, 2, 1], "rowband", flush, wk)
        if args.trace and wk == 0:
            events += chrome_trace("AR slot S=64 groups [1,1,1,1]", *r1, 64, 1)
            events += chrome_trace("AR rowband S=64 groups [1,2,1]", *r2, 64, 2)
        one(ctx, "reducescatter", 8192, 8192, 1024, 256, 64, [2, 4, 6, 4], "auto", flush, wk)
        one(ctx, "alltoall", 1024, 4096, 14336, 128, 64, [1, 1], "auto", flush, wk)
    ctx.close()
    if args.trace:
        import json
        with open(args.trace, "w") as f:
            json.dump({"traceEvents": events, "displayTimeUnit": "ns"}, f)


if __name__ == "__main__":
    main()
