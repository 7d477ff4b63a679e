#!/usr/bin/env python
"""Benchmark of the overlapped GEMM + collective layer (BASELINE.json metric):
overlapped GEMM+AllReduce us per layer, speedup vs the same GEMM followed by a
non-overlapped NCCL call, and % of roofline.

Workload (BASELINE.json configs[1]): Llama-3-8B row-parallel down-proj,
M=4096 tokens, N=4096, K=14336/TP, bf16, AllReduce at TP = --gpus.
At --gpus 1 this is TP=1 (K=14336, the AllReduce is a 1-rank NCCL call).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl fo|reference]

One JSON line on rank 0.  Timing: W untimed warm-up steps, then K steps, each
bracketed by (barrier,) an L2 flush (256 MiB write, outside the timed span) and
CUDA events on the launching stream; per-step device time, max over ranks;
the value is the median step (mean, p10, p90 in step_stats_us).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

# stdout must carry exactly one JSON line: NCCL's init banner ("NCCL version
# ...", printed when NCCL_DEBUG=VERSION, e.g. set by the image) goes to stderr
if os.environ.get("NCCL_DEBUG", "").upper() in ("", "VERSION"):
    os.environ["NCCL_DEBUG"] = "WARN"


class _StdoutToStderr:
    """Route C-level stdout (NCCL/driver prints) to stderr inside the block."""

    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)
        return self

    def __exit__(self, *a):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)


M_TOK, N_HID, K_FFN = 4096, 4096, 14336
BM, BN = 256, 256   # tcgen05 cta_group::2 tile (CTA pair)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="fo", choices=["fo", "reference"])
    ap.add_argument("--workers", type=int, default=None,
                    help="S = concurrent tile workers (CTA pairs); default: fewest workers with the same wave count as all SMs")
    ap.add_argument("--groups", default=None, help="explicit wave-group partition, e.g. 1,1,2 (default: Alg. 1)")
    ap.add_argument("--tail-split", type=int, default=0, help="FO_OPT_TAIL_SPLIT with --workers/--groups")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-shards", action="store_true", help="skip the other configs' per-rank layers")
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="target CPU work for the oracle sample")
    ap.add_argument("--emulate-world", type=int, default=0,
                    help="DEV ONLY: one process acting as rank 0 of N with the emulated-link evaluation backend "
                         "(fo_ctx_create_emulated; timing model, not NVLink) — exercises the N>1 code paths on one GPU")
    return ap.parse_args()


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def workload(n):
    K = K_FFN // n
    return dict(workload=f"llama3-8b-down-proj-allreduce-tp{n}", M=M_TOK, N=N_HID, K_loc=K, K=K_FFN, tp=n,
                collective="allreduce", tile=f"{BM}x{BN}", dtype="bf16")


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling (to a file, 50 ms period) of SM clocks and throttle
    reasons while the timed region runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        import tempfile
        self.device, self.proc = device, None
        self.path = tempfile.mktemp(prefix="fo_clocks_", suffix=".csv")

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50", "-f", self.path], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 8:
                    rows.append(parts)
            os.unlink(self.path)
        except Exception:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(r[0]) for r in rows if num(r[0])]
        mx = [num(r[1]) for r in rows if num(r[1])]
        pw = [num(r[2]) for r in rows if num(r[2])]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower() == "active"})
        load = [s for s in sm if s > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows), "power_w_max": max(pw) if pw else None}


# --------------------------------------------------------------------------- CPU oracle baseline
def cpu_oracle_sample(wl, n, target_s):
    """Time the CPU oracle (as it stands) on a bounded sample of the workload:
    the full pipeline (n fp64 rank GEMMs -> AR pre-reorder -> explicit per-group
    AllReduce -> post-reorder) for `rows` output rows of every rank; scaled to
    the full M.  Returns (us per full layer, description, threads)."""
    import torch

    import synthetic
    from oracle import pipeline as opl
    from oracle import plan as op

    M, N, K = wl["M"], wl["N"], wl["K_loc"]

    def run(rows):
        As, Bts = [], []
        for r in range(n):
            A, Bt = synthetic.float_inputs(rows, N, K, seed=synthetic.rank_seed(20000, n, r))
            As.append(A)
            Bts.append(Bt)
        tiles = (rows // BM) * (N // BN)
        pl = op.make_plan(rows, N, BM, BN, min(tiles, 148), None)
        t0 = time.perf_counter()
        opl.run_allreduce(As, Bts, pl)
        return time.perf_counter() - t0

    t1 = run(BM)
    rows = int(min(M, max(BM, BM * round(target_s / max(t1, 1e-3)))))
    rows = max(BM, (rows // BM) * BM)
    t = run(rows) if rows != BM else t1
    us = t * 1e6 * (M / rows)
    threads = torch.get_num_threads()
    try:
        import numpy.__config__  # noqa: F401
        cores = len(os.sched_getaffinity(0))
    except Exception:
        cores = os.cpu_count()
    desc = (f"oracle run_allreduce on {rows} of {M} rows x all {N} cols, K={K}, {n} simulated rank(s): "
            f"{t:.2f} s, scaled x{M / rows:.1f} to the full layer")
    return us, desc, cores or threads


# --------------------------------------------------------------------------- reference arm
def reference_arm(args, wl, rank, world):
    if rank != 0:
        return
    K, W = args.steps, args.warmup
    per = max(0.5, min(10.0, 120.0 / max(1, K + W)))
    times, desc, cores = [], "", 1
    for i in range(W + K):
        us, desc, cores = cpu_oracle_sample(wl, world, per)
        if i >= W:
            times.append(us)
    v = statistics.mean(times)
    line = {"impl": "reference", "metric": "overlapped GEMM+AllReduce us per layer", "value": round(v, 1),
            "unit": "us", "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": round(v / 1e3, 3),
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {k: wl[k] for k in ("workload", "M", "N", "K_loc", "tp", "collective")},
            "cpu_baseline": {"value": round(v, 1), "unit": "us", "cores": cores, "kind": "oracle", "sample": desc},
            "e2e": {"value": round(v, 1), "unit": "us", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU arm
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    emulate = args.emulate_world > 1 and "WORLD_SIZE" not in os.environ
    if emulate:
        world, rank = args.emulate_world, 0
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and "WORLD_SIZE" in os.environ:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    wl = workload(world)
    if args.impl == "reference":
        return reference_arm(args, wl, rank, world)

    import torch
    import torch.distributed as dist

    import paper_2504_19519_b200 as fo

    torch.cuda.set_device(local)
    # under torchrun (even at one process) the distributed plumbing is live
    use_dist = "WORLD_SIZE" in os.environ and "MASTER_ADDR" in os.environ
    if use_dist:
        with _StdoutToStderr():
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    peaks, peak_src = load_peaks()
    sms = fo.device_sm_count(local)
    M, N, K = wl["M"], wl["N"], wl["K_loc"]
    tiles = (M // BM) * (N // BN)
    cg = BM // 128
    if args.workers:
        S = args.workers
    else:
        # waves are quantised: keep T of the full-GPU grid, use the fewest workers
        # achieving it; the SMs this frees are left to NCCL (R18)
        T_full = -(-tiles // (sms // cg))
        S = -(-tiles // T_full)
    comm_sms = sms - cg * S    # the NCCL CTA cap (SMs a quantisation-aware S leaves free)

    # ---- inputs (synthetic, seeded; SURVEY §8(d) recipe), resident in HBM
    import synthetic
    A_h, B_h = synthetic.float_inputs(M, N, K, seed=synthetic.rank_seed(20000, world, rank))
    A = A_h.cuda()
    Bt = B_h.cuda()
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    # ---- NCCL context of the library (unique id broadcast over the process group)
    def emu_ctx(cap):
        c = fo.Context.emulated(local, rank, world, 770.0, 6.0, ctas=min(max(cap, 16), 32))
        c.nccl_max_ctas = cap
        return c
    if emulate:
        ctx = emu_ctx(max(1, comm_sms))
        ctxs = [ctx, emu_ctx(max(comm_sms + 12, 32))]
        ctx_seq = emu_ctx(0)
    elif use_dist:
        obj = [fo.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    else:
        uid = fo.unique_id()
    if not emulate:
        with _StdoutToStderr():
            ctx = fo.Context.create(local, rank, world, uid, nccl_max_ctas=max(1, comm_sms) if world > 1 else 0)
        # a second overlapped-op communicator with a wider CTA cap: the tuner
        # searches the SM split (GEMM workers vs NCCL CTAs) across both
        ctxs = [ctx]
    if world > 1 and not emulate:
        if use_dist:
            obj = [fo.unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            uid2 = obj[0]
        else:
            uid2 = fo.unique_id()
        with _StdoutToStderr():
            ctxs.append(fo.Context.create(local, rank, world, uid2, nccl_max_ctas=max(comm_sms + 12, 32)))
    # the sequential baseline's NCCL call runs alone, so it gets NCCL's default
    # CTA count (its own communicator) instead of the overlapped op's SM cap
    if emulate:
        pass
    elif world > 1:
        if use_dist:
            obj = [fo.unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            uid_seq = obj[0]
        else:
            uid_seq = fo.unique_id()
        with _StdoutToStderr():
            ctx_seq = fo.Context.create(local, rank, world, uid_seq)
    else:
        ctx_seq = ctx

    def barrier():
        if use_dist:
            dist.barrier(device_ids=[local])

    # device time: after the flush + barrier + sync the stream is pre-loaded
    # with a ~100 us sleep kernel, so the work is already queued when the start
    # event executes and the events bracket device work only (the ~12 us host
    # enqueue of a call, tools/host_overhead.py, is excluded); the e2e number
    # keeps everything, host included
    PRELOAD_CYCLES = 200_000

    def timed(fn, steps, warm, preload=True):
        for _ in range(warm):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(steps):
            flush.zero_()
            barrier()
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if preload:
                torch.cuda._sleep(PRELOAD_CYCLES)
            s.record()
            fn()
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e) * 1e3)
        med = statistics.median(ts)
        if use_dist:
            t = torch.tensor([med], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            med = t.item()
        return med, ts

    def dist_stats(v):
        q = sorted(v)

        def pct(f):  # nearest-rank percentile
            return q[min(len(q) - 1, max(0, int(round(f * (len(q) - 1)))))]
        return {"mean": round(statistics.mean(q), 2), "median": round(statistics.median(q), 2),
                "p10": round(pct(0.1), 2), "p90": round(pct(0.9), 2), "n": len(q)}

    stats_out = {}

    def timed_multi(fns, steps, warm):
        """Interleaved timing: every iteration runs each variant once (flush +
        barrier + events around each), so all variants see the same clocks."""
        for _ in range(warm):
            for f in fns.values():
                f()
        torch.cuda.synchronize()
        ts = {k: [] for k in fns}
        for _ in range(steps):
            for k, f in fns.items():
                flush.zero_()
                barrier()
                torch.cuda.synchronize()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda._sleep(PRELOAD_CYCLES)
                s.record()
                f()
                e.record()
                torch.cuda.synchronize()
                ts[k].append(s.elapsed_time(e) * 1e3)
        if use_dist:
            # per-step max over ranks (a step ends when its slowest rank does)
            ts_t = torch.tensor([ts[k] for k in fns], device="cuda", dtype=torch.float64)
            dist.all_reduce(ts_t, op=dist.ReduceOp.MAX)
            ts = {k: ts_t[i].tolist() for i, k in enumerate(fns)}
        stats_out.update({k: dist_stats(v) for k, v in ts.items()})
        # the median step: a host stall longer than the ~100 us preload (e.g.
        # while nvidia-smi samples the clocks) inflates one step by
        # milliseconds and would dominate a mean of 20
        return {k: statistics.median(v) for k, v in ts.items()}

    # ---- offline + online stages of Alg. 1 (untimed, tuner.tune_layer): GEMM
    # duration per candidate wave width S and layout, the NCCL curve on the
    # library's communicator, Alg. 1 over the wave groups; the fused-op layer
    # is tuned with its per-group fused op folded into the curve (R28)
    from paper_2504_19519_b200 import tuner as fot
    if args.workers or args.groups:
        T = (tiles + S - 1) // S
        gplan0 = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=BM, tile_n=BN, workers=S, swizzle=0)
        gemm_us, _ = timed(lambda: fo.gemm_stage(gplan0, A, Bt, out), 5, 2)
        curve = ctx.sample_curve("allreduce", [1 << s for s in range(18, 27)], iters=5)
        groups = tuple(int(x) for x in args.groups.split(",")) if args.groups else \
            fo.tune_search(gemm_us, tiles, S, BM * BN * 2, curve)[0]
        pred = fo.tune_predict(groups, gemm_us, tiles, S, BM * BN * 2, curve)
        spec = dict(coll="allreduce", m=M, n=N, k=K, tile_m=BM, tile_n=BN, workers=S, swizzle=0,
                    group_waves=list(groups), ar_layout="auto")
        if args.tail_split:
            spec["options"] = {"tail_split": args.tail_split}
        nspec = dict(spec, post="add_rmsnorm")
        pred_n = pred
        curve_bw = None
        nctx = ctx
    else:
        shapes = [(BM, BN), (128, 256)]      # CTA-pair 256x256 and single-CTA 128x256 tiles
        # the uncapped communicator too: a single group overlaps nothing and
        # runs best as the sequential plan (all SMs, NCCL's default CTAs)
        tune_ctxs = ctxs + ([ctx_seq] if ctx_seq is not ctx else [])
        ch = fot.tune_layer(M, N, K, tune_ctxs, "allreduce", "none", device=local, tile_shapes=shapes)
        chn = fot.tune_layer(M, N, K, tune_ctxs, "allreduce", "add_rmsnorm", device=local, tile_shapes=shapes)
        if rank == 0:
            for name, c in (("plain", ch), ("fused", chn)):
                for cand in c.candidates[:6]:
                    print(f"[tune_layer {name}] S={cand[0]} layout={cand[1]} groups={cand[2]} "
                          f"predicted {cand[3]:.1f} us" + (f", measured {cand[5]:.1f} us" if len(cand) > 5 else ""),
                          file=sys.stderr)
        S, groups, pred = ch.workers, tuple(ch.groups), ch.predicted_us
        curve_bw = ch.curve
        ctx, nctx = tune_ctxs[ch.ctx_index], tune_ctxs[chn.ctx_index]   # the communicators the tuner chose
        spec, nspec, pred_n = ch.spec(M, N, K, "allreduce"), chn.spec(M, N, K, "allreduce", "add_rmsnorm"), \
            chn.predicted_us
    # the chosen tile shape (tune_layer searches it; the explicit --workers /
    # --groups path keeps 256x256)
    BMc, BNc = spec["tile_m"], spec["tile_n"]
    cgc = BMc // 128
    tiles_c = (M // BMc) * (N // BNc)
    T = (tiles_c + S - 1) // S
    plan = fo.Plan(rank=rank, world=world, **spec)
    # fused-op convention (R17): the same layer followed by
    # residual add + RMSNorm, fused into the (per-band) post-communication pass
    nplan = fo.Plan(rank=rank, world=world, **nspec)
    groups_n = nspec["group_waves"]
    resid = synthetic.normal_bf16((M, N), 1.0, 7, device="cuda")
    gamma = synthetic.normal_bf16((N,), 1.0, 8, device="cuda")
    out2 = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    out_cb = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    # the GEMM-only timing uses exactly the overlapped plan's execution order
    gplan = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=BMc, tile_n=BNc, workers=S,
                    tile_order=plan.export_order(), options=spec.get("options"))
    # the sequential baseline: the overlapped plan at one rank (same thing);
    # at N > 1 the GEMM alone on the whole GPU (every 256x256 CTA pair, split
    # tail), its output then one NCCL call with NCCL's default CTAs — not the
    # overlapped plan's narrower wave width
    if world > 1:
        # the standalone GEMM's best wave width: all pairs with the split tail
        # for long K, the fewest pairs with the full wave count for short K
        # (measured, profiles/r02_tp_shard_probe.txt)
        long_k = K >= 3584
        S_seq = sms // 2 if long_k else -(-((M // 256) * (N // 256)) // -(-((M // 256) * (N // 256)) // (sms // 2)))
        T_seq = -(-((M // 256) * (N // 256)) // S_seq)
        seq_spec = dict(coll="allreduce", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S_seq, swizzle=0,
                        group_waves=[T_seq], ar_layout="auto", options={"tail_split": -1} if long_k else None)
        seqplan = fo.Plan(rank=rank, world=world, **seq_spec)
        nseqplan = fo.Plan(rank=rank, world=world, **dict(seq_spec, post="add_rmsnorm"))
    else:
        seqplan, nseqplan = plan, nplan

    # ---- full-size spot check (N=1: sampled rows vs an fp64 torch CPU product; not the oracle)
    fo.run(ctx, plan, A, Bt, out)
    torch.cuda.synchronize()
    spot = None
    if world == 1:
        rows = torch.randperm(M, generator=torch.Generator().manual_seed(0))[:8]
        ref = A_h[rows].double() @ B_h.double().t()
        got = out[rows.cuda()].double().cpu()
        rms = ref.pow(2).mean().sqrt()
        spot = {"rows": 8, "max_rel_err": float(((got - ref).abs() / torch.maximum(ref.abs(), rms)).max())}

    # ---- timed: overlapped, sequential, GEMM kernel alone
    l0 = fo.kernel_launch_count()
    fo.run(ctx, plan, A, Bt, out)
    torch.cuda.synchronize()
    launches_per_step = fo.kernel_launch_count() - l0
    with ClockSampler(local) as clk:
        m = timed_multi({"ov": lambda: fo.run(ctx, plan, A, Bt, out),
                         "seq": lambda: fo.run_sequential(ctx_seq, seqplan, A, Bt, out),
                         "gemm": lambda: fo.gemm_stage(gplan, A, Bt, out),
                         "ov_norm": lambda: fo.run(nctx, nplan, A, Bt, out2, resid, gamma),
                         "seq_norm": lambda: fo.run_sequential(ctx_seq, nseqplan, A, Bt, out2, resid, gamma),
                         # library comparator (not on the product path): the same GEMM through cuBLAS
                         "cublas": lambda: torch.matmul(A, Bt.t(), out=out_cb)},
                        args.steps, args.warmup)
    ov_us, seq_us, gk_us, cb_us = m["ov"], m["seq"], m["gemm"], m["cublas"]
    main_stats = dict(stats_out)   # (later timed_multi calls reuse the keys)
    launches = launches_per_step * args.steps

    # ---- the other BASELINE.json configs' per-rank layers (their exchange
    # needs the other ranks): the GEMM writing row-major C, the same GEMM with
    # the layer's pre-communication reorder + signal epilogue (AR slot / RS
    # subtiles / A2A pools — the paper's epilogue overhead),
    # and cuBLAS on the same shard, interleaved
    shards = {}
    if world == 1 and not args.no_shards:
        for name, Ms, Ns, Ks, coll in (("llama3-8b-down-proj tp2 shard (AR)", 4096, 4096, 7168, "allreduce"),
                                       ("llama3-8b-down-proj tp4 shard (AR)", 4096, 4096, 3584, "allreduce"),
                                       ("llama3-8b-down-proj tp8 shard (AR)", 4096, 4096, 1792, "allreduce"),
                                       ("llama3-70b-o-proj tp8 shard (RS)", 8192, 8192, 1024, "reducescatter"),
                                       ("mixtral-8x7b-w2 ep8 expert (A2A)", 1024, 4096, 14336, "alltoall")):
            As_, Bs_ = synthetic.float_inputs(Ms, Ns, Ks, seed=synthetic.cell_seed(Ms, Ns, Ks), device="cuda")
            Cs_ = torch.empty(Ms, Ns, dtype=torch.bfloat16, device="cuda")
            t_ = (Ms // BM) * (Ns // BN)
            smax = sms // cg
            # two wave widths, both timed: the fewest workers with the full
            # GPU's wave count, and the full GPU with the last partial wave
            # split along K (R34) when it qualifies; the faster one is reported
            variants = [(-(-t_ // -(-t_ // smax)), 0)]
            R_ = t_ - (-(-t_ // smax) - 1) * smax
            if 0 < R_ < smax and 2 * R_ <= smax and Ks >= 128 and variants[0][0] != smax:
                variants.append((smax, -1))
            best = None
            for Sw, ts_ in variants:
                Tw = -(-t_ // Sw)
                opts_ = {"tail_split": ts_} if ts_ else None
                kw_ = dict(coll=coll, m=Ms, n=Ns, k=Ks, tile_m=BM, tile_n=BN, workers=Sw, swizzle=0,
                           group_waves=[1] * Tw, ar_layout="slot" if coll == "allreduce" else "auto")
                if coll == "alltoall":
                    kw_["row_dst"] = np.zeros(Ms, np.int32)
                    sp_ = fo.Plan(rank=0, world=1, peers=[kw_], options=opts_, **kw_)
                else:
                    sp_ = fo.Plan(options=opts_, **kw_)
                gp_ = fo.Plan(coll="nocomm", m=Ms, n=Ns, k=Ks, tile_m=BM, tile_n=BN, workers=Sw,
                              tile_order=sp_.export_order(), options=opts_)
                send_ = torch.empty(sp_.info["send_elems"], dtype=torch.bfloat16, device="cuda")
                mm = timed_multi({"gemm": lambda: fo.gemm_stage(gp_, As_, Bs_, Cs_),
                                  "epi": lambda: fo.gemm_stage(sp_, As_, Bs_, send_),
                                  "cublas": lambda: torch.matmul(As_, Bs_.t(), out=Cs_)}, 10, 2)
                if best is None or mm["gemm"] < best[2]["gemm"]:
                    best = (Sw, ts_, mm, Tw)
                del send_
            Sw, ts_, mm, Tw = best
            fl_ = 2.0 * Ms * Ns * Ks
            shards[name] = {"M": Ms, "N": Ns, "K_loc": Ks, "workers": Sw, "waves": Tw, "tail_split": ts_,
                            "gemm_us": round(mm["gemm"], 2), "gemm_tflops": round(fl_ / mm["gemm"] / 1e6, 1),
                            "reorder_epilogue_us": round(mm["epi"], 2),
                            "epilogue_overhead_pct": round(100.0 * (mm["epi"] / mm["gemm"] - 1.0), 2),
                            "cublas_us": round(mm["cublas"], 2)}
            # this rank's side of the layer in the paper's layout (SLOT: the
            # epilogue reorder + the post-communication pass over the output)
            # and in ROWBAND (H11a / R40 / R41: the collective lands
            # the rows in the output, no post pass); the collective moves the
            # same bytes in both (n=8 ranks' plans for RS / A2A, rank 0's side)
            nr_ = 8 if coll != "allreduce" else 1
            lay_t = {}
            try:
                fns_ = {}
                for lay in ("slot", "rowband"):
                    Ntl = Ns // BN
                    gw = [1] * Tw if Sw % Ntl == 0 else [Tw]
                    kl = dict(coll=coll, m=Ms, n=Ns, k=Ks, tile_m=BM, tile_n=BN, workers=Sw, swizzle=0,
                              group_waves=gw, ar_layout=lay)
                    if coll == "alltoall":
                        rds_ = [synthetic.balanced_moe_row_dst(Ms // nr_, nr_)] * nr_
                        lp = fo.Plan(rank=0, world=nr_, peers=[dict(kl, row_dst=r_) for r_ in rds_],
                                     options={"tail_split": ts_} if ts_ else None, row_dst=rds_[0], **kl)
                    else:
                        lp = fo.Plan(rank=0, world=nr_ if coll == "reducescatter" else 1,
                                     options={"tail_split": ts_} if ts_ else None, **kl)
                    snd = torch.empty(max(1, lp.info["send_elems"]), dtype=torch.bfloat16, device="cuda")
                    rcv = torch.zeros(max(1, lp.info["recv_elems"]), dtype=torch.bfloat16, device="cuda")
                    o_ = torch.empty(lp.info["out_rows"], Ns, dtype=torch.bfloat16, device="cuda")
                    fns_[lay + "_epi"] = (lambda lp=lp, snd=snd: fo.gemm_stage(lp, As_, Bs_, snd))
                    if lay == "slot":
                        fns_["slot_post"] = (lambda lp=lp, rcv=rcv, o_=o_: fo.post_stage(lp, rcv, o_))
                mt = timed_multi(fns_, 10, 2)
                for lay in ("slot", "rowband"):
                    post_ = mt.get(lay + "_post", 0.0)
                    lay_t[lay] = {"epilogue_us": round(mt[lay + "_epi"], 2), "post_us": round(post_, 2),
                                  "rank_work_us": round(mt[lay + "_epi"] + post_, 2)}
            except Exception as ex:  # pragma: no cover - evidence only
                lay_t = {"error": str(ex)[:200]}
            shards[name]["layouts"] = lay_t
            del As_, Bs_, Cs_

    # ---- e2e through the public API with host (pinned) buffers
    A_pin = A_h.pin_memory()
    out_pin = torch.empty(M, N, dtype=torch.bfloat16).pin_memory()

    # the host path is PCIe-bound: the plan that hides most of it has one wave
    # per group in row bands of ~1/8 of the output (the GEMM starts on the
    # first A chunk, keeps pace with the 8 chunk copies, and every band goes
    # back to the host right after its collective; the exposed tail is one
    # band's GEMM + D2H — profiles/r01_e2e_probe2.txt)
    Nt_, Mt_ = N // BN, M // BM
    S_e = Nt_ * max(1, Mt_ // 8)
    if S_e > sms // cg:
        S_e = S if S % Nt_ == 0 else max(Nt_, (min(tiles, sms // cg) // Nt_) * Nt_)
    T_e = (tiles + S_e - 1) // S_e
    e2e_spec = dict(coll="allreduce", m=M, n=N, k=K, tile_m=BM, tile_n=BN, workers=S_e, swizzle=1,
                    group_waves=[1] * T_e, ar_layout="rowband")
    eplan = fo.Plan(rank=rank, world=world, **e2e_spec)

    def e2e_step():  # the C-ABI host-buffer entry point: H2D of the activations + overlapped op + D2H
        fo.run_host(ctx, eplan, A_pin, Bt, out_pin)  # weights (Bt) are model state resident in HBM

    # latency: one call alone (flush, barrier, sync around it)
    e2e_lat_us, _ = timed(e2e_step, max(3, args.steps // 2), 2, preload=False)
    # throughput: K calls issued back to back (FO_OPT_HOST_PIPELINE bit 2: two
    # staging sets, so call i+1's H2D overlaps call i), one sync at the end;
    # every step still copies its activations in and its output out
    n_e2e = max(3, args.steps // 2)
    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    flush.zero_()
    barrier()
    torch.cuda.synchronize()
    s_e, e_e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s_e.record()
    for _ in range(n_e2e):
        e2e_step()
    e_e.record()
    torch.cuda.synchronize()
    e2e_us = s_e.elapsed_time(e_e) * 1e3 / n_e2e
    if use_dist:
        t_ = torch.tensor([e2e_us], device="cuda", dtype=torch.float64)
        dist.all_reduce(t_, op=dist.ReduceOp.MAX)
        e2e_us = t_.item()

    flops = 2.0 * M * N * K
    achieved = flops / (gk_us * 1e-6) / 1e12
    peak = peaks["bf16_tflops"]
    # NVLink: the measured peer-copy bandwidth per direction of this pool's
    # B200s (B200_PROFILING.md: 770 GB/s; 900 GB/s nominal)
    nvlink_gbs, nvlink_src = 770.0, "measured peer copy per direction, B200_PROFILING.md (900 nominal)"
    S_B = M * N * 2
    bus_ring = 2.0 * (world - 1) / world * S_B      # nccl-tests bus bytes of an AllReduce
    bus_nvls = 1.0 * (world - 1) / world * S_B      # what crosses each link with in-switch reduction
    gemm_roof_us = flops / (peak * 1e12) * 1e6
    layer_roof_us = max(gemm_roof_us, bus_ring / (nvlink_gbs * 1e9) * 1e6)
    layer_roof_nvls_us = max(gemm_roof_us, bus_nvls / (nvlink_gbs * 1e9) * 1e6)
    # the CTA cap's cost: the same collective on the uncapped communicator
    uncapped = None
    if world > 1:
        uncapped = [[sz] + [round(x, 1) for x in ctx_seq.time_collective_bw("allreduce", sz, 5)]
                    for sz in (1 << 22, 1 << 23, 1 << 24, S_B)]
    # PAPER.md:622 perfect-overlap bound from the measured pieces: the GEMM
    # (same order, same S) and the collective of the full output / of the last
    # wave on the library's communicator
    comm_full_us = ctx.time_collective("allreduce", S_B, 5)
    last_wave_bytes = (tiles_c - (T - 1) * S) * BMc * BNc * 2
    comm_last_us = ctx.time_collective("allreduce", last_wave_bytes, 5)
    if gk_us >= comm_full_us:
        pob_us = gk_us + comm_last_us
    else:
        pob_us = gk_us / T + comm_full_us
    traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "gemm_traffic.json")))
        ts_key = "/ts" if (spec.get("options") or {}).get("tail_split") else ""
        traffic = tr.get(f"{M}x{N}x{K}/{BMc}x{BNc}/S{S}{ts_key}")
    except Exception:
        pass

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            us, desc, cores = cpu_oracle_sample(wl, world, args.cpu_seconds)
            cpu = {"value": round(us, 1), "unit": "us", "cores": cores, "kind": "oracle", "sample": desc}
        except Exception as e:  # pragma: no cover
            cpu = {"value": None, "unit": "us", "cores": None, "kind": "oracle", "sample": f"failed: {e}"}

    if rank == 0:
        line = {
            "metric": "overlapped GEMM+AllReduce us per layer",
            "value": round(ov_us, 2), "unit": "us", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ov_us / 1e3, 4), "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded N(0,1) activations, N(0,0.02^2) weights)"
            + ("; EMULATED NVLink (--emulate-world: one GPU, collectives = link-model kernels; NOT a measurement)"
               if emulate else ""),
            "config": {**{k: wl[k] for k in ("workload", "M", "N", "K_loc", "tp", "collective")},
                       "tile": f"{BMc}x{BNc}", "workers": S, "comm_sms": sms - cgc * S,
                       "nccl_max_ctas": getattr(ctx, "nccl_max_ctas", None) if world > 1 else None,
                       "waves": T, "groups": list(groups), "swizzle_order": "auto (DESIGN.md R25)",
                       "tail_split": (spec.get("options") or {}).get("tail_split", 0),
                       "ar_layout": "rowband" if plan.info["ar_layout"] == 1 else "slot",
                       "l2": "flushed (256 MiB write) before every timed step", "parallelism": f"tp{world}",
                       "timing": "device time: CUDA events on the launching stream, pre-loaded by a ~100 us sleep "
                                 "kernel so host enqueue latency (~12 us per call) is excluded; e2e includes it; "
                                 "value = median of the timed steps (each the max over ranks), step_stats_us has "
                                 "mean/p10/p90"},
            "note": ("N=1: the overlapped op is the GEMM followed by a 1-rank NCCL AllReduce that moves no data, so "
                     "speedup_vs_sequential is ~1 by construction; the multi-rank exchange runs at N>1"
                     if world == 1 else f"TP={world}: every rank's GEMM overlaps its wave groups' NCCL AllReduce"),
            "speedup_vs_sequential": round(seq_us / ov_us, 4), "sequential_us": round(seq_us, 2),
            "sequential_config": ("the overlapped plan's GEMM writing row-major C, then one NCCL AllReduce"
                                  if world == 1 else
                                  f"GEMM alone at its best wave width (S={seqplan.info['workers']} CTA pairs"
                                  f"{', split tail' if K >= 3584 else ''}), then one NCCL AllReduce on a "
                                  "communicator with NCCL's default CTA count"),
            # SURVEY ambiguity 17 / DESIGN R17: strict (incl. the post-communication
            # reorder; the headline), the paper's (excl. it) and the fused op
            "latency_conventions": {
                "strict_us": round(ov_us, 2),
                "paper_us": round(ov_us, 2) if plan.info["ar_layout"] == 1 else None,
                "fused_us": round(m["ov_norm"], 2), "fused_sequential_us": round(m["seq_norm"], 2),
                "note": ("ROWBAND plan: the AllReduce runs in place in C, no post-communication reorder exists, so "
                         "the strict and the paper convention coincide" if plan.info["ar_layout"] == 1 else
                         "slot plan: the per-group reorder overlaps the later groups; excluded time not separable")},
            "tflops": round(world * flops / (ov_us * 1e-6) / 1e12, 1),
            "layer_roofline_us": round(layer_roof_us, 2), "frac_of_layer_roofline": round(layer_roof_us / ov_us, 4),
            "layer_roofline": {"gemm_us": round(gemm_roof_us, 2),
                               "allreduce_ring_us": round(bus_ring / (nvlink_gbs * 1e9) * 1e6, 2),
                               "allreduce_nvls_us": round(bus_nvls / (nvlink_gbs * 1e9) * 1e6, 2),
                               "max_ring_us": round(layer_roof_us, 2), "max_nvls_us": round(layer_roof_nvls_us, 2),
                               "nvlink_gbs": nvlink_gbs, "nvlink_source": nvlink_src,
                               "tensor_peak_tflops": peak, "tensor_peak_source": f"{peak_src} bf16_tflops (burst)"},
            "perfect_overlap_bound_us": round(pob_us, 2), "frac_of_perfect_overlap": round(pob_us / ov_us, 4),
            "perfect_overlap_inputs": {"gemm_us": round(gk_us, 2), "comm_full_us": round(comm_full_us, 2),
                                       "comm_last_wave_us": round(comm_last_us, 2), "waves": T,
                                       "rule": "PAPER.md:622: GEMM + last-wave comm if GEMM-bound, else "
                                               "first-wave GEMM + full comm"},
            "step_stats_us": {k: main_stats.get(k) for k in ("ov", "seq", "gemm", "cublas")},
            "nccl_allreduce_curve": ({"unit": "bytes, algbw GB/s, busbw GB/s (nccl-tests convention)",
                                      "comm": f"library communicator, maxCTAs="
                                              f"{getattr(ctx, 'nccl_max_ctas', 0) if world > 1 else 'default'}",
                                      "points": [[int(b), round(a, 1), round(bb, 1)] for b, a, bb in curve_bw]}
                                     if curve_bw else None),
            "nccl_allreduce_uncapped": ({"unit": "bytes, us, busbw GB/s", "comm": "NCCL default CTA count",
                                         "points": uncapped} if uncapped else None),
            "alg1_predicted_us": round(pred, 2), "spot_check": spot,
            "fused_add_rmsnorm": {"overlapped_us": round(m["ov_norm"], 2), "sequential_us": round(m["seq_norm"], 2),
                                  "speedup": round(m["seq_norm"] / m["ov_norm"], 4), "groups": list(groups_n),
                                  "workers": nspec["workers"],
                                  "layout": "rowband" if nplan.info["ar_layout"] == 1 else "slot",
                                  "alg1_predicted_us": round(pred_n, 2),
                                  "note": "GEMM+AR+residual add+RMSNorm; " + (
                                      "overlapped runs the fused op per row band right after its collective"
                                      if len(groups_n) > 1 and nplan.info["ar_layout"] == 1 else
                                      "the tuner's fastest plan has one group: the fused op runs once after "
                                      "the collective (as in the sequential form)")},
            "roofline": {"bound": "tensor", "kernel": f"fo_gemm_tcgen05_kernel<{BNc},{cgc}>", "achieved": round(achieved, 1),
                         "peak": peak, "unit": "TFLOP/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                         "traffic_source": "dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed "
                                           "ncu --set full capture of this shape/plan (profiles/gemm_traffic.json)"
                                           if traffic else None,
                         "peak_source": f"{peak_src} bf16_tflops (burst; kernel timed alone per step)",
                         "frac_of_sustained_peak": round(achieved / peaks.get("bf16_tflops_sustained", peak), 4),
                         "kernel_us": round(gk_us, 2), "flops_per_launch": flops,
                         "cublas_us": round(cb_us, 2), "frac_of_cublas_same_loop": round(cb_us / gk_us, 4)},
            "cpu_baseline": cpu,
            "e2e": {"value": round(e2e_us, 1), "unit": "us",
                    "h2d_bytes_per_step": int(M * K * 2), "d2h_bytes_per_step": int(M * N * 2),
                    "latency_us": round(e2e_lat_us, 1), "steps_back_to_back": n_e2e,
                    "workers": S_e, "groups": [1] * T_e, "ar_layout": "rowband",
                    "note": "fo_run_host per step: activations A host->device (pinned; 8 tile-row chunks "
                            "the GEMM producer waits on), output device->host per row band right after "
                            "its collective; weights resident in HBM. value = per-step time of steps "
                            "issued back to back (two staging sets: a step's H2D overlaps the previous "
                            "step), latency_us = one step alone"},
            "shard_layers_n1": shards or None,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    for c in {id(x): x for x in ctxs + [ctx_seq]}.values():   # every distinct context once
        c.close()
    if use_dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
