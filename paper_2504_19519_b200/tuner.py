"""Offline tuner driver (Alg. 1) and the pre-searched plan
cache with nearest-neighbour reuse for unseen sizes (NEXT f1).

Offline stage:
  (1) computation - the GEMM duration of our persistent kernel at wave width S
      (measured with CUDA events, L2 flushed), T = ceil(tiles / S);
  (2) communication - the (bytes, GB/s) curve of the collective, sampled at
      log-spaced sizes on the process group's NCCL (world 1: no exchange);
  (3) resource contention - S = SMs left after `comm_sms` (Alg. 1 line 3).
Online stage: fo_tune_search (C++, enumeration or the exact DP, R24).

The cache is a JSON file keyed "MxNxK/coll/g<world>"; a miss reuses the
nearest cached shape when its distance |dlog2 M| + |dlog2 N| + |dlog2 K| is at
most 1.5 (SPEC.md:339 idea), else tunes and stores.
"""
from __future__ import annotations

import json
import math
import os
from dataclasses import asdict, dataclass, field
from typing import Callable, Optional

from . import Plan, device_sm_count, gemm_stage, tune_predict, tune_search

TILE_M, TILE_N = 256, 256


@dataclass
class TunedPlan:
    M: int
    N: int
    K: int
    coll: str
    world: int
    tile_m: int
    tile_n: int
    workers: int
    swizzle: int
    groups: list
    predicted_us: float
    gemm_us: float
    curve: list = field(default_factory=list)
    source: str = "tuned"  # "tuned" | "neighbour:<key>"

    def spec(self) -> dict:
        return dict(coll=self.coll, m=self.M, n=self.N, k=self.K, tile_m=self.tile_m, tile_n=self.tile_n,
                    workers=self.workers, swizzle=self.swizzle, group_waves=list(self.groups))


def key_of(M, N, K, coll, world) -> str:
    return f"{M}x{N}x{K}/{coll}/g{world}"


def default_workers(tiles: int, sms: int, cg: int = 2) -> int:
    """Fewest workers with the wave count of the full GPU (the freed SMs are left to NCCL)."""
    t_full = -(-tiles // max(1, sms // cg))
    return -(-tiles // t_full)


def measure_gemm_us(M, N, K, workers, swizzle=0, tile_m=TILE_M, tile_n=TILE_N, iters=10) -> float:
    """Offline stage (1): our GEMM's duration at wave width S (CUDA events, L2 flushed)."""
    import torch

    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    Bt = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
    C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    plan = Plan(coll="nocomm", m=M, n=N, k=K, tile_m=tile_m, tile_n=tile_n, workers=workers, swizzle=swizzle)
    for _ in range(3):
        gemm_stage(plan, A, Bt, C)
    tot = 0.0
    for _ in range(iters):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        gemm_stage(plan, A, Bt, C)
        e.record()
        torch.cuda.synchronize()
        tot += s.elapsed_time(e) * 1e3
    return tot / iters


def sample_curve(coll: str, group=None, sizes=None, iters=5, ctx=None) -> list:
    """Offline stage (2): NCCL bandwidth vs message size.  With `ctx`, on the
    library's own communicator and comm stream (its CTA cap included — what the
    hot path will see); else on the torch.distributed group.  World 1 without a
    context has no exchange: a flat, very high curve."""
    import torch
    import torch.distributed as dist

    if ctx is not None:
        return ctx.sample_curve(coll, sizes, iters)
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return [(1 << 10, 1e6), (1 << 30, 1e6)]
    n = dist.get_world_size(group)
    sizes = sizes or [1 << s for s in range(16, 28)]
    out = []
    for sz in sizes:
        x = torch.empty(sz // 2, dtype=torch.bfloat16, device="cuda")
        y = torch.empty(sz // 2 // n, dtype=torch.bfloat16, device="cuda")

        def op():
            if coll == "reducescatter":
                dist.reduce_scatter_tensor(y, x, group=group)
            else:
                dist.all_reduce(x, group=group)

        for _ in range(2):
            op()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(iters):
            op()
        e.record()
        torch.cuda.synchronize()
        t_us = s.elapsed_time(e) * 1e3 / iters
        out.append((sz, sz / (t_us * 1e-6) / 1e9))
    return out


def tune(M, N, K, coll="allreduce", world=1, comm_sms=None, group=None, swizzle=0, device=0, ctx=None) -> TunedPlan:
    """Run the offline + online stages of Alg. 1 for one layer shape."""
    sms = device_sm_count(device)
    tiles = (M // TILE_M) * (N // TILE_N)
    S = default_workers(tiles, sms) if comm_sms is None else (sms - comm_sms) // 2
    dur = measure_gemm_us(M, N, K, S, swizzle)
    curve = sample_curve(coll, group, ctx=ctx)
    groups, pred = tune_search(dur, tiles, S, TILE_M * TILE_N * 2, curve)
    return TunedPlan(M, N, K, coll, world, TILE_M, TILE_N, S, swizzle, list(groups), pred, dur, curve)


def distance(a, b) -> float:
    return sum(abs(math.log2(x) - math.log2(y)) for x, y in zip(a, b))


class PlanCache:
    """Pre-searched plans for representative sizes + nearest-neighbour reuse
    ("pre-search for representative GEMM sizes, and apply
    nearest-neighbor matching for unseen cases during execution")."""

    def __init__(self, path: Optional[str] = None, threshold: float = 1.5):
        self.path, self.threshold = path, threshold
        self.entries: dict = {}
        if path and os.path.exists(path):
            with open(path) as f:
                self.entries = json.load(f)

    def save(self):
        if self.path:
            with open(self.path, "w") as f:
                json.dump(self.entries, f, indent=1, sort_keys=True)

    def put(self, tp: TunedPlan):
        self.entries[key_of(tp.M, tp.N, tp.K, tp.coll, tp.world)] = asdict(tp)

    def nearest(self, M, N, K, coll, world):
        best, best_d = None, math.inf
        for k, e in self.entries.items():
            if e["coll"] != coll or e["world"] != world:
                continue
            d = distance((M, N, K), (e["M"], e["N"], e["K"]))
            if d < best_d or (d == best_d and best is not None and k < best[0]):
                best, best_d = (k, e), d
        return best, best_d

    def lookup_or_tune(self, M, N, K, coll="allreduce", world=1,
                       tuner: Callable[..., TunedPlan] = tune, **kw) -> TunedPlan:
        k = key_of(M, N, K, coll, world)
        if k in self.entries:
            return TunedPlan(**self.entries[k])
        near, d = self.nearest(M, N, K, coll, world)
        if near is not None and d <= self.threshold:
            e = dict(near[1])
            tp = TunedPlan(**e)
            # reuse the neighbour's choices (workers, swizzle, groups) if they fit this shape
            tiles = (M // tp.tile_m) * (N // tp.tile_n)
            T = -(-tiles // tp.workers)
            if sum(tp.groups) == T:
                return TunedPlan(M, N, K, coll, world, tp.tile_m, tp.tile_n, tp.workers, tp.swizzle, tp.groups,
                                 tp.predicted_us, tp.gemm_us, tp.curve, f"neighbour:{near[0]}")
        tp = tuner(M, N, K, coll=coll, world=world, **kw)
        self.put(tp)
        self.save()
        return tp


def a2a_wave_bytes(specs: list, elem_bytes: int = 2):
    """Per-rank, per-wave bytes each rank sends off-rank in an All-to-All plan
    set (the census of PAPER.md:392, one plan per wave): [ranks][T]."""
    import numpy as np

    from . import Plan

    n = len(specs)
    out = []

    def waves(s):
        return -(-(s["m"] // s["tile_m"]) * (s["n"] // s["tile_n"]) // s["workers"])
    # experts with no rows (m = 0, R45) send nothing in every wave
    Ts = {waves(s) for s in specs if s["m"] > 0}
    if len(Ts) > 1:
        raise ValueError("imbalance-aware search needs a common wave count (pad experts to a common tile count)")
    Tc = Ts.pop() if Ts else 0
    per_wave = [dict(s, group_waves=[1] * Tc if s["m"] > 0 else [0] * Tc) for s in specs]
    for r, sp in enumerate(specs):
        plan = Plan(rank=r, world=n, peers=per_wave, **per_wave[r])
        sc, _ = plan.export_a2a_counts()          # [T, n] subtokens per (wave, destination)
        sc = sc.astype(np.float64)
        sc[:, r] = 0.0                            # the self part is a local copy
        out.append((sc.sum(axis=1) * sp["tile_n"] * elem_bytes).tolist())
    return out


def tune_alltoall(specs: list, durations: list, curve: list, s1=2, sp=4, prune=True):
    """A2A imbalance extension of Alg. 1 (R26): one
    common partition for all expert ranks from their GEMM durations and their
    per-wave send bytes."""
    from . import tune_search_multi

    wb = a2a_wave_bytes(specs)
    return tune_search_multi(durations, wb, curve, s1=s1, sp=sp, prune=prune)


def effective_curve(curve: list, post_us_per_byte: float, post_fixed_us: float = 0.0) -> list:
    """Fold a per-group post-communication op (the fused add / RMSNorm that runs
    right after each group's collective) into the bandwidth curve Alg. 1 sees:
    the latency of a group of b bytes becomes collective(b) + post(b), with
    post(b) = post_fixed_us + post_us_per_byte * b (measured offline)."""
    out = []
    for b, bw in curve:
        t = b / (bw * 1e9) * 1e6 + post_fixed_us + post_us_per_byte * b
        out.append((b, b / (t * 1e-6) / 1e9))
    return out


def insitu_curve(ctx, spec: dict, A, Bt, out, T: int, S: int, tile_bytes: int, base_curve: list,
                 group_sizes=(1, 2, 4), iters: int = 3, run_args=()) -> list:
    """Offline stage (3), resource contention, measured: the
    comm-stream work of a group while the GEMM runs.  For g in `group_sizes`
    (waves) the layer runs with groups (g, T-g); the comm stream's timestamps
    around group 0's collective (+ its per-group post pass, when `spec` has a
    fused op: then `run_args` = (residual, gamma)) give its in-situ latency at
    g waves' bytes — group 0 never queues behind an earlier group's work.
    Those points replace the standalone curve's samples in their size range;
    the standalone samples above it stay (groups that large run mostly after
    the GEMM).  DESIGN.md R42.  spec: the layer's fo.Plan keyword arguments
    without group_waves."""
    import statistics

    import torch

    from . import Plan, run
    pts = []
    for g in group_sizes:
        if g >= T:
            break
        plan = Plan(group_waves=[g, T - g], **spec)
        ts = torch.zeros(4, dtype=torch.int64, device="cuda")
        plan.set_debug(None, ts)
        d = []
        for _ in range(iters):
            run(ctx, plan, A, Bt, out, *run_args)
            torch.cuda.synchronize()
            t = ts.cpu().tolist()
            d.append((t[1] - t[0]) / 1e3)
        plan.close()
        b = g * S * tile_bytes
        pts.append((b, b / (statistics.median(d) * 1e-6) / 1e9))
    if not pts:
        return list(base_curve)
    lo, hi = min(p[0] for p in pts), max(p[0] for p in pts)
    keep = [(b, bw) for b, bw in base_curve if b < lo or b > hi]
    return sorted(keep + pts)


def predict_insitu(groups, duration_us, tiles, S, tile_bytes, icurve, base_curve) -> float:
    """Alg. 1's prediction with the in-situ curve for the groups whose
    comm-stream work overlaps the GEMM and the standalone curve for the last
    group, which runs after the GEMM (R42).  The recurrence adds the last
    group's latency as its final term (t = max(acc_p, acc_m) + t_m(G_P)), so
    swapping that one term is exact."""
    G = list(groups)
    pred = tune_predict(G, duration_us, tiles, S, tile_bytes, icurve)
    last = tiles - S * (sum(G) - G[-1])
    if last <= 0:
        return pred
    # a one-group prediction with zero duration is exactly that group's latency
    lat_i = tune_predict([G[-1]], 0.0, last, S, tile_bytes, icurve)
    lat_b = tune_predict([G[-1]], 0.0, last, S, tile_bytes, base_curve)
    return pred - lat_i + lat_b


# collectives with a ROWBAND layout (AR: in place; RS: scattered straight into
# the output, R40)
BANDED = ("allreduce", "reducescatter")


@dataclass
class LayerChoice:
    workers: int
    swizzle: int
    groups: list
    layout: str          # "rowband" | "slot" (AllReduce / ReduceScatter) | "auto" (All-to-All)
    predicted_us: float
    gemm_us: float
    candidates: list     # (workers, tile:layout[+tailsplit], groups, predicted_us, gemm_us[, measured_us])
    tail_split: int = 0  # FO_OPT_TAIL_SPLIT of the chosen plan (0 off, -1 auto)
    tile_m: int = TILE_M
    tile_n: int = TILE_N
    curve: list = field(default_factory=list)  # (bytes, algbw GB/s, busbw GB/s) on the chosen context's communicator
    ctx_index: int = 0   # which of the contexts passed to tune_layer (their NCCL CTA caps) the plan runs on

    def spec(self, M, N, K, coll, post="none") -> dict:
        d = dict(coll=coll, m=M, n=N, k=K, tile_m=self.tile_m, tile_n=self.tile_n, workers=self.workers,
                 swizzle=self.swizzle, group_waves=list(self.groups),
                 ar_layout=self.layout if coll in BANDED else "auto", post=post)
        if self.tail_split:
            d["options"] = {"tail_split": self.tail_split}
        return d


def candidate_workers(tiles: int, Nt: int, sms: int, coll: str, cg: int = 2) -> list:
    """Offline stage (3) candidates for the wave width S (T is set
    by the SMs the collective leaves): the fewest workers with the full GPU's
    wave count, the full GPU, and (AllReduce / ReduceScatter) the widest S whose
    waves are whole tile-rows (groups are then row bands: no reorder at all,
    DESIGN.md H11a, R40)."""
    smax = sms // cg
    cands = {default_workers(tiles, sms, cg), min(smax, tiles)}
    if coll in BANDED and Nt <= smax:
        cands.add((smax // Nt) * Nt)
    return sorted(c for c in cands if c >= 1)


def compositions(T: int) -> list:
    """All 2^(T-1) partitions of T waves into consecutive groups."""
    out = []
    for mask in range(1 << max(T - 1, 0)):
        part, run = [], 0
        for w in range(T):
            run += 1
            if w == T - 1 or (mask >> w) & 1:
                part.append(run)
                run = 0
        out.append(part)
    return out


def tune_layer(M, N, K, ctx, coll="allreduce", post="none", tile_m=TILE_M, tile_n=TILE_N, device=0,
               sizes=None, iters=10, min_comm_sms=16, verify=8, all_partitions_T=7,
               tile_shapes=None, insitu=None) -> LayerChoice:
    """Joint choice of S (wave width), layout and wave groups for one layer
    (AllReduce / ReduceScatter; world from the context).

    For each candidate S and layout: measure the GEMM in that plan's execution
    order (offline stage (1)), use the collective's curve sampled on the
    context's communicator (stage (2)), fold the per-group post work into it
    (R28: the reorder of a slot layout and/or the fused op), run Alg. 1, and
    add any post pass that cannot run per group (RMSNorm on a slot layout).
    For T <= all_partitions_T every partition is predicted (not only Alg. 1's
    pick); the `verify` best predictions over all (S, layout, partition) are
    then run for real (fo_run) and the fastest wins: the predictor does not
    model the contention between the GEMM and per-group post kernels.  At world > 1 every decision is rank 0's
    (broadcast over the default process group) so all ranks build the same
    plan.

    `ctx` may be a list of contexts on the same ranks whose communicators
    differ in their NCCL CTA cap (`nccl_max_ctas`): the SM split between the
    persistent GEMM and the collective is then
    searched too — every S that leaves a context's CTAs their SMs is a
    candidate with that context's sampled curve, and the measured
    verification picks the context (`LayerChoice.ctx_index`).

    `insitu` (default: world > 1, or a fused op): Alg. 1 sees the collective's
    (+ per-group op's) curve sampled while the GEMM runs on the candidate's S
    workers (insitu_curve, R42) for the group sizes that overlap the GEMM —
    measured on emulated NVLink it cuts the prediction error from 6.7% to 3.0%
    and the pick reaches the measured optimum
    (profiles/r02_predictor_emulated.txt)."""
    import torch

    from . import post_stage

    sms = device_sm_count(device)
    ctxs = list(ctx) if isinstance(ctx, (list, tuple)) else [ctx]
    ctx = ctxs[0]
    world = ctx.world
    caps = [int(getattr(c, "nccl_max_ctas", 0) or 0) for c in ctxs]
    # tile shapes searched (PAPER.md:460 leaves the GEMM configuration to the
    # tuner): those that tile the output and, for RS, split by world
    shapes = [(tm, tn) for tm, tn in (tile_shapes or [(tile_m, tile_n)])
              if M % tm == 0 and N % tn == 0 and (coll != "reducescatter" or tm % world == 0)]
    if not shapes:
        raise ValueError("no tile shape divides the layer")
    curves_bw = [c.sample_curve_bw(coll, sizes or [1 << s for s in range(18, 28)], iters=3) for c in ctxs]
    curves = [[(b, alg) for b, alg, _ in cb] for cb in curves_bw]

    def ctx_ok(ci, S, cg):
        """S leaves the SMs context ci's collective needs (world 1: anything)."""
        if world == 1:
            return True
        return sms - cg * S >= max(min_comm_sms, caps[ci])
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    Bt = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
    out_rows = M if coll == "allreduce" else M // world
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    res = torch.randn(out_rows, N, device="cuda").to(torch.bfloat16)
    gam = torch.randn(N, device="cuda").to(torch.bfloat16)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def timeit_many(fns, rounds):
        """Device time of each fn: round-robin (one flushed run of each per
        round) with the stream pre-loaded by a sleep kernel, medians — clock /
        power drift hits every candidate alike and host enqueue is excluded."""
        for f in fns:
            for _ in range(2):
                f()
        torch.cuda.synchronize()
        ts = [[] for _ in fns]
        for _ in range(rounds):
            for i, f in enumerate(fns):
                flush.zero_()
                s0, e0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda._sleep(200_000)
                s0.record()
                f()
                e0.record()
                torch.cuda.synchronize()
                ts[i].append(s0.elapsed_time(e0) * 1e3)
        return [sorted(v)[len(v) // 2] for v in ts]

    post_cache = {}

    def post_us(layout, op, tm, tn):
        """Full-output post pass of `layout` with `op`, measured standalone."""
        if op == "none" and layout == "rowband":
            return 0.0
        key = (layout, op, tm, tn)
        if key not in post_cache:
            t_ = (M // tm) * (N // tn)
            pl = Plan(coll=coll, m=M, n=N, k=64, tile_m=tm, tile_n=tn, workers=min(t_, sms // max(1, tm // 128)),
                      swizzle=1, ar_layout=layout if coll in BANDED else "auto", post=op, rank=ctx.rank,
                      world=world)
            recv = torch.zeros(pl.info["recv_elems"], dtype=torch.bfloat16, device="cuda")
            o = torch.empty(pl.info["out_rows"], N, dtype=torch.bfloat16, device="cuda")
            post_cache[key] = timeit_many([lambda: post_stage(pl, recv, o, res, gam)], iters)[0]
        return post_cache[key]

    out_bytes = out_rows * N * 2
    layouts = ("rowband", "slot") if coll in BANDED else ("auto",)
    evaluated = []
    # offline stage (1): the GEMM in each candidate's execution order, all
    # candidates (tile shape x S x layout x tail split) timed together
    probes = []
    for tm, tn in shapes:
        Nt = N // tn
        tiles = (M // tm) * Nt
        cg = max(1, tm // 128)
        cands = candidate_workers(tiles, Nt, sms, coll, cg)
        full = set()
        if world > 1:
            # the collective's kernels need SMs the persistent GEMM leaves free
            # (Alg. 1 line 3); without them nothing overlaps.  Each context's
            # widest S that leaves its CTAs their SMs is a candidate too
            allc = set(cands)
            cands = sorted(allc | {(sms - max(min_comm_sms, c)) // cg for c in caps})
            cands = [c for c in cands if c >= 1 and any(ctx_ok(ci, c, cg) for ci in range(len(ctxs)))] \
                or [min(cands)]
            # a single group overlaps nothing: the whole GEMM, then the
            # collective with every SM — so the wave widths that leave NCCL no
            # SMs are candidates for it alone, on any context (the plan is then
            # the sequential one and the tuner never picks worse than it)
            full = {c for c in allc if c not in cands}
            cands = sorted(set(cands) | full)
        for S in cands:
            T = -(-tiles // S)
            for layout in layouts:
                # multi-group ROWBAND needs waves of whole tile-rows; one group of
                # every tile is a band (the whole output) for any S and order
                single_only = (layout == "rowband" and S % Nt != 0) or S in full
                swz = 1 if (layout == "rowband" and not single_only) else 0
                probe = Plan(coll=coll, m=M, n=N, k=K, tile_m=tm, tile_n=tn, workers=S, swizzle=swz,
                             group_waves=[T], ar_layout=layout if layout != "auto" else "auto", rank=ctx.rank,
                             world=world)
                # the last partial wave split along K over the idle workers
                # (FO_OPT_TAIL_SPLIT auto: when 2R <= S for R tail tiles)
                R = tiles - (T - 1) * S
                for split in ((0, -1) if 0 < R and 2 * R <= S and K >= 128 else (0,)):
                    gp = Plan(coll="nocomm", m=M, n=N, k=K, tile_m=tm, tile_n=tn, workers=S,
                              tile_order=probe.export_order(), options={"tail_split": split} if split else None)
                    probes.append((S, T, layout, single_only, swz, gp, split, tm, tn, tiles))
    durs = timeit_many([(lambda gp=pr[5]: gemm_stage(gp, A, Bt, out)) for pr in probes], iters)
    # in-situ curves (R42): at world > 1, and wherever a fused op runs per
    # group beside the GEMM (its cost there is bounded by the free SMs, far
    # above its standalone cost: profiles/r02_band_post_probe.txt)
    use_insitu = (world > 1 or post != "none") if insitu is None else bool(insitu)
    icurves = {}

    def curve_for(ci, S, T, layout, swz, tm, tn, op, base):
        """`base` (the context's curve with the per-group op folded in),
        contended by the GEMM at this S: the in-situ points of group 0's
        comm-stream work incl. the op (R42), cached per (context, S, tile,
        layout, op)."""
        if not use_insitu or T < 2:
            return base
        key = (ci, S, tm, tn, layout, op)
        if key not in icurves:
            sp = dict(coll=coll, m=M, n=N, k=K, tile_m=tm, tile_n=tn, workers=S, swizzle=swz,
                      ar_layout=layout if layout != "auto" else "auto", rank=ctx.rank, world=world, post=op)
            icurves[key] = insitu_curve(ctxs[ci], sp, A, Bt, out, T, S, tm * tn * 2, base, iters=3,
                                        run_args=(res, gam) if op != "none" else ())
        return icurves[key]
    for (S, T, layout, single_only, swz, _, split, tm, tn, tiles), dur in zip(probes, durs):
        norm = post in ("add_rmsnorm", "add_rmsnorm_res")
        per_group_op = post if (layout == "rowband" or not norm) else "none"
        per_group = post_us(layout if layout != "auto" else "slot", per_group_op, tm, tn) / out_bytes
        tail = post_us("slot", post, tm, tn) if (layout != "rowband" and norm) else 0.0
        for ci in range(len(ctxs)):
            if not single_only and not ctx_ok(ci, S, max(1, tm // 128)):
                continue
            # (a single group does not overlap the GEMM: the standalone curve)
            base = effective_curve(curves[ci], per_group)
            eff = base if single_only else curve_for(ci, S, T, layout, swz, tm, tn, per_group_op, base)
            if single_only:
                pred = tune_predict([T], dur, tiles, S, tm * tn * 2, eff)
                evaluated.append((S, layout, [T], pred + tail, dur, swz, split, tm, tn, ci))
                continue
            G, pred = tune_search(dur, tiles, S, tm * tn * 2, eff)
            if eff is not base:   # in-situ curve: the last group is charged at the standalone one
                pred = predict_insitu(G, dur, tiles, S, tm * tn * 2, eff, base)
            evaluated.append((S, layout, list(G), pred + tail, dur, swz, split, tm, tn, ci))
            if T <= all_partitions_T:
                for comp in compositions(T):
                    if comp != list(G):
                        p2 = (predict_insitu(comp, dur, tiles, S, tm * tn * 2, eff, base) if eff is not base
                              else tune_predict(comp, dur, tiles, S, tm * tn * 2, eff))
                        evaluated.append((S, layout, comp, p2 + tail, dur, swz, split, tm, tn, ci))
    import torch.distributed as dist

    def agree(obj):
        if world > 1 and dist.is_initialized():
            box = [obj]
            dist.broadcast_object_list(box, src=0)
            return box[0]
        return obj

    evaluated = sorted(evaluated, key=lambda e: e[3])
    # the verified set: the best prediction of every (S, layout) (the
    # predictor ranks across wave widths only through noisy GEMM durations),
    # the single-group plan (no overlap: the whole GEMM, then one collective —
    # so the chosen split is never one measured slower than not splitting),
    # then the global ranking, up to `verify` plans
    nv = max(1, verify)
    chosen = []
    for e in evaluated:
        if not any(c[0] == e[0] and c[1] == e[1] and c[6:10] == e[6:10] for c in chosen):
            chosen.append(e)
    single = [e for e in evaluated if len(e[2]) == 1]
    if single:
        best1 = min(single, key=lambda e: (e[1] != "rowband", e[3]))
        if best1 not in chosen:
            chosen.append(best1)
    for e in evaluated:
        if len(chosen) >= nv:
            break
        if e not in chosen:
            chosen.append(e)
    evaluated = chosen + [e for e in evaluated if e not in chosen]
    evaluated, nv = agree((evaluated, len(chosen)))
    from . import run as fo_run

    # verification: the candidates' fo_run timed round-robin, medians
    runs = []
    for (S, layout, G, pred, dur, swz, split, tm, tn, ci) in evaluated[:nv]:
        spec = dict(coll=coll, m=M, n=N, k=K, tile_m=tm, tile_n=tn, workers=S, swizzle=swz,
                    group_waves=G, ar_layout=layout if layout != "auto" else "auto", post=post)
        pl = Plan(rank=ctx.rank, world=world, options={"tail_split": split} if split else None, **spec)
        o = torch.empty(pl.info["out_rows"], N, dtype=torch.bfloat16, device="cuda")
        args = (res, gam) if post != "none" else (None, None)
        runs.append((pl, o, args, ctxs[ci]))
    measured = timeit_many([(lambda r=r: fo_run(r[3], r[0], A, Bt, r[1], *r[2])) for r in runs], max(3, iters))
    if world > 1 and dist.is_initialized():
        tt = torch.tensor(measured, device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        measured = tt.tolist()
    k = min(range(len(measured)), key=lambda i: measured[i])
    best = evaluated[k]
    cands = [(e[0], f"{e[7]}x{e[8]}:" + e[1] + ("+tailsplit" if e[6] else "") +
              (f"+ctas{caps[e[9]]}" if len(ctxs) > 1 else ""), e[2], e[3], e[4]) +
             ((measured[i],) if i < len(measured) else ()) for i, e in enumerate(evaluated)]
    return LayerChoice(best[0], best[5], best[2], best[1], best[3], best[4], cands, best[6], best[7], best[8],
                       curves_bw[best[9]], best[9])
