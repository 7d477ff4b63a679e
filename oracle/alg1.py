"""Oracle for the offline tuner: Alg. 1 "Grouping tuning algorithm"
(PAPER.md:451-489), the design space, its pruning
 and the perfect-overlap bound.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Readings: R13 - at i = 1 the previous group G_0 does not exist and
its communication latency is 0; R14 - `duration` is the GEMM duration measured
at the actual wave width S, T = ceil(tiles / S); R15 - the bandwidth curve is
interpolated linearly in log2(bytes) and clamped at its end points; R16 -
ties go to fewer groups, then the lexicographically smaller partition.

Pins (tests/test_oracle_alg1.py): |space| = 2^(T-1), T=8 -> 128;
(1,2,2) and (2,3) are in the T=5 space; pruned sizes for
T=1..12 by an independent count; hand traces of the recurrence
((1,1,1,1) -> 50, (4) -> 80, comm-bound (1,1,1,1) -> 85 = the
PAPER.md:622 bound); single group == GEMM + full comm; the bytes -> us
conversion of interp_latency_us by hand (1 MB at 1 GB/s = 1000 us, 4 MB at
400 GB/s = 10 us); both branches of perfect_overlap_bound by hand values of
PAPER.md:622's sentence, and its GEMM-bound branch attained by the finest
partition when each wave's communication hides under the next wave.
"""
from __future__ import annotations

import math


def candidates(T: int):
    """All partitions: a binary communicate/not decision after each of the
    waves W_1..W_{T-1}; W_T always communicates."""
    out = []
    for mask in range(1 << (T - 1)):
        part, run = [], 0
        for w in range(T):
            run += 1
            last = (w == T - 1)
            if last or (mask >> w) & 1:
                part.append(run)
                run = 0
        out.append(tuple(part))
    return out


def pruned_candidates(T: int, S1: int = 2, SP: int = 4):
    """|G_1| <= S1 and |G_P| <= SP.  For T = 1 the single
    group is both first and last; it is kept whatever the caps (the space must
    not be empty)."""
    if T == 1:
        return [(1,)]
    return [c for c in candidates(T) if c[0] <= S1 and c[-1] <= SP]


def interp_bandwidth(curve, nbytes: float) -> float:
    """curve: list of (bytes, GB/s) with strictly increasing bytes.  Linear in
    log2(bytes) between samples, clamped outside (R15)."""
    xs = [math.log2(b) for b, _ in curve]
    ys = [bw for _, bw in curve]
    x = math.log2(nbytes)
    if x <= xs[0]:
        return ys[0]
    if x >= xs[-1]:
        return ys[-1]
    for k in range(len(xs) - 1):
        if xs[k] <= x <= xs[k + 1]:
            f = (x - xs[k]) / (xs[k + 1] - xs[k])
            return ys[k] + f * (ys[k + 1] - ys[k])
    raise AssertionError("unreachable")


def interp_latency_us(curve, nbytes: float) -> float:
    """Alg. 1 line 14: latency of a message of `nbytes` (0 bytes -> 0 us)."""
    if nbytes <= 0:
        return 0.0
    return nbytes / (interp_bandwidth(curve, nbytes) * 1e9) * 1e6


def group_bytes(partition, S: int, ntiles: int, tile_bytes: int):
    """get_data_size(G): bytes of the tiles in each group (the last wave may be partial)."""
    out, W = [], 0
    for g in partition:
        lo = S * W
        W += g
        hi = min(S * W, ntiles)
        out.append((hi - lo) * tile_bytes)
    return out


def predict(partition, duration_us: float, T: int, sizes, comm_latency) -> float:
    """Alg. 1 lines 10-22 for one candidate G.

    sizes[i]: data size of group i; comm_latency(bytes) -> us."""
    t_acc_p = 0.0
    t_acc_m = 0.0
    for i, g in enumerate(partition):
        t_m = comm_latency(sizes[i - 1]) if i > 0 else 0.0       # lines 12-14 (R13)
        t_p = duration_us / T * g                                 # line 16
        t_acc_m = max(t_acc_p, t_acc_m) + t_m                     # line 18 (old t_acc_p)
        t_acc_p = t_acc_p + t_p
    t_acc_m = max(t_acc_p, t_acc_m) + comm_latency(sizes[-1])     # lines 20-21
    return t_acc_m


def search(T: int, duration_us: float, sizes_of, comm_latency, S1=2, SP=4, prune=True):
    """Alg. 1 lines 7-26: argmin of the prediction over the (pruned) candidates.
    sizes_of(partition) -> per-group data sizes.  Tie-break R16."""
    cands = pruned_candidates(T, S1, SP) if prune else candidates(T)
    best, best_t = None, math.inf
    for G in cands:
        t = predict(G, duration_us, T, sizes_of(G), comm_latency)
        key = (t, len(G), G)
        if best is None or key < (best_t, len(best), best):
            best, best_t = G, t
    return best, best_t


def perfect_overlap_bound(duration_us: float, T: int, comm_full_us: float, comm_last_wave_us: float) -> float:
    """GEMM + last-wave communication if GEMM takes more time,
    else first-wave GEMM + the full communication."""
    if duration_us >= comm_full_us:
        return duration_us + comm_last_wave_us
    return duration_us / T + comm_full_us


# ------------------------------------------------------------------ A2A imbalance extension
def predict_multi(partition, durations, wave_bytes, comm_latency) -> float:
    """"the prediction algorithm is extended by taking the maximum
    across all GPUs for the accumulated latencies (t_p^acc and t_m^acc)".

    Reading R26: every rank r runs the same wave partition over T
    waves (experts padded to a common tile count), with its own GEMM duration
    durations[r] and its own A2A bytes per wave wave_bytes[r][w].  Alg. 1's
    loop runs per rank from the shared (maxed) accumulators, and after every
    step each accumulator is the maximum over the ranks."""
    R = len(durations)
    T = len(wave_bytes[0])
    bounds, W = [], 0
    for g in partition:
        bounds.append((W, W + g))
        W += g
    if W != T:
        raise ValueError("partition does not cover the T waves")

    def t_m(r, i):  # comm latency of group i on rank r
        lo, hi = bounds[i]
        return comm_latency(sum(wave_bytes[r][lo:hi]))

    t_acc_p = [0.0] * R
    t_acc_m = 0.0
    for i, g in enumerate(partition):
        p_max = max(t_acc_p)
        t_acc_m = max(max(p_max, t_acc_m) + (t_m(r, i - 1) if i > 0 else 0.0) for r in range(R))
        t_acc_p = [t_acc_p[r] + durations[r] / T * g for r in range(R)]
    p_max = max(t_acc_p)
    return max(max(p_max, t_acc_m) + t_m(r, len(partition) - 1) for r in range(R))


def search_multi(T, durations, wave_bytes, comm_latency, S1=2, SP=4, prune=True):
    """Argmin of predict_multi over the (pruned) candidates; tie-break R16."""
    cands = pruned_candidates(T, S1, SP) if prune else candidates(T)
    best, best_t = None, math.inf
    for G in cands:
        t = predict_multi(G, durations, wave_bytes, comm_latency)
        if best is None or (t, len(G), G) < (best_t, len(best), best):
            best, best_t = G, t
    return best, best_t
