"""The n > 1 exchange, checked call by call on CPU (no GPU, no NCCL).

fo_run and fo_run_sequential issue exactly the calls of the plan's schedule
(fo_plan_export_calls; runtime.cu exec_calls).  Here every rank's schedule at
world 1..8 is executed by tests/comm_sim.py with NCCL's semantics on numpy
buffers that hold the ORACLE's pre-reordered send buffers (oracle/reorder.py
O5, integer data), and the resulting receive buffers must equal the oracle's
explicit per-group collectives (oracle/collectives.py O6) element for element
(PAPER.md:368 one call per group on its contiguous range; PAPER.md:381-392 the
AR / RS / A2A layouts).  The simulator also fails on anything real NCCL would
hang on or reject: ranks issuing different collective sequences or counts,
unmatched send/recv pairs, ranges outside a buffer.  The sequential schedules
must produce the plain definitions (AR sum; RS contiguous rows, NCCL's
standard layout; A2A all-to-all-v order).
"""
import numpy as np
import pytest

import comm_sim
import paper_2504_19519_b200 as fo
from oracle import collectives as oc
from oracle import plan as op
from oracle import reorder as orr


def _partition(rng, T):
    cuts = sorted(rng.choice(np.arange(1, T), size=rng.integers(0, T), replace=False).tolist()) if T > 1 else []
    bounds = [0] + cuts + [T]
    return [b - a for a, b in zip(bounds[:-1], bounds[1:])]


def _case(rng, world, coll):
    BM = int(rng.choice([128, 256]))
    BN = int(rng.choice([64, 128, 256]))
    Mt, Nt = int(rng.integers(1, 5)), int(rng.integers(1, 5))
    M, N = BM * Mt, BN * Nt
    tiles = Mt * Nt
    S = int(rng.integers(1, tiles + 1))
    T = -(-tiles // S)
    part = _partition(rng, T)
    if rng.random() < 0.5:
        order, swz = rng.permutation(tiles).astype(np.int32), 1
    else:
        order, swz = None, int(rng.integers(1, Mt + 1))
    return BM, BN, M, N, S, part, order, swz


def _oracle_plan(M, N, BM, BN, S, part, order, swz):
    return op.make_plan(M, N, BM, BN, S, part, order=order, swizzle=swz)


def _ints(rng, shape):
    return rng.integers(-4, 5, size=shape).astype(np.float64)


def _lib_plan(rank, world, **spec):
    return fo.Plan(rank=rank, world=world, **spec)


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("layout", ["slot", "rowband"])
def test_allreduce_schedule(world, layout):
    rng = np.random.default_rng(100 + world + (7 if layout == "rowband" else 0))
    for _ in range(12):
        BM, BN, M, N, S, part, order, swz = _case(rng, world, "allreduce")
        if layout == "rowband":
            # raster order, waves of whole tile-rows: every group is a row band
            Nt = N // BN
            S = Nt * int(rng.integers(1, M // BM + 1))
            T = -(-(M // BM) * Nt // S)
            part, order, swz = _partition(rng, T), None, 1
        opl = _oracle_plan(M, N, BM, BN, S, part, order, swz)
        spec = dict(coll="allreduce", m=M, n=N, k=64, tile_m=BM, tile_n=BN, workers=S, tile_order=order,
                    swizzle=swz, group_waves=part, ar_layout=layout)
        plans = [_lib_plan(r, world, **spec) for r in range(world)]
        Ys = [_ints(rng, (M, N)) for _ in range(world)]
        sends = [orr.ar_pre(Y, opl, layout) for Y in Ys]
        want = oc.allreduce_groups(sends, orr.group_elem_ranges(opl, layout))
        bufname = "out" if layout == "rowband" else "send"
        bufs = [{bufname: s.copy()} for s in sends]
        steps = comm_sim.run([p.export_calls(0) for p in plans], bufs)
        assert steps == len(part)                       # one collective per wave group
        for r in range(world):
            np.testing.assert_array_equal(bufs[r][bufname], want[r])
        # sequential: one AllReduce of row-major C in place
        seq = [{"out": Y.reshape(-1).copy()} for Y in Ys]
        assert comm_sim.run([p.export_calls(1) for p in plans], seq) == 1
        total = sum(Ys).reshape(-1)
        for r in range(world):
            np.testing.assert_array_equal(seq[r]["out"], total)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("layout", ["slot", "rowband"])
def test_reducescatter_schedule(world, layout):
    rng = np.random.default_rng(200 + world + (7 if layout == "rowband" else 0))
    for _ in range(12):
        BM, BN, M, N, S, part, order, swz = _case(rng, world, "reducescatter")
        if layout == "rowband":
            # raster order, waves of whole tile-rows: ascending bands (R40)
            Nt = N // BN
            S = Nt * int(rng.integers(1, M // BM + 1))
            T = -(-(M // BM) * Nt // S)
            part, order, swz = _partition(rng, T), None, 1
        opl = _oracle_plan(M, N, BM, BN, S, part, order, swz)
        spec = dict(coll="reducescatter", m=M, n=N, k=64, tile_m=BM, tile_n=BN, workers=S, tile_order=order,
                    swizzle=swz, group_waves=part, ar_layout=layout)
        plans = [_lib_plan(r, world, **spec) for r in range(world)]
        assert all(p.info["ar_layout"] == (1 if layout == "rowband" else 0) for p in plans)
        Ys = [_ints(rng, (M, N)) for _ in range(world)]
        sends = [orr.rs_pre(Y, opl, world, layout) for Y in Ys]
        want = oc.reduce_scatter_groups(sends, orr.group_elem_ranges(opl, layout))
        bufs = []
        for r in range(world):
            if layout == "rowband":
                # the band's rows land in `out` (at one rank the GEMM wrote it: in place)
                b = {"out": sends[r].copy() if world == 1 else np.full(M // world * N, np.nan),
                     "send": sends[r].copy()}
            else:
                b = {"send": sends[r].copy()}
                b["recv"] = b["send"] if world == 1 else np.full(plans[r].info["recv_elems"], np.nan)
            bufs.append(b)
        assert comm_sim.run([p.export_calls(0) for p in plans], bufs) == len(part)
        for r in range(world):
            got = bufs[r]["out" if layout == "rowband" else "recv"][:plans[r].info["recv_elems"]]
            np.testing.assert_array_equal(got, want[r])
            if layout == "rowband":   # received in output order: no post-communication reorder
                np.testing.assert_array_equal(got.reshape(M // world, N), orr.rs_post(want[r], opl, world, layout))
        # sequential: ncclReduceScatter of row-major C -> contiguous rows
        seq = [{"scratch": Y.reshape(-1).copy(), "out": np.full(M // world * N, np.nan)} for Y in Ys]
        assert comm_sim.run([p.export_calls(1) for p in plans], seq) == 1
        total = sum(Ys)
        for r in range(world):
            np.testing.assert_array_equal(seq[r]["out"], total[r * M // world:(r + 1) * M // world].reshape(-1))


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("routing", ["random", "sorted", "skewed", "empty_expert"])
@pytest.mark.parametrize("layout", ["slot", "rowband"])
def test_alltoall_schedule(world, routing, layout):
    """empty_expert: the last source (and the first, at world >= 3) has no rows
    — an expert no token was routed to — and takes part with P empty groups
    (R45)."""
    if routing == "empty_expert" and world == 1:
        pytest.skip("needs a peer")
    rng = np.random.default_rng(300 + world + {"random": 0, "sorted": 50, "skewed": 90, "empty_expert": 130}[routing])
    for _ in range(6):
        BM = int(rng.choice([128, 256]))
        BN = int(rng.choice([64, 128]))
        N = BN * int(rng.integers(1, 4))
        Ms = [BM * int(rng.integers(1, 4)) for _ in range(world)]          # imbalanced experts
        if routing == "empty_expert":
            Ms[-1] = 0
            if world >= 3:
                Ms[0] = 0
        S = int(rng.integers(1, 3))
        if layout == "rowband":
            S = N // BN      # raster, one tile-row per wave: ascending bands on every source (R41)
        Ts = [-(-(m // BM) * (N // BN) // S) for m in Ms]
        P = int(rng.integers(1, min(t for t in Ts if t) + 1))             # a common number of groups
        parts = []
        for T in Ts:
            if T == 0:
                parts.append([0] * P)
                continue
            cuts = sorted(rng.choice(np.arange(1, T), size=P - 1, replace=False).tolist()) if P > 1 else []
            b = [0] + cuts + [T]
            parts.append([y - x for x, y in zip(b[:-1], b[1:])])
        rds = []
        for s in range(world):
            if routing == "random":
                rd = rng.integers(0, world, size=Ms[s])
            elif routing == "skewed":
                rd = np.minimum(rng.geometric(0.6, size=Ms[s]) - 1, world - 1)
            elif routing == "sorted":
                rd = np.sort(rng.integers(0, world, size=Ms[s]))
            else:
                rd = rng.integers(0, world, size=Ms[s])
            rds.append(rd.astype(np.int32))
        swz = [1 if layout == "rowband" else 1 + s % 2 for s in range(world)]
        specs = [dict(coll="alltoall", m=Ms[s], n=N, k=64, tile_m=BM, tile_n=BN, workers=S, swizzle=swz[s],
                      group_waves=parts[s], row_dst=rds[s], ar_layout=layout) for s in range(world)]
        plans = [fo.Plan(rank=r, world=world, peers=specs, **specs[r]) for r in range(world)]
        opls = [op.make_plan(Ms[s], N, BM, BN, S, parts[s], swizzle=swz[s]) for s in range(world)]
        Ys = [_ints(rng, (Ms[s], N)) for s in range(world)]
        osends = [orr.a2a_pre(Ys[s], opls[s], rds[s], world, layout) for s in range(world)]
        orecv = oc.alltoall_groups(osends, P)
        bufs = []
        for r in range(world):
            b = {"send": np.concatenate([osends[r].pools[d].reshape(-1) for d in range(world)])}
            b["recv"] = b["send"] if world == 1 else np.full(plans[r].info["recv_elems"], np.nan)
            bufs.append(b)
        comm_sim.run([p.export_calls(0) for p in plans], bufs)
        for d in range(world):
            if layout == "rowband":
                # the receive layout is the output: the all-to-all-v rows themselves
                want = np.concatenate([Ys[s][rds[s] == d] for s in range(world)], axis=0).reshape(-1)
                np.testing.assert_array_equal(bufs[d]["recv"], want)
                continue
            want = np.concatenate([a.reshape(-1) for _, a in orecv[d]]) if orecv[d] else np.zeros(0)
            np.testing.assert_array_equal(bufs[d]["recv"][:want.size], want)
        # sequential: runs of one destination, all-to-all-v output order
        seq = [{"scratch": Ys[r].reshape(-1).copy(), "out": np.full(plans[r].info["out_rows"] * N, np.nan)}
               for r in range(world)]
        comm_sim.run([p.export_calls(1) for p in plans], seq)
        for d in range(world):
            want = np.concatenate([Ys[s][rds[s] == d] for s in range(world)], axis=0).reshape(-1)
            np.testing.assert_array_equal(seq[d]["out"], want)


def test_schedule_groups_and_order():
    """Every overlapped call carries its wave group, groups appear in order,
    and a plan with P groups issues exactly P collectives (AR / RS)."""
    p = fo.Plan(coll="reducescatter", m=1024, n=512, k=64, tile_m=256, tile_n=128, workers=3, swizzle=2,
                group_waves=[1, 2, 3], rank=1, world=4)
    calls = p.export_calls(0)
    assert [c["group"] for c in calls] == [0, 1, 2]
    assert all(c["kind"] == "reducescatter" for c in calls)
    for j, c in enumerate(calls):
        pb, pe, eb, ee = p.group(j)
        assert (c["src_off"], c["dst_off"], c["count"]) == (eb, eb // 4, (ee - eb) // 4)
    assert p.export_calls(1) == [dict(kind="reducescatter", group=-1, peer=-1, src_buf="scratch", dst_buf="out",
                                      src_off=0, dst_off=0, count=1024 * 512 // 4)]


def test_simulator_catches_mismatches():
    """The checker itself: a rank with a different count, a missing
    collective, or an unmatched send must be reported, not silently run."""
    base = dict(coll="allreduce", m=512, n=256, k=64, tile_m=128, tile_n=128, workers=2, swizzle=1,
                group_waves=[2, 2], ar_layout="slot")
    plans = [fo.Plan(rank=r, world=2, **base) for r in range(2)]
    good = [p.export_calls(0) for p in plans]
    bufs = [{"send": np.zeros(512 * 256)} for _ in range(2)]
    bad = [list(good[0]), [dict(c) for c in good[1]]]
    bad[1][0]["count"] += 1
    with pytest.raises(comm_sim.ScheduleError):
        comm_sim.run(bad, bufs)
    with pytest.raises(comm_sim.ScheduleError):
        comm_sim.run([good[0], good[1][:1]], bufs)
    p2p = [[dict(kind="group_start"), dict(kind="send", peer=1, src_buf="send", src_off=0, count=4),
            dict(kind="group_end")],
           [dict(kind="group_start"), dict(kind="recv", peer=0, dst_buf="send", dst_off=0, count=8),
            dict(kind="group_end")]]
    with pytest.raises(comm_sim.ScheduleError):
        comm_sim.run(p2p, bufs)
