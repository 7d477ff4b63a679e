"""Multi-process (gloo, world size 2 and 4, CPU) test of the n > 1 host logic.

Each process builds its plan through paper_2504_19519_b200.dist (peer census
over the process group for All-to-All), fills its send buffer through the
plan's exported send map, then executes the plan's exported communication
schedule (fo_plan_export_calls — the exact calls fo_run issues on NCCL) with
gloo collectives and point-to-point messages on CPU tensors in place of NCCL
(a TEST of the plan's multi-rank contract, not a product path), and compares
every rank's output (through the exported receive map) with the oracle's plain
definition; the sequential schedule likewise.  Bit-exact on integer data.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(n, r, M, N, K):
    rng = np.random.default_rng(1000 + 17 * r + M)
    return rng.integers(-3, 4, size=(M, K)).astype(float), rng.integers(-3, 4, size=(N, K)).astype(float)


def _gloo_exec(calls, bufs, rank, world):
    """Execute a plan's exported schedule over gloo (test stand-in for NCCL):
    AllReduce in place; ReduceScatter as an AllReduce of the send range keeping
    this rank's chunk (gloo has no ReduceScatter); each GROUP_START..GROUP_END
    as isend/irecv pairs matched by gloo in issue order; local copies."""
    def view(name, off, cnt):
        b = bufs[name]
        assert 0 <= off and off + cnt <= b.size, (name, off, cnt, b.size)
        return b[off:off + cnt]

    i = 0
    while i < len(calls):
        c = calls[i]
        if c["kind"] == "allreduce":
            t = torch.from_numpy(view(c["src_buf"], c["src_off"], c["count"]).copy())
            dist.all_reduce(t)
            view(c["dst_buf"], c["dst_off"], c["count"])[:] = t.numpy()
        elif c["kind"] == "reducescatter":
            t = torch.from_numpy(view(c["src_buf"], c["src_off"], world * c["count"]).copy())
            dist.all_reduce(t)
            view(c["dst_buf"], c["dst_off"], c["count"])[:] = t.numpy()[rank * c["count"]:(rank + 1) * c["count"]]
        elif c["kind"] == "local_copy":
            view(c["dst_buf"], c["dst_off"], c["count"])[:] = view(c["src_buf"], c["src_off"], c["count"]).copy()
        elif c["kind"] == "group_start":
            reqs, landing = [], []
            i += 1
            while calls[i]["kind"] != "group_end":
                c = calls[i]
                if c["kind"] == "send":
                    reqs.append(dist.isend(torch.from_numpy(view(c["src_buf"], c["src_off"], c["count"]).copy()),
                                           c["peer"]))
                else:
                    t = torch.zeros(c["count"], dtype=torch.float64)
                    reqs.append(dist.irecv(t, c["peer"]))
                    landing.append((t, c))
                i += 1
            for q in reqs:
                q.wait()
            for t, c in landing:
                view(c["dst_buf"], c["dst_off"], c["count"])[:] = t.numpy()
        else:
            raise AssertionError(f"unexpected call {c}")
        i += 1


def _worker(rank, port, coll, errq, WORLD=2, layout="slot"):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=WORLD)
        from oracle import pipeline as opl

        import paper_2504_19519_b200 as fo  # noqa: F401
        from paper_2504_19519_b200 import dist as fodist

        N, K, BN = 256, 8, 128
        if coll == "alltoall":
            Ms = [384, 256, 512, 256][:WORLD]    # imbalanced experts; T >= 2 each
            M = Ms[rank]
            rds = [np.random.default_rng(5 + s).integers(0, WORLD, size=Ms[s]).astype(np.int32) for s in range(WORLD)]
            tiles = (M // 128) * (N // BN)
            S = 2
            T = (tiles + S - 1) // S
            if layout == "rowband":   # raster, one tile-row per wave (R41)
                S = N // BN
                T = (tiles + S - 1) // S
            spec = dict(coll="alltoall", m=M, n=N, k=64, tile_n=BN, workers=S, swizzle=2 if layout == "slot" else 1,
                        group_waves=[1, T - 1], row_dst=rds[rank], ar_layout=layout)
        else:
            M = 512
            spec = dict(coll=coll, m=M, n=N, k=64, tile_n=BN, workers=3, swizzle=2, group_waves=[1, 1, 1],
                        ar_layout="slot")
            if layout == "rowband":   # raster, one tile-row per wave (H11a / R40)
                spec.update(workers=N // BN, swizzle=1, group_waves=[1, 1, 2], ar_layout="rowband")
        plan = fodist.make_plan(**spec)
        assert plan.info["ar_layout"] == (1 if layout == "rowband" else 0)
        A, Bt = _inputs(WORLD, rank, M, N, K)
        Y = A @ Bt.T
        send = np.zeros(plan.info["send_elems"])
        send[plan.export_send_map()] = Y.reshape(-1)
        recv = np.zeros(plan.info["recv_elems"])
        # the plan's own communication schedule (fo_plan_export_calls, what
        # fo_run issues on NCCL), driven through gloo's collectives and
        # point-to-point messages; ROWBAND AR reduces C in place and RS
        # scatters into `out` (both the output layout)
        bufs = {"send": send, "recv": recv, "out": None}
        if layout == "rowband" and coll == "allreduce":
            bufs = {"send": None, "recv": None, "out": send}
        elif layout == "rowband" and coll == "reducescatter":
            bufs = {"send": send, "recv": None, "out": recv}
        _gloo_exec(plan.export_calls(0), bufs, rank, WORLD)
        if coll == "allreduce":
            recv = send
        out = recv[plan.export_recv_map()].reshape(plan.info["out_rows"], N)
        seq_out = np.full(plan.info["out_rows"] * N, np.nan)
        seq_bufs = {"out": seq_out, "scratch": Y.reshape(-1).copy()}
        if coll == "allreduce":
            seq_bufs["out"] = Y.reshape(-1).copy()
        _gloo_exec(plan.export_calls(1), seq_bufs, rank, WORLD)
        seq_out = seq_bufs["out"].reshape(plan.info["out_rows"], N)
        As, Bts = zip(*[_inputs(WORLD, r, (Ms[r] if coll == "alltoall" else M), N, K) for r in range(WORLD)])
        if coll == "allreduce":
            want = opl.plain_allreduce(list(As), list(Bts))[rank]
        elif coll == "reducescatter":
            want = opl.plain_reducescatter(list(As), list(Bts), 128)[rank]
        else:
            want = opl.plain_alltoall(list(As), list(Bts), rds)[rank]
        assert np.array_equal(out, want), f"rank {rank}: mismatch"
        if coll == "reducescatter":   # the sequential RS: NCCL's contiguous rows
            full = opl.plain_allreduce(list(As), list(Bts))[rank]
            want = full[rank * (M // WORLD):(rank + 1) * (M // WORLD)]
        assert np.array_equal(seq_out, want), f"rank {rank}: sequential mismatch"
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        import traceback
        errq.put(f"rank {rank}: {e}\n{traceback.format_exc()}")
        raise


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("coll", ["allreduce", "reducescatter", "alltoall"])
@pytest.mark.parametrize("layout", ["slot", "rowband"])
def test_multi_rank_plan_contract(coll, world, layout):
    from paper_2504_19519_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, coll, errq, world, layout)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, "\n".join(errs)
    assert all(p.exitcode == 0 for p in procs)
