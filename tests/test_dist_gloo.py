"""Multi-process (gloo, world size 2 and 4, CPU) test of the n > 1 host logic.

Each process builds its plan through paper_2504_19519_b200.dist (peer census
over the process group for All-to-All), then runs the method's data movement
with the plan's exported maps and group ranges, using gloo collectives on CPU
tensors in place of NCCL (this is a TEST of the plan's multi-rank contract, not
a product path), and compares every rank's output with the oracle's plain
definition.  Bit-exact on integer data.
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


def _worker(rank, port, coll, errq, WORLD=2):
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
            spec = dict(coll="alltoall", m=M, n=N, k=64, tile_n=BN, workers=S, swizzle=2,
                        group_waves=[1, T - 1], row_dst=rds[rank])
        else:
            M = 512
            spec = dict(coll=coll, m=M, n=N, k=64, tile_n=BN, workers=3, swizzle=2, group_waves=[1, 1, 1],
                        ar_layout="slot")
        plan = fodist.make_plan(**spec)
        A, Bt = _inputs(WORLD, rank, M, N, K)
        Y = A @ Bt.T
        send = np.zeros(plan.info["send_elems"])
        send[plan.export_send_map()] = Y.reshape(-1)
        P = plan.info["num_groups"]
        recv = np.zeros(plan.info["recv_elems"])
        if coll == "allreduce":
            for j in range(P):
                _, _, b, e = plan.group(j)
                t = torch.from_numpy(send[b:e].copy())
                dist.all_reduce(t)
                recv[b:e] = t.numpy()
        elif coll == "reducescatter":
            for j in range(P):
                _, _, b, e = plan.group(j)
                t = torch.from_numpy(send[b:e].copy())
                dist.all_reduce(t)                       # RS emulated as AR + keep my chunk
                c = (e - b) // WORLD
                recv[b // WORLD:b // WORLD + c] = t.numpy()[rank * c:(rank + 1) * c]
        else:
            sc, rc = plan.export_a2a_counts()
            pool_base = np.concatenate([[0], np.cumsum(sc.sum(axis=0))])
            start = np.vstack([np.zeros((1, WORLD), int), np.cumsum(sc, axis=0)[:-1]])
            roff = np.concatenate([[0], np.cumsum(rc.reshape(-1))])[:-1].reshape(P, WORLD)
            for j in range(P):
                reqs = []
                for d in range(WORLD):
                    a = (pool_base[d] + start[j, d]) * BN
                    if d == rank:
                        b0 = roff[j, d] * BN
                        recv[b0:b0 + sc[j, d] * BN] = send[a:a + sc[j, d] * BN]
                        continue
                    if sc[j, d]:
                        reqs.append(dist.isend(torch.from_numpy(send[a:a + sc[j, d] * BN].copy()), d))
                bufs = {}
                for s in range(WORLD):
                    if s != rank and rc[j, s]:
                        bufs[s] = torch.zeros(int(rc[j, s]) * BN, dtype=torch.float64)
                        reqs.append(dist.irecv(bufs[s], s))
                for q in reqs:
                    q.wait()
                for s, b in bufs.items():
                    b0 = roff[j, s] * BN
                    recv[b0:b0 + rc[j, s] * BN] = b.numpy()
        out = recv[plan.export_recv_map()].reshape(plan.info["out_rows"], N)
        As, Bts = zip(*[_inputs(WORLD, r, (Ms[r] if coll == "alltoall" else M), N, K) for r in range(WORLD)])
        if coll == "allreduce":
            want = opl.plain_allreduce(list(As), list(Bts))[rank]
        elif coll == "reducescatter":
            want = opl.plain_reducescatter(list(As), list(Bts), 128)[rank]
        else:
            want = opl.plain_alltoall(list(As), list(Bts), rds)[rank]
        assert np.array_equal(out, want), f"rank {rank}: mismatch"
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        import traceback
        errq.put(f"rank {rank}: {e}\n{traceback.format_exc()}")
        raise


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("coll", ["allreduce", "reducescatter", "alltoall"])
def test_multi_rank_plan_contract(coll, world):
    from paper_2504_19519_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, coll, errq, world)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, "\n".join(errs)
    assert all(p.exitcode == 0 for p in procs)
