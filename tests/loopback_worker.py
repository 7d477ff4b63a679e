"""World-W run of the library's multi-rank data path on ONE GPU (test
infrastructure, launched by tests/test_gpu_loopback.py in a subprocess).

W in-process ranks share one B200 through the loopback communicator
(fo_loopback_create / fo_ctx_create_loopback): every rank has its own context
(comm + post streams), plan, caller stream and inputs, and every rank's calls
are issued from its own host thread, exactly as W processes would each issue
theirs.  The ranks' GEMMs, counter-triggered group calls on the comm
streams, last-group calls on the caller streams, receive buffers and post
passes all run for real; only the transport differs from NCCL.

Inputs are in the exact-integer regime (A, B in {-1, 0, 1}, <= 256 nonzeros per
output row over all ranks), so every partial sum is exact in bf16 and the
outputs must equal the ORACLE's plain definitions (oracle/pipeline.py O8) bit
for bit: AllReduce = sum_r C_r; ReduceScatter = rows R_k (fo_run) /
contiguous rows (fo_run_sequential); All-to-All = concat over sources
(all-to-all-v order); AllGather + row exchange = the AllReduce.

usage: loopback_worker.py W  -> prints "loopback W=<W>: OK" and exits 0.
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from concurrent.futures import ThreadPoolExecutor  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402
import synthetic  # noqa: E402
from oracle import pipeline as opl  # noqa: E402


TRACE = os.environ.get("FO_LOOPBACK_TRACE") == "1"


def main(W):
    torch.cuda.set_device(0)
    grp = fo.LoopbackGroup(0, W)
    ctxs = grp.contexts()
    streams = [torch.cuda.Stream() for _ in range(W)]
    bad = []

    def check(name, got, want):
        g = got.double().cpu().numpy() if isinstance(got, torch.Tensor) else got
        if g.shape != want.shape or not np.array_equal(g, want):
            diff = np.abs(g - want).max() if g.shape == want.shape else f"shape {g.shape} vs {want.shape}"
            print(f"MISMATCH W={W} {name}: {diff}", flush=True)
            bad.append(name)

    pool = ThreadPoolExecutor(W)

    def each(fn):
        """Issue fn(r) for every rank from its own host thread on its own
        stream — as W processes would; a host call that blocks in one rank
        (a synchronous allocation or copy) never stops the others from issuing
        the calls its kernels wait for — then wait for all of them."""
        def one(r):
            torch.cuda.set_device(0)
            if TRACE:
                print(f"[host] t={int(time.time() * 1000) % 1000000} ms rank {r} issue", file=sys.stderr, flush=True)
            with torch.cuda.stream(streams[r]):
                fn(r)
            if TRACE:
                print(f"[host] t={int(time.time() * 1000) % 1000000} ms rank {r} issued", file=sys.stderr, flush=True)
            streams[r].synchronize()
        for f in [pool.submit(one, r) for r in range(W)]:
            f.result()

    M, N, K, BM, BN = 1024, 512, 256, 256, 128           # 16 tiles; S = 4 -> 4 waves
    S = 4
    inp = [synthetic.exact_inputs(M, N, K, seed=synthetic.rank_seed(61, W, r), nnz_per_row=max(1, 256 // W))
           for r in range(W)]
    As = [a.double().numpy() for a, _ in inp]
    Bts = [b.double().numpy() for _, b in inp]
    Ad = [a.cuda() for a, _ in inp]
    Bd = [b.cuda() for _, b in inp]
    torch.cuda.synchronize()
    full = opl.plain_allreduce(As, Bts)[0]
    for coll, layout, groups, split in (("allreduce", "slot", [1, 2, 1], 0), ("allreduce", "rowband", [1, 1, 2], 0),
                                        ("allreduce", "rowband", [4], 0), ("allreduce", "slot", [2, 2], -1),
                                        ("reducescatter", "auto", [2, 1, 1], 0),
                                        ("reducescatter", "rowband", [1, 1, 2], 0),
                                        ("reducescatter", "auto", [1, 3], -1)):
        if coll == "reducescatter" and BM % W:
            continue
        spec = dict(coll=coll, m=M, n=N, k=K, tile_m=BM, tile_n=BN, workers=S,
                    swizzle=1 if layout == "rowband" else 2, group_waves=groups, ar_layout=layout)
        # the split tail needs workers idle in the last wave: 3 full waves of 5 + 1
        if split:
            spec["workers"] = 5
            spec["group_waves"] = [1, 3] if coll == "reducescatter" else [2, 2]
        plans = [fo.Plan(rank=r, world=W, options={"tail_split": split} if split else None, **spec)
                 for r in range(W)]
        for p in plans:     # no rank allocates while another's collective is in flight
            p.prepare(sequential=True, host=True)
        name = f"{coll}/{layout}/{spec['group_waves']}/split={split}"
        print(f"[W={W}] {name}", flush=True)
        if coll == "allreduce":
            want = full
        else:
            want = opl.plain_reducescatter(As, Bts, BM)
        outs = [torch.full((p.info["out_rows"], N), float("nan"), dtype=torch.bfloat16, device="cuda")
                for p in plans]
        torch.cuda.synchronize()
        for trig in (1, 0):
            for p in plans:
                p.set_option("last_group_in_order", trig)
            for _ in range(3):
                each(lambda r: fo.run(ctxs[r], plans[r], Ad[r], Bd[r], outs[r], stream=streams[r]))
            for r in range(W):
                check(f"{name}/in_order={trig}/rank{r}", outs[r], want if coll == "allreduce" else want[r])
        seq = [torch.full_like(o, float("nan")) for o in outs]
        torch.cuda.synchronize()
        each(lambda r: fo.run_sequential(ctxs[r], plans[r], Ad[r], Bd[r], seq[r], stream=streams[r]))
        for r in range(W):
            w = full if coll == "allreduce" else full[r * (M // W):(r + 1) * (M // W)]
            check(f"{name}/sequential/rank{r}", seq[r], w)
        if coll == "reducescatter":
            gath = [torch.empty(M, N, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
            torch.cuda.synchronize()
            each(lambda r: fo.run_allgather(ctxs[r], plans[r], outs[r], gath[r], stream=streams[r]))
            for r in range(W):
                check(f"{name}/allgather+rowexchange/rank{r}", gath[r], full)
        # fo_run_host: host activations (chunked H2D the GEMM waits on, two staging sets)
        # (W <= 4: with its three copy streams a rank has six streams, and
        # more than 32 streams alias the device's hardware queues, where one
        # rank's pending stream wait can block another rank's launch — a
        # one-process artefact; with NCCL every rank is its own process)
        # (RS rowband: its bands land in `out` row-major, so each band goes back
        # to the host right after its ReduceScatter, as for AR rowband)
        if (coll == "allreduce" or layout == "rowband") and not split and W <= 4:
            hosts = [[torch.full((p.info["out_rows"], N), float("nan"), dtype=torch.bfloat16).pin_memory()
                      for _ in range(2)] for p in plans]
            A_h = [a.pin_memory() for a, _ in inp]
            for i in range(2):
                each(lambda r: fo.run_host(ctxs[r], plans[r], A_h[r], Bd[r], hosts[r][i], stream=streams[r]))
            for r in range(W):
                for i in range(2):
                    check(f"{name}/run_host[{i}]/rank{r}", hosts[r][i], full if coll == "allreduce" else want[r])
        for p in plans:
            p.close()
    # ---- All-to-All: imbalanced experts, random routing, same P on every rank;
    # then the same with the last expert receiving no tokens (m = 0: P empty
    # groups, no GEMM) and rank 0 receiving no rows (R45)
    for empty in (False, True):
        rng = np.random.default_rng(7 + W)
        Ms = [256 * int(rng.integers(2, 5)) for _ in range(W)]   # >= 2 tile-rows: two one-row waves
        if empty:
            Ms[-1] = 0
        # the empty variant also routes no row to rank 0: an empty output (NULL out)
        rds = [rng.integers(1 if empty else 0, W, size=Ms[s]).astype(np.int32) for s in range(W)]
        inp = [synthetic.exact_inputs(max(Ms[s], 256), N, K, seed=synthetic.rank_seed(71, W, s), nnz_per_row=128)
               for s in range(W)]
        inp = [(a[:Ms[s]].contiguous(), b) for s, (a, b) in enumerate(inp)]
        As = [a.double().numpy() for a, _ in inp]
        Bts = [b.double().numpy() for _, b in inp]
        Ad = [a.cuda() for a, _ in inp]
        Bd = [b.cuda() for _, b in inp]
        want = opl.plain_alltoall(As, Bts, rds)
        # the paper's subtoken pools (S = 2) and R41's rows received straight into
        # the output (raster, one tile-row per wave)
        for layout, S2, swz in (("slot", 2, 2), ("rowband", N // BN, 1)):
            specs = []
            for s in range(W):
                T = -(-(Ms[s] // BM) * (N // BN) // S2)
                specs.append(dict(coll="alltoall", m=Ms[s], n=N, k=K, tile_m=BM, tile_n=BN, workers=S2, swizzle=swz,
                                  group_waves=[1, T - 1] if T else [0, 0], row_dst=rds[s], ar_layout=layout))
            plans = [fo.Plan(rank=r, world=W, peers=specs, **specs[r]) for r in range(W)]
            assert all(p.info["ar_layout"] == (1 if layout == "rowband" else 0) for p in plans)
            print(f"[W={W}] alltoall/{layout} Ms={Ms}", flush=True)
            tag = "alltoall-empty" if empty else "alltoall"
            for p in plans:
                p.prepare(sequential=True)
            outs = [torch.full((p.info["out_rows"], N), float("nan"), dtype=torch.bfloat16, device="cuda")
                    for p in plans]
            torch.cuda.synchronize()
            for _ in range(3):
                each(lambda r: fo.run(ctxs[r], plans[r], Ad[r], Bd[r], outs[r], stream=streams[r]))
            for r in range(W):
                check(f"{tag}/{layout}/rank{r}", outs[r], want[r])
            seq = [torch.full_like(o, float("nan")) for o in outs]
            torch.cuda.synchronize()
            each(lambda r: fo.run_sequential(ctxs[r], plans[r], Ad[r], Bd[r], seq[r], stream=streams[r]))
            for r in range(W):
                check(f"{tag}/{layout}/sequential/rank{r}", seq[r], want[r])
            # the MoE combine as the post pass (R31): top-2 with weights 1 and 0
            # over a permutation of the A2A output rows — the combined rows are the
            # A2A rows in the permuted order, exactly (fp32 1*x + 0*y, one rounding)
            perms = [np.random.default_rng(50 + r).permutation(p.info["out_rows"]).astype(np.int32) for r, p in
                     enumerate(plans)]
            idxs = [torch.from_numpy(np.stack([pm, pm[::-1].copy()], 1)).cuda() for pm in perms]
            ws = [torch.tensor([[1.0, 0.0]], device="cuda").repeat(len(pm), 1).contiguous() for pm in perms]
            comb = [torch.full((len(pm), N), float("nan"), dtype=torch.bfloat16, device="cuda") for pm in perms]
            torch.cuda.synchronize()
            for _ in range(2):
                each(lambda r: fo.run_combine(ctxs[r], plans[r], Ad[r], Bd[r], comb[r], idxs[r], ws[r], stream=streams[r]))
            for r in range(W):
                check(f"{tag}/{layout}/combine/rank{r}", comb[r], want[r][perms[r]])
            for p in plans:
                p.close()
    for c in ctxs:
        c.close()
    grp.close()
    print(f"loopback W={W}: " + ("OK" if not bad else f"{len(bad)} mismatches"), flush=True)
    return 0 if not bad else 1


if __name__ == "__main__":
    sys.exit(main(int(sys.argv[1])))
