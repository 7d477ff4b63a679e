"""A tensor-parallel transformer block's communication-bearing half, end to
end on the library (second workload): Llama-3-8B shapes,
synthetic weights, world = TP ranks (torchrun; one rank works too).

    h     = x + AllReduce(attn_out @ Wo_shardᵀ)          o_proj, row-parallel
    n     = RMSNorm(h) · γ                              fused: fo_run post=add_rmsnorm_res
                                                        (writes n, updates x -> h in place)
    a     = silu(n @ Wg_shardᵀ) · (n @ Wu_shardᵀ)          gate/up, column-parallel: our GEMM with the
                                                        SwiGLU fused into its epilogue (FO_OPT_GEMM_SWIGLU;
                                                        weight rows interleaved in blocks of 128)
    y     = h + AllReduce(a @ Wd_shardᵀ)                 down-proj, row-parallel: fo_run post=add

The attention core is not part of this (its output is a synthetic input);
every other step runs in the library's kernels.
Both collective layers run overlapped (fo_run, tuned plans) and sequential
(fo_run_sequential: GEMM -> one NCCL call -> the same fused op); the block
time is reported for each.  Correctness: tests/test_gpu_graph.py runs a small
block at TP = 1 (NCCL) and TP = 2 (loopback, one GPU) against the oracle's TP
block (oracle/block.py).

    python tools/tp_block.py [--tokens 4096]
    python -m torch.distributed.run --nproc-per-node N tools/tp_block.py
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402
import synthetic  # noqa: E402
from paper_2504_19519_b200 import tuner as fot  # noqa: E402


def block_weights(H, I, rank, world, device="cuda"):
    """Rank `rank`'s synthetic shard weights (seeded; device = where they are drawn)."""
    Hl, Il = H // world, I // world
    seed = synthetic.rank_seed(50000, world, rank)
    Wo = synthetic.normal_bf16((H, Hl), 0.02, seed + 1, device=device)        # [out H, in H/tp]
    # gate/up rows interleaved in blocks of 128: [g0..127, u0..127, g128..255, ...]
    Wgu = synthetic.normal_bf16((2 * Il, H), 0.02, seed + 2, device=device)
    Wd = synthetic.normal_bf16((H, Il), 0.02, seed + 3, device=device)        # [out H, in I/tp]
    gamma = synthetic.normal_bf16((H,), 1.0, 50001, device=device)
    return Wo, Wgu, Wd, gamma


class Block:
    def __init__(self, ctx, T, H, I, rank, world, tuned=True, device=0, weights=None):
        assert H % world == 0 and I % world == 0
        self.ctx, self.T, self.H, self.I, self.world = ctx, T, H, I, world
        Hl, Il = H // world, I // world
        Wo, Wgu, Wd, gamma = weights if weights is not None else block_weights(H, I, rank, world)
        self.Wo, self.Wgu, self.Wd, self.gamma = Wo.cuda(), Wgu.cuda(), Wd.cuda(), gamma.cuda()
        if tuned:
            co = fot.tune_layer(T, H, Hl, ctx, "allreduce", "add_rmsnorm_res", device=device, iters=5)
            cd = fot.tune_layer(T, H, Il, ctx, "allreduce", "add", device=device, iters=5)
            self.p_o = fo.Plan(rank=rank, world=world, **co.spec(T, H, Hl, "allreduce", "add_rmsnorm_res"))
            self.p_d = fo.Plan(rank=rank, world=world, **cd.spec(T, H, Il, "allreduce", "add"))
        else:
            def simple(K, post):
                # two waves, one group each (per-band fused op on the ROWBAND layout)
                tiles = (T // 256) * (H // 256)
                S = max(1, min(64, -(-tiles // 2)))
                return fo.Plan(rank=rank, world=world, coll="allreduce", m=T, n=H, k=K, tile_m=256, tile_n=256,
                               workers=S, swizzle=0, group_waves=[1] * (-(-tiles // S)), post=post)
            self.p_o, self.p_d = simple(Hl, "add_rmsnorm_res"), simple(Il, "add")
        tiles_gu = (T // 256) * (2 * Il // 256)
        self.p_gu = fo.Plan(coll="nocomm", m=T, n=2 * Il, k=H, tile_m=256, tile_n=256,
                            workers=-(-tiles_gu // -(-tiles_gu // 74)), swizzle=0, options={"gemm_swiglu": 1, "tail_split": -1})
        self.n = torch.empty(T, H, dtype=torch.bfloat16, device="cuda")
        self.a = torch.empty(T, Il, dtype=torch.bfloat16, device="cuda")
        self.y = torch.empty(T, H, dtype=torch.bfloat16, device="cuda")

    def forward(self, attn_out, x, overlapped=True):
        """x is the block input (residual stream); it is updated in place to h."""
        run = fo.run if overlapped else fo.run_sequential
        run(self.ctx, self.p_o, attn_out, self.Wo, self.n, x, self.gamma)
        fo.gemm_stage(self.p_gu, self.n, self.Wgu, self.a)      # a = silu(gate) * up, fused
        run(self.ctx, self.p_d, self.a, self.Wd, self.y, x)
        return self.y


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=4096)
    ap.add_argument("--hidden", type=int, default=4096)
    ap.add_argument("--inter", type=int, default=14336)
    ap.add_argument("--steps", type=int, default=20)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if "MASTER_ADDR" in os.environ:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        from paper_2504_19519_b200 import dist as fodist
        ctx = fodist.make_context(local, nccl_max_ctas=16)
    else:
        ctx = fo.Context.create(local, 0, 1, fo.unique_id())
    T, H, I = args.tokens, args.hidden, args.inter
    blk = Block(ctx, T, H, I, rank, world, device=local)
    attn = synthetic.normal_bf16((T, H // world), 1.0, 7, device="cuda")
    x0 = synthetic.normal_bf16((T, H), 1.0, 8, device="cuda")
    x = x0.clone()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    res = {}
    for ov in (True, False):
        for _ in range(3):
            x.copy_(x0)
            blk.forward(attn, x, ov)
        torch.cuda.synchronize()
    ts = {True: [], False: []}
    for _ in range(args.steps):
        for ov in (True, False):
            x.copy_(x0)
            flush.zero_()
            if world > 1:
                dist.barrier(device_ids=[local])
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(200_000)
            s.record()
            blk.forward(attn, x, ov)
            e.record()
            torch.cuda.synchronize()
            ts[ov].append(s.elapsed_time(e) * 1e3)
    res = {k: statistics.median(v) for k, v in ts.items()}
    if world > 1:
        t = torch.tensor([res[True], res[False]], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res = {True: t[0].item(), False: t[1].item()}
    flops = 2.0 * T * H * (H // world) + 2.0 * T * (2 * I // world) * H + 2.0 * T * H * (I // world)
    if rank == 0:
        print(json.dumps({"block": "llama3-8b o_proj + MLP, TP=%d" % world, "tokens": T,
                          "overlapped_us": round(res[True], 1), "sequential_us": round(res[False], 1),
                          "speedup": round(res[False] / res[True], 4),
                          "tflops_per_rank": round(flops / (res[True] * 1e-6) / 1e12, 1),
                          "o_proj_plan": {"workers": blk.p_o.info["workers"], "groups": blk.p_o.info["num_groups"]},
                          "down_plan": {"workers": blk.p_d.info["workers"], "groups": blk.p_d.info["num_groups"]}}))
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
