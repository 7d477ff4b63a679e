"""Post-communication reorder kernel timing (dev tool): achieved HBM GB/s per
map / op, against MEASURED_PEAKS.json's copy bandwidth.

Timing: CUDA events around one launch on a stream pre-loaded with a ~100 us
sleep kernel (so the host-side launch cost — ctypes + driver, several us —
is not inside the events; without it a 10 us kernel reads as 15-18 us), medians
of `iters`.  Cache state before each launch (--flush):
  read   stream a 512 MiB buffer through a read-only kernel: L2 holds clean
         lines of another buffer (cold, nothing to write back) — the state a
         kernel meets after unrelated reads;
  write  zero a 512 MiB buffer (round-1 method): L2 full of DIRTY lines that
         the timed kernel's misses must write back first (~100 MB of extra
         HBM writes inside the timed region for a 67 MB kernel).
Each line is followed by torch's own copy_ / add over the same bytes with no
reordering (what a library elementwise kernel achieves at that size).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def timeit(fn, flush_fn, iters=30, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        flush_fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(100_000)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    return sorted(ts)[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--flush", default="read,write")
    ap.add_argument("--iters", type=int, default=30)
    args = ap.parse_args()
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        peak = 6650.0
    buf = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    fbuf = buf.view(torch.float32)
    flushes = {"read": lambda: fbuf.amax(), "write": lambda: buf.zero_()}
    cases = [
        ("AR slot 4096x4096 256x256 S64", dict(coll="allreduce", m=4096, n=4096, k=64, tile_m=256, tile_n=256,
                                                workers=64, swizzle=2, group_waves=[1, 2, 1], ar_layout="slot"), 1, 0),
        ("RS slot n=8 8192x8192 256x256 S64", dict(coll="reducescatter", m=8192, n=8192, k=64, tile_m=256, tile_n=256,
                                                    workers=64, group_waves=[2, 4, 6, 4], ar_layout="slot"), 8, 0),
        ("A2A slot n=8 1024x4096 256x256", None, 8, 0),
        ("AR slot 8192x8192 256x256 S64", dict(coll="allreduce", m=8192, n=8192, k=64, tile_m=256, tile_n=256,
                                                workers=64, swizzle=2, group_waves=[4, 4, 8], ar_layout="slot"), 1, 0),
        # ROWBAND plans (H11a, R40): the post pass is only the fused op, on rows in place
        ("AR rowband 4096x4096 S64", dict(coll="allreduce", m=4096, n=4096, k=64, tile_m=256, tile_n=256,
                                          workers=64, swizzle=1, group_waves=[1, 2, 1], ar_layout="rowband"), 1, 0),
        ("RS rowband n=8 8192x8192 S64", dict(coll="reducescatter", m=8192, n=8192, k=64, tile_m=256, tile_n=256,
                                              workers=64, swizzle=1, group_waves=[2, 4, 6, 4], ar_layout="rowband"),
         8, 0),
        ("AR rowband 8192x8192 S64", dict(coll="allreduce", m=8192, n=8192, k=64, tile_m=256, tile_n=256,
                                          workers=64, swizzle=1, group_waves=[4, 4, 8], ar_layout="rowband"), 1, 0),
    ]
    print(f"# HBM peak {peak:.0f} GB/s (MEASURED_PEAKS.json); GB/s = algorithmic bytes (read + write) / median time",
          flush=True)
    for fl in args.flush.split(","):
        flush_fn = flushes[fl]
        print(f"## flush={fl}", flush=True)
        for name, spec, world, rank in cases:
            if spec is None:
                rng = np.random.default_rng(0)
                specs = []
                for s in range(world):
                    rd = np.sort(rng.integers(0, world, size=1024)).astype(np.int32)
                    specs.append(dict(coll="alltoall", m=1024, n=4096, k=64, tile_m=256, tile_n=256, workers=32,
                                      group_waves=[1, 1], row_dst=rd, ar_layout="slot"))
                plan_args = [(dict(specs[rank], post=op), dict(rank=rank, world=world, peers=specs))
                             for op in ("none", "add", "add_rmsnorm")]
            else:
                ops = ("add_rmsnorm",) if spec["ar_layout"] == "rowband" else ("none", "add", "add_rmsnorm")
                plan_args = [(dict(spec, post=op), dict(rank=rank, world=world)) for op in ops]
            for sp, kw in plan_args:
                plan = fo.Plan(**kw, **sp)
                rows, N = plan.info["out_rows"], plan.info["out_cols"]
                recv = torch.randn(plan.info["recv_elems"], device="cuda").to(torch.bfloat16)
                out = torch.empty(rows, N, dtype=torch.bfloat16, device="cuda")
                res = torch.randn(rows, N, device="cuda").to(torch.bfloat16)
                gam = torch.randn(N, device="cuda").to(torch.bfloat16)
                nb = 2 * rows * N * 2 + (rows * N * 2 if sp["post"] != "none" else 0)
                src = recv[:rows * N].view(rows, N)
                variants = [("", 1)] if sp["post"] != "add_rmsnorm" else [(" bulk", 1), (" regs", 0)]
                for tag, bulk in variants:
                    plan.set_option("post_bulk", bulk)
                    t = timeit(lambda: fo.post_stage(plan, recv, out, res, gam), flush_fn, args.iters)
                    if sp["post"] == "none":
                        tr = timeit(lambda: out.copy_(src), flush_fn, args.iters)
                        ref = "torch copy_"
                    else:
                        tr = timeit(lambda: torch.add(src, res, out=out), flush_fn, args.iters)
                        ref = "torch add"
                    print(f"{name:34s} post={sp['post'] + tag:17s} {t:8.2f} us {nb / t / 1e3:7.0f} GB/s "
                          f"({nb / t / 1e3 / peak:.2f} of peak) | {ref:11s} {tr:8.2f} us {nb / tr / 1e3:7.0f} GB/s "
                          f"({nb / tr / 1e3 / peak:.2f})  [{nb / 1e6:.1f} MB]", flush=True)
                if sp["post"] == "add_rmsnorm":
                    # the unfused library form: torch add, then torch's rms_norm (two HBM passes)
                    def unfused():
                        y = torch.add(src, res)
                        torch.nn.functional.rms_norm(y, (N,), gam, 1e-5)
                    tu = timeit(unfused, flush_fn, args.iters)
                    print(f"{'':34s} {'torch add + F.rms_norm (unfused)':34s} {tu:8.2f} us", flush=True)


if __name__ == "__main__":
    main()
