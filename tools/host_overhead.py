"""Host-side enqueue cost of the public entry points (dev tool): wall time of
the Python call (ctypes marshalling + the library's host work + launches),
measured while the GPU is busy with earlier work so nothing blocks, and the
device time of the same calls with the queue pre-loaded by a sleep kernel
(host launch latency excluded)."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402
import synthetic  # noqa: E402


def main():
    torch.cuda.set_device(0)
    ctx = fo.Context.create(0, 0, 1, fo.unique_id())
    M, N, K = 4096, 4096, 14336
    A, Bt = synthetic.float_inputs(M, N, K, seed=1, device="cuda")
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    plan = fo.Plan(coll="allreduce", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=64, swizzle=0,
                   group_waves=[4], ar_layout="rowband")
    plan4 = fo.Plan(coll="allreduce", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=64, swizzle=1,
                    group_waves=[1, 1, 1, 1], ar_layout="rowband")
    gp = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=64, swizzle=0)
    fns = {"fo_run [4]": lambda: fo.run(ctx, plan, A, Bt, out),
           "fo_run [1,1,1,1]": lambda: fo.run(ctx, plan4, A, Bt, out),
           "fo_run_sequential": lambda: fo.run_sequential(ctx, plan, A, Bt, out),
           "fo_gemm_stage": lambda: fo.gemm_stage(gp, A, Bt, out),
           "torch.matmul": lambda: torch.matmul(A, Bt.t(), out=out)}
    for f in fns.values():
        f()
    torch.cuda.synchronize()
    for name, f in fns.items():
        host = []
        for _ in range(20):
            torch.cuda._sleep(5_000_000)  # keep the GPU busy: nothing below blocks
            t0 = time.perf_counter()
            f()
            host.append((time.perf_counter() - t0) * 1e6)
            torch.cuda.synchronize()
        dev = []
        for _ in range(20):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(2_000_000)  # pre-load: the events bracket device time only
            s.record()
            f()
            e.record()
            torch.cuda.synchronize()
            dev.append(s.elapsed_time(e) * 1e3)
        print(f"{name:20s} host enqueue median {statistics.median(host):7.1f} us   device (pre-loaded) median "
              f"{statistics.median(dev):7.1f} us", flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
