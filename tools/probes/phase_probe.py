"""GEMM phase trace (dev probe; needs the instrumented build made by
tools/probes/phase_patch.py, whose kernel writes %globaltimer stamps after
the per-tile area of the debug buffer): per stamp, the min / median / max over
CTAs of (stamp - first CTA's entry), median over runs, L2 flushed by a write.

    python tools/probes/phase_probe.py tools/probes/phase [M N K S ts]...
"""
import os
import sys

root = sys.argv[1]
sys.path.insert(0, root)
sys.path.insert(1, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import torch  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402
import synthetic  # noqa: E402

NAMES = ["entry", "setup done", "1st TMA issued", "MMA 1st full", "MMA last commit", "epi last tfull",
         "epi stores issued", "epi signalled", "epi bulk done", "exit barrier", "barriers init'd",
         "TMEM allocated", "thread 0 at sync", "prologue start", "1st stage issued"]


def main():
    torch.cuda.set_device(0)
    noflush = "--noflush" in sys.argv
    args = [int(v) for v in sys.argv[2:] if v != "--noflush"] or [1024, 4096, 4096, 64, 0]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for c in range(0, len(args), 5):
        M, N, K, S, ts = args[c:c + 5]
        A, Bt = synthetic.float_inputs(M, N, K, seed=1, device="cuda")
        C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        p = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, swizzle=0,
                    options={"tail_split": ts} if ts else None)
        tiles = (M // 256) * (N // 256)
        grid = 2 * S
        buf = torch.zeros(tiles + grid * 16, dtype=torch.int64, device="cuda")
        runs = []
        for it in range(8):
            buf.zero_()
            if not noflush:
                flush.zero_()
            torch.cuda.synchronize()
            fo.gemm_stage_timed(p, A, Bt, C, buf)
            torch.cuda.synchronize()
            st = buf[tiles:].view(grid, 16)[:, :len(NAMES)].cpu()
            if it >= 2:
                runs.append(st)
        print(f"== {M}x{N}x{K} S={S} ts={ts} tiles={tiles}" + (" (no L2 flush)" if noflush else ""))
        for i, name in enumerate(NAMES):
            mins, meds, maxs = [], [], []
            for st in runs:
                t0 = st[:, 0][st[:, 0] > 0].min()
                v = st[:, i]
                v = v[v > 0]
                if len(v) == 0:
                    continue
                d = (v - t0).double() / 1e3
                mins.append(d.min().item())
                meds.append(d.median().item())
                maxs.append(d.max().item())
            if mins:
                med = lambda x: sorted(x)[len(x) // 2]  # noqa: E731
                print(f"  {name:18s} min {med(mins):8.2f} med {med(meds):8.2f} max {med(maxs):8.2f}")


if __name__ == "__main__":
    main()
