"""A/B of two GEMM builds with ns-resolution kernel durations (dev probe).

The CUDA event clock on these boxes ticks in ~2.05 us steps and the one-wave
shapes repeat to within a tick, so event means cannot resolve sub-2-us changes.
This runs the ab_gemm.py cases `--reps` times each for the build under
`<package root>`; run it under

    ncu --metrics gpu__time_duration.sum --clock-control none --cache-control all \
        --csv --log-file OUT.csv python tools/probes/ab_ncu.py <root>

(ncu flushes the caches before every launch: cold L2 as in the bench) and
summarise with `python tools/probes/ab_ncu.py --parse OUT.csv [OUT2.csv ...]`."""
import csv
import os
import statistics
import sys

CASES = [(4096, 4096, 14336, 74, -1), (1024, 4096, 4096, 64, 0), (1024, 4096, 14336, 64, 0),
         (4096, 4096, 1792, 64, 0), (8192, 8192, 1024, 64, 0), (2048, 4096, 4096, 64, 0)]
REPS = 10


def run(root):
    sys.path.insert(0, root)
    sys.path.insert(1, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
    import torch
    import paper_2504_19519_b200 as fo
    import synthetic
    torch.cuda.set_device(0)
    for (M, N, K, S, ts) in CASES:
        A, Bt = synthetic.float_inputs(M, N, K, seed=1, device="cuda")
        C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        p = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, swizzle=0,
                    options={"tail_split": ts} if ts else None)
        for _ in range(REPS):
            fo.gemm_stage(p, A, Bt, C)
        torch.cuda.synchronize()


def parse(paths):
    for path in paths:
        rows = []
        with open(path) as f:
            lines = [ln for ln in f if ln.startswith('"')]
        for r in csv.DictReader(lines):
            if "fo_gemm_tcgen05" in r["Kernel Name"] and r["Metric Name"] == "gpu__time_duration.sum":
                v = float(r["Metric Value"].replace(",", ""))
                rows.append(v / 1e3 if r["Metric Unit"] in ("ns", "nsecond") else v)
        out = []
        for i, (M, N, K, S, ts) in enumerate(CASES):
            v = rows[i * REPS:(i + 1) * REPS]
            if v:
                out.append(f"{M}x{N}x{K}/S{S}: {statistics.median(v):.2f}")
        print(path, " ".join(out))


if __name__ == "__main__":
    if sys.argv[1] == "--parse":
        parse(sys.argv[2:])
    else:
        run(sys.argv[1])
