import sys, os, numpy as np, torch
sys.path.insert(0, "/root/repo" if os.path.exists("/root/repo") else ".")
import paper_2504_19519_b200 as fo, synthetic
M, N, K = 4096, 4096, 14336
A, Bt = synthetic.float_inputs(M, N, K, seed=1, device="cuda")
out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
S = 74
plan = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, options={"tail_split": -1})
ts = torch.zeros(256, dtype=torch.int64, device="cuda")
res = []
for it in range(7):
    flush.zero_(); torch.cuda.synchronize()
    fo.gemm_stage_timed(plan, A, Bt, out, ts); torch.cuda.synchronize()
    t = ts.cpu().numpy().astype(np.int64); t = (t - t.min()) / 1e3
    w2 = t[2 * S:3 * S]            # wave-2 finish per worker (worker = position % S)
    tail = t[3 * S:]               # tail tile r: slices on workers 2r, 2r+1
    slice_us = np.median(tail - np.maximum(w2[0:68:2], w2[1:68:2]))
    # static: tile r done at max(w2[2r], w2[2r+1]) + slice_us ; dynamic: slices to the earliest finishers in order
    static_end = max(np.max(np.maximum(w2[0:68:2], w2[1:68:2]) + slice_us), w2.max())
    order = np.sort(w2)
    dyn_end = max(np.max(np.maximum(order[0:68:2], order[1:68:2]) + slice_us), w2.max())
    res.append((t.max(), slice_us, static_end, dyn_end, w2.min(), np.median(w2), w2.max()))
    print(f"run {it}: measured end {t.max():.1f}  slice+fold {slice_us:.1f}  model static {static_end:.1f}  dynamic {dyn_end:.1f}  wave2 finish min/med/max {w2.min():.1f}/{np.median(w2):.1f}/{w2.max():.1f}")
# which workers are slow: rank by mean wave-2 finish
