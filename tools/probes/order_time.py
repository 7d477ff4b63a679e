"""Time of the bench GEMM under several tile orders (device-time means of 20)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2504_19519_b200 as fo  # noqa: E402
import synthetic  # noqa: E402
M, N, K = 4096, 4096, 14336
torch.cuda.set_device(0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
A, Bt = synthetic.float_inputs(M, N, K, seed=1, device="cuda")
C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
v = {}
for swz in (7, 8, 9, -1):
    p = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=74, swizzle=swz, options={"tail_split": -1})
    v[f"swz{swz}"] = (lambda p=p: fo.gemm_stage(p, A, Bt, C))
for f in v.values():
    f()
torch.cuda.synchronize()
ts = {k: [] for k in v}
for _ in range(20):
    for k, f in v.items():
        flush.zero_()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(200_000)
        s.record()
        f()
        e.record()
        torch.cuda.synchronize()
        ts[k].append(s.elapsed_time(e) * 1e3)
print(" ".join(f"{k}: {sum(x) / len(x):.1f} us" for k, x in ts.items()))
