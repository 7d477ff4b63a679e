# r02 evidence run: bench line, ncu launch list of the bench step, ncu --set full of the bench GEMM
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
echo bench rc=$?
tail -c 600 gpurun_out/r02_bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-shards > /dev/null 2>&1
echo ncu-list rc=$?
cat > /tmp/one.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
import paper_2504_19519_b200 as fo
M, N, K = 4096, 4096, 14336
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
Bt = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
p = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=74, swizzle=0, options={"tail_split": -1})
for _ in range(3): fo.gemm_stage(p, A, Bt, C)
torch.cuda.synchronize()
PY
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fo_gemm -s 2 -c 1 -o gpurun_out/r02_gemm_full python /tmp/one.py > /dev/null 2>&1
echo ncu-full rc=$?
