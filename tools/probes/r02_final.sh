# end-of-round evidence on HEAD: GPU suite + smoke, bench line, ncu launch list of the bench step, ncu --set full of the bench GEMM
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/f_gpu_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/f_gpu_tests.log
timeout 600 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo bench rc=$?
timeout 600 python bench.py --impl reference > gpurun_out/f_bench_ref.json 2> gpurun_out/f_bench_ref.err; echo ref rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-shards > /dev/null 2>&1; echo ncu-list rc=$?
cat > /tmp/one.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
import paper_2504_19519_b200 as fo
import synthetic
M, N, K = 4096, 4096, 14336
A, Bt = synthetic.float_inputs(M, N, K, seed=1, device="cuda")
C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
p = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=74, swizzle=0, options={"tail_split": -1})
for _ in range(3): fo.gemm_stage(p, A, Bt, C)
torch.cuda.synchronize()
PY
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fo_gemm -s 2 -c 1 -o gpurun_out/f_gemm_full python /tmp/one.py > /dev/null 2>&1; echo ncu-full rc=$?
