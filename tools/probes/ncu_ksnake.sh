set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python tools/gemm_ab_probe.py > gpurun_out/ksnake.txt 2>&1; cat gpurun_out/ksnake.txt
# dram bytes of the bench shape, forward vs snake
cat > /tmp/one.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
import paper_2504_19519_b200 as fo
snake = int(sys.argv[1]); S = int(sys.argv[2]); ts = int(sys.argv[3])
M, N, K = 4096, 4096, 14336
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
Bt = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
p = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S, swizzle=0, options={"tail_split": ts, "k_snake": snake} if ts else {"k_snake": snake})
for _ in range(3): fo.gemm_stage(p, A, Bt, C)
torch.cuda.synchronize()
PY
for cfg in "0 74 -1" "1 74 -1" "0 64 0" "1 64 0"; do
  set -- $cfg
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:fo_gemm -s 2 -c 1 --csv python /tmp/one.py $1 $2 $3 2>/dev/null | grep -E "dram__bytes|gpu__time" | awk -F'","' -v c="$cfg" '{print c, $(NF-2), $NF}'
done
