# mode-0 regression check (previous build vs this, events + ncu) and the L2-hint probe on more shapes
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for i in 1 2; do
  timeout 600 python tools/probes/ab_gemm.py tools/probes/ab_old >> gpurun_out/ab_ev.txt 2>&1
  timeout 600 python tools/probes/ab_gemm.py . >> gpurun_out/ab_ev.txt 2>&1
done
for b in old new; do
  root=$([ $b = old ] && echo tools/probes/ab_old || echo .)
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control all --csv --log-file gpurun_out/ab_$b.csv python tools/probes/ab_ncu.py $root > /dev/null 2>&1
done
python tools/probes/ab_ncu.py --parse gpurun_out/ab_old.csv gpurun_out/ab_new.csv > gpurun_out/ab_ncu.txt 2>&1
timeout 900 python tools/probes/l2hint_probe.py > gpurun_out/l2_time3.txt 2>&1
cat gpurun_out/ab_ev.txt gpurun_out/ab_ncu.txt gpurun_out/l2_time3.txt
