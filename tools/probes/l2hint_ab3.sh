# mode-0 regression check after moving the hint setup out of the prologue (ncu ns resolution, two runs per build)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for i in 1 2; do for b in old new; do
  root=$([ $b = old ] && echo tools/probes/ab_old || echo .)
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control all --csv --log-file gpurun_out/ab3_${b}_$i.csv python tools/probes/ab_ncu.py $root > /dev/null 2>&1
done; done
python tools/probes/ab_ncu.py --parse gpurun_out/ab3_old_1.csv gpurun_out/ab3_new_1.csv gpurun_out/ab3_old_2.csv gpurun_out/ab3_new_2.csv
