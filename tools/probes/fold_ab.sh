# split-tail fold with the partials staged by one cp.async batch: tail-split parity, then ncu A/B vs the previous build
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_fuzz.py tests/test_gpu_parity.py -q -x -k "tail or split or fuzz or bench_plan" > gpurun_out/fold_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/fold_tests.log
for i in 1 2; do for b in old new; do
  root=$([ $b = old ] && echo tools/probes/ab_old || echo .)
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control all --csv --log-file gpurun_out/fold_${b}_$i.csv python tools/probes/ab_ncu.py $root > /dev/null 2>&1
done; done
python tools/probes/ab_ncu.py --parse gpurun_out/fold_old_1.csv gpurun_out/fold_new_1.csv gpurun_out/fold_old_2.csv gpurun_out/fold_new_2.csv
python tools/probes/tail_trace.py 2>&1 | head -6
