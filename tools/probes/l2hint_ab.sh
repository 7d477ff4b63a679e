# FO_OPT_L2_HINTS A/B: gemm parity subset, device time, ncu dram bytes per mode
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -x > gpurun_out/l2_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/l2_tests.log
timeout 600 python tools/probes/l2hint_probe.py > gpurun_out/l2_time.txt 2>&1; echo time rc=$?
timeout 600 python tools/probes/l2hint_probe.py > gpurun_out/l2_time2.txt 2>&1; echo time2 rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:fo_gemm --csv python tools/probes/l2hint_probe.py ncu > gpurun_out/l2_ncu.csv 2> gpurun_out/l2_ncu.err; echo ncu rc=$?
cat gpurun_out/l2_time.txt gpurun_out/l2_time2.txt
