# multicast vs plain pairs at S=64 on the bench shape, ncu: time, clock, tensor active, L2->SM sectors; + combine tests (launch caching)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "combine" > gpurun_out/mc_cmb.log 2>&1; echo cmb rc=$?; tail -1 gpurun_out/mc_cmb.log
timeout 900 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,lts__t_sectors_srcunit_tex.sum,dram__bytes_read.sum --clock-control none --cache-control all --csv python tools/probes/mc_ncu.py 4096 4096 14336 > gpurun_out/mc.csv 2> gpurun_out/mc.err; echo ncu rc=$?
