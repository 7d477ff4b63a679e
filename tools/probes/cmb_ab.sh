# A/B of the MoE combine kernel: combine parity tests, loopback world 2, combine_probe old build vs this build
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "combine" > gpurun_out/cmb_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/cmb_tests.log
CUDA_MODULE_LOADING=EAGER timeout 300 python tests/loopback_worker.py 2 > gpurun_out/cmb_loop.log 2>&1; echo loop rc=$?; tail -3 gpurun_out/cmb_loop.log
(echo "## old"; timeout 300 python tools/combine_probe.py tools/probes/ab_old; echo "## new"; timeout 300 python tools/combine_probe.py; echo "## old again"; timeout 300 python tools/combine_probe.py tools/probes/ab_old; echo "## new again"; timeout 300 python tools/combine_probe.py) > gpurun_out/cmb_probe.txt 2>&1
grep -v "^$" gpurun_out/cmb_probe.txt | grep "k=2\|##" | grep -v index
