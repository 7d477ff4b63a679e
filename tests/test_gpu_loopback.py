"""The multi-rank data path at world 2, 4 and 8 on one B200 (loopback
communicator, tests/loopback_worker.py): fo_run (both triggers, split tail),
fo_run_sequential, fo_run_allgather and fo_run_host for AllReduce (slot /
rowband / single group), ReduceScatter and imbalanced All-to-All, every rank's
output bit-exact vs the oracle's plain definitions.  Each world runs in its own
subprocess under a timeout (a schedule mismatch traps the device instead of
hanging; the process dies, the GPU stays usable)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_loopback_world(world):
    # eager module loading: a lazily loaded kernel's first launch may wait for
    # running kernels, i.e. for another in-process rank's call at its barrier
    env = dict(os.environ, CUDA_DEVICE_MAX_CONNECTIONS="32", CUDA_MODULE_LOADING="EAGER")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "loopback_worker.py"), str(world)], cwd=ROOT,
                       env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and f"loopback W={world}: OK" in r.stdout, r.stdout[-4000:] + r.stderr[-4000:]
