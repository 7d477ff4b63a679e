"""Real multi-GPU parity (NCCL over NVLink): tests/mgpu_worker.py on 2, 4 and
8 ranks of one box, every rank's fo_run / fo_run_sequential output bit-exact
vs the plain collective (n = 1 runs the same worker through torchrun on one
GPU).  Skipped when the box has fewer GPUs (the round's
gpurun boxes have one; the n > 1 host logic is covered by test_dist_gloo and
the kernels rank by rank by test_gpu_parity / test_gpu_fuzz)."""
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_multi_gpu_parity(n):
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs, {torch.cuda.device_count()} visible")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "tests", "mgpu_worker.py")]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "multi-GPU parity: OK" in r.stdout
