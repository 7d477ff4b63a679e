"""bench.py's JSON-line contract (the driver parses it): the reference arm
(the CPU oracle, runs anywhere) and, on a GPU, our arm with every key the
contract names — roofline, cpu_baseline, e2e, gpu_launches, clocks."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config"}


def _run(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT, capture_output=True,
                       text=True, timeout=timeout)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "3"], 600)
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["steps"] == 1 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["higher_is_better"] is False and d["value"] > 0
    assert d["config"]["workload"]
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_gpu_arm_contract():
    d = _run(["--steps", "5", "--warmup", "3"], 1200)
    assert BASE_KEYS <= set(d)
    assert "impl" not in d or d["impl"] != "reference"
    assert d["steps"] == 5 and d["warmup"] == 3 and d["n_gpus"] == 1 and d["value"] > 0
    assert d["dtype"] == "bf16" and d["config"]["workload"]
    rf = d["roofline"]
    assert rf["bound"] in ("hbm", "tensor", "alu") and rf["unit"] in ("GB/s", "TFLOP/s")
    assert rf["achieved"] > 0 and rf["peak"] > 0
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-3
    assert d["cpu_baseline"]["kind"] == "oracle"
    e = d["e2e"]
    assert e["value"] > 0 and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    lc = d["latency_conventions"]   # SURVEY ambiguity 17: strict headline, paper's, fused
    assert lc["strict_us"] == d["value"] and lc["fused_us"] > 0
    assert lc["paper_us"] is None or lc["paper_us"] <= lc["strict_us"]
    assert d["perfect_overlap_bound_us"] > 0 and d["step_stats_us"]["ov"]["p10"] <= d["step_stats_us"]["ov"]["p90"]


@pytest.mark.gpu
@pytest.mark.parametrize("n", [2, 8])
def test_gpu_arm_n_gt_1_code_paths_emulated(n):
    """bench.py's N>1 code paths (tuner across two CTA caps with in-situ
    curves, the sequential baseline at its own wave width on an uncapped
    communicator, e2e, perfect-overlap bound, max-over-ranks plumbing) run on
    one GPU with --emulate-world (the emulated-link evaluation backend, R42);
    the line says so in `data`.  Only the real multi-GPU run (torchrun, NCCL)
    measures NVLink."""
    d = _run(["--emulate-world", str(n), "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-shards"], 1200)
    assert BASE_KEYS <= set(d)
    assert d["n_gpus"] == n and d["value"] > 0 and "EMULATED" in d["data"]
    assert d["config"]["tp"] == n and d["config"]["K_loc"] == 14336 // n
    assert d["sequential_us"] > 0 and d["layer_roofline"]["allreduce_ring_us"] > 0
    assert d["nccl_allreduce_uncapped"]["points"]
    assert d["e2e"]["h2d_bytes_per_step"] == 4096 * (14336 // n) * 2
