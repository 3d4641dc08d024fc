"""bench.py keeps the driver's JSON contract (one line, the required keys).

GPU: runs the small C1 workload through bench.py for a few steps; CPU: the
reference arm (the oracle) on a tiny sample.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REQUIRED = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
            "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config"]


def _run(args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args,
                         capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "2", "--warmup", "1", "--ref-seconds", "2",
              "--workload", "C1"])
    for k in REQUIRED:
        assert k in d, k
    assert d["impl"] == "reference"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["value"] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("workload", ["C1", "C2"])
def test_our_arm_line(workload):
    d = _run(["--workload", workload, "--steps", "20", "--warmup", "3", "--no-cpu-baseline",
              "--e2e-iters", "3", "--e2e-steps", "1"])
    for k in REQUIRED + ["roofline", "e2e", "gpu_launches", "clocks", "stage_ms"]:
        assert k in d, k
    r = d["roofline"]
    for k in ["bound", "achieved", "peak", "unit", "frac", "traffic"]:
        assert k in r, k
    assert d["gpu_launches"] > 0 and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["config"]["workload"] == workload
