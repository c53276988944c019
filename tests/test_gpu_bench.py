"""bench.py's small workloads run end to end on the GPU and print the contract's
JSON line (the default config-3 line is produced by the driver's own bench run)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    return json.loads(lines[0])


def test_bench_c1_latency_line():
    d = run_bench("--workload", "c1", "--steps", "20", "--warmup", "3")
    assert d["indices_match_inverse_cdf"] is True
    assert d["higher_is_better"] is False and d["value"] > 0
    assert d["launches_per_step"] == 2 and d["gpu_launches"] > 0
    for k in ("metric", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "config", "clocks"):
        assert k in d, k
