"""bench.py's N > 1 code paths on a one-GPU lease: two
torchrun ranks on cuda:0 over gloo (RTF_DIST_BACKEND=gloo, RTF_ONE_DEVICE=1;
collectives staged through host memory, the fused build's peer stores through
CUDA IPC).  The timings are meaningless here; the lines must be well formed
and every rank's build must succeed."""
import json
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(extra):
    env = dict(os.environ, RTF_DIST_BACKEND="gloo", RTF_ONE_DEVICE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "3",
           "--no-cpu-baseline", *extra]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_c3_sharded_two_ranks():
    d = _run(["--samples", str(1 << 22)])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak"
    assert d["config"]["n"] == 2 << 24 and d["config"]["m"] == 2 << 22
    assert d["config"]["n_pos"] > 0 and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 4 << 24


def test_bench_c4_sharded_two_ranks():
    d = _run(["--workload", "c4", "--samples", str(1 << 22)])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
