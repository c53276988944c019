"""The C ABI without Python: examples/rtf_demo.c, compiled with gcc against
include/rtf.h and librtf.so, builds and samples on the GPU; and the
build + sample pair captured in a CUDA graph replays to identical results
(rtf.h: every call is stream-ordered and launch-only)."""
import os
import subprocess

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from workloads import philox_xi, power_law  # noqa: E402

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_demo(tmp_path):
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_1901_05423_b200._build_lib import build_library
    lib = build_library()
    exe = str(tmp_path / "rtf_demo")
    subprocess.check_call(["gcc", "-O2", "-o", exe, os.path.join(ROOT, "examples", "rtf_demo.c"),
                           "-I" + os.path.join(ROOT, "include"), "-I/usr/local/cuda/include",
                           "-L" + os.path.dirname(lib), "-lrtf", "-L/usr/local/cuda/lib64",
                           "-lcudart", "-lm", "-Wl,-rpath," + os.path.dirname(lib)])
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr + out.stdout
    assert "ok" in out.stdout


def test_cuda_graph_capture():
    import paper_1901_05423_b200 as rtf
    p = torch.from_numpy(power_law(1 << 20, "A")).cuda()
    f = rtf.Forest(p.numel(), 1 << 18)
    xi = torch.from_numpy(philox_xi(1 << 20, seed=5).view(np.int32)).cuda()
    out = torch.empty_like(xi)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        f.build(p, stream=s)
        f.sample(xi, out, stream=s)
    torch.cuda.synchronize()
    ref = out.clone()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        f.build(p, stream=s)
        f.sample(xi, out, stream=s)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    # new data in the same buffers: the replayed build picks it up
    p.copy_(torch.from_numpy(power_law(1 << 20, "D")))
    g.replay()
    torch.cuda.synchronize()
    f2 = rtf.build(p, 1 << 18)
    assert torch.equal(out, f2.sample(xi))
