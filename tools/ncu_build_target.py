"""Minimal ncu target: three C3 builds (n = 2^24, m = 2^22, bench.py's
workload) so that `ncu -k regex:k_build -s 2 -c 1` captures a warm launch.
  python tools/ncu_build_target.py [c3|c2]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1901_05423_b200 as rtf  # noqa: E402

wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
p = torch.from_numpy(bench.make_p(wl)).cuda()
f = rtf.Forest(wl["n"], wl["m"])
for _ in range(3):
    f.build(p)
torch.cuda.synchronize()
assert f.status() == 0
