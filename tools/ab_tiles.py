"""Build time of the default tiles vs RTF_BUILD_SMALL_TILES (256-entry tiles,
one warp per CTA) for several n: python tools/ab_tiles.py"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1901_05423_b200 as rtf  # noqa: E402
from workloads import power_law  # noqa: E402

cases = [("c2", torch.from_numpy(bench.make_p(bench.WORKLOADS["c2"])).cuda(), 1 << 21)]
for lg in (18, 20, 22, 24):
    cases.append((f"A n=2^{lg}", torch.from_numpy(power_law(1 << lg, "A")).cuda(), 1 << (lg - 2)))
for name, p, m in cases:
    res = []
    for flags in (0, 1):
        f = rtf.Forest(p.numel(), m, flags)
        for _ in range(3):
            f.build(p)
        ts = []
        for _ in range(20):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); f.build(p); b.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        res.append(statistics.median(ts) * 1e3)
    print(f"{name:12s} default {res[0]:8.1f} us   small tiles {res[1]:8.1f} us", flush=True)
