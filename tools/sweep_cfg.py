"""Experiment: time the build under RTF_EXPERIMENT_CFG variants (set per process)
and check the result against the oracle once.  Usage: python tools/sweep_cfg.py CFG"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_1901_05423_b200 as rtf  # noqa: E402
from workloads import power_law  # noqa: E402

cfg = os.environ.get("RTF_EXPERIMENT_CFG", "0")
n, m = 1 << 24, 1 << 22
p = power_law(n, "A")
pd = torch.from_numpy(p).cuda()
f = rtf.Forest(n, m)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    f.build(pd)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    f.build(pd)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ref = oracle.build(p, m)
nodes = f.nodes_numpy()
ok = (np.array_equal(nodes["key"], ref.key) and np.array_equal(nodes["c0"], ref.child0)
      and np.array_equal(nodes["c1"], ref.child1) and f.table_numpy().tobytes() == ref.table2().tobytes())
print(f"cfg {cfg}: build median {np.median(ts)*1e3:.1f} us  min {min(ts)*1e3:.1f} us  parity={ok}")
