"""Run the config-3 (or --workload) build a few times: a target for ncu captures
of k_build alone (tools/gpu_prof_build.sh)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1901_05423_b200 as rtf  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c3")
ap.add_argument("--reps", type=int, default=4)
a = ap.parse_args()
wl = bench.WORKLOADS[a.workload]
p = torch.from_numpy(bench.make_p(wl)).cuda()
f = rtf.build(p, wl["m"])
for _ in range(a.reps):
    f.build(p)
torch.cuda.synchronize()
print("status", f.status(), "n_pos", f.n_pos())
