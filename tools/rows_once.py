"""Run the config-5 batched build a few times (an ncu target for k_build_rows)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench
import paper_1901_05423_b200 as rtf
wl = bench.WORKLOADS["c5"]
p = torch.from_numpy(bench.make_p(wl)).cuda()
f = rtf.RowsForest(wl["rows"], wl["n_row"], wl["m"])
for _ in range(3):
    f.build(p)
torch.cuda.synchronize()
print("ok")
