"""Table-1-style measurement on one B200: the power-law / exponential families
A-D (workloads.power_law) at n = 2^24, m = 2^22, 2^28 Philox
samples: build time, sampling rate, loads (max, avg, avg_32: Table 1's
columns) with and without the two-interval / packed flags, the
worst case over every 32-bit xi before and after the fallback (R21), and the
GPU baselines on the same CDF (binary search, Eytzinger binary search,
cutpoint + binary)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1901_05423_b200 as rtf  # noqa: E402
from workloads import power_law  # noqa: E402

n, m, S = 1 << 24, 1 << 22, 1 << 28
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=5):
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


xi = rtf.philox(S, seed=0x5EED)
out = torch.empty_like(xi)
rows = []
for fam in "ABCD":
    p = torch.from_numpy(power_law(n, fam)).cuda()
    f = rtf.Forest(n, m)
    f.build(p)
    tb = timed(lambda: f.build(p))
    ts = timed(lambda: f.sample(xi, out))
    loads, plain = f.sample_loads(xi[: 1 << 20], plain=True)
    loads, plain = loads.double(), plain.double()
    cdf = rtf.build_cdf(p)
    cut = cdf.cutpoint(m)
    ey = cdf.eytzinger()
    bs, cb, eb = torch.empty_like(out), torch.empty_like(out), torch.empty_like(out)
    tbs = timed(lambda: cdf.sample(xi, bs), 3)
    tcb = timed(lambda: cut.sample(xi, cb, binary=True), 3)
    tey = timed(lambda: ey.sample(xi, eb), 3)
    assert torch.equal(bs, out) and torch.equal(cb, out) and torch.equal(eb, out)
    f.build_fallback()
    depth, _ = f.cell_depths()
    tab = f.table_numpy()
    marked = (tab["ref"] >= 0) & (tab["key32"] >> 30 == 3)
    kk = tab["key32"].astype("int64") & 0x3FFFFFFF
    bis = np.where(marked, np.ceil(np.log2(kk + 1)).astype(np.int64), 0)
    worst = (int(depth.max()) + 1, int(np.where(marked, bis, depth).max()) + 1)
    del ey
    rows.append({
        "family": fam, "n_pos": f.n_pos(), "build_ms": round(tb, 4),
        "build_G_entries_s": round(n / tb / 1e6, 2),
        "sample_G_s": round(S / ts / 1e6, 1), "bsearch_G_s": round(S / tbs / 1e6, 1),
        "eytzinger_G_s": round(S / tey / 1e6, 1),
        "cutpoint_binary_G_s": round(S / tcb / 1e6, 1),
        "speedup_vs_best_bsearch": round(min(tbs, tey) / ts, 2),
        "worst_case_loads_all_xi": {"radix": worst[0], "with_fallback": worst[1],
                                    "cells_marked": int(marked.sum())},
        "loads": {"max": int(loads.max()), "avg": round(loads.mean().item(), 3),
                  "avg32": round(loads.view(-1, 32).max(1).values.mean().item(), 3)},
        "loads_without_flag": {"avg": round(plain.mean().item(), 3),
                               "avg32": round(plain.view(-1, 32).max(1).values.mean().item(), 3)},
    })
    print(json.dumps(rows[-1]), flush=True)
