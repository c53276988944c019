"""Host-buffer sampling (rtf_sample_host) at several staging chunk sizes, next
to the raw pinned H2D / D2H copy rates and a concurrent H2D + D2H pair: how far
the e2e pipeline is from the PCIe floor.  C3 forest, 2^28 Philox xi.
  python tools/e2e_chunks.py"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1901_05423_b200 as rtf  # noqa: E402

wl = bench.WORKLOADS["c3"]
p = torch.from_numpy(bench.make_p(wl)).cuda()
f = rtf.Forest(wl["n"], wl["m"]).build(p)
S = 1 << 28
xi = rtf.philox(S, seed=0x5EED)
xi_h = torch.empty(S, dtype=torch.int32).pin_memory()
xi_h.copy_(xi.cpu())
out_h = torch.empty(S, dtype=torch.int32).pin_memory()
dev_a = torch.empty(S, dtype=torch.int32, device="cuda")
dev_b = torch.empty(S, dtype=torch.int32, device="cuda")


def wall(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts)


GB = 4 * S / 1e9
t = wall(lambda: dev_a.copy_(xi_h, non_blocking=True))
print(f"H2D 1 GB pinned: {GB / t:.1f} GB/s")
t = wall(lambda: out_h.copy_(dev_b, non_blocking=True))
print(f"D2H 1 GB pinned: {GB / t:.1f} GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def both():
    with torch.cuda.stream(s1):
        dev_a.copy_(xi_h, non_blocking=True)
    with torch.cuda.stream(s2):
        out_h.copy_(dev_b, non_blocking=True)
    s1.synchronize()
    s2.synchronize()


t = wall(both)
print(f"H2D + D2H concurrent, 1 GB each: {t * 1e3:.1f} ms -> floor {S / t / 1e9:.2f} G samples/s")
for lg in (18, 20, 22, 23, 24, 25):
    chunk = 1 << lg
    xs = torch.empty(2 * chunk, dtype=torch.int32, device="cuda")
    os_ = torch.empty(2 * chunk, dtype=torch.int32, device="cuda")
    t = wall(lambda: rtf.sample_host(f, xi_h, out_h, xs, os_))
    ok = torch.equal(out_h[: 1 << 20].cuda(), f.sample(xi[: 1 << 20]))
    print(f"sample_host chunk 2^{lg}: {t * 1e3:.1f} ms = {S / t / 1e9:.2f} G samples/s  exact={ok}")
