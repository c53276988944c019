"""A/B of config-4 sampling between library builds: python tools/ab_c4.py LIB [LIB...]
Each library runs in its own subprocess (RTF_AB_LIB): one 2^28 build, then
2^30 Philox samples, median of 3 device-timed batches."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child():
    sys.path.insert(0, ROOT)
    import ctypes
    from paper_1901_05423_b200 import _lib
    _lib.LIB_PATH = os.environ["RTF_AB_LIB"]
    probe = ctypes.CDLL(_lib.LIB_PATH)
    for k in list(_lib.PROTOTYPES):
        if not hasattr(probe, k):
            del _lib.PROTOTYPES[k]
    import torch
    import bench
    import paper_1901_05423_b200 as rtf
    wl = bench.WORKLOADS["c4"]
    p = torch.from_numpy(bench.make_p(wl)).cuda()
    f = rtf.build(p, wl["m"])
    xi = rtf.philox(1 << 30, seed=0x5EED)
    out = torch.empty_like(xi)
    f.sample(xi, out)
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); f.sample(xi, out); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    print(f"{os.path.basename(_lib.LIB_PATH):22s} c4 sample 2^30 {ts[1]:.3f} ms "
          f"({(1 << 30) / ts[1] / 1e6:.1f} G samples/s)", flush=True)


if __name__ == "__main__":
    if os.environ.get("RTF_AB_LIB"):
        child()
    else:
        for lib in sys.argv[1:]:
            env = dict(os.environ, RTF_AB_LIB=os.path.abspath(lib))
            subprocess.run([sys.executable, os.path.abspath(__file__)], env=env, check=False)
