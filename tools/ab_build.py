"""A/B timing between library builds: python tools/ab_build.py LIB [LIB...]
Each library runs in its own subprocess (RTF_AB_LIB); prints median build times
for c3/c2 and the c3 sampling time."""
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
    res = []
    for wlname in ("c3", "c2"):
        wl = bench.WORKLOADS[wlname]
        p = torch.from_numpy(bench.make_p(wl)).cuda()
        f = rtf.Forest(wl["n"], wl["m"])
        for _ in range(3):
            f.build(p)
        ts = []
        for _ in range(30):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); f.build(p); b.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ts.sort()
        res.append(f"{wlname} build {ts[15]*1e3:7.1f} us (min {ts[0]*1e3:7.1f})")
        if wlname == "c2":
            xi = rtf.philox(1 << 26, seed=0x5EED)
            out = torch.empty_like(xi)
            f.sample(xi, out)
            ts = []
            for _ in range(7):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(); f.sample(xi, out); b.record(); torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            ts.sort()
            res.append(f"c2 sample 2^26 {ts[3]*1e3:.1f} us")
        if wlname == "c3":
            xi = rtf.philox(1 << 28, seed=0x5EED)
            out = torch.empty_like(xi)
            f.sample(xi, out)
            ts = []
            for _ in range(5):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(); f.sample(xi, out); b.record(); torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            ts.sort()
            res.append(f"c3 sample 2^28 {ts[2]:.3f} ms")
    print(f"{os.path.basename(_lib.LIB_PATH):22s}", " | ".join(res), flush=True)


if __name__ == "__main__":
    if os.environ.get("RTF_AB_LIB"):
        child()
    else:
        for lib in sys.argv[1:]:
            env = dict(os.environ, RTF_AB_LIB=os.path.abspath(lib))
            subprocess.run([sys.executable, os.path.abspath(__file__)], env=env, check=False)
