"""A/B of the config-5 rows build and rows sampling between library builds (child processes)."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if os.environ.get("RTF_AB_LIB"):
    sys.path.insert(0, ROOT)
    import ctypes
    from paper_1901_05423_b200 import _lib
    _lib.LIB_PATH = os.environ["RTF_AB_LIB"]
    import torch, bench, statistics
    import paper_1901_05423_b200 as rtf
    wl = bench.WORKLOADS["c5"]
    p = torch.from_numpy(bench.make_p(wl)).cuda()
    f = rtf.RowsForest(wl["rows"], wl["n_row"], wl["m"])
    for _ in range(3): f.build(p)
    ts = []
    for _ in range(15):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); f.build(p); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    print(f"{os.path.basename(_lib.LIB_PATH):22s} c5 build {statistics.median(ts):.4f} ms (min {min(ts):.4f})", flush=True)
    # 2048-entry rows (the 2-D env map's conditionals): 1024 x 2048
    p2 = torch.rand(1024 * 2048, generator=torch.Generator().manual_seed(3)).cuda()
    f2 = rtf.RowsForest(1024, 2048, 2048)
    for _ in range(3): f2.build(p2)
    ts = []
    for _ in range(15):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); f2.build(p2); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    print(f"{os.path.basename(_lib.LIB_PATH):22s} 1024x2048 rows build {statistics.median(ts):.4f} ms (min {min(ts):.4f})", flush=True)
else:
    for lib in sys.argv[1:]:
        subprocess.run([sys.executable, os.path.abspath(__file__)], env=dict(os.environ, RTF_AB_LIB=os.path.abspath(lib)))
