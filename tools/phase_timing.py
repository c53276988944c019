"""Per-phase cycle breakdown of k_build (debug aid, not part of the product).

Builds tools/librtf_timing.so with -DRTF_PHASE_TIMING (thread 0 of every CTA
accumulates clock64() deltas per phase), runs the config-3 build a few times
and prints the mean cycles per CTA per phase.

  python tools/phase_timing.py --build      # here (nvcc cross-compiles)
  python tools/phase_timing.py              # on the GPU box
"""
import argparse
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
LIB = os.path.join(ROOT, "tools", "librtf_timing.so")
SLOTS = ["A scale (+barrier)", "B totals (+barrier)", "C spine (+barrier)",
         "D1 wait+quantise+warp scan (+bar 1)", "D2 scan/keys/lambda/table/records (+bar 2)",
         "D3 forest links (+bar 3)", "D4 record stores + spine row", "D tail (barrier wait)",
         "E cross-tile + runs"]


def build():
    from paper_1901_05423_b200 import _build_lib as b
    cmd = [b.NVCC, *b.NVCC_FLAGS, "-DRTF_PHASE_TIMING", "-o", LIB, *b.sources()]
    subprocess.check_call(cmd)
    print(LIB)


def run(reps, workload):
    import numpy as np
    import torch
    import paper_1901_05423_b200 as rtf
    from paper_1901_05423_b200 import _lib
    _lib.LIB_PATH = LIB
    rtf.lib()
    fn = ctypes.CDLL(LIB).rtf_debug_phase_cycles
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
    import bench
    wl = bench.WORKLOADS[workload]
    p = torch.from_numpy(bench.make_p(wl)).cuda()
    f = rtf.build(p, wl["m"])
    torch.cuda.synchronize()
    rows = 8192
    buf = np.zeros((rows, 16), np.uint64)
    fn(buf.ctypes.data, rows, 1)  # reset after warm-up
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    for _ in range(reps):
        f.build(p)
    stop.record()
    torch.cuda.synchronize()
    print(f"{workload}: {start.elapsed_time(stop) / reps * 1e3:.1f} us per build ({reps} builds)")
    fn(buf.ctypes.data, rows, 0)
    extra = buf[:, 9:11].astype(np.float64) / reps
    # slot 14: phase E's cross-tile links (slot 8 then holds the long runs only)
    buf[:, 8] += buf[:, 14]
    e1 = buf[:, 14].astype(np.float64) / reps
    used = buf[:, :9].sum(axis=1) > 0
    per = buf[used, :9].astype(np.float64) / reps
    tot = per.sum(axis=1)
    print(f"CTAs {used.sum()}, mean cycles per CTA per build {tot.mean():.0f} "
          f"(min {tot.min():.0f}, max {tot.max():.0f})")
    for s, name in enumerate(SLOTS):
        col = per[:, s]
        print(f"  {name:30s} mean {col.mean():9.0f}  max {col.max():9.0f}  "
              f"{100 * col.mean() / tot.mean():5.1f} %")
    # per-tile timeline of the last build (globaltimer, ns)
    try:
        tf = ctypes.CDLL(LIB).rtf_debug_tile_ns
        tf.argtypes = [ctypes.c_void_p, ctypes.c_int]
        nt = (wl["n"] + 4095) // 4096
        tb = np.zeros((min(nt, 65536), 3), np.uint64)
        tf(tb.ctypes.data, tb.shape[0])
        st = tb[:, 0].astype(np.int64)
        en = tb[:, 1].astype(np.int64)
        t0 = st.min()
        dur = (en - st) / 1e3
        nb = 16
        print(f"  tiles {nt}: phase D span {(en.max() - t0) / 1e3:.1f} us from the first tile start; "
              f"tile duration us (mean / p90 / max) {dur.mean():.2f} / {np.percentile(dur, 90):.2f} / {dur.max():.2f}")
        for k in range(nb):
            sl = slice(k * nt // nb, (k + 1) * nt // nb)
            print(f"    tiles {sl.start:6d}-{sl.stop - 1:6d}: mean {dur[sl].mean():6.2f} us  max {dur[sl].max():6.2f}")
        cta = tb[:, 2].astype(np.int64)
        last_end = np.zeros(cta.max() + 1, np.int64)
        np.maximum.at(last_end, cta, en)
        le = (last_end[last_end > 0] - t0) / 1e3
        print(f"  per-CTA last tile end (us from start): min {le.min():.1f} median {np.median(le):.1f} "
              f"max {le.max():.1f}")
        order = np.argsort(en)[-8:]
        print("  last tiles to finish: " + ", ".join(f"t{int(t)} ({dur[t]:.1f} us, ends {(en[t] - t0) / 1e3:.1f})"
                                                  for t in order))
        np.save(os.path.join(ROOT, "gpurun_out", f"tiles_{workload}.npy"), tb)
    except AttributeError:
        pass
    ex = extra[used]
    if e1[used].max() > 0:
        print(f"  E split: cross-tile links mean {e1[used].mean():.0f} max {e1[used].max():.0f}; "
              f"long runs mean {per[:, 8].mean() - e1[used].mean():.0f} cycles per CTA")
    spread = buf[used, 11:14].astype(np.float64) / reps
    print("  warp arrival spread at phase D's block barriers (last - first, cycles per CTA per build): "
          + ", ".join(f"barrier {k + 1} {spread[:, k].mean():.0f}" for k in range(3)))
    try:
        lw = np.zeros((3, 32), np.uint64)
        ctypes.CDLL(LIB).rtf_debug_last_warp(ctypes.c_void_p(lw.ctypes.data))
        for k in range(3):
            tot_k = max(1, int(lw[k].sum()))
            top = np.argsort(lw[k])[::-1][:4]
            print(f"  barrier {k + 1}: last to arrive " + ", ".join(
                f"warp {int(w)} {100 * int(lw[k][w]) / tot_k:.0f}%" for w in top))
    except AttributeError:
        pass
    print(f"  (issuer waiting for the TMA store to read the stage: mean {ex[:, 0].mean():.0f}; "
          f"thread 0 waiting for the weights' TMA load: mean {ex[:, 1].mean():.0f} cycles per CTA)")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--build", action="store_true")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--workload", default="c3")
    a = ap.parse_args()
    if a.build:
        build()
    else:
        run(a.reps, a.workload)
