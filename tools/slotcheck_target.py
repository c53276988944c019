"""Slot-arrival check of the forest build (tests/test_gpu_slotcheck.py).

Runs builds through tools/librtf_slotcheck.so, a librtf.so compiled with
-DRTF_SLOT_CHECK: every link write of the cooperative build (phase D's staged
links, phase E's cross-tile links) and of the row kernel (Alg. 1's
atomicExch protocol) also counts, per record child field, how often it was
written and, per record, how often it was linked as an internal node.

Checked, per build:
  * no child field is written twice (a write-write race shows here even when
    the two writers happen to store the same bytes);
  * every internal node (a record that is not the first leaf of its cell) is
    linked exactly once and no anchor is linked (Alg. 1: each
    internal node has one parent; a cell root is the right child of its
    anchor, R5);
  * the records and table equal the oracle's (so the counted writes are the
    ones that built the right forest).

This stands in for compute-sanitizer's racecheck on pools where the sanitizer
is unavailable.  Prints "slot check ok" on success.
"""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
LIB = os.path.join(ROOT, "tools", "librtf_slotcheck.so")


def build_variant():
    from paper_1901_05423_b200 import _build_lib as b
    deps = b._deps()
    if os.path.exists(LIB) and all(os.path.getmtime(d) <= os.path.getmtime(LIB) for d in deps):
        return
    tmp = LIB + f".tmp{os.getpid()}"
    subprocess.check_call([b.NVCC, *b.NVCC_FLAGS, "-DRTF_SLOT_CHECK", "-o", tmp, *b.sources()])
    os.replace(tmp, LIB)


def main():
    build_variant()
    import numpy as np
    import torch

    import oracle
    import paper_1901_05423_b200 as rtf
    from paper_1901_05423_b200 import _lib
    from workloads import env_map, power_law, random_small

    _lib.LIB_PATH = LIB
    rtf.lib()
    setbuf = ctypes.CDLL(LIB).rtf_debug_slot_buffers
    setbuf.argtypes = [ctypes.c_void_p, ctypes.c_void_p]

    def counted(run, records):
        fields = torch.zeros(2 * (records + 1), dtype=torch.int32, device="cuda")
        nodes = torch.zeros(records + 1, dtype=torch.int32, device="cuda")
        assert setbuf(fields.data_ptr(), nodes.data_ptr()) == 0
        out = run()
        torch.cuda.synchronize()
        assert setbuf(None, None) == 0
        return out, fields.cpu().numpy(), nodes.cpu().numpy()

    def check(fields, nodes, cell, what):
        k = cell.size
        anchor = np.ones(k, bool)
        anchor[1:] = cell[1:] != cell[:-1]
        assert fields.max(initial=0) <= 1, f"{what}: a child field written {fields.max()} times"
        want = np.where(anchor, 0, 1)
        bad = np.flatnonzero(nodes[:k] != want)
        assert bad.size == 0, f"{what}: {bad.size} records linked wrongly, first {bad[:5]} " \
                              f"counts {nodes[bad[:5]]} anchors {anchor[bad[:5]]}"
        assert nodes[k:].sum() == 0, f"{what}: links beyond the last record"
        return int(fields.sum()), int(nodes.sum())

    rng = np.random.default_rng(11)
    cases = [
        ("power law A, n=2^20, m=2^18", power_law(1 << 20, "A"), 1 << 18),
        ("power law C, n=300000, m=70001", power_law(300000, "C"), 70001),
        ("random with zeros, n=70000, m=9000", random_small(rng, 70000, 0.4), 9000),
        ("env map 512x256, m=n", env_map(512, 256, seed=4), 512 * 256),
        ("m=1 (one tree), n=50000", random_small(rng, 50000, 0.1), 1),
        ("packed cells, n=150000, m=2^17", random_small(rng, 150000, zero_frac=0.05, dyn=3.0), 1 << 17),
        ("row kernel, n=3000, m=1024", power_law(3000, "A"), 1024),
    ]
    for name, p, m in cases:
        ref = oracle.build(p, m)
        pd = torch.from_numpy(np.ascontiguousarray(p, np.float32)).cuda()
        flag_sets = [rtf.RTF_BUILD_DEFAULT] if p.size <= 4096 else [rtf.RTF_BUILD_DEFAULT,
                                                                     rtf.RTF_BUILD_SMALL_TILES]
        for flags in flag_sets:
            f, fields, nodes = counted(lambda: rtf.build(pd, m, flags), p.size)
            rec = f.nodes_numpy()
            assert rec.size == ref.n_pos
            assert np.array_equal(rec["key"], ref.key) and np.array_equal(rec["c0"], ref.child0) \
                and np.array_equal(rec["c1"], ref.child1), f"{name}: forest differs from the oracle"
            nf, nn = check(fields, nodes, ref.cell, f"{name} flags={flags}")
            print(f"{name:40s} flags={flags}: {nn} node links, {nf} field writes, each once")
    # batched rows: Alg. 1's atomicExch protocol in shared memory, every row
    rows, n_row, m_row = 64, 1024, 256
    pr = np.exp(2.0 * rng.standard_normal((rows, n_row))).astype(np.float32)
    pr[::7, ::3] = 0.0
    refr = oracle.build_rows(pr, rows, n_row, m_row)
    prd = torch.from_numpy(pr).cuda()
    rf, fields, nodes = counted(lambda: rtf.build_rows(prd, m_row), rows * n_row)
    rec = rf.nodes_numpy()
    for r in range(rows):
        k = int(refr["n_pos"][r])
        sl = slice(r * n_row, r * n_row + k)
        assert np.array_equal(rec["c0"][sl], refr["child0"][sl]) and \
            np.array_equal(rec["c1"][sl], refr["child1"][sl]), f"row {r} differs from the oracle"
        check(fields[2 * r * n_row: 2 * (r * n_row + k)], nodes[r * n_row: r * n_row + n_row],
              refr["cell"][sl], f"row {r}")
        # Alg. 1 in the row kernel writes every child field but the anchors'
        # child0 exactly once
        cell = refr["cell"][sl]
        anchor = np.ones(k, bool)
        anchor[1:] = cell[1:] != cell[:-1]
        fr = fields[2 * r * n_row: 2 * (r * n_row + k)].reshape(k, 2)
        assert np.all(fr[:, 1] == 1) and np.all(fr[~anchor, 0] == 1), f"row {r}: a field never written"
    print(f"rows {rows} x {n_row}: every child field written exactly once")
    print("slot check ok")


if __name__ == "__main__":
    main()
