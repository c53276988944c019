"""Slot-arrival check: a debug build of librtf.so
(-DRTF_SLOT_CHECK) counts every link write of the cooperative build and of
the row kernel; tools/slotcheck_target.py checks that no child field is
written twice (a write-write race) and that every internal node is linked
exactly once (Alg. 1), and that the forest equals the oracle's.
Race detection on pools where compute-sanitizer is unavailable."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_slot_arrival_check():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "slotcheck_target.py")],
                       capture_output=True, text=True, timeout=1800, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "slot check ok" in out, out[-4000:]
