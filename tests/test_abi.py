"""CPU checks of the C ABI: librtf.so loads, exports every function include/rtf.h
declares, and the host-only calls / argument validation behave as documented
(no device work is issued by any call here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rtf.h")


@pytest.fixture(scope="module")
def L():
    from paper_1901_05423_b200._build_lib import build_library
    build_library()
    from paper_1901_05423_b200 import _lib
    return _lib.load()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(rtf_[a-z_0-9]+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_paper_calls():
    names = declared_functions()
    for must in ("rtf_build", "rtf_sample", "rtf_build_rows", "rtf_sample_rows",
                 "rtf_forest_bytes", "rtf_workspace_bytes", "rtf_forest_status"):
        assert must in names
    assert len(names) >= 18


def test_every_declared_symbol_is_exported(L):
    from paper_1901_05423_b200 import _lib
    out = subprocess.check_output(["nm", "-D", "--defined-only", _lib.LIB_PATH], text=True)
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    for name in declared_functions():
        assert name in exported, name
        assert hasattr(L, name)
        assert name in _lib.PROTOTYPES, f"binding lacks a prototype for {name}"


def test_library_is_sm100a(L):
    from paper_1901_05423_b200 import _lib
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                                  text=True)
    assert "sm_100a" in out


def test_host_only_sizes(L):
    c0 = L.rtf_launch_count()  # earlier tests in the same process may have launched
    fb = L.rtf_forest_bytes(1 << 24, 1 << 22, 1)
    assert fb >= 16 * (1 << 24) + 4 * (1 << 22) + 40
    assert fb % 256 == 0
    assert L.rtf_forest_bytes(1024, 1024, 65536) >= 65536 * (16 * 1024 + 4 * 1024 + 40)
    # per tile: a prefix (16 B) and a spine row; the run queue; nothing per entry
    # (otherBounds, lives in shared memory per tile)
    wb = L.rtf_workspace_bytes(1 << 24, 1 << 22, 0)
    assert 4096 * (16 + 256) < wb < (1 << 24)
    assert L.rtf_status_string(0) == b"RTF_OK"
    assert b"sm_100a" in L.rtf_version()
    assert L.rtf_quad_bytes(1 << 24) == 32 << 24
    assert L.rtf_launch_count() == c0


def test_argument_validation_before_launch(L):
    from paper_1901_05423_b200 import _lib
    c0 = L.rtf_launch_count()
    v = _lib.rtf_forest()
    EINVAL, ETOOLARGE = _lib.RTF_EINVAL, _lib.RTF_ETOOLARGE
    assert L.rtf_build(None, 10, 4, 0, None, 0, None, 0, None, ctypes.byref(v)) == EINVAL
    assert L.rtf_forest_view(None, 0, 1, 1, 1, ctypes.byref(v)) == EINVAL
    fake = ctypes.c_void_p(1 << 20)  # never dereferenced: checks fail first
    assert L.rtf_forest_view(fake, 1 << 30, 0, 4, 1, ctypes.byref(v)) == EINVAL
    assert L.rtf_forest_view(fake, 1 << 30, 1 << 31, 4, 1, ctypes.byref(v)) == ETOOLARGE
    assert L.rtf_forest_view(fake, 16, 10, 4, 1, ctypes.byref(v)) == _lib.RTF_ENOSPACE
    assert L.rtf_forest_view(ctypes.c_void_p((1 << 20) + 8), 1 << 30, 10, 4, 1,
                             ctypes.byref(v)) == EINVAL  # misaligned
    assert L.rtf_build_rows(fake, 10, 5000, 16, fake, 1 << 40, None, ctypes.byref(v)) == ETOOLARGE
    assert L.rtf_sample(None, None, 0, None, None) == EINVAL
    assert L.rtf_build(fake, 10, 4, 7, fake, 1 << 30, fake, 1 << 30, None,
                       ctypes.byref(v)) == EINVAL  # unknown flag
    assert L.rtf_build_quad(None, fake, 1 << 30, None) == EINVAL
    assert L.rtf_sample_quad(None, fake, None, 0, None, None) == EINVAL
    assert L.rtf_launch_count() == c0


def test_python_binding_fails_loudly_without_library(tmp_path, monkeypatch):
    from paper_1901_05423_b200 import _lib
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(ImportError):
        _lib.load()


def test_product_package_never_imports_the_oracle():
    """The product path shares no code with oracle/ (DESIGN.md section 3)."""
    pkg = os.path.join(ROOT, "paper_1901_05423_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "rtf_oracle" not in src and "liboracle" not in src, f
