"""Build a variant of librtf.so with extra nvcc defines for A/B timing:
  python tools/build_variant.py NAME -DFOO=1 ...   ->  tools/librtf_NAME.so"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1901_05423_b200 import _build_lib as b  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(ROOT, "tools", f"librtf_{name}.so")
subprocess.check_call([b.NVCC, *b.NVCC_FLAGS, *defs, "-o", out, *b.sources()])
print(out)
