# build librtf.so of a git revision (default HEAD) into tools/librtf_<name>.so for A/B
REV=${1:-HEAD}; NAME=${2:-head}
D=$(mktemp -d); git archive "$REV" paper_1901_05423_b200 include | tar -x -C "$D"
python - "$D" "$NAME" <<'PY'
import sys, glob, os, subprocess
sys.path.insert(0, os.getcwd())
from paper_1901_05423_b200 import _build_lib as b
d, name = sys.argv[1], sys.argv[2]
srcs = sorted(glob.glob(os.path.join(d, "paper_1901_05423_b200", "csrc", "*.cu")))
subprocess.check_call([b.NVCC, *b.NVCC_FLAGS, "-o", f"tools/librtf_{name}.so", *srcs])
print(f"tools/librtf_{name}.so")
PY
rm -rf "$D"
