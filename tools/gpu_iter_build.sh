# build iteration on the GPU box: parity tests, then per-phase cycles (debug
# library) and the product build time for configs 3 and 2
TAG=${1:-it}
timeout 800 python -m pytest tests -m gpu -x -q --tb=short > gpurun_out/pt_$TAG.log 2>&1; rc=$?
tail -4 gpurun_out/pt_$TAG.log
if [ $rc -ne 0 ]; then echo "TESTS FAILED rc=$rc"; grep -m5 -B5 "Error\|assert" gpurun_out/pt_$TAG.log | head -60; exit 1; fi
python tools/phase_timing.py --reps 20 2>&1
python tools/phase_timing.py --reps 20 --workload c2 2>&1
