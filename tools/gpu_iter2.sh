# build iteration: GPU parity tests (stop on first failure), then phase cycles + build time c3/c2, short bench
TAG=${1:-it}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --tb=short > gpurun_out/pt_$TAG.log 2>&1; rc=$?
tail -4 gpurun_out/pt_$TAG.log
if [ $rc -ne 0 ]; then echo "TESTS FAILED rc=$rc"; grep -m3 -B2 -A12 "Error\|assert" gpurun_out/pt_$TAG.log | head -80; exit 1; fi
timeout 300 python tools/phase_timing.py --reps 20 2>&1
timeout 300 python tools/phase_timing.py --reps 20 --workload c2 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_$TAG.json')); print('build', d['build'], 'sample', d['sampling']['value'], 'bsearch', d['sampling']['bsearch']['value'], 'cutbin', d['sampling']['cutpoint_binary'], 'cutlin', d['sampling']['cutpoint_linear'])"
