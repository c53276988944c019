# quick iteration on the GPU box: parity tests, a short bench, per-kernel launch times
set -x
TAG=${1:-iter}
timeout 900 python -m pytest tests -m gpu -x -q --tb=short > gpurun_out/pytest_$TAG.log 2>&1; rc=$?
tail -25 gpurun_out/pytest_$TAG.log
if [ $rc -ne 0 ]; then echo "TESTS FAILED rc=$rc"; exit 1; fi
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc=$?
tail -3 gpurun_out/bench_$TAG.err
cat gpurun_out/bench_$TAG.json
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --samples 67108864 > /dev/null 2>&1; echo ncu rc=$?
