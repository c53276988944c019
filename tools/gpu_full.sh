# full round check: all GPU tests, default bench, config-4 bench, launch list
set -x
TAG=${1:-full}
timeout 1200 python -m pytest tests -m gpu -q --tb=short > gpurun_out/pytest_$TAG.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc=$?
tail -3 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
timeout 600 python bench.py --workload c4 --steps 3 --warmup 3 > gpurun_out/bench_c4_$TAG.json 2> gpurun_out/bench_c4_$TAG.err; echo bench_c4 rc=$?
tail -3 gpurun_out/bench_c4_$TAG.err; cat gpurun_out/bench_c4_$TAG.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2>&1; echo ref rc=$?
tail -2 gpurun_out/bench_ref_$TAG.json
