# HEAD check on the GPU box: smoke, all GPU tests, default bench, per-phase cycles
TAG=${1:-chk}
mkdir -p gpurun_out
python __graft_entry__.py --smoke > gpurun_out/smoke_$TAG.log 2>&1; echo smoke rc=$?; tail -3 gpurun_out/smoke_$TAG.log
timeout 1200 python -m pytest tests -m gpu -q --tb=short > gpurun_out/pytest_$TAG.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc=$?
tail -3 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
timeout 300 python tools/phase_timing.py --reps 20 2>&1
timeout 300 python tools/phase_timing.py --reps 20 --workload c2 2>&1
