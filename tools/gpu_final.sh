# final round evidence at HEAD: smoke, all GPU tests, default bench (+ c2), ncu launch list,
# ncu --set full of k_build and k_sample, phase timing
TAG=${1:-r02c}
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke_$TAG.log
timeout 1800 python -m pytest tests -m gpu -q --tb=short > gpurun_out/pytest_$TAG.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/pytest_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc=$?
timeout 600 python bench.py --workload c2 --no-e2e > gpurun_out/bench_c2_$TAG.json 2> gpurun_out/bench_c2_$TAG.err; echo bench_c2 rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1; echo ncu_launch rc=$?
bash tools/gpu_ncu_kernels.sh $TAG k_build:3 k_sample:3
timeout 300 python tools/phase_timing.py --reps 20 > gpurun_out/phase_$TAG.txt 2>&1
timeout 300 python tools/phase_timing.py --reps 20 --workload c2 >> gpurun_out/phase_$TAG.txt 2>&1; echo phase rc=$?
