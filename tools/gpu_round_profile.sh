# round evidence on the GPU box: all GPU tests, default bench (+ c2, c4 at N=1, reference arm),
# ncu launch list of the default bench command, ncu --set full of k_build and k_sample
TAG=${1:-r01}
mkdir -p gpurun_out
python __graft_entry__.py --smoke > gpurun_out/smoke_$TAG.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke_$TAG.log
timeout 1500 python -m pytest tests -m gpu -q --tb=short > gpurun_out/pytest_$TAG.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc=$?; tail -2 gpurun_out/bench_$TAG.err
timeout 600 python bench.py --workload c2 --no-e2e > gpurun_out/bench_c2_$TAG.json 2> gpurun_out/bench_c2_$TAG.err; echo bench_c2 rc=$?
timeout 900 python bench.py --workload c4 --steps 3 --warmup 3 > gpurun_out/bench_c4_$TAG.json 2> gpurun_out/bench_c4_$TAG.err; echo bench_c4 rc=$?; tail -2 gpurun_out/bench_c4_$TAG.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo ref rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1; echo ncu_launch rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_build|k_sample|k_bsearch|k_sample_cutpoint|k_eytzinger|k_fallback" -s 8 -c 5 \
  -o gpurun_out/${TAG}_full python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --samples 268435456 > gpurun_out/ncu_full_$TAG.log 2>&1; echo ncu_full rc=$?
ls gpurun_out
