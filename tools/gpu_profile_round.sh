# round profiling: launch list of the bench command + ncu --set full of the top kernels
set -x
R=${1:-r01}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${R}_launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline \
  > gpurun_out/${R}_launches_bench.log 2>&1; echo launches rc=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_build|k_sample|k_bsearch" \
  -s 3 -c 4 -o gpurun_out/${R}_full python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline \
  > gpurun_out/${R}_full.log 2>&1; echo full rc=$?
tail -3 gpurun_out/${R}_full.log
