# ncu --set full (+ source) of one k_build launch and one k_sample launch (config 3),
# plus the launch list of the default bench command
TAG=${1:-p}
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_build -s 2 -c 1 \
  -o gpurun_out/prof_build_$TAG python tools/build_once.py > gpurun_out/prof_build_$TAG.log 2>&1; echo ncu_build rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sample -s 3 -c 1 \
  -o gpurun_out/prof_sample_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof_sample_$TAG.log 2>&1; echo ncu_sample rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo ncu_launches rc=$?
