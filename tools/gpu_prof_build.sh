# ncu --set full (+ source counters) of one k_build launch of config 3
set -x
TAG=${1:-build}
WL=${2:-c3}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_build -s 2 -c 1 \
  -o gpurun_out/prof_$TAG python tools/build_once.py --workload $WL > gpurun_out/prof_$TAG.log 2>&1
echo ncu rc=$?
tail -3 gpurun_out/prof_$TAG.log
