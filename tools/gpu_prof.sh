# ncu --set full on the build kernels (one timed step of the bench)
set -x
TAG=${1:-prof}
REGEX=${2:-"k_scale|k_tile_totals|k_scan_build|k_cross_tile"}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$REGEX" -s ${3:-12} -c ${4:-4} -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --samples 67108864 > gpurun_out/prof_$TAG.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/prof_$TAG.log
