# ncu --set full of one k_sample launch (config 3) + key metrics
TAG=${1:-s}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sample -s 3 -c 1 \
  -o gpurun_out/prof_sample_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof_sample_$TAG.log 2>&1; echo ncu_sample rc=$?
python tools/ncu_summary.py gpurun_out/prof_sample_$TAG.ncu-rep
