# ncu --set full of the main-path kernels: one k_build (config 3) and one k_sample (2^28 config-3 samples)
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_build -s 2 -c 1 \
  -o gpurun_out/${TAG}_build python tools/build_once.py > gpurun_out/ncu_build_$TAG.log 2>&1; echo ncu_build rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_sample$" -s 3 -c 1 \
  -o gpurun_out/${TAG}_sample python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --samples 268435456 > gpurun_out/ncu_sample_$TAG.log 2>&1; echo ncu_sample rc=$?
python tools/ncu_summary.py gpurun_out/${TAG}_build.ncu-rep
python tools/ncu_summary.py gpurun_out/${TAG}_sample.ncu-rep
