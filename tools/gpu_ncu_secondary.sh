# ncu --set full of the secondary workloads' kernels: k_build_rows (config 5), k_sample_2d (2-D)
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:k_build_rows -s 1 -c 1 \
  -o gpurun_out/${TAG}_rows python tools/rows_once.py > gpurun_out/ncu_rows_$TAG.log 2>&1; echo ncu_rows rc=$?
timeout 600 ncu --set full --clock-control none -k regex:k_sample_2d -s 2 -c 1 \
  -o gpurun_out/${TAG}_2d python bench.py --workload c2d --steps 1 --warmup 3 > gpurun_out/ncu_2d_$TAG.log 2>&1; echo ncu_2d rc=$?
python tools/ncu_summary.py gpurun_out/${TAG}_rows.ncu-rep
python tools/ncu_summary.py gpurun_out/${TAG}_2d.ncu-rep
