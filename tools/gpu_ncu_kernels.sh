# ncu --set full of selected kernels of the default bench command, one report each:
#   bash tools/gpu_ncu_kernels.sh TAG kernel:skip [kernel:skip ...]
TAG=$1; shift
mkdir -p gpurun_out
for KS in "$@"; do
  K=${KS%%:*}; S=${KS##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"${K}" -s $S -c 1 \
    -o gpurun_out/${TAG}_${K} python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --samples 268435456 > gpurun_out/ncu_${K}_$TAG.log 2>&1; echo ncu $K rc=$?
done
