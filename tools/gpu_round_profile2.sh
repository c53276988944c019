# round evidence on the GPU box: default bench (+ c2, c4 at N=1, reference arm),
# ncu launch list of the default bench command, ncu --set full of each main kernel
# (one capture per kernel, separate reports: TAG_<kernel>.ncu-rep)
TAG=${1:-r02}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc=$?; tail -2 gpurun_out/bench_$TAG.err
timeout 600 python bench.py --workload c2 --no-e2e > gpurun_out/bench_c2_$TAG.json 2> gpurun_out/bench_c2_$TAG.err; echo bench_c2 rc=$?
timeout 900 python bench.py --workload c4 --steps 3 --warmup 3 > gpurun_out/bench_c4_$TAG.json 2> gpurun_out/bench_c4_$TAG.err; echo bench_c4 rc=$?; tail -2 gpurun_out/bench_c4_$TAG.err
timeout 600 python bench.py --workload c5 --steps 3 --warmup 3 > gpurun_out/bench_c5_$TAG.json 2> gpurun_out/bench_c5_$TAG.err; echo bench_c5 rc=$?
timeout 600 python bench.py --workload c2d --steps 3 --warmup 3 > gpurun_out/bench_c2d_$TAG.json 2> gpurun_out/bench_c2d_$TAG.err; echo bench_c2d rc=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo ref rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1; echo ncu_launch rc=$?
# kernel regex : launches to skip (the bench's first calls warm up / check equality)
for KS in "k_build:3" "k_sample:3" "k_bsearch:1" "k_eytzinger:1" "k_sample_cutpoint:1" "k_fallback_depth:0" "k_sample4:1"; do
  K=${KS%%:*}; S=${KS##*:}; N=$K
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"${K}" -s $S -c 1 \
    -o gpurun_out/${TAG}_${N} python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --samples 268435456 > gpurun_out/ncu_${N}_$TAG.log 2>&1; echo ncu $N rc=$?
done
ls gpurun_out
