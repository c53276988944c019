# per-phase cycles of k_build (timing build) + one ncu --set full of k_build on c3
TAG=${1:-ph}
mkdir -p gpurun_out
timeout 300 python tools/phase_timing.py --reps 20 > gpurun_out/phase_$TAG.txt 2>&1
timeout 300 python tools/phase_timing.py --reps 20 --workload c2 >> gpurun_out/phase_$TAG.txt 2>&1
cat gpurun_out/phase_$TAG.txt
bash tools/gpu_prof_build.sh $TAG c3
python tools/ncu_summary.py gpurun_out/prof_$TAG.ncu-rep
