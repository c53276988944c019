mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q --tb=short > gpurun_out/pytest_s3.log 2>&1; echo tests rc=$?; tail -5 gpurun_out/pytest_s3.log
timeout 600 python bench.py > gpurun_out/bench_s3.json 2> gpurun_out/bench_s3.err; echo bench rc=$?
timeout 300 python tools/phase_timing.py --reps 20 > gpurun_out/phase_s3.txt 2>&1; cat gpurun_out/phase_s3.txt
bash tools/gpu_prof_build.sh s3 c3
python tools/src_hotspots.py gpurun_out/prof_s3.ncu-rep > gpurun_out/hot_s3.txt 2>&1; head -80 gpurun_out/hot_s3.txt
