mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --tb=short -k "host" > gpurun_out/pytest_s5.log 2>&1; echo tests rc=$?; tail -5 gpurun_out/pytest_s5.log
timeout 300 python tools/phase_timing.py --reps 20 > gpurun_out/phase_s5.txt 2>&1; cat gpurun_out/phase_s5.txt
timeout 300 python tools/phase_timing.py --reps 20 --workload c2 >> gpurun_out/phase_s5.txt 2>&1; tail -30 gpurun_out/phase_s5.txt
