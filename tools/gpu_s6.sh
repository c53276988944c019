mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -m gpu -x -q --tb=short > gpurun_out/pytest_s6.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/pytest_s6.log
L=paper_1901_05423_b200/librtf.so
timeout 900 python tools/ab_build.py tools/librtf_scalar.so $L tools/librtf_run128.so tools/librtf_scalar.so $L tools/librtf_run128.so 2>&1
timeout 300 python tools/phase_timing.py --reps 20 > gpurun_out/phase_s6.txt 2>&1; cat gpurun_out/phase_s6.txt
