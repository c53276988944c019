mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slotcheck.py -m gpu -x -q --tb=short > gpurun_out/pytest_s8.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/pytest_s8.log
L=paper_1901_05423_b200/librtf.so
timeout 900 python tools/ab_build.py tools/librtf_inorder.so $L tools/librtf_zigzag.so tools/librtf_inorder.so $L tools/librtf_zigzag.so 2>&1
timeout 300 python tools/phase_timing.py --reps 20 > gpurun_out/phase_s8.txt 2>&1; cat gpurun_out/phase_s8.txt
timeout 300 python tools/phase_timing.py --reps 20 --workload c2 > gpurun_out/phase_s8c2.txt 2>&1; grep -v "^    tiles" gpurun_out/phase_s8c2.txt
