timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slotcheck.py -m gpu -x -q --tb=short 2>&1 | tail -2
L=paper_1901_05423_b200/librtf.so
timeout 900 python tools/ab_build.py tools/librtf_head.so $L tools/librtf_head.so $L tools/librtf_head.so $L 2>&1
timeout 300 python tools/phase_timing.py --reps 20 2>&1 | grep -E "spread|last to|us per build|D[0-9 ]|tail|issuer"
