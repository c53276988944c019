timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --tb=short 2>&1 | tail -2
L=paper_1901_05423_b200/librtf.so
timeout 900 python tools/ab_build.py tools/librtf_head.so $L tools/librtf_head.so $L tools/librtf_head.so $L 2>&1
