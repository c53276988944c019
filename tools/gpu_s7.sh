mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --tb=short > gpurun_out/pytest_s7.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/pytest_s7.log
L=paper_1901_05423_b200/librtf.so
timeout 900 python tools/ab_build.py tools/librtf_oldatom.so $L tools/librtf_zigzag.so tools/librtf_oldatom.so $L tools/librtf_zigzag.so 2>&1
