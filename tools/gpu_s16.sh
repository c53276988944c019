timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slotcheck.py -m gpu -x -q --tb=short 2>&1 | tail -2
L=paper_1901_05423_b200/librtf.so
timeout 900 python tools/ab_build.py tools/librtf_nocoop.so $L tools/librtf_nocoop.so $L tools/librtf_nocoop.so $L 2>&1
timeout 600 python bench.py --workload c2 --no-e2e > gpurun_out/bench_c2_s16.json 2> gpurun_out/bench_c2_s16.err; echo bench_c2 rc=$?
