# build iteration: parity tests (stop at the first failure), phase cycles, short bench
python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -x -q 2>&1 | tail -15 > gpurun_out/it_tests.txt
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-c2 > gpurun_out/it_bench.json 2> gpurun_out/it_bench.err
python tools/phase_timing.py 2>&1 | tail -12 > gpurun_out/it_phase.txt
python tools/phase_timing.py --workload c2 2>&1 | tail -12 >> gpurun_out/it_phase.txt
cat gpurun_out/it_tests.txt gpurun_out/it_phase.txt
python -c "import json; d=json.load(open('gpurun_out/it_bench.json')); print('BUILD', d['value'], 'G entries/s')"
