mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_slotcheck.py tests/test_gpu_parity.py tests/test_gpu_sanitize.py -m gpu -x -q --tb=short > gpurun_out/pytest_s4.log 2>&1; echo tests rc=$?; tail -15 gpurun_out/pytest_s4.log
timeout 600 python bench.py > gpurun_out/bench_s4.json 2> gpurun_out/bench_s4.err; echo bench rc=$?
python -c "
import json;d=json.load(open('gpurun_out/bench_s4.json'));print(d['value'], d['build'], json.dumps(d['e2e']))"
