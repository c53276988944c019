mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --tb=short > gpurun_out/pytest_s11.log 2>&1; echo tests rc=$?; tail -4 gpurun_out/pytest_s11.log
timeout 600 python bench.py > gpurun_out/bench_s11.json 2> gpurun_out/bench_s11.err; echo bench rc=$?
python -c "
import json;d=json.load(open('gpurun_out/bench_s11.json'));print(d['value'], d['build'], d['ms_per_step'], json.dumps(d['e2e']), d['roofline']['frac'])"
timeout 300 python tools/phase_timing.py --reps 20 > gpurun_out/phase_s11.txt 2>&1; cat gpurun_out/phase_s11.txt
