# quick GPU check: selected tests (args) + default bench
TAG=${1:-q}; shift
mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu --tb=short "$@" > gpurun_out/pytest_$TAG.log 2>&1; echo pytest rc=$?; tail -15 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc=$?; tail -3 gpurun_out/bench_$TAG.err
python - <<PY
import json
d=json.load(open("gpurun_out/bench_$TAG.json"))
print("build", d["build"], "sample", d["sampling"]["value"], "eyt", d["sampling"].get("bsearch_eytzinger"), "bs", d["sampling"]["bsearch"]["value"], "cb", d["sampling"]["cutpoint_binary"]["value"])
print("c2", d.get("config2_envmap"))
PY
