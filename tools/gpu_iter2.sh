# selected parity tests (stop at first failure), then A/B timing of library variants
TAG=${1:-it}; shift
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_2d.py tests/test_gpu_quad.py -m gpu -x -q --tb=short > gpurun_out/pytest_$TAG.log 2>&1; echo tests rc=$?; tail -15 gpurun_out/pytest_$TAG.log
timeout 600 python tools/ab_build.py paper_1901_05423_b200/librtf.so "$@" 2>&1
