# parity subset, then A/B of HEAD (tools/librtf_head.so) against the working tree's librtf.so, then phase timing
TESTS=${1:-"tests/test_gpu_parity.py"}
timeout 1200 python -m pytest $TESTS -m gpu -x -q --tb=short 2>&1 | tail -2
L=paper_1901_05423_b200/librtf.so
timeout 900 python tools/ab_build.py tools/librtf_head.so $L tools/librtf_head.so $L tools/librtf_head.so $L 2>&1
timeout 300 python tools/phase_timing.py --reps 20 2>&1 | grep -E "us per build|E split|tail|E cross"
