timeout 300 python tools/phase_timing.py --reps 20 2>&1 | grep -v "^    tiles"
