bash tools/gpu_round_profile2.sh r02b
timeout 300 python tools/phase_timing.py --reps 20 > gpurun_out/phase_r02b.txt 2>&1
timeout 300 python tools/phase_timing.py --reps 20 --workload c2 >> gpurun_out/phase_r02b.txt 2>&1
timeout 900 python tools/families.py > gpurun_out/families_r02b.jsonl 2> gpurun_out/families_r02b.err; echo families rc=$?
