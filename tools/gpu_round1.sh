set -x
python __graft_entry__.py --smoke 2>&1 | tail -5
timeout 1200 python -m pytest tests -m gpu -q --tb=short 2>&1 | tail -30
timeout 900 python bench.py > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err; echo bench rc=$?
tail -5 gpurun_out/bench_r01.err
cat gpurun_out/bench_r01.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_ncu.log 2>&1; echo ncu1 rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_scale|k_tile_totals|k_scan_build|k_cross_tile|k_sample|k_bsearch" -s 12 -c 7 -o gpurun_out/prof_r01 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --samples 268435456 > gpurun_out/prof.log 2>&1; echo ncu2 rc=$?
tail -3 gpurun_out/prof.log
