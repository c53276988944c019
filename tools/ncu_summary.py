"""Key metrics per kernel from an ncu report (raw page) + top stall reasons."""
import csv, io, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
want = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'lts__t_sector_hit_rate.pct', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__occupancy_limit_shared_mem',
        'launch__occupancy_limit_registers', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__inst_executed.sum',
        'sm__inst_executed.avg.per_cycle_elapsed', 'lts__t_sectors.sum', 'launch__grid_size',
        'smsp__thread_inst_executed_per_inst_executed.ratio']
stall = [c for c in h if c.startswith('smsp__average_warp_latency_issue_stalled') or c.startswith('smsp__pcsamp_warps_issue_stalled_')]
for r in rows[2:]:
    print('----', r[h.index('Kernel Name')][:70])
    for w in want[1:]:
        if w in h:
            print(f'  {w}: {r[h.index(w)]}')
    st = []
    for c in stall:
        if c.startswith('smsp__pcsamp_warps_issue_stalled_') and not c.endswith('not_issued'):
            try:
                st.append((float(r[h.index(c)].replace(',', '')), c.replace('smsp__pcsamp_warps_issue_stalled_', '')))
            except ValueError:
                pass
    st.sort(reverse=True)
    tot = sum(s for s, _ in st) or 1
    print('  stalls:', ', '.join(f'{n} {100*s/tot:.0f}%' for s, n in st[:7]))
