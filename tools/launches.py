"""Summarise an ncu --csv launch list: per-kernel time of the last occurrence."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]
ki, mi, vi, ui, ii = (h.index(x) for x in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit', 'ID'))
launch = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    launch.setdefault(int(r[ii]), {'name': r[ki]})[r[mi]] = (float(r[vi].replace(',', '')), r[ui])
last = list(launch.items())[-int(sys.argv[2]) if len(sys.argv) > 2 else -14:]
for i, d in last:
    t = d.get('gpu__time_duration.sum', (0, ''))
    rd = d.get('dram__bytes_read.sum', (0, ''))
    wr = d.get('dram__bytes_write.sum', (0, ''))
    print(f"{i:4d} {d['name'][:58]:58s} {t[0]:12.0f} {t[1]:4s} rd {rd[0]:10.2f} {rd[1]:6s} wr {wr[0]:10.2f} {wr[1]}")
