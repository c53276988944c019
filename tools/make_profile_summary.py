"""Turn the round's ncu outputs (gpurun_out/) into committed summaries under profiles/:
  profiles/<R>_launches.csv    per-launch device times of the bench command (ncu, cold, serialised)
  profiles/<R>_ncu_full.csv     key metrics per profiled kernel (ncu --set full)
  profiles/ncu_traffic.json     dram bytes per launch (read by bench.py's roofline "traffic")
Usage: python tools/make_profile_summary.py r01"""
import csv, io, json, os, subprocess, sys

R = sys.argv[1] if len(sys.argv) > 1 else "r01"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
os.makedirs(P, exist_ok=True)

# launch list
rows = list(csv.reader(open(os.path.join(G, f"{R}_launches.csv"))))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, vi, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
with open(os.path.join(P, f"{R}_launches.csv"), "w", newline="") as f:
    w = csv.writer(f)
    w.writerow(["launch_id", "kernel", "gpu_time_us"])
    for r in rows[hi + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            w.writerow([r[ii], r[ki][:90], f"{float(r[vi].replace(',', '')) / 1000:.2f}"])

# full captures: the main-path kernels (tools/gpu_ncu_main.sh) and the baselines
# (tools/gpu_round_profile.sh)
rows, h, units = [], None, None
import glob as _glob
_reps = [f"{R}_build.ncu-rep", f"{R}_sample.ncu-rep", f"{R}_full.ncu-rep"] + sorted(
    os.path.basename(x) for x in _glob.glob(os.path.join(G, f"{R}_k_*.ncu-rep")))
for rep in _reps:
    if not os.path.exists(os.path.join(G, rep)):
        continue
    out = subprocess.run(["ncu", "-i", os.path.join(G, rep), "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(out)))
    if h is None:
        h, units = rr[0], rr[1]
        rows = [h, units]
    idx = [rr[0].index(c) if c in rr[0] else None for c in h]
    sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tsc = {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}
    for r in rr[2:]:
        row = []
        for c, i in zip(h, idx):
            v = r[i] if i is not None else ""
            if c.startswith("dram__bytes_") and v:  # per-report units -> bytes
                v = str(int(float(v.replace(",", "")) * sc.get(rr[1][i], 1)))
            if c == "gpu__time_duration.sum" and v:  # per-report units -> us
                v = f"{float(v.replace(',', '')) * tsc.get(rr[1][i], 1):.3f}"
            row.append(v)
        rows.append(row)
for c in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
    units[h.index(c)] = "byte"
units[h.index("gpu__time_duration.sum")] = "us"
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed.avg.per_cycle_elapsed",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "lts__t_sectors.sum"]
cols = [c for c in want if c in h]
tr = {}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
with open(os.path.join(P, f"{R}_ncu_full.csv"), "w", newline="") as f:
    w = csv.writer(f)
    w.writerow(cols)
    w.writerow([units[h.index(c)] for c in cols])
    for r in rows[2:]:
        w.writerow([r[h.index(c)] for c in cols])
        name = r[h.index("Kernel Name")].replace("void ", "").replace("rtf::", "")
        rd = float(r[h.index("dram__bytes_read.sum")].replace(",", "")) * scale.get(units[h.index("dram__bytes_read.sum")], 1)
        wr = float(r[h.index("dram__bytes_write.sum")].replace(",", "")) * scale.get(units[h.index("dram__bytes_write.sum")], 1)
        if name.startswith("k_sample<0, 0") or name.startswith("k_sample<0>"):
            # the profiled launch is 2^28 config-3 samples (tools/gpu_ncu_main.sh)
            tr.setdefault("k_sample_per_sample", round((rd + wr) / 2**28, 3))
            continue
        key = "build" if name.startswith("k_build<512, 8, 0") else \
              "k_bsearch" if name.startswith("k_bsearch") else None
        if key and key not in tr:
            tr[key] = int(rd + wr)
json.dump({"c3_powerlaw": tr, "note": f"dram read+write bytes from ncu --set full ({R}): per launch "
           "for the build (n = 2^24) and k_bsearch (2^28 samples), per sample for k_sample "
           "(measured on a 2^28-sample launch)"},
          open(os.path.join(P, "ncu_traffic.json"), "w"), indent=1)
print(open(os.path.join(P, f"{R}_ncu_full.csv")).read())
print(json.load(open(os.path.join(P, "ncu_traffic.json"))))
