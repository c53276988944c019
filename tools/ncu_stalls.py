"""Per-source-line stall-reason breakdown from an ncu report (source page).
  python tools/ncu_stalls.py REPORT [--top N] [--file rtf_build.cu]"""
import argparse
import csv
import io
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--top", type=int, default=25)
ap.add_argument("--file", default="rtf_build.cu")
a = ap.parse_args()
out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
rows, hdr, fname, cur = [], None, "?", None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Name":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    if r[0].isdigit():  # a source line: the SASS rows below it add up into it
        cur = [fname, int(r[0]), r[1].strip(), 0.0, 0.0, {}]
        rows.append(cur)
        continue
    if cur is None or len(r) < 5 or not r[2].startswith("0x"):
        continue
    def num(i):
        try:
            return float(r[i] or 0)
        except ValueError:
            return 0.0
    cur[3] += num(4)
    cur[4] += num(7)
    for i, k in enumerate(hdr):
        if k.startswith("stall_") and "Not Issued" not in k and i < len(r):
            cur[5][k[6:]] = cur[5].get(k[6:], 0.0) + num(i)
tot = sum(x[3] for x in rows) or 1
agg = {}
for x in rows:
    for k, v in x[5].items():
        agg[k] = agg.get(k, 0) + v
print("all lines:", ", ".join(f"{k} {100*v/tot:.1f}%" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
for f, ln, src, samp, inst, st in sorted(rows, key=lambda x: -x[3])[: a.top]:
    top = ", ".join(f"{k} {100*v/max(samp,1):.0f}%" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3] if v)
    print(f"{f:14s}{ln:5d} {100*samp/tot:5.1f}%  [{top}]  {src[:60]}")
