"""Per-source-line instruction counts and stall samples from an ncu report
(`ncu -i R --page source --csv --print-source cuda,sass`).

  python tools/src_hotspots.py gpurun_out/prof_b1.ncu-rep [--top 40] [--ranges a-b,c-d]
"""
import argparse
import csv
import io
import subprocess


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    rows = []
    fname = "?"
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No") or r[0] == "":
            continue
        try:
            line = int(r[0])
            inst = int(r[7]) if r[7] not in ("-", "") else 0
            samp = int(r[6]) if r[6] not in ("-", "") else 0
        except (ValueError, IndexError):
            continue
        rows.append((fname, line, r[1].strip(), inst, samp))
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--ranges", default="")
    a = ap.parse_args()
    rows = load(a.rep)
    ti = sum(r[3] for r in rows) or 1
    ts = sum(r[4] for r in rows) or 1
    print(f"total warp instructions {ti:,}  stall samples {ts:,}")
    for f, ln, src, inst, samp in sorted(rows, key=lambda r: -r[3])[:a.top]:
        print(f"{f:16s}{ln:5d} {100 * inst / ti:5.1f}% inst {100 * samp / ts:5.1f}% samp  {src[:70]}")
    for rg in filter(None, a.ranges.split(",")):
        lo, hi = map(int, rg.split("-"))
        sel = [r for r in rows if r[0].startswith("rtf_build") and lo <= r[1] <= hi]
        print(f"lines {lo}-{hi}: {100 * sum(r[3] for r in sel) / ti:5.1f}% inst "
              f"{100 * sum(r[4] for r in sel) / ts:5.1f}% samples")


if __name__ == "__main__":
    main()
