"""Quadratic error of 2-D sampling vs the number of samples (the methodology of
the paper's Fig. 'convergence': e = sum_i (p_i - c_i / n)^2 over the
pixels, c_i = samples that realised pixel i), for the synthetic 2048 x 1024 env
map through rtf_build_2d / rtf_sample_2d.

Two point sets per n = 2^k:
  * qmc: the n-point Hammersley set (k / n, radical inverse_2(k)) -- xi1 picks
    the row through the marginal, xi2 the column (component by component,
    P:1523-1529).  The inverse mapping is monotone, so the set's stratification
    survives (the paper's argument for inversion over the alias method);
  * mc: Philox4x32-10 pseudo-random pairs.
  * qmc_alias / mc_alias: the same two point sets through the 2-D alias
    baseline (rtf_sample_alias_2d), whose tables give every row and pixel
    exactly the xi counts the inverse mapping gives it (baselines.alias_2d
    over the same fixed-point CDFs): the difference is the mapping alone.
    The paper's figure shows the alias method losing the Hammersley set's
    advantage.

  python tools/convergence.py [--kmin 14] [--kmax 26] [--out profiles/r01_convergence.jsonl]
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def bitrev32(x):
    import torch
    x = x.to(torch.int64)
    r = torch.zeros_like(x)
    for b in range(32):
        r |= ((x >> b) & 1) << (31 - b)
    return r


def main():
    import numpy as np
    import torch

    import paper_1901_05423_b200 as rtf
    from workloads import env_map

    ap = argparse.ArgumentParser()
    ap.add_argument("--kmin", type=int, default=14)
    ap.add_argument("--kmax", type=int, default=26)
    ap.add_argument("--W", type=int, default=2048)
    ap.add_argument("--H", type=int, default=1024)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_convergence.jsonl"))
    a = ap.parse_args()
    W, H = a.W, a.H
    dev = torch.device("cuda", 0)
    img = env_map(W, H)
    p = torch.from_numpy(img.astype(np.float64) / img.astype(np.float64).sum()).to(dev)
    f = rtf.build_2d(torch.from_numpy(img).reshape(H, W).to(dev), W, H)
    assert f.status() == 0
    import baselines
    t = torch.from_numpy(img).reshape(H, W).to(dev)
    K_marg = rtf.build_cdf(torch.from_numpy(f.weights()).to(dev)).cdf.cpu().numpy().view(np.uint64)
    K_rows = [rtf.build_cdf(t[y].contiguous()).cdf.cpu().numpy().view(np.uint64)
              if bool((t[y] > 0).any()) else None for y in range(H)]
    al = rtf.Alias2D(*baselines.alias_2d(K_marg, K_rows), W, H, device=dev)
    rows = []
    for k in range(a.kmin, a.kmax + 1):
        n = 1 << k
        idx = torch.arange(n, dtype=torch.int64, device=dev)
        sets = {
            "qmc": ((idx << (32 - k)).to(torch.int32),
                    bitrev32(idx).to(torch.int32)),
            "mc": (rtf.philox(n, seed=0x5EED, start=0, device=dev),
                   rtf.philox(n, seed=0x5EED, start=n, device=dev)),
        }
        row = {"n": n}
        for name, (x1, x2) in sets.items():
            pix = f.sample(x1.contiguous(), x2.contiguous(), with_pos=False)
            c = torch.bincount(pix.to(torch.int64), minlength=W * H).to(torch.float64)
            row[f"e_{name}"] = float(((p - c / n) ** 2).sum())
            pa = al.sample(x1.contiguous(), x2.contiguous())
            c = torch.bincount(pa.to(torch.int64), minlength=W * H).to(torch.float64)
            row[f"e_{name}_alias"] = float(((p - c / n) ** 2).sum())
        row["e_mc_expected"] = float((p * (1 - p)).sum() / n)
        rows.append(row)
        print(json.dumps(row), flush=True)
    # least-squares slopes of log2 e vs log2 n
    def slope(key):
        xs = [math.log2(r["n"]) for r in rows]
        ys = [math.log2(r[key]) for r in rows]
        mx, my = sum(xs) / len(xs), sum(ys) / len(ys)
        return sum((x - mx) * (y - my) for x, y in zip(xs, ys)) / sum((x - mx) ** 2 for x in xs)
    summary = {"slope_qmc": round(slope("e_qmc"), 3), "slope_mc": round(slope("e_mc"), 3),
               "slope_qmc_alias": round(slope("e_qmc_alias"), 3),
               "slope_mc_alias": round(slope("e_mc_alias"), 3),
               "ratio_mc_over_qmc_at_nmax": round(rows[-1]["e_mc"] / rows[-1]["e_qmc"], 2),
               "ratio_qmc_alias_over_qmc_at_nmax":
                   round(rows[-1]["e_qmc_alias"] / rows[-1]["e_qmc"], 2),
               "image": f"workloads.env_map({W}, {H}), mx = {W}, my = {H}",
               "error": "e = sum_i (p_i - c_i / n)^2, p = image / sum(image) (float64)"}
    print(json.dumps(summary), flush=True)
    with open(a.out, "w") as fo:
        for r in rows:
            fo.write(json.dumps(r) + "\n")
        fo.write(json.dumps(summary) + "\n")


if __name__ == "__main__":
    main()
