#!/usr/bin/env python
"""Benchmark of the radix-tree-forest hot path on B200.

One step = one pass of the whole hot path over one batch of synthetic input:
  build (rtf_build: p resident in HBM -> guide table + forest, 4 kernels) and
  sample (rtf_sample: 2^30 xi resident in HBM -> 2^30 original indices).
Default workload: config 3 (power law p_i ~ ((i+1)/n)^20, n = 2^24, m = 2^22,
2^30 Philox4x32-10 xi per GPU).  L2 is flushed (512 MiB write) between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c3|c2]
  python bench.py --impl reference ...    # the CPU oracle arm

`value` = forest build throughput (G entries/s, whole job); the sampling
throughput, its binary-search baseline, roofline fractions, the CPU oracle
baseline, end-to-end (host buffer) numbers and clocks are extra keys.
Multi-GPU (torchrun): config 3 (default) is weak-scaled WITHOUT redundant
work: one distribution of N x 2^24 entries built by the sharded protocol (the
cross-GPU scan of shard totals, per-shard builds storing into the owner's
buffer over NVLink), each rank sampling its own xi stratum; config 4 is the
strong-scaled sharded build of one n = 2^28 distribution; the env-map and rows
workloads run one independent problem per GPU.  Times are max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "forest build G entries/s; sampling G samples/s (vs binary search) at 1/2/4/8 B200"
L2_FLUSH_BYTES = 512 << 20

WORKLOADS = {
    "c1": dict(name="c1_teaser", n=16, m=8, samples=1024,
               desc="config 1 (teaser, Fig. 1): n=16 weights (2,4,10,24,3,1,1,2,1,1,1,2,3,1,4,4), "
                    "m=8, 1024 Hammersley points (dim 0 = k/1024); latency-bound"),
    "c3": dict(name="c3_powerlaw", n=1 << 24, m=1 << 22, samples=1 << 30,
               desc="config 3: power law p_i ~ ((i+1)/n)^20 (family A), n=2^24, m=2^22, "
                    "2^30 Philox4x32-10 xi per GPU"),
    "c2": dict(name="c2_envmap", n=2048 * 1024, m=2048 * 1024, samples=1 << 26,
               desc="config 2: 2048x1024 synthetic env-map luminance, m=n, 2^26 Sobol xi per GPU"),
    # m = 2^22: the 32 MB table stays L2-resident (m = 2^26 -> a 512 MB table read
    # at random from DRAM: 39.6 G samples/s on one B200)
    "c4": dict(name="c4_spikes", n=1 << 28, m=1 << 22, samples=1 << 32,
               desc="config 4: n=2^28 spiky (4 spikes x 0.24 + uniform 0.04), m=2^22; sharded "
                    "build (cross-GPU scan of shard totals), each rank keeping the cells of its "
                    "xi stratum; 2^32 Philox xi split over the GPUs"),
    "c2d": dict(name="c2_envmap_2d", n=2048 * 1024, m=2048, W=2048, H=1024, my=1024,
                samples=1 << 26,
                desc="2-D (Sec.6 P:1523-1529): the 2048x1024 env map as marginal over rows "
                     "(my=1024 cells) + 1024 row forests (mx=2048 cells); 2^26 Philox (xi1, xi2) "
                     "pairs -> pixel + sub-pixel position"),
    "c5": dict(name="c5_rows", n=65536 * 1024, m=1024, rows=65536, n_row=1024, samples=1 << 26,
               desc="config 5: 65536 independent rows of n=1024 (p = exp(3 N(0,1)), every 16th row "
                    "4 spikes), m_row=1024, one CTA per row; 2^26 (row, Philox xi) samples"),
}


def make_p(wl, rank=0):
    """The workload's weights; rank r > 0 of a multi-GPU run of the env-map or
    rows workloads gets its own independent problem (seed + r): independent
    problems are the unit those workloads shard over (weak scaling)."""
    from workloads import env_map, power_law, spikes
    if wl["name"] == "c3_powerlaw":
        return power_law(wl["n"], "A")
    if wl["name"] == "c4_spikes":
        return spikes(wl["n"])
    if wl["name"] == "c5_rows":
        from workloads import rows_lognormal
        return rows_lognormal(wl["rows"], wl["n_row"], seed=7 + rank)
    return env_map(seed=1 + rank)


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(kernel: str, workload: str):
    """dram bytes per launch of `kernel` from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(path):
        return None
    d = json.load(open(path))
    return d.get(workload, {}).get(kernel)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        # one streaming nvidia-smi (-lms) instead of one process per sample
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            return
        for line in self._proc.stdout:
            row = [x.strip() for x in line.split(",")]
            if len(row) >= 3:  # skip error / blank lines
                self.rows.append(row)
            if self._stop.is_set():
                break

    def __enter__(self):
        self._proc = None
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        time.sleep(0.3)  # the first sample lands before the timed region
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._proc is not None:
            self._proc.terminate()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if len(r) > 3 + k and r[3 + k].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ============================================================================ GPU arm

def init_dist(world, local):
    """Device and process group of this rank.  One process per GPU over NCCL;
    RTF_DIST_BACKEND=gloo with RTF_ONE_DEVICE=1 runs every rank on cuda:0 (the
    single-GPU multi-process test of the N > 1 code path: collectives staged
    through host memory, meaningless timings)."""
    import torch
    import torch.distributed as dist
    one = os.environ.get("RTF_ONE_DEVICE") == "1"
    dev = torch.device("cuda", 0 if one else local)
    torch.cuda.set_device(dev)
    if world > 1:
        backend = os.environ.get("RTF_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    return dev


def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_1901_05423_b200 as rtf
    from workloads import sobol0_xi

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1 and args.workload == "c3":
        return run_gpu_c3_sharded(args)
    dev = init_dist(world, local)

    wl = WORKLOADS[args.workload]
    n, m, S = wl["n"], wl["m"], wl["samples"]
    if args.samples:
        S = args.samples
    p_host = make_p(wl, rank)
    p = torch.from_numpy(p_host).to(dev)
    forest = rtf.Forest(n, m)
    if wl["name"] == "c2_envmap":  # Sobol dim 0, this rank's slice of the sequence
        xi = torch.from_numpy(sobol0_xi(S, start=rank * S).view(np.int32)).to(dev)
    else:  # Philox, this rank's counter range
        xi = rtf.philox(S, seed=0x5EED, start=rank * S, device=dev)
    out = torch.empty(S, dtype=torch.int32, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def step(ev=None):
        if ev:
            ev[0].record(stream)
        forest.build(p)
        if ev:
            ev[1].record(stream)
        forest.sample(xi, out)
        if ev:
            ev[2].record(stream)

    for _ in range(args.warmup):
        step()
        flush.zero_()
    torch.cuda.synchronize()
    assert forest.status() == 0

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    sampler = ClockSampler(dev.index)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = rtf.launch_count()
    with sampler:
        for k in range(args.steps):
            step(evs[k])
            flush.zero_()  # L2 flush between timed steps (not inside the events)
        torch.cuda.synchronize()
    launches = rtf.launch_count() - l0
    if world > 1:
        dist.barrier()
    build_ms = [e[0].elapsed_time(e[1]) for e in evs]
    sample_ms = [e[1].elapsed_time(e[2]) for e in evs]
    tb, ts = sum(build_ms), sum(sample_ms)
    if world > 1:  # max over ranks
        t = torch.tensor([tb, ts], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tb, ts = t.tolist()
    K = args.steps
    build_gs = world * n * K / (tb * 1e-3) / 1e9
    sample_gs = world * S * K / (ts * 1e-3) / 1e9

    # ------------------------------------------------ replication alternative (N > 1)
    # each rank rebuilds its forest (no collective on the
    # data path); for comparison, the cost of replicating rank 0's forest over
    # NVLink instead (ncclBroadcast of the whole forest buffer), max over ranks.
    replication = None
    if world > 1:
        fbuf = forest._buf.forest
        rts = []
        for _ in range(3):
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            dist.broadcast(fbuf, src=0)
            e1.record(stream)
            torch.cuda.synchronize()
            rts.append(e0.elapsed_time(e1))
        t = torch.tensor([statistics.median(rts)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        replication = {"ms_broadcast": round(t.item(), 4), "bytes": int(fbuf.numel()),
                       "ms_rebuild": round(tb / args.steps, 4),
                       "note": "the bench rebuilds per rank; this is the NCCL alternative"}
        forest.build(p)  # every rank's own forest again (the broadcast overwrote it)
        torch.cuda.synchronize()

    # ------------------------------------------------ baseline: binary search on the same CDF
    cdf = rtf.build_cdf(p)
    bs_out = torch.empty_like(out)
    cdf.sample(xi, bs_out)
    torch.cuda.synchronize()
    eq = bool(torch.equal(bs_out, out))
    bs_ms = []
    for _ in range(max(2, min(3, K))):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        cdf.sample(xi, bs_out)
        e1.record(stream)
        torch.cuda.synchronize()
        bs_ms.append(e0.elapsed_time(e1))
    tbs = statistics.median(bs_ms)
    if world > 1:
        t = torch.tensor([tbs], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tbs = t.item()
    bsearch_gs = world * S / (tbs * 1e-3) / 1e9

    # ------------------------------------------------ baselines: cutpoint + binary / + linear
    def time_call(fn, reps):
        ts_ = []
        for _ in range(reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize()
            ts_.append(e0.elapsed_time(e1))
        return statistics.median(ts_)

    cut = cdf.cutpoint(m)
    cb_out = torch.empty_like(out)
    cut.sample(xi, cb_out, binary=True)
    torch.cuda.synchronize()
    cb_eq = bool(torch.equal(cb_out, out))
    t_cb = time_call(lambda: cut.sample(xi, cb_out, binary=True), max(2, min(3, K)))
    S_lin = min(S, 1 << 26)  # bounded: the linear scan is unbounded on skewed cells
    cl_out = torch.empty(S_lin, dtype=torch.int32, device=dev)
    cut.sample(xi[:S_lin], cl_out, binary=False)
    torch.cuda.synchronize()
    cl_eq = bool(torch.equal(cl_out, out[:S_lin]))
    t_cl = time_call(lambda: cut.sample(xi[:S_lin], cl_out, binary=False), 2)
    if world > 1:
        t = torch.tensor([t_cb, t_cl], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_cb, t_cl = t.tolist()
    cutbin_gs = world * S / (t_cb * 1e-3) / 1e9
    cutlin_gs = world * S_lin / (t_cl * 1e-3) / 1e9

    # ------------------------------------------------ baseline: Eytzinger binary search
    # (breadth-first key order, top 13 levels in shared memory per CTA)
    ey = cdf.eytzinger()
    ey_out = torch.empty_like(out)
    ey.sample(xi, ey_out)
    torch.cuda.synchronize()
    ey_eq = bool(torch.equal(ey_out, out))
    t_ey = time_call(lambda: ey.sample(xi, ey_out), max(2, min(3, K)))
    if world > 1:
        t = torch.tensor([t_ey], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_ey = t.item()
    eyt_gs = world * S / (t_ey * 1e-3) / 1e9
    del ey, ey_out

    # ------------------------------------------------ baseline: the alias method (Sec.2.6)
    # host-built table over the same xi grid (baselines/alias.c); every item
    # receives exactly its inverse-CDF xi count (checked here), not the same xi
    import baselines
    K_host = cdf.cdf.cpu().numpy().view(np.uint64)
    prob, alias, ak = baselines.alias_table(K_host)
    kc = (K_host + np.uint64((1 << 31) - 1)) >> np.uint64(31)
    want_cnt = np.diff(np.append(kc, np.uint64(1 << 32)).astype(np.int64))
    s_b = float(1 << (32 - ak))
    got_cnt = (np.bincount(np.arange(prob.size), weights=prob.astype(np.float64), minlength=prob.size)
               + np.bincount(alias, weights=s_b - prob.astype(np.float64), minlength=prob.size))
    alias_exact = bool(np.array_equal(got_cnt[:n].astype(np.int64), want_cnt)
                       and not np.any(got_cnt[n:]))
    al = rtf.Alias(prob, alias, ak, device=dev)
    al_out = torch.empty_like(out)
    al.sample(xi, al_out)
    t_al = time_call(lambda: al.sample(xi, al_out), max(2, min(3, K)))
    if world > 1:
        t = torch.tensor([t_al], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_al = t.item()
    alias_gs = world * S / (t_al * 1e-3) / 1e9
    alias_same = float((al_out == out).float().mean().item())
    del al, al_out, K_host

    # context only: torch.searchsorted on a float32 CDF -- a
    # library binary search, not bit-exact with the fixed-point CDF
    S_ts = min(S, 1 << 28)
    cdf32 = torch.cumsum(p.double(), 0)
    cdf32 = (cdf32 / cdf32[-1]).float()
    xf = (xi[:S_ts].to(torch.int64) & 0xFFFFFFFF).to(torch.float64).mul_(2.0 ** -32).float()
    ts_out = torch.searchsorted(cdf32, xf, right=True)
    t_ts = time_call(lambda: torch.searchsorted(cdf32, xf, right=True, out=ts_out), 2)
    ts_agree = float((ts_out.to(torch.int32) == out[:S_ts]).float().mean().item())
    del cdf32, xf, ts_out
    if world > 1:
        t = torch.tensor([t_ts], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_ts = t.item()
    torch_ss_gs = world * S_ts / (t_ts * 1e-3) / 1e9

    # ------------------------------------------------ load statistics (E[visits], avg_32)
    loads, loads_p = forest.sample_loads(xi[: 1 << 20], plain=True)
    loads, loads_p = loads.double(), loads_p.double()
    e_loads = loads.mean().item()
    avg32 = loads.view(-1, 32).max(dim=1).values.mean().item()
    max_loads = int(loads.max().item())
    e_loads_p = loads_p.mean().item()
    avg32_p = loads_p.view(-1, 32).max(dim=1).values.mean().item()

    # ------------------------------------------------ roofline
    peak, peak_src = peaks()
    n_pos = forest.n_pos()
    # SURVEY.md 8(d)'s algorithmic bytes (a 4-B table reference): per sample
    # 4 (xi) + 4 (out) + 4 (table) + 16 E[v], E[v] = node records visited after
    # the table (e_loads counts the table load too); per build entry 4 (p) +
    # 16 (record) + 4 m / n (table).  The implementation's own 8-B table cell
    # and n' records are reported beside them ("implementation_bytes").
    bytes_sample = 4 + 4 + 4 + 16 * (e_loads - 1.0)
    bytes_sample_impl = 4 + 4 + 8 + 16 * (e_loads - 1.0)
    t_sample_launch = ts / K * 1e-3
    ach_s = S * bytes_sample / t_sample_launch / 1e9
    bytes_build = 4 * n + 16 * n + 4 * m
    bytes_build_impl = 4 * n + 16 * n_pos + 8 * m
    t_build = tb / K * 1e-3
    ach_b = bytes_build / t_build / 1e9

    # ------------------------------------------------ end to end through host buffers
    e2e = None
    if not args.no_e2e:
        import torch as T
        p_pin = T.from_numpy(p_host).pin_memory()
        p_stage = T.empty(n, dtype=T.float32, device=dev)
        f2 = rtf.Forest(n, m)
        rtf.build_host(f2, p_pin, p_stage)
        ts_e = []
        for _ in range(K):
            flush.zero_()
            T.cuda.synchronize()
            t0 = time.perf_counter()
            st = rtf.build_host(f2, p_pin, p_stage)
            ts_e.append(time.perf_counter() - t0)
            assert st == 0
        te = sum(ts_e)
        S_e = min(S, 1 << 28)
        xi_h = T.empty(S_e, dtype=T.int32).pin_memory()
        xi_h.copy_(xi[:S_e].cpu())
        out_h = T.empty(S_e, dtype=T.int32).pin_memory()
        chunk = 1 << 24
        xs = T.empty(2 * chunk, dtype=T.int32, device=dev)
        os_ = T.empty(2 * chunk, dtype=T.int32, device=dev)
        rtf.sample_host(f2, xi_h, out_h, xs, os_)
        ts_s = []
        for _ in range(max(2, min(3, K))):
            t0 = time.perf_counter()
            rtf.sample_host(f2, xi_h, out_h, xs, os_)
            ts_s.append(time.perf_counter() - t0)
        tss = statistics.median(ts_s)
        if world > 1:
            t = T.tensor([te, tss], dtype=T.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            te, tss = t.tolist()
        e2e = {"value": round(world * n * K / te / 1e9, 4), "unit": "G entries/s",
               "h2d_bytes_per_step": 4 * n, "d2h_bytes_per_step": 40,
               "path": "rtf_build_host: pinned host p -> device copy -> build -> header read back",
               "sampling": {"value": round(world * S_e / tss / 1e9, 4), "unit": "G samples/s",
                            "samples": S_e, "h2d_bytes_per_step": 4 * S_e,
                            "d2h_bytes_per_step": 4 * S_e,
                            "path": "rtf_sample_host: pinned host xi -> 3-stream pipeline -> "
                                    "pinned host out"}}

    quad = quad_summary(forest, xi, out, flush)
    fallback = fallback_summary(forest, p, xi, out, flush)
    forest.build(p)  # unmarked again
    xi_gen = None
    if wl["name"] != "c2_envmap":  # the Philox input, timed apart from sampling
        xi2 = torch.empty_like(xi)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rtf.philox(S, seed=0x5EED, start=rank * S, out=xi2)
        e1.record()
        torch.cuda.synchronize()
        xi_gen = {"kernel": "k_philox (Philox4x32-10)", "ms": round(e0.elapsed_time(e1), 4),
                  "identical_to_timed_xi": bool(torch.equal(xi2, xi))}
        del xi2
    result = {
        "metric": METRIC,
        "value": round(build_gs, 4),
        "unit": "G entries/s",
        "n_gpus": world,
        "steps": K,
        "warmup": args.warmup,
        "ms_per_step": round((tb + ts) / K, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u64",
        "data": "synthetic",
        "config": {"workload": wl["desc"], "n": n, "m": m, "samples_per_gpu": S,
                   "n_pos": n_pos,
                   "l2": f"flushed between steps ({L2_FLUSH_BYTES >> 20} MiB write, untimed)",
                   "parallelism": f"independent problems x{world}: GPU r builds and samples "
                                  "its own distribution (seed 1 + r), no collective on the data "
                                  "path",
                   "value_is": "build entries per second: n * n_gpus * steps / sum of build "
                               "times (max over ranks)"},
        "build": {"value": round(build_gs, 4), "unit": "G entries/s",
                  "ms_per_build": round(tb / K, 5)},
        "sampling": {"value": round(sample_gs, 4), "unit": "G samples/s",
                     "ms_per_batch": round(ts / K, 4),
                     "bsearch": {"value": round(bsearch_gs, 4), "unit": "G samples/s",
                                 "ms_per_batch": round(tbs, 4), "identical_indices": eq},
                     "bsearch_eytzinger": {"value": round(eyt_gs, 4), "unit": "G samples/s",
                                           "ms_per_batch": round(t_ey, 4),
                                           "identical_indices": ey_eq,
                                           "what": "binary search in breadth-first key order, "
                                                   "top 13 levels in shared memory"},
                     "alias_method": {"value": round(alias_gs, 4), "unit": "G samples/s",
                                      "ms_per_batch": round(t_al, 4), "buckets": 1 << ak,
                                      "exact_counts": alias_exact,
                                      "same_index_fraction": round(alias_same, 6),
                                      "what": "Walker/Vose alias table over the same 32-bit xi "
                                              "grid (host-built): exact per-item xi counts, "
                                              "but not monotone (Sec.2.6 P:203-239)"},
                     "speedup_vs_bsearch": round(sample_gs / max(bsearch_gs, eyt_gs), 3),
                     "speedup_vs_bsearch_plain": round(sample_gs / bsearch_gs, 3),
                     "cutpoint_binary": {"value": round(cutbin_gs, 4), "unit": "G samples/s",
                                         "ms_per_batch": round(t_cb, 4), "cells": m,
                                         "identical_indices": cb_eq},
                     "cutpoint_linear": {"value": round(cutlin_gs, 4), "unit": "G samples/s",
                                         "ms_per_batch": round(t_cl, 4), "samples": S_lin,
                                         "identical_indices": cl_eq},
                     "torch_searchsorted_f32": {"value": round(torch_ss_gs, 4),
                                                "unit": "G samples/s", "samples": S_ts,
                                                "agreement": round(ts_agree, 6),
                                                "note": "context only: float32 CDF, not "
                                                        "bit-exact"},
                     "quad_records": quad,
                     "fallback": fallback,
                     "xi_generation": xi_gen,
                     "loads_per_sample": {"avg": round(e_loads, 4), "avg32": round(avg32, 4),
                                          "max": max_loads, "of": 1 << 20,
                                          "without_two_interval_flag": {
                                              "avg": round(e_loads_p, 4),
                                              "avg32": round(avg32_p, 4)}}},
        "roofline": {"kernel": "k_sample (Alg. 2)", "bound": "hbm",
                     "achieved": round(ach_s, 2), "peak": peak, "unit": "GB/s",
                     "frac": round(ach_s / peak, 4),
                     "traffic": (round(ncu_traffic("k_sample_per_sample", wl["name"]) * S)
                                 if ncu_traffic("k_sample_per_sample", wl["name"]) else None),
                     "algorithmic_bytes_per_unit": round(bytes_sample, 3),
                     "bytes_definition": "SURVEY.md 8(d): 4 xi + 4 out + 4 table + 16 E[v]",
                     "implementation_bytes_per_unit": round(bytes_sample_impl, 3),
                     "unit_of_work": "sample", "peak_source": peak_src,
                     "limiter": "not HBM: scattered 8/16-B loads, one L1TEX->L2 request each; "
                                "ncu l1tex__m_l1tex2xbar_req_cycles_active = 81% of peak "
                                "(profiles/r01_summary.md, DESIGN.md 5.3)"},
        "roofline_build": {"kernel": "k_build (one cooperative kernel: scale, tile totals, "
                                     "spine scan, tiles + in-tile forest, cross-tile links)",
                           "bound": "hbm",
                           "achieved": round(ach_b, 2), "peak": peak, "unit": "GB/s",
                           "frac": round(ach_b / peak, 4),
                           "traffic": ncu_traffic("build", wl["name"]),
                           "algorithmic_bytes_per_launch": bytes_build,
                           "bytes_definition": "SURVEY.md 8(d): 4 p + 16 record + 4 m/n table "
                                               "per entry",
                           "implementation_bytes_per_launch": bytes_build_impl,
                           "limiter": "issue and block barriers: ~231 thread-instructions per "
                                      "entry, issue active 53 %, 32 warps/SM, barrier the largest "
                                      "stall; DRAM far below peak (profiles/r02c_summary.md, "
                                      "DESIGN.md 5.2)",
                           "peak_source": peak_src},
        "gpu_launches": launches,
        "clocks": sampler.summary(),
    }
    if e2e:
        result["e2e"] = e2e
    if replication:
        result["replication"] = replication
    if wl["name"] == "c3_powerlaw" and not args.no_c2:
        result["config2_envmap"] = c2_summary(args, dev, stream, flush, world)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:  # the oracle baseline: N = 1 only
        result["cpu_baseline"] = cpu_baseline(p_host, m, xi[: 1 << 22].cpu().numpy().view(np.uint32),
                                              cdf.cdf.cpu().numpy().view(np.uint64))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(result), flush=True)


def quad_summary(forest, xi, out, flush, reps=3):
    """The 4-ary collapsed records (rtf_build_quad / rtf_sample_quad)
    on the same forest and xi: device time of the collapse and of one batch (L2
    flushed before each launch, median of reps), and index equality with the
    binary descent's out."""
    import torch
    out4 = torch.empty_like(out)

    def timed(fn):
        ts = []
        for _ in range(reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts)

    t_q = timed(lambda: forest.build_quad())
    t_s = timed(lambda: forest.sample_quad(xi, out4))
    same = bool(torch.equal(out, out4))
    del out4
    return {"value": round(xi.numel() / (t_s * 1e-3) / 1e9, 4), "unit": "G samples/s",
            "ms_per_batch": round(t_s, 4), "build_quad_ms": round(t_q, 4),
            "identical_indices": same,
            "what": "4-ary collapsed 32-B records: one load per two levels (P:1537-1539)"}


def fallback_summary(forest, p, xi, out, flush, reps=3):
    """The degenerate-cell fallback (reading R21; rtf_build_fallback): device
    time of the marking pass and of one batch through the marked table (L2
    flushed before each launch, median of reps), index equality with out, and
    the worst case over EVERY 32-bit xi (the per-cell depths the pass
    measures): node reads + 1 table read with the radix trees alone and with
    the marked cells bisected.  The forest is rebuilt afterwards by the caller
    if it is sampled again unmarked."""
    import numpy as np
    import torch
    out_f = torch.empty_like(out)

    def timed(fn, reps=reps):
        ts = []
        for _ in range(reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts)

    def fb_once():
        forest.build(p)  # untimed: an unmarked table for every measured pass
        torch.cuda.synchronize()
        return timed(lambda: forest.build_fallback(), reps=1)

    t_f = statistics.median(fb_once() for _ in range(reps))
    depth, last = forest.cell_depths()  # of the last pass, on an unmarked table
    tab = forest.table_numpy()
    marked = (tab["ref"] >= 0) & (tab["key32"] >> 30 == 3)
    k = (tab["key32"].astype(np.int64) & 0x3FFFFFFF)
    bis = np.where(marked, np.ceil(np.log2(k + 1)).astype(np.int64), 0)
    worst_radix = int(depth.max()) + 1
    worst_fb = int(np.where(marked, bis, depth).max()) + 1
    t_s = timed(lambda: forest.sample(xi, out_f))
    same = bool(torch.equal(out, out_f))
    loads = forest.sample_loads(xi[: 1 << 20]).double()
    del out_f
    return {"value": round(xi.numel() / (t_s * 1e-3) / 1e9, 4), "unit": "G samples/s",
            "ms_per_batch": round(t_s, 4), "build_fallback_ms": round(t_f, 4),
            "cells_marked": int(marked.sum()), "identical_indices": same,
            "worst_case_loads_all_xi": {"radix": worst_radix, "with_fallback": worst_fb},
            "loads_per_sample": {"avg": round(loads.mean().item(), 4),
                                 "max": int(loads.max().item()), "of": 1 << 20},
            "what": "cells deeper than bisection + 4 reads searched by bisection "
                    "(P:983-984, P:1516-1518, P:1545-1548)"}


def c2_summary(args, dev, stream, flush, world):
    """BASELINE configs[1] in the same run: the 2048x1024 env map (n = m = 2^21),
    build + 2^26 Sobol samples, binary search on the same CDF.  Device-timed
    like the headline (CUDA events, L2 flushed between steps), max over ranks."""
    import torch
    import torch.distributed as dist

    import paper_1901_05423_b200 as rtf
    from workloads import sobol0_xi
    wl = WORKLOADS["c2"]
    n, m, S = wl["n"], wl["m"], wl["samples"]
    rank = int(os.environ.get("RANK", "0"))
    p = torch.from_numpy(make_p(wl)).to(dev)
    f = rtf.Forest(n, m, device=dev)
    xi = torch.from_numpy(sobol0_xi(S, start=rank * S).view(np.int32)).to(dev)
    out = torch.empty(S, dtype=torch.int32, device=dev)
    cdf = rtf.build_cdf(p)
    bs = torch.empty_like(out)

    def timed(fn, reps):
        ts_ = []
        for _ in range(reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize()
            ts_.append(e0.elapsed_time(e1))
        return statistics.median(ts_)

    for _ in range(3):
        f.build(p)
        f.sample(xi, out)
    cdf.sample(xi, bs)
    torch.cuda.synchronize()
    assert f.status() == 0
    tb = timed(lambda: f.build(p), max(args.steps, 5))
    ts = timed(lambda: f.sample(xi, out), max(args.steps, 5))
    tbs = timed(lambda: cdf.sample(xi, bs), 3)
    eq = bool(torch.equal(out, bs))
    ey = cdf.eytzinger()
    ey.sample(xi, bs)
    torch.cuda.synchronize()
    ey_eq = bool(torch.equal(out, bs))
    tey = timed(lambda: ey.sample(xi, bs), 3)
    del ey
    if world > 1:
        t = torch.tensor([tb, ts, tbs, tey], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tb, ts, tbs, tey = t.tolist()
    peak, _ = peaks()
    loads = f.sample_loads(xi[: 1 << 20]).double().mean().item()
    bytes_b = 4 * n + 16 * n + 4 * m
    bytes_s = 4 + 4 + 4 + 16 * (loads - 1.0)
    quad = quad_summary(f, xi, out, flush)
    return {"workload": wl["desc"],
            "build": {"value": round(world * n / (tb * 1e-3) / 1e9, 4), "unit": "G entries/s",
                      "ms_per_build": round(tb, 5),
                      "roofline_frac": round(bytes_b / (tb * 1e-3) / 1e9 / peak, 4)},
            "sampling": {"value": round(world * S / (ts * 1e-3) / 1e9, 4), "unit": "G samples/s",
                         "ms_per_batch": round(ts, 4),
                         "roofline_frac": round(S * bytes_s / (ts * 1e-3) / 1e9 / peak, 4),
                         "quad_records": quad},
            "bsearch": {"value": round(world * S / (tbs * 1e-3) / 1e9, 4), "unit": "G samples/s",
                        "identical_indices": eq},
            "bsearch_eytzinger": {"value": round(world * S / (tey * 1e-3) / 1e9, 4),
                                  "unit": "G samples/s", "identical_indices": ey_eq},
            "timing": "median of >= 5 device-timed runs, L2 flushed before each"}


def run_gpu_c3_sharded(args):
    """Config 3 at N > 1 GPUs, weak scaling without redundant work: ONE
    power-law distribution (family A) of n = N 2^24 entries and m = N 2^22
    cells, 2^24 entries per GPU.  The build is the sharded protocol
    (north star: "a cross-GPU scan of per-shard totals plus a per-shard build
    over contiguous cell ranges"; paper_1901_05423_b200.sharded, fused: the
    build kernel stores each record and table cell straight into the buffer
    of the rank owning its cell, over NVLink symmetric memory); rank r keeps
    the cells [r m/N, (r+1) m/N) and samples 2^30 xi of that stratum.  Every
    collective runs inside the timed build (CUDA events, max over ranks)."""
    import torch
    import torch.distributed as dist

    import paper_1901_05423_b200 as rtf
    from paper_1901_05423_b200 import sharded

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = init_dist(world, local)
    wl = WORKLOADS["c3"]
    n_local, S = wl["n"], (args.samples or wl["samples"])
    n, m = world * n_local, world * wl["m"]
    base = rank * n_local
    # this rank's shard of ((i+1)/n)^20 (family A over the whole n; the scale is
    # irrelevant: quantisation normalises by the largest weight)
    i = np.arange(base, base + n_local, dtype=np.float64)
    p_local = torch.from_numpy(np.exp(20.0 * np.log((i + 1.0) / n)).astype(np.float32)).to(dev)
    del i
    comm = sharded.DistComm()
    # the fused protocol needs CUDA symmetric memory (NVLink peer mappings); if
    # the runtime cannot provide it, the ranged protocol with NCCL send/recv
    # (another GPU path, same result bytes) is timed instead and named in config
    fused, fused_note = True, None
    try:
        shards = sharded.make_shards_local(p_local, n, m, rank, world, base, alloc=comm.alloc)
        sharded.build_sharded(shards, comm, ranged=True, fused=True)
        torch.cuda.synchronize()
    except Exception as e:  # noqa: BLE001 -- uniform across ranks (the same runtime)
        fused, fused_note = False, f"symmetric memory unavailable ({type(e).__name__}): NCCL send/recv"
        shards = sharded.make_shards_local(p_local, n, m, rank, world, base)
    forest = rtf.Forest.from_buffer(n, m, shards[0].forest)
    xi = sharded.ranged_xi(rtf.philox(S, seed=0x5EED, start=rank * S, device=dev), rank, world, m)
    out = torch.empty(S, dtype=torch.int32, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def step(ev=None):
        if ev:
            ev[0].record(stream)
        sharded.build_sharded(shards, comm, ranged=True, fused=fused)
        if ev:
            ev[1].record(stream)
        forest.sample(xi, out)
        if ev:
            ev[2].record(stream)

    for _ in range(args.warmup):
        step()
        flush.zero_()
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    sampler = ClockSampler(dev.index)
    dist.barrier()
    torch.cuda.synchronize()
    l0 = rtf.launch_count()
    with sampler:
        for k in range(args.steps):
            step(evs[k])
            flush.zero_()
        torch.cuda.synchronize()
    launches = rtf.launch_count() - l0
    dist.barrier()
    tb = sum(e[0].elapsed_time(e[1]) for e in evs)
    ts = sum(e[1].elapsed_time(e[2]) for e in evs)
    t = torch.tensor([tb, ts], dtype=torch.float64, device=dev)
    comm.allreduce_max([t])
    tb, ts = t.tolist()
    # the slots this rank holds and a sampled check of its indices (untimed)
    j0, j1 = sharded.slots_of(shards[0])
    g0, g1 = shards[0].cells
    cnt = torch.tensor([j1 - j0], dtype=torch.int64, device=dev)
    comm.allreduce_sum([cnt])
    K = args.steps
    build_gs = n * K / (tb * 1e-3) / 1e9
    sample_gs = S * world * K / (ts * 1e-3) / 1e9
    peak, peak_src = peaks()
    bytes_rank = 4 * n_local + 16 * n_local + 4 * (m // world)  # SURVEY.md 8(d), per GPU
    result = {
        "metric": METRIC, "value": round(build_gs, 4), "unit": "G entries/s", "n_gpus": world,
        "steps": K, "warmup": args.warmup, "ms_per_step": round((tb + ts) / K, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic",
        "config": {"workload": f"config 3 weak-scaled: one power law ((i+1)/n)^20 over "
                               f"n = {world} x 2^24 entries, m = {world} x 2^22, 2^30 Philox xi "
                               "per GPU (each GPU samples its stratum)",
                   "n": n, "m": m, "n_per_gpu": n_local, "samples_per_gpu": S,
                   "n_pos": int(cnt.item()),
                   "l2": f"flushed between steps ({L2_FLUSH_BYTES >> 20} MiB write, untimed)",
                   "parallelism": f"sharded build over {world} GPUs: MAX all-reduce of the "
                                  "scale word, all-gather of shard totals (the cross-GPU scan), "
                                  "per-shard build storing records / table cells into the owning "
                                  "rank's buffer (symmetric memory over NVLink), MAX all-reduce "
                                  "of the slot boundaries, all-gather of tile spine rows, "
                                  "per-rank finish; rank r keeps cells [r m/N, (r+1) m/N)",
                   "protocol": "fused (peer stores)" if fused else fused_note,
                   "value_is": "entries of the one distribution per second (n K / max over "
                               "ranks of the summed build times)"},
        "build": {"value": round(build_gs, 4), "unit": "G entries/s",
                  "ms_per_build": round(tb / K, 5)},
        "sampling": {"value": round(sample_gs, 4), "unit": "G samples/s",
                     "ms_per_batch": round(ts / K, 4)},
        "roofline": {"kernel": "sharded build, per GPU (all calls incl. exchanges)",
                     "bound": "hbm",
                     "achieved": round(bytes_rank / (tb / K * 1e-3) / 1e9, 2), "peak": peak,
                     "unit": "GB/s", "frac": round(bytes_rank / (tb / K * 1e-3) / 1e9 / peak, 4),
                     "traffic": None, "peak_source": peak_src},
        "gpu_launches": launches, "clocks": sampler.summary(),
    }
    if not args.no_e2e:  # end to end: each rank's p shard from pinned host memory, the
        # sharded build, the status word read back; wall clock, max over ranks
        p_pin = p_local.cpu().pin_memory()
        te = []
        for _ in range(K):
            flush.zero_()
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            p_local.copy_(p_pin, non_blocking=True)
            sharded.build_sharded(shards, comm, ranged=True, fused=True)
            st = forest.status()
            te.append(time.perf_counter() - t0)
            assert st == 0
        t = torch.tensor([sum(te)], dtype=torch.float64, device=dev)
        comm.allreduce_max([t])
        result["e2e"] = {"value": round(n * K / t.item() / 1e9, 4), "unit": "G entries/s",
                         "h2d_bytes_per_step": 4 * n_local, "d2h_bytes_per_step": 40,
                         "path": "per rank: pinned host p shard -> device, sharded build "
                                 "(all collectives), header status read back"}
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(result), flush=True)


def run_gpu_c4(args):
    """Config 4: strong scaling of one n = 2^28 distribution over N GPUs.  Each
    rank holds its shard of p; the build is the sharded protocol of
    paper_1901_05423_b200.sharded (NCCL through DistComm); every rank then
    samples 2^32 / N xi from its replicated forest."""
    import torch
    import torch.distributed as dist

    import paper_1901_05423_b200 as rtf
    from paper_1901_05423_b200 import sharded

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = init_dist(world, local)
    wl = WORKLOADS["c4"]
    n, m = wl["n"], wl["m"]
    S = (args.samples or wl["samples"]) // world
    base, n_local = sharded.shard_range(n, world, rank)
    # this rank's shard of spikes(n): uniform background + the spikes it holds
    bg = (1.0 - 4 * 0.24) / (n - 4)
    p_local = torch.full((n_local,), bg, dtype=torch.float32, device=dev)
    for k in range(4):
        pos = (2 * k + 1) * n // 8
        if base <= pos < base + n_local:
            p_local[pos - base] = 0.24
    comm = sharded.DistComm() if world > 1 else sharded.LocalComm()
    fused = not args.c4_replicate and not args.c4_nccl and world > 1
    shards = sharded.make_shards_local(p_local, n, m, rank, world, base,
                                       alloc=comm.alloc if fused else None)
    forest = rtf.Forest.from_buffer(n, m, shards[0].forest)
    ranged = not args.c4_replicate
    xi = rtf.philox(S, seed=0x5EED, start=rank * S, device=dev)
    if ranged:  # this rank samples its own xi range (its cell slice), stratified
        xi = sharded.ranged_xi(xi, rank, world, m)
    out = torch.empty(S, dtype=torch.int32, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def step(ev=None):
        if ev:
            ev[0].record(stream)
        sharded.build_sharded(shards, comm, ranged=ranged, fused=fused)
        if ev:
            ev[1].record(stream)
        forest.sample(xi, out)
        if ev:
            ev[2].record(stream)

    for _ in range(args.warmup):
        step()
        flush.zero_()
    torch.cuda.synchronize()
    assert forest.status() == 0
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    sampler = ClockSampler(dev.index)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = rtf.launch_count()
    with sampler:
        for k in range(args.steps):
            step(evs[k])
            flush.zero_()
        torch.cuda.synchronize()
    launches = rtf.launch_count() - l0
    tb = sum(e[0].elapsed_time(e[1]) for e in evs)
    ts = sum(e[1].elapsed_time(e[2]) for e in evs)
    if world > 1:
        t = torch.tensor([tb, ts], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tb, ts = t.tolist()
    K = args.steps
    build_gs = n * K / (tb * 1e-3) / 1e9
    sample_gs = S * world * K / (ts * 1e-3) / 1e9
    peak, peak_src = peaks()
    bytes_build = 4 * n + 16 * n + 4 * m
    quad = quad_summary(forest, xi, out, flush) if world == 1 else None
    m26 = c4_m26_summary(p_local, n, flush) if world == 1 and not args.no_m26 else None
    result = {
        "metric": METRIC, "value": round(build_gs, 4), "unit": "G entries/s", "n_gpus": world,
        "steps": K, "warmup": args.warmup, "ms_per_step": round((tb + ts) / K, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic",
        "config": {"workload": wl["desc"], "n": n, "m": m, "samples_total": S * world,
                   "l2": f"flushed between steps ({L2_FLUSH_BYTES >> 20} MiB write, untimed)",
                   "parallelism": (f"sharded build over {world} GPU(s); ranged: rank r keeps "
                                   "the cells [r m/N, (r+1) m/N) and samples that xi stratum; "
                                   + ("records and table cells stored by the build kernel "
                                      "straight into their owner's buffer (symmetric memory)"
                                      if fused else "records by grouped send/recv, table "
                                      "reduce-scatter")
                                   if ranged else
                                   f"sharded build over {world} GPU(s) + replicated forest; "
                                   "sampling split across GPUs")},
        "sampling": {"value": round(sample_gs, 4), "unit": "G samples/s",
                     "ms_per_batch": round(ts / K, 4),
                     "quad_records": quad if quad else "single-GPU forest only"},
        "m_2_26": m26 if m26 else "single GPU only (or --no-m26)",
        "roofline_build": {"kernel": "sharded build (all calls, incl. exchanges)",
                           "bound": "hbm", "achieved": round(bytes_build / (tb / K * 1e-3) / 1e9, 2),
                           "peak": peak, "unit": "GB/s",
                           "frac": round(bytes_build / (tb / K * 1e-3) / 1e9 / peak, 4),
                           "traffic": None, "peak_source": peak_src},
        "gpu_launches": launches, "clocks": sampler.summary(),
    }
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(result), flush=True)


def c4_m26_summary(p, n, flush, S=1 << 30, reps=3):
    """Config 4's distribution with the table size SURVEY.md proposes, m =
    2^26 (a 512 MB table that no longer stays in L2), built once by rtf_build
    on one GPU: build time, 2^30 Philox samples through the binary records,
    the 4-ary records and the fallback-marked table (each median of reps, L2
    flushed before every launch), identical indices."""
    import torch

    import paper_1901_05423_b200 as rtf
    m = 1 << 26

    def timed(fn):
        ts = []
        for _ in range(reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts)

    f = rtf.Forest(n, m, device=p.device)
    tb = timed(lambda: f.build(p))
    xi = rtf.philox(S, seed=0x5EED, device=p.device)
    out = torch.empty_like(xi)
    ts = timed(lambda: f.sample(xi, out))
    quad = quad_summary(f, xi, out, flush, reps)
    fb = fallback_summary(f, p, xi, out, flush, reps)
    del f, xi, out
    torch.cuda.empty_cache()
    return {"m": m, "build": {"ms": round(tb, 4), "value": round(n / (tb * 1e-3) / 1e9, 4),
                              "unit": "G entries/s"},
            "sampling": {"value": round(S / (ts * 1e-3) / 1e9, 4), "unit": "G samples/s",
                         "ms_per_batch": round(ts, 4), "samples": S},
            "quad_records": quad, "fallback": fb,
            "note": "one forest (rtf_build), not the sharded protocol; 512 MB table"}


def run_gpu_2d(args):
    """2-D sampling: build = rtf_build_2d (rows, row weights,
    marginal), sample = rtf_sample_2d with positions.  Replicas for N > 1."""
    import torch
    import torch.distributed as dist

    import paper_1901_05423_b200 as rtf
    from workloads import env_map

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = init_dist(world, local)
    wl = WORKLOADS["c2d"]
    W, H, mx, my = wl["W"], wl["H"], wl["m"], wl["my"]
    S = args.samples or wl["samples"]
    p = torch.from_numpy(env_map(W, H, seed=1 + rank)).to(dev)
    f = rtf.Forest2D(W, H, mx, my, device=dev)
    xi1 = rtf.philox(S, seed=0x5EED, start=2 * rank * S, device=dev)
    xi2 = rtf.philox(S, seed=0x5EED, start=(2 * rank + 1) * S, device=dev)
    pix = torch.empty(S, dtype=torch.int32, device=dev)
    pos = torch.empty((S, 2), dtype=torch.float32, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def step(ev=None):
        if ev:
            ev[0].record(stream)
        f.build(p)
        if ev:
            ev[1].record(stream)
        f.sample(xi1, xi2, pix, pos)
        if ev:
            ev[2].record(stream)

    for _ in range(args.warmup):
        step()
        flush.zero_()
    torch.cuda.synchronize()
    assert f.status() == 0
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    sampler = ClockSampler(dev.index)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = rtf.launch_count()
    with sampler:
        for k in range(args.steps):
            step(evs[k])
            flush.zero_()
        torch.cuda.synchronize()
    launches = rtf.launch_count() - l0
    tb = sum(e[0].elapsed_time(e[1]) for e in evs)
    ts = sum(e[1].elapsed_time(e[2]) for e in evs)
    if world > 1:
        t = torch.tensor([tb, ts], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tb, ts = t.tolist()
    K = args.steps
    build_gs = world * W * H * K / (tb * 1e-3) / 1e9
    sample_gs = world * S * K / (ts * 1e-3) / 1e9
    result = {
        "metric": METRIC, "value": round(build_gs, 4), "unit": "G entries/s", "n_gpus": world,
        "steps": K, "warmup": args.warmup, "ms_per_step": round((tb + ts) / K, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic",
        "config": {"workload": wl["desc"], "W": W, "H": H, "mx": mx, "my": my,
                   "samples_per_gpu": S,
                   "l2": f"flushed between steps ({L2_FLUSH_BYTES >> 20} MiB write, untimed)",
                   "parallelism": f"independent problems x{world}: GPU r its own env map "
                                  "(seed 1 + r)"},
        "build": {"value": round(build_gs, 4), "unit": "G entries/s", "ms_per_build": round(tb / K, 5),
                  "launches": "rows build + row weights + marginal build"},
        "sampling": {"value": round(sample_gs, 4), "unit": "G 2-D samples/s",
                     "ms_per_batch": round(ts / K, 4),
                     "output": "pixel (int32) + sub-pixel position (2 x float32) per sample"},
        "gpu_launches": launches, "clocks": sampler.summary(),
    }
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(result), flush=True)


def run_gpu_c1(args):
    """Config 1: the teaser distribution (16 weights, 8 cells, 1024 Hammersley
    points).  Latency-bound: reports microseconds per build + sample step,
    launched eagerly and as one replayed CUDA graph."""
    import torch

    import paper_1901_05423_b200 as rtf
    from workloads import TEASER_WEIGHTS, hammersley_xi

    local = int(os.environ.get("LOCAL_RANK", "0"))
    if int(os.environ.get("RANK", "0")) != 0:
        return  # one GPU's latency: the other ranks have nothing to add
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    wl = WORKLOADS["c1"]
    p = torch.tensor(TEASER_WEIGHTS, dtype=torch.float32, device=dev)
    xi_host, _ = hammersley_xi(wl["samples"])
    xi = torch.from_numpy(np.ascontiguousarray(xi_host, dtype=np.uint32).view(np.int32)).to(dev)
    forest = rtf.Forest(wl["n"], wl["m"], device=dev)
    out = torch.empty(wl["samples"], dtype=torch.int32, device=dev)
    stream = torch.cuda.Stream(device=dev)
    K = max(args.steps, 100)

    def step():
        forest.build(p, stream=stream)
        forest.sample(xi, out, stream=stream)

    def timed(fn):
        with torch.cuda.stream(stream):
            for _ in range(args.warmup):
                fn()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            stream.synchronize()
            a.record(stream)
            for _ in range(K):
                fn()
            b.record(stream)
            b.synchronize()
        return a.elapsed_time(b) * 1e3 / K

    sampler = ClockSampler(dev.index)
    with sampler:
        l0 = rtf.launch_count()
        eager_us = timed(step)
        launches = (rtf.launch_count() - l0) // (K + args.warmup)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            step()
            stream.synchronize()
            with torch.cuda.graph(g, stream=stream):
                step()
        graph_us = timed(g.replay)
    torch.cuda.synchronize()
    ok = np.array_equal(out.cpu().numpy(), np.searchsorted(
        np.cumsum(np.array(TEASER_WEIGHTS, dtype=np.int64)) * (1 << 26), xi_host.astype(np.int64),
        side="right"))
    result = {
        "metric": "config 1 latency: build + 1024 samples", "value": round(graph_us, 3),
        "unit": "us per step (CUDA graph)", "n_gpus": 1, "steps": K, "warmup": args.warmup,
        "ms_per_step": round(graph_us / 1e3, 6), "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": wl["desc"], "n": wl["n"], "m": wl["m"], "samples": wl["samples"],
                   "l2": "not flushed (a 200-byte problem; latency is the quantity)"},
        "eager_us_per_step": round(eager_us, 3), "graph_us_per_step": round(graph_us, 3),
        "launches_per_step": launches, "indices_match_inverse_cdf": bool(ok),
        "gpu_launches": launches * K, "clocks": sampler.summary(),
    }
    print(json.dumps(result), flush=True)


def run_gpu_c5(args):
    """Config 5: batched rebuilds of 65536 independent rows (rtf_build_rows, one CTA
    per row, everything in shared memory) + sampling (row, xi) pairs.  Rows are
    independent, so N GPUs each take their own 65536 rows (weak scaling)."""
    import torch
    import torch.distributed as dist

    import paper_1901_05423_b200 as rtf

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = init_dist(world, local)
    wl = WORKLOADS["c5"]
    rows, n_row, m_row = wl["rows"], wl["n_row"], wl["m"]
    S = args.samples or wl["samples"]
    p_host = make_p(wl, rank)
    p = torch.from_numpy(p_host).to(dev)
    forest = rtf.RowsForest(rows, n_row, m_row, device=dev)
    row = torch.from_numpy((np.arange(S, dtype=np.uint64) * 2654435761 % rows)
                           .astype(np.uint32).view(np.int32)).to(dev)
    xi = rtf.philox(S, seed=0x5EED, start=rank * S, device=dev)
    out = torch.empty(S, dtype=torch.int32, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def step(ev=None):
        if ev:
            ev[0].record(stream)
        forest.build(p)
        if ev:
            ev[1].record(stream)
        forest.sample(row, xi, out)
        if ev:
            ev[2].record(stream)

    for _ in range(args.warmup):
        step()
        flush.zero_()
    torch.cuda.synchronize()
    forest.headers()
    assert forest.last_status == 0
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    sampler = ClockSampler(dev.index)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = rtf.launch_count()
    with sampler:
        for k in range(args.steps):
            step(evs[k])
            flush.zero_()
        torch.cuda.synchronize()
    launches = rtf.launch_count() - l0
    tb = sum(e[0].elapsed_time(e[1]) for e in evs)
    ts = sum(e[1].elapsed_time(e[2]) for e in evs)
    if world > 1:
        t = torch.tensor([tb, ts], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tb, ts = t.tolist()
    K = args.steps
    N = rows * n_row
    build_gs = world * N * K / (tb * 1e-3) / 1e9
    sample_gs = world * S * K / (ts * 1e-3) / 1e9
    peak, peak_src = peaks()
    n_pos = int(forest.headers()["n_pos"].astype(np.int64).sum())
    bytes_build = 4 * N + 16 * N + 4 * m_row * rows
    ach_b = bytes_build / (tb / K * 1e-3) / 1e9
    result = {
        "metric": METRIC, "value": round(build_gs, 4), "unit": "G entries/s", "n_gpus": world,
        "steps": K, "warmup": args.warmup, "ms_per_step": round((tb + ts) / K, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic",
        "config": {"workload": wl["desc"], "rows": rows, "n_row": n_row, "m_row": m_row,
                   "samples_per_gpu": S,
                   "l2": f"flushed between steps ({L2_FLUSH_BYTES >> 20} MiB write, untimed)",
                   "parallelism": f"independent problems x{world}: GPU r builds its own rows "
                                  "(seed 7 + r)"},
        "build": {"value": round(build_gs, 4), "unit": "G entries/s", "ms_per_build": round(tb / K, 5)},
        "sampling": {"value": round(sample_gs, 4), "unit": "G samples/s",
                     "ms_per_batch": round(ts / K, 4)},
        "roofline_build": {"kernel": "k_build_rows (one CTA per row)", "bound": "hbm",
                           "achieved": round(ach_b, 2), "peak": peak, "unit": "GB/s",
                           "frac": round(ach_b / peak, 4), "traffic": None,
                           "algorithmic_bytes_per_launch": bytes_build, "peak_source": peak_src},
        "gpu_launches": launches, "clocks": sampler.summary(),
    }
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(result), flush=True)


def host_cpu():
    """The host CPU model and its logical CPU count."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"model": model, "nproc": os.cpu_count(),
            "affinity": len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity")
            else os.cpu_count()}


def cpu_baseline(p_host, m, xi_sample, cdf_host):
    """The CPU oracle as it stands (single thread), on a bounded sample; plus
    the OpenMP binary search (baselines/cpu_bsearch.c) on the same CDF."""
    import baselines
    import oracle
    n = p_host.size
    reps, tb = 0, 0.0
    while tb < 8.0 and reps < 6:
        t0 = time.perf_counter()
        f = oracle.build(p_host, m)
        tb += time.perf_counter() - t0
        reps += 1
    t0 = time.perf_counter()
    f.sample(xi_sample)
    tsm = time.perf_counter() - t0
    baselines.bsearch(cdf_host, xi_sample[:1024])  # warm-up (thread pool)
    xs = np.tile(xi_sample, 4)
    t0 = time.perf_counter()
    baselines.bsearch(cdf_host, xs)
    tbs = time.perf_counter() - t0
    return {"value": round(n * reps / tb / 1e9, 6), "unit": "G entries/s", "cores": 1,
            "kind": "oracle", "host": host_cpu(),
            "sample": f"{reps} full oracle builds of the same n={n} input; sampling "
                      f"{xi_sample.size} of the same xi",
            "sampling": {"value": round(xi_sample.size / tsm / 1e9, 6), "unit": "G samples/s"},
            "bsearch_openmp": {"value": round(xs.size / tbs / 1e9, 6), "unit": "G samples/s",
                               "cores": baselines.threads(),
                               "sample": f"{xs.size} xi, binary search on the full u64 CDF "
                                         "(baselines/cpu_bsearch.c)"}}


# ============================================================================ reference arm

def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    from workloads import philox_xi, sobol0_xi
    wl = WORKLOADS[args.workload]
    n, m = wl["n"], wl["m"]
    p = make_p(wl)
    S_ref = 1 << 20
    xi = philox_xi(S_ref, seed=0x5EED) if wl["name"] == "c3_powerlaw" else sobol0_xi(S_ref)
    for _ in range(args.warmup if args.warmup < 2 else 1):
        oracle.build(p, m)
    tb, ts = 0.0, 0.0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        f = oracle.build(p, m)
        t1 = time.perf_counter()
        f.sample(xi)
        t2 = time.perf_counter()
        tb += t1 - t0
        ts += t2 - t1
    value = n * args.steps / tb / 1e9
    result = {
        "metric": METRIC, "value": round(value, 6), "unit": "G entries/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round((tb + ts) / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": wl["desc"], "n": n, "m": m,
                   "samples_per_step": S_ref,
                   "note": "CPU oracle (oracle/rtf_oracle.c, serial, 1 thread): each step = one "
                           "full build of the same input + a bounded sample of 2^20 xi"},
        "cpu_baseline": {"value": round(value, 6), "unit": "G entries/s", "cores": 1,
                         "kind": "oracle", "host": host_cpu(),
                         "sample": f"full n={n} build per step; sampling {S_ref} xi per step",
                         "sampling": {"value": round(S_ref * args.steps / ts / 1e9, 6),
                                      "unit": "G samples/s"}},
        "e2e": {"value": round(value, 6), "unit": "G entries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(result), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="rtf", choices=["rtf", "reference"])
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--samples", type=int, default=0, help="override samples per GPU")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c2", action="store_true", help="skip the config-2 summary")
    ap.add_argument("--c4-replicate", action="store_true",
                    help="config 4: replicate the whole forest instead of ranged sharding")
    ap.add_argument("--no-m26", action="store_true",
                    help="config 4: skip the m = 2^26 single-forest summary")
    ap.add_argument("--c4-nccl", action="store_true",
                    help="config 4 ranged: move records with NCCL send/recv instead of the "
                         "fused peer stores")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl != "reference":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "c4":
        run_gpu_c4(args)
    elif args.workload == "c5":
        run_gpu_c5(args)
    elif args.workload == "c1":
        run_gpu_c1(args)
    elif args.workload == "c2d":
        run_gpu_2d(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
