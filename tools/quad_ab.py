"""Binary (rtf_sample) vs 4-ary collapsed records (rtf_sample_quad) on configs 3,
2 and 4: per-launch device times with the L2 flushed before each launch."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    import paper_1901_05423_b200 as rtf
    from workloads import spikes

    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    def timed(fn, reps=7):
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

    cases = [("c3", bench.make_p(bench.WORKLOADS["c3"]), 1 << 22),
             ("c2", bench.make_p(bench.WORKLOADS["c2"]), 2048 * 1024),
             ("c4", spikes(1 << 28), 1 << 22)]
    S = 1 << 28
    xi = rtf.philox(S, seed=0x5EED)
    out = torch.empty(S, dtype=torch.int32, device="cuda")
    out4 = torch.empty(S, dtype=torch.int32, device="cuda")
    for name, p_host, m in cases:
        p = torch.from_numpy(p_host).cuda()
        f = rtf.build(p, m)
        t_build = timed(lambda: f.build(p))
        f.build_quad()
        t_quad = timed(lambda: f.build_quad())
        t_s = timed(lambda: f.sample(xi, out))
        t_s4 = timed(lambda: f.sample_quad(xi, out4))
        same = bool(torch.equal(out, out4))
        print(f"{name}: build {t_build:.3f} ms, build_quad {t_quad:.3f} ms | 2^28 samples: binary "
              f"{t_s:.3f} ms ({S / t_s / 1e6:.1f} G/s), quad {t_s4:.3f} ms ({S / t_s4 / 1e6:.1f} G/s)"
              f", identical {same}", flush=True)
        del f, p
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
