/* cpu_bsearch.c -- host-core binary-search baseline (SURVEY.md 8(d) "CPU side"):
 * out[k] = the last i with cdf[i] <= xi[k] 2^31 over the full fixed-point CDF
 * (the search of Sec.2.2, an upper_bound on the same u64 keys the
 * GPU baseline k_bsearch searches), OpenMP over all host cores.  A reported
 * baseline for bench.py, not part of the product path and not the oracle. */
#include <stdint.h>
#include <omp.h>

int cpu_bsearch_threads(void) { return omp_get_max_threads(); }

void cpu_bsearch(const uint64_t *cdf, uint32_t n, const uint32_t *xi, uint64_t count,
                 int32_t *out) {
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < (int64_t)count; ++k) {
        const uint64_t x = (uint64_t)xi[k] << 31;
        uint32_t base = 0, len = n;
        while (len > 1) {
            const uint32_t half = len >> 1;
            base = (cdf[base + half] <= x) ? base + half : base;
            len -= half;
        }
        out[k] = (int32_t)base;
    }
}
