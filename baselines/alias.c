/* alias.c -- host construction of an alias table (Walker's method with Vose's
 * worklists, Sec.2.6 P:203-239 of the paper, one of its comparison systems)
 * over the SAME 32-bit xi grid as the forest: item i owns exactly
 *   c_i = ceil(K_{i+1} / 2^31) - ceil(K_i / 2^31)        (K_n = 2^63)
 * of the 2^32 xi values (the counts the inverse mapping gives it), and the
 * table realises those counts exactly in integers.  2^k >= n buckets of
 * s = 2^(32-k) xi values each; bucket b < n starts with its own item b,
 * buckets b >= n with none.  A xi lands in bucket b = xi >> (32-k) at offset
 * o = xi & (s-1) and returns b if o < prob[b], else alias[b].  A reported
 * baseline for bench.py (sampled by rtf_sample_alias on the GPU), not the
 * product path and not the oracle. */
#include <stdint.h>
#include <stdlib.h>

/* From per-item xi counts c[0..n) (summing to 2^32) into 2^k >= n buckets;
 * returns 0, or -1 on allocation failure. */
int alias_build_counts(const uint64_t *cnt, uint32_t n, int k, uint32_t *prob, int32_t *alias) {
    const uint64_t nb = 1ull << k, s = 1ull << (32 - k);
    uint64_t *c = (uint64_t *)malloc(sizeof(uint64_t) * nb);
    uint32_t *small = (uint32_t *)malloc(sizeof(uint32_t) * nb);
    uint32_t *large = (uint32_t *)malloc(sizeof(uint32_t) * nb);
    if (!c || !small || !large) {
        free(c); free(small); free(large);
        return -1;
    }
    for (uint64_t b = 0; b < nb; ++b) c[b] = b < n ? cnt[b] : 0;
    uint64_t ns = 0, nl = 0;
    for (uint64_t b = nb; b-- > 0;) {  /* worklists as stacks, lowest index on top */
        if (c[b] < s) small[ns++] = (uint32_t)b;
        else large[nl++] = (uint32_t)b;
    }
    while (ns > 0 && nl > 0) {
        const uint32_t l = small[--ns], g = large[--nl];
        prob[l] = (uint32_t)c[l];
        alias[l] = (int32_t)g;
        c[g] -= s - c[l];
        if (c[g] < s) small[ns++] = g;
        else large[nl++] = g;
    }
    /* the rest hold exactly s (in exact integers nothing is left over) */
    while (nl > 0) {
        const uint32_t g = large[--nl];
        prob[g] = (uint32_t)s;
        alias[g] = (int32_t)g;
    }
    while (ns > 0) {
        const uint32_t l = small[--ns];
        prob[l] = (uint32_t)c[l];  /* only c = s can remain */
        alias[l] = (int32_t)l;
    }
    free(c); free(small); free(large);
    return 0;
}

/* From the full fixed-point CDF K[0..n): c_i = ceil(K_{i+1}/2^31) -
 * ceil(K_i/2^31) (K_n = 2^63).  Returns k (log2 of the bucket count), or -1. */
int alias_build(const uint64_t *K, uint32_t n, uint32_t *prob, int32_t *alias) {
    int k = 1;
    while ((1ull << k) < (uint64_t)n) ++k;
    uint64_t *c = (uint64_t *)malloc(sizeof(uint64_t) * (n ? n : 1));
    if (!c) return -1;
    for (uint32_t b = 0; b < n; ++b) {
        const uint64_t lo = (K[b] + 0x7fffffffull) >> 31;
        const uint64_t hi = b + 1 < n ? (K[b + 1] + 0x7fffffffull) >> 31 : (1ull << 32);
        c[b] = hi - lo;
    }
    const int r = alias_build_counts(c, n, k, prob, alias);
    free(c);
    return r ? -1 : k;
}
