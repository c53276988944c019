// rtf_sample.cu -- Alg. 2 sampler, the binary-search baseline and
// the Philox input generator.
//
// k_sample: every thread owns 4 samples (one 16-B load of xi, one 16-B store of
// out) and advances their 4 descents in lock-step so up to 4 independent node
// loads are in flight per thread.  Per visit one 16-B record (key + both
// children, the interleaving of P:1082-1083) is read through the read-only path.
#include "rtf_device.cuh"
#include "rtf_internal.h"

namespace rtf {

constexpr int kSampleThreads = 256;
// A valid forest needs at most 64 node visits (<= 63 internal levels, since the
// split level strictly decreases from a cell root to a leaf, plus the anchor).
// The descent is bounded so a corrupted buffer cannot hang the GPU; such
// samples return kCorrupt.
constexpr int kMaxVisits = 64;
constexpr int32_t kCorrupt = INT32_MIN;

__device__ __forceinline__ int32_t descend_step(const rtf_node* __restrict__ nodes, int32_t j,
                                                uint64_t x63) {
    const ulonglong2 r = __ldg(reinterpret_cast<const ulonglong2*>(nodes + j));
    return (int32_t)(x63 < r.x ? (uint32_t)r.y : (uint32_t)(r.y >> 32));
}

// Degenerate-cell fallback (reading R21): a marked cell (key32 = 3 << 30 | k,
// ref = its first leaf a) is searched by bisection of the index interval
// [a-1, a+k) of the intervals overlapping it (Sec.6), at most
// ceil(log2(k + 1)) record reads.  The answer's leaf reference comes from the
// probed records as prefilled by the build: ~orig(a-1) is the anchor's child0,
// ~orig(j) the child1 of record j when leaf j hangs right of gap j-1, else
// the child0 of record j+1 (then probed as the upper bound).
constexpr uint32_t kBisectFlag = 0xC0000000u;  // both top bits: never a packed cell's
constexpr uint32_t kFallbackSlack = 4;

__device__ __forceinline__ int32_t bisect_cell(const rtf_node* __restrict__ nodes, int32_t a,
                                               uint32_t k, uint64_t x63, int32_t* visits) {
    int32_t lo = a - 1, hi = a + (int32_t)k;  // key_lo <= x63 < key_hi
    int32_t c1_lo = 0, c0_hi = 0;
    while (hi - lo > 1) {
        const int32_t mid = (lo + hi) >> 1;  // lo >= -1 and hi < 2^31: no overflow
        const ulonglong2 r = __ldg(reinterpret_cast<const ulonglong2*>(nodes + mid));
        if (r.x <= x63) {
            lo = mid;
            c1_lo = (int32_t)(uint32_t)(r.y >> 32);
        } else {
            hi = mid;
            c0_hi = (int32_t)(uint32_t)r.y;
        }
        if (visits) ++*visits;
    }
    return (lo == a - 1 || c1_lo >= 0) ? c0_hi : c1_lo;
}

// Alg. 2's first step on a guide-table cell (rtf_ref): a node reference, a
// packed three-interval cell (R20) or a leaf that a two-interval cell (R18)
// splits with one comparison (table_step, rtf_device.cuh).  A marked cell
// (R21) returns kBisect: the caller bisects it after its lock-step descents,
// so the bisection adds no registers to them.  (kBisect = INT32_MIN is no leaf
// reference: ~orig >= INT32_MIN + 1 for orig < 2^31 - 1.)
constexpr int32_t kBisect = INT32_MIN;

template <bool FB = true>
__device__ __forceinline__ int32_t cell_step(const rtf_ref* __restrict__ table, uint32_t m,
                                             uint32_t xmask, uint32_t x) {
    const int2 e = __ldg(reinterpret_cast<const int2*>(table) + (uint32_t)(((uint64_t)x * m) >> 32));
    if (FB && e.y >= 0 && ((uint32_t)e.x & kBisectFlag) == kBisectFlag) return kBisect;
    return table_step(e, x, x & xmask);
}

// the answer for xi = x in a marked cell (a leaf reference)
__device__ __noinline__ int32_t bisect_xi(const rtf_ref* __restrict__ table,
                                          const rtf_node* __restrict__ nodes, uint32_t m, uint32_t x,
                                          int32_t* visits) {
    const int2 e = __ldg(reinterpret_cast<const int2*>(table) + (uint32_t)(((uint64_t)x * m) >> 32));
    return bisect_cell(nodes, e.y, (uint32_t)e.x & ~kBisectFlag, (uint64_t)x << 31, visits);
}

template <bool ROWS, bool FB>
__device__ __forceinline__ int32_t sample_one(const rtf_node* __restrict__ nodes,
                                              const rtf_ref* __restrict__ table,
                                              const rtf_header* __restrict__ hdr, uint32_t n,
                                              uint32_t m, uint32_t xmask, uint32_t r, uint32_t x) {
    if (ROWS) {  // a poisoned row's cells are {0, INT32_MIN}: the answer is INT32_MAX
        nodes += (size_t)r * n;
        table += (size_t)r * m;
    }
    int32_t j = cell_step<FB>(table, m, xmask, x);
    if (FB && j == kBisect) return ~bisect_xi(table, nodes, m, x, nullptr);
    const uint64_t x63 = (uint64_t)x << 31;
    for (int d = 0; j >= 0 && d < kMaxVisits; ++d) j = descend_step(nodes, j, x63);
    return j >= 0 ? kCorrupt : ~j;
}

// float xi in [0, 1) -> u32 fixed point floor(xi 2^32) (exact: a power-of-two
// scaling, then truncation; reading R11); out-of-range values saturate
__device__ __forceinline__ uint32_t xi_bits(uint32_t v, bool f32) {
    return f32 ? __float2uint_rz(__uint_as_float(v) * 4294967296.0f) : v;
}

// FB: the table may hold cells marked by rtf_build_fallback (R21); the
// unmarked sampler carries no code for them (registers stay at 32).
template <bool ROWS, bool F32 = false, bool FB = false>
__global__ void __launch_bounds__(kSampleThreads, FB ? 8 : 0)
    k_sample(const rtf_node* __restrict__ nodes, const rtf_ref* __restrict__ table,
             const rtf_header* __restrict__ hdr, uint32_t n, uint32_t m, uint32_t xmask,
             const uint32_t* __restrict__ row, const uint32_t* __restrict__ xi, uint64_t count,
             int32_t* __restrict__ out, bool vec) {
    const uint64_t gt = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t gs = (uint64_t)gridDim.x * blockDim.x;
    const bool bad = !ROWS && hdr->status != 0;
    // The kernel is bound by the L1TEX -> L2 request rate (about one request
    // per clock per SM for scattered loads; ncu): what counts
    // is loads per sample, which the two-interval cells cut.  (L2 evict-first
    // on the xi/out streams was measured slower: 8.0 vs 7.4 ms for config 3.)
    uint64_t done = 0;
    if (vec) {
        const uint64_t nq = count >> 2;
        for (uint64_t q = gt; q < nq; q += gs) {
            const uint4 xv = ld_stream_u4(xi + 4 * q);
            const uint32_t x[4] = {xi_bits(xv.x, F32), xi_bits(xv.y, F32), xi_bits(xv.z, F32),
                                   xi_bits(xv.w, F32)};
            int32_t j[4];
            const rtf_node* nb[4];
            uint64_t x63[4];
            bool dead[4];
            uint4 rv = make_uint4(0, 0, 0, 0);
            if (ROWS) rv = ld_stream_u4(row + 4 * q);
            const uint32_t rr[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const rtf_node* nk = nodes;
                const rtf_ref* tk = table;
                dead[k] = bad;
                if (ROWS) {
                    nk += (size_t)rr[k] * n;
                    tk += (size_t)rr[k] * m;
                }
                nb[k] = nk;
                x63[k] = (uint64_t)x[k] << 31;
                j[k] = dead[k] ? -1 : cell_step<FB>(tk, m, xmask, x[k]);
            }
            for (int it = 0; (j[0] & j[1] & j[2] & j[3]) >= 0 && it < kMaxVisits; ++it) {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (j[k] >= 0) j[k] = descend_step(nb[k], j[k], x63[k]);
            }
            if (FB && ((j[0] == kBisect) | (j[1] == kBisect) | (j[2] == kBisect) | (j[3] == kBisect))) {
#pragma unroll
                for (int k = 0; k < 4; ++k)  // marked cells (R21), after the lock-step descents
                    if (j[k] == kBisect)
                        j[k] = bisect_xi(ROWS ? table + (size_t)rr[k] * m : table, nb[k], m, x[k], nullptr);
            }
            int4 o;
            o.x = dead[0] ? INT32_MAX : (j[0] >= 0 ? kCorrupt : ~j[0]);
            o.y = dead[1] ? INT32_MAX : (j[1] >= 0 ? kCorrupt : ~j[1]);
            o.z = dead[2] ? INT32_MAX : (j[2] >= 0 ? kCorrupt : ~j[2]);
            o.w = dead[3] ? INT32_MAX : (j[3] >= 0 ? kCorrupt : ~j[3]);
            __stcs(reinterpret_cast<int4*>(out + 4 * q), o);
        }
        done = nq << 2;
    }
    for (uint64_t k = done + gt; k < count; k += gs) {
        const uint32_t r = ROWS ? row[k] : 0u;
        out[k] = bad ? INT32_MAX : sample_one<ROWS, FB>(nodes, table, hdr, n, m, xmask, r, xi_bits(xi[k], F32));
    }
}

// Load counts (a measurement aid, not the sampler): 1 table cell + 1 per node
// visited (Table 1's convention); loads_plain: the same without
// the two-interval and packed-cell flags (a flagged cell costs its anchor
// visit, a packed one its anchor and root visits too).
__global__ void __launch_bounds__(kSampleThreads)
    k_sample_loads(const rtf_node* __restrict__ nodes, const rtf_ref* __restrict__ table,
                   uint32_t m, uint32_t xmask, const uint32_t* __restrict__ xi, uint64_t count,
                   int32_t* __restrict__ loads, int32_t* __restrict__ loads_plain) {
    const uint64_t gs = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count; k += gs) {
        const uint32_t x = xi[k];
        const uint32_t g = (uint32_t)(((uint64_t)x * m) >> 32);
        // without the flags a two-interval cell costs its anchor visit too,
        // a packed cell its anchor and root visits
        const rtf_ref e = table[g];
        const int32_t extra =
            (e.key32 == 0 || (e.ref >= 0 && (e.key32 & kBisectFlag) == kBisectFlag)) ? 0 : (e.ref < 0 ? 1 : 2);
        int32_t l = 1;
        int32_t j = cell_step(table, m, xmask, x);
        if (j == kBisect) j = bisect_xi(table, nodes, m, x, &l);
        for (; j >= 0 && l <= kMaxVisits; ++l) j = descend_step(nodes, j, (uint64_t)x << 31);
        loads[k] = l;
        if (loads_plain) loads_plain[k] = l + extra;
    }
}

// ------------------------------------------------------------ degenerate-cell fallback pass (R21)
// K1, one thread per leaf j: the last leaf of each cell (last[cell]); for a
// leaf reachable by a 32-bit xi (ceil(key_j / 2^31) < ceil(key_{j+1} / 2^31))
// the node visits Alg. 2 makes for xi_j = ceil(key_j / 2^31) through an
// anchor cell, maximised per cell of xi_j (depth[]).  Every xi reaching leaf j
// follows the same path, so depth[g] is the most visits of any xi of cell g
// (but the anchor's left child: 1).
__global__ void __launch_bounds__(kSampleThreads)
    k_fallback_depth(const rtf_node* __restrict__ nodes, const rtf_ref* __restrict__ table,
                     const rtf_header* __restrict__ hdr, uint32_t n, uint32_t m,
                     uint32_t* __restrict__ depth, uint32_t* __restrict__ last) {
    const uint32_t n_pos = hdr->status ? 0u : min(hdr->n_pos, n);
    const uint32_t gs = gridDim.x * blockDim.x;
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n_pos; j += gs) {
        const uint64_t key = __ldg(&nodes[j].key);
        const uint64_t kn = j + 1 < n_pos ? __ldg(&nodes[j + 1].key) : kOne63;
        const uint32_t c = cell_of(key, m);
        if (j + 1 == n_pos || cell_of(kn, m) != c) last[c] = j;
        const uint64_t x = (key + 0x7fffffffull) >> 31, xn = (kn + 0x7fffffffull) >> 31;
        if (x >= xn) continue;  // no 32-bit xi reaches leaf j
        const uint32_t g = (uint32_t)((x * m) >> 32);
        const int2 e = __ldg(reinterpret_cast<const int2*>(table) + g);
        if (e.y < 0 || e.x != 0) continue;  // not an anchor cell
        const uint64_t x63 = x << 31;
        int32_t v = 0, node = e.y;
        for (; node >= 0 && v < kMaxVisits; ++v) {
            const ulonglong2 r = __ldg(reinterpret_cast<const ulonglong2*>(nodes + node));
            node = (int32_t)(x63 < r.x ? (uint32_t)r.y : (uint32_t)(r.y >> 32));
        }
        atomicMax(&depth[g], (uint32_t)v);
    }
}

// K2, one thread per cell: an anchor cell (key32 = 0, ref = a) with k leaves
// is marked when it holds k < 2^30 leaves and its depth exceeds
// ceil(log2(k + 1)) + kFallbackSlack.
__global__ void k_fallback_mark(rtf_ref* __restrict__ table, uint32_t m,
                                const uint32_t* __restrict__ depth, const uint32_t* __restrict__ last) {
    const uint32_t gs = gridDim.x * blockDim.x;
    for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < m; g += gs) {
        const rtf_ref e = table[g];
        if (e.ref < 0 || e.key32 != 0) continue;
        const uint32_t k = last[g] - (uint32_t)e.ref + 1u;
        const uint32_t bis = 32u - (uint32_t)__clz((int)k);  // ceil(log2(k + 1))
        if (k < (1u << 30) && depth[g] > bis + kFallbackSlack) st_cell(table, g, kBisectFlag | k, e.ref);
    }
}


// ------------------------------------------------------------ binary-search baseline

__global__ void __launch_bounds__(kSampleThreads)
    k_bsearch(const uint64_t* __restrict__ cdf, uint32_t n, const rtf_header* __restrict__ hdr,
              const uint32_t* __restrict__ xi, uint64_t count, int32_t* __restrict__ out,
              bool vec) {
    const uint64_t gt = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t gs = (uint64_t)gridDim.x * blockDim.x;
    const bool bad = hdr->status != 0;
    uint64_t done = 0;
    if (vec) {
        const uint64_t nq = count >> 2;
        for (uint64_t q = gt; q < nq; q += gs) {
            const uint4 xv = ld_stream_u4(xi + 4 * q);
            const uint64_t x63[4] = {(uint64_t)xv.x << 31, (uint64_t)xv.y << 31,
                                     (uint64_t)xv.z << 31, (uint64_t)xv.w << 31};
            uint32_t base[4] = {0, 0, 0, 0};
            uint32_t len = n;
            while (len > 1) {  // last index with cdf <= x (cdf[0] = 0)
                const uint32_t half = len >> 1;
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (__ldg(cdf + base[k] + half) <= x63[k]) base[k] += half;
                len -= half;
            }
            int4 o;
            o.x = bad ? INT32_MAX : (int32_t)base[0];
            o.y = bad ? INT32_MAX : (int32_t)base[1];
            o.z = bad ? INT32_MAX : (int32_t)base[2];
            o.w = bad ? INT32_MAX : (int32_t)base[3];
            __stcs(reinterpret_cast<int4*>(out + 4 * q), o);
        }
        done = nq << 2;
    }
    for (uint64_t k = done + gt; k < count; k += gs) {
        const uint64_t x63 = (uint64_t)xi[k] << 31;
        uint32_t base = 0, len = n;
        while (len > 1) {
            const uint32_t half = len >> 1;
            if (__ldg(cdf + base + half) <= x63) base += half;
            len -= half;
        }
        out[k] = bad ? INT32_MAX : (int32_t)base;
    }
}

// ------------------------------------------------------------ Eytzinger binary-search baseline
// The binary search of Sec.2.2 laid out for a GPU: the keys
// cdf[1..n-1] (cdf[0] = 0 is below every xi) as a complete binary search tree
// of height H = ceil(log2 n) in breadth-first order (node k at depth d holds the
// key of in-order rank (2 (k - 2^d) + 1) 2^(H-1-d) - 1, ranks >= n - 1 hold
// +inf).  After H comparisons "go right iff key <= x" the node index minus 2^H
// is the number of keys <= x, i.e. the last i with cdf[i] <= x: no index array.
// The top levels (up to 2^13 - 1 keys, 64 KB) sit in shared memory per CTA,
// so only the lower levels are global (L2 / HBM) loads.

constexpr int kEytThreads = 256;
constexpr int kEytSmemLevels = 13;

__global__ void k_eytzinger_build(const uint64_t* __restrict__ cdf, uint32_t n, uint32_t H,
                                  uint64_t* __restrict__ eyt) {
    const uint64_t slots = 1ull << H;  // index 0 unused
    const uint64_t gs = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = 1 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < slots; k += gs) {
        const uint32_t d = 63u - (uint32_t)__clzll((long long)k);
        const uint64_t rank = ((2ull * (k - (1ull << d)) + 1ull) << (H - 1u - d)) - 1ull;
        eyt[k] = rank + 1 < n ? cdf[rank + 1] : ~0ull;
    }
}

__global__ void __launch_bounds__(kEytThreads, 3)
    k_eytzinger(const uint64_t* __restrict__ eyt, uint32_t H, const rtf_header* __restrict__ hdr,
                const uint32_t* __restrict__ xi, uint64_t count, int32_t* __restrict__ out,
                bool vec) {
    extern __shared__ uint64_t s_top[];  // s_top[k] = eyt[k], k < 2^L
    const uint32_t L = H < (uint32_t)kEytSmemLevels ? H : (uint32_t)kEytSmemLevels;
    for (uint32_t k = threadIdx.x; k < (1u << L); k += blockDim.x) s_top[k] = eyt[k];
    __syncthreads();
    const bool bad = hdr->status != 0;
    const uint64_t gt = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t gs = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t top = 1ull << H;
    uint64_t done = 0;
    if (vec) {
        const uint64_t nq = count >> 2;
        for (uint64_t q = gt; q < nq; q += gs) {
            const uint4 xv = ld_stream_u4(xi + 4 * q);
            const uint64_t x63[4] = {(uint64_t)xv.x << 31, (uint64_t)xv.y << 31,
                                     (uint64_t)xv.z << 31, (uint64_t)xv.w << 31};
            uint64_t k[4] = {1, 1, 1, 1};
            for (uint32_t d = 0; d < L; ++d) {
#pragma unroll
                for (int s = 0; s < 4; ++s) k[s] = 2 * k[s] + (s_top[k[s]] <= x63[s] ? 1 : 0);
            }
            for (uint32_t d = L; d < H; ++d) {
#pragma unroll
                for (int s = 0; s < 4; ++s) k[s] = 2 * k[s] + (__ldg(eyt + k[s]) <= x63[s] ? 1 : 0);
            }
            int4 o;
            o.x = bad ? INT32_MAX : (int32_t)(k[0] - top);
            o.y = bad ? INT32_MAX : (int32_t)(k[1] - top);
            o.z = bad ? INT32_MAX : (int32_t)(k[2] - top);
            o.w = bad ? INT32_MAX : (int32_t)(k[3] - top);
            __stcs(reinterpret_cast<int4*>(out + 4 * q), o);
        }
        done = nq << 2;
    }
    for (uint64_t i = done + gt; i < count; i += gs) {
        const uint64_t x63 = (uint64_t)xi[i] << 31;
        uint64_t k = 1;
        for (uint32_t d = 0; d < H; ++d) k = 2 * k + ((d < L ? s_top[k] : __ldg(eyt + k)) <= x63 ? 1 : 0);
        out[i] = bad ? INT32_MAX : (int32_t)(k - top);
    }
}

// ------------------------------------------------------------ alias baseline
// The alias method (Walker, Vose; Sec.2.6, a comparison system of
// the paper) over the same 32-bit xi grid: 2^k buckets of 2^(32-k) xi each,
// entry {prob, alias} (host-built, baselines/alias.c); xi -> bucket b = xi >>
// (32-k), offset o = xi mod 2^(32-k), answer o < prob ? b : alias.  Each
// item receives exactly the xi count the inverse mapping gives it, but not
// the same xi: the mapping is not monotone.  One 8-B load per xi.
__global__ void __launch_bounds__(kSampleThreads)
    k_alias(const uint2* __restrict__ tab, uint32_t k, const uint32_t* __restrict__ xi,
            uint64_t count, int32_t* __restrict__ out, bool vec) {
    const uint64_t gt = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t gs = (uint64_t)gridDim.x * blockDim.x;
    const uint32_t sh = 32u - k, om = (uint32_t)((1ull << sh) - 1ull);
    auto one = [&](uint32_t x) -> int32_t {
        const uint2 e = __ldg(tab + (x >> sh));
        return (x & om) < e.x ? (int32_t)(x >> sh) : (int32_t)e.y;
    };
    uint64_t done = 0;
    if (vec) {
        const uint64_t nq = count >> 2;
        for (uint64_t q = gt; q < nq; q += gs) {
            const uint4 xv = ld_stream_u4(xi + 4 * q);
            int4 o;
            o.x = one(xv.x);
            o.y = one(xv.y);
            o.z = one(xv.z);
            o.w = one(xv.w);
            __stcs(reinterpret_cast<int4*>(out + 4 * q), o);
        }
        done = nq << 2;
    }
    for (uint64_t i = done + gt; i < count; i += gs) out[i] = one(xi[i]);
}

// ------------------------------------------------------------ cutpoint baselines
// The guide-table methods the paper compares against (Sec.2.3, Table 1
// P:1458-1482): cut[g] = the answer for the smallest xi of cell g (an index
// into the full CDF), then a linear scan (cutpoint + linear) or a binary
// search bounded by cut[g+1] (cutpoint + binary).  Same fixed-point CDF and
// the same results as k_bsearch / k_sample.

__device__ __forceinline__ uint32_t last_le(const uint64_t* __restrict__ cdf, uint32_t base,
                                            uint32_t len, uint64_t x63) {
    while (len > 1) {  // last index in [base, base + len) with cdf <= x63
        const uint32_t half = len >> 1;
        if (__ldg(cdf + base + half) <= x63) base += half;
        len -= half;
    }
    return base;
}

__global__ void k_cutpoint_build(const uint64_t* __restrict__ cdf, uint32_t n, uint32_t m,
                                 uint32_t* __restrict__ cut) {
    const uint32_t gs = gridDim.x * blockDim.x;
    for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g <= m; g += gs) {
        if (g == m) {
            cut[m] = n - 1;
            continue;
        }
        const uint64_t xmin = (((uint64_t)g << 32) + m - 1) / m;  // ceil(g 2^32 / m)
        cut[g] = last_le(cdf, 0, n, xmin << 31);
    }
}

template <bool BINARY>
__global__ void __launch_bounds__(kSampleThreads)
    k_sample_cutpoint(const uint64_t* __restrict__ cdf, uint32_t n,
                      const rtf_header* __restrict__ hdr, const uint32_t* __restrict__ cut,
                      uint32_t m, const uint32_t* __restrict__ xi, uint64_t count,
                      int32_t* __restrict__ out) {
    const uint64_t gs = (uint64_t)gridDim.x * blockDim.x;
    const bool bad = hdr->status != 0;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count; k += gs) {
        const uint32_t x = xi[k];
        const uint64_t x63 = (uint64_t)x << 31;
        const uint32_t g = (uint32_t)(((uint64_t)x * m) >> 32);
        uint32_t i = __ldg(cut + g);
        if (BINARY) {
            i = last_le(cdf, i, __ldg(cut + g + 1) - i + 1, x63);
        } else {
            while (i + 1 < n && __ldg(cdf + i + 1) <= x63) ++i;
        }
        out[k] = bad ? INT32_MAX : (int32_t)i;
    }
}

// ------------------------------------------------------------ Philox4x32-10 input generator

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    }
    return c;
}

__global__ void k_philox(uint64_t seed, uint64_t start, uint64_t count, uint32_t* __restrict__ out) {
    const uint64_t b0 = start >> 2, b1 = (start + count + 3) >> 2;
    const uint64_t gs = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t b = b0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; b < b1; b += gs) {
        const uint4 r = philox4x32_10(make_uint4((uint32_t)b, (uint32_t)(b >> 32), 0u, 0u),
                                      (uint32_t)seed, (uint32_t)(seed >> 32));
        const uint32_t v[4] = {r.x, r.y, r.z, r.w};
        const uint64_t k0 = b << 2;
        if (k0 >= start && k0 + 4 <= start + count && ((k0 - start) & 3) == 0 &&
            (((uintptr_t)(out + (k0 - start))) & 15) == 0) {
            *reinterpret_cast<uint4*>(out + (k0 - start)) = r;
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint64_t k = k0 + i;
                if (k >= start && k < start + count) out[k - start] = v[i];
            }
        }
    }
}

// ------------------------------------------------------------ launchers

#ifndef RTF_SAMPLE_GRID_PER_SM
#define RTF_SAMPLE_GRID_PER_SM 64
#endif
static inline uint32_t grid_for(uint64_t work_items) {
    const uint64_t want = (work_items + kSampleThreads - 1) / kSampleThreads;
    return (uint32_t)std::max<uint64_t>(
        1, std::min<uint64_t>(want, (uint64_t)device_sms() * RTF_SAMPLE_GRID_PER_SM));
}

cudaError_t launch_fallback(const rtf_forest& f, uint32_t* depth, uint32_t* last, cudaStream_t st,
                            int* launches) {
    cudaError_t e = cudaMemsetAsync(depth, 0, sizeof(uint32_t) * (size_t)f.m, st);
    if (e != cudaSuccess) return e;
    k_fallback_depth<<<grid_for(f.n), kSampleThreads, 0, st>>>(f.nodes, f.table, f.header, f.n,
                                                               f.m, depth, last);
    ++*launches;
    k_fallback_mark<<<grid_for(f.m), kSampleThreads, 0, st>>>(f.table, f.m, depth, last);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_sample(const rtf_forest& f, const uint32_t* row, const uint32_t* xi,
                          uint64_t count, int32_t* out, cudaStream_t st, int* launches) {
    if (count == 0) return cudaSuccess;
    bool vec = (((uintptr_t)xi | (uintptr_t)out) & 15u) == 0;
    if (row) vec = vec && (((uintptr_t)row & 15u) == 0);
    const uint32_t grid = grid_for(vec ? (count + 3) / 4 : count);
    if (row)
        k_sample<true><<<grid, kSampleThreads, 0, st>>>(f.nodes, f.table, f.header, f.n, f.m,
                                                        xoff_mask(f.m), row, xi, count, out, vec);
    else if (f.flags & RTF_FOREST_MARKED)
        k_sample<false, false, true><<<grid, kSampleThreads, 0, st>>>(
            f.nodes, f.table, f.header, f.n, f.m, xoff_mask(f.m), nullptr, xi, count, out, vec);
    else
        k_sample<false><<<grid, kSampleThreads, 0, st>>>(f.nodes, f.table, f.header, f.n, f.m,
                                                         xoff_mask(f.m), nullptr, xi, count, out,
                                                         vec);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_sample_f32(const rtf_forest& f, const float* xi, uint64_t count, int32_t* out,
                              cudaStream_t st, int* launches) {
    if (count == 0) return cudaSuccess;
    const bool vec = (((uintptr_t)xi | (uintptr_t)out) & 15u) == 0;
    if (f.flags & RTF_FOREST_MARKED) {
        k_sample<false, true, true><<<grid_for(vec ? (count + 3) / 4 : count), kSampleThreads, 0, st>>>(
            f.nodes, f.table, f.header, f.n, f.m, xoff_mask(f.m), nullptr,
            reinterpret_cast<const uint32_t*>(xi), count, out, vec);
        ++*launches;
        return cudaGetLastError();
    }
    k_sample<false, true><<<grid_for(vec ? (count + 3) / 4 : count), kSampleThreads, 0, st>>>(
        f.nodes, f.table, f.header, f.n, f.m, xoff_mask(f.m), nullptr,
        reinterpret_cast<const uint32_t*>(xi), count, out, vec);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_sample_loads(const rtf_forest& f, const uint32_t* xi, uint64_t count,
                                int32_t* loads, int32_t* loads_plain, cudaStream_t st,
                                int* launches) {
    if (count == 0) return cudaSuccess;
    k_sample_loads<<<grid_for(count), kSampleThreads, 0, st>>>(f.nodes, f.table, f.m,
                                                              xoff_mask(f.m), xi, count, loads,
                                                              loads_plain);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_bsearch(const uint64_t* cdf, uint32_t n, const rtf_header* hdr,
                           const uint32_t* xi, uint64_t count, int32_t* out, cudaStream_t st,
                           int* launches) {
    if (count == 0) return cudaSuccess;
    const bool vec = (((uintptr_t)xi | (uintptr_t)out) & 15u) == 0;
    k_bsearch<<<grid_for(vec ? (count + 3) / 4 : count), kSampleThreads, 0, st>>>(cdf, n, hdr, xi,
                                                                                  count, out, vec);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_eytzinger_build(const uint64_t* cdf, uint32_t n, uint64_t* eyt,
                                   cudaStream_t st, int* launches) {
    const uint32_t H = (uint32_t)ceil_log2_u32(n);
    if (H == 0) return cudaSuccess;
    k_eytzinger_build<<<grid_for(1ull << H), kSampleThreads, 0, st>>>(cdf, n, H, eyt);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_eytzinger(const uint64_t* eyt, uint32_t n, const rtf_header* hdr,
                             const uint32_t* xi, uint64_t count, int32_t* out, cudaStream_t st,
                             int* launches) {
    if (count == 0) return cudaSuccess;
    const uint32_t H = (uint32_t)ceil_log2_u32(n);
    const uint32_t L = std::min<uint32_t>(H, kEytSmemLevels);
    const size_t smem = sizeof(uint64_t) << L;
    static std::atomic<bool> attr_set[kMaxDevices] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < kMaxDevices && !attr_set[dev].load(std::memory_order_relaxed)) {
        cudaError_t e = cudaFuncSetAttribute(k_eytzinger, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)(sizeof(uint64_t) << kEytSmemLevels));
        if (e != cudaSuccess) return e;
        attr_set[dev].store(true, std::memory_order_relaxed);
    }
    const bool vec = (((uintptr_t)xi | (uintptr_t)out) & 15u) == 0;
    const uint64_t items = vec ? (count + 3) / 4 : count;
    const uint64_t want = (items + kEytThreads - 1) / kEytThreads;
    const uint32_t grid = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(want, 3ull * device_sms()));
    k_eytzinger<<<grid, kEytThreads, smem, st>>>(eyt, H, hdr, xi, count, out, vec);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_alias(const uint2* tab, uint32_t k, const uint32_t* xi, uint64_t count,
                         int32_t* out, cudaStream_t st, int* launches) {
    if (count == 0) return cudaSuccess;
    const bool vec = (((uintptr_t)xi | (uintptr_t)out) & 15u) == 0;
    k_alias<<<grid_for(vec ? (count + 3) / 4 : count), kSampleThreads, 0, st>>>(tab, k, xi, count,
                                                                                out, vec);
    ++*launches;
    return cudaGetLastError();
}

// 2-D alias baseline (the comparison of the paper's convergence figure,
// P:900-970): xi1 through the marginal table picks the row y, xi2 through row
// y's table (2^kx buckets at rows + y 2^kx) picks the column x.  Two dependent
// 8-B loads per pair.
__global__ void __launch_bounds__(kSampleThreads)
    k_alias_2d(const uint2* __restrict__ marg, uint32_t ky, const uint2* __restrict__ rows,
               uint32_t kx, uint32_t W, const uint32_t* __restrict__ xi1,
               const uint32_t* __restrict__ xi2, uint64_t count, int32_t* __restrict__ pixel) {
    const uint64_t gs = (uint64_t)gridDim.x * blockDim.x;
    const uint32_t shy = 32u - ky, omy = (uint32_t)((1ull << shy) - 1ull);
    const uint32_t shx = 32u - kx, omx = (uint32_t)((1ull << shx) - 1ull);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gs) {
        const uint32_t a = __ldcs(xi1 + i), b = __ldcs(xi2 + i);
        const uint2 ey = __ldg(marg + (a >> shy));
        const uint32_t y = (a & omy) < ey.x ? (a >> shy) : ey.y;
        const uint2 ex = __ldg(rows + ((uint64_t)y << kx) + (b >> shx));
        const uint32_t x = (b & omx) < ex.x ? (b >> shx) : ex.y;
        __stcs(pixel + i, (int32_t)(y * W + x));
    }
}

cudaError_t launch_alias_2d(const uint2* marg, uint32_t ky, const uint2* rows, uint32_t kx,
                            uint32_t W, const uint32_t* xi1, const uint32_t* xi2, uint64_t count,
                            int32_t* pixel, cudaStream_t st, int* launches) {
    if (count == 0) return cudaSuccess;
    k_alias_2d<<<grid_for(count), kSampleThreads, 0, st>>>(marg, ky, rows, kx, W, xi1, xi2, count,
                                                           pixel);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_cutpoint_build(const uint64_t* cdf, uint32_t n, uint32_t m, uint32_t* cut,
                                  cudaStream_t st, int* launches) {
    k_cutpoint_build<<<grid_for((uint64_t)m + 1), kSampleThreads, 0, st>>>(cdf, n, m, cut);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_cutpoint(const uint64_t* cdf, uint32_t n, const rtf_header* hdr,
                            const uint32_t* cut, uint32_t m, bool binary, const uint32_t* xi,
                            uint64_t count, int32_t* out, cudaStream_t st, int* launches) {
    if (count == 0) return cudaSuccess;
    if (binary)
        k_sample_cutpoint<true><<<grid_for(count), kSampleThreads, 0, st>>>(cdf, n, hdr, cut, m,
                                                                            xi, count, out);
    else
        k_sample_cutpoint<false><<<grid_for(count), kSampleThreads, 0, st>>>(cdf, n, hdr, cut, m,
                                                                             xi, count, out);
    ++*launches;
    return cudaGetLastError();
}

// ------------------------------------------------------------ ranged sharding helper

// counts[k] = number of leaves among nodes[j0, j0 + cnt) whose cell
// floor(key m / 2^63) lies below bounds[k] (keys increase, so a binary search)
__global__ void k_count_cells(const rtf_node* __restrict__ nodes, uint32_t j0, uint32_t cnt,
                              uint32_t m, const uint32_t* __restrict__ bounds, uint32_t nb,
                              uint32_t* __restrict__ counts) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nb) return;
    const uint32_t g = bounds[k];
    uint32_t lo = 0, hi = cnt;  // first local leaf with cell >= g
    while (lo < hi) {
        const uint32_t mid = lo + (hi - lo) / 2;
        if (cell_of(nodes[j0 + mid].key, m) < g) lo = mid + 1;
        else hi = mid;
    }
    counts[k] = lo;
}

cudaError_t launch_count_cells(const rtf_node* nodes, uint32_t j0, uint32_t cnt, uint32_t m,
                               const uint32_t* bounds, uint32_t nb, uint32_t* counts,
                               cudaStream_t st, int* launches) {
    k_count_cells<<<(nb + 127) / 128, 128, 0, st>>>(nodes, j0, cnt, m, bounds, nb, counts);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_philox(uint64_t seed, uint64_t start, uint64_t count, uint32_t* out,
                          cudaStream_t st, int* launches) {
    if (count == 0) return cudaSuccess;
    k_philox<<<grid_for((count + 3) / 4 + 1), kSampleThreads, 0, st>>>(seed, start, count, out);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace rtf
