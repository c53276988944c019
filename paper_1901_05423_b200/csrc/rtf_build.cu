// rtf_build.cu -- the forest build: 4 kernels on the caller's stream.
//
//   K1 k_scale        read p once: max weight bits (for E), NaN/Inf/negative flags;
//                     the last block folds the partials into one scale word and
//                     resets the per-build counters.
//   K2 k_tile_totals  per super-tile (kSubs K3 tiles): quantise (w), sum W, count
//                     positives, last positive index; single-pass reduce-then-scan:
//                     the last CTA to finish scans the super-tile aggregates and
//                     writes every K3 tile's exclusive prefix (the parallel prefix
//                     sum of P:239), T, n' and the reciprocal of T.
//   K3 k_scan_build   persistent, TMA-fed tiles: block scan + tile prefix -> W_j,
//                     compaction, one exact division per leaf (key_j); per owned
//                     leaf: cell, split level lambda_j, guide-table anchors and
//                     short runs; Alg. 1 for every leaf
//                     of the tile except its first and last ("phase 1",
//                     shared-memory atomicExch); coalesced flush of 16-B records.
//   K4 k_cross_tile   "phase 2": the <= 2 pending edge leaves per tile continue
//                     Alg. 1 with global atomicExch, consuming the deposits the
//                     tiles flushed; plus the long empty-cell runs of the table.
// The result bytes do not depend on the schedule.

#include "rtf_device.cuh"
#include "rtf_internal.h"

namespace rtf {

constexpr uint32_t kShortRun = 32;  // empty-cell runs up to this length: written in place
constexpr uint32_t kChunk = 2048;   // longer runs: queued in chunks of this many cells
constexpr int kSubs = 2;            // K3 tiles per K2 super-tile

// workspace counters
enum : int { kCtrDoneK2 = 0, kCtrQueue = 1, kCtrDoneK1 = 3 };

struct RunChunk {
    uint32_t start, len;
    int32_t value;
    uint32_t pad;
};

struct PendingLeaf {
    int32_t j;    // compacted leaf index, -1 if none
    int32_t ref;  // ~orig(j)
};

// ============================================================== K1: scale and validate

__global__ void __launch_bounds__(256) k_scale(const float* __restrict__ p, uint32_t n,
                                               uint32_t* __restrict__ maxpart,
                                               uint32_t* __restrict__ counters,
                                               uint32_t* __restrict__ scale_word, bool vec) {
    const uint32_t gt = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t gs = gridDim.x * blockDim.x;
    if (gt == 0) counters[kCtrQueue] = 0;
    uint32_t mx = 0, fl = 0;
    auto visit = [&](float x) {
        const uint32_t b = __float_as_uint(x);
        if (x != x) fl |= RTF_DATA_NAN;
        else if (fabsf(x) == __int_as_float(0x7f800000)) fl |= RTF_DATA_INF;
        else if (x < 0.0f) fl |= RTF_DATA_NEG;
        else if (x > 0.0f) mx = max(mx, b);
    };
    if (vec) {
        const uint32_t n4 = n >> 2;
        uint32_t q = gt;
        for (; q + 3 * gs < n4; q += 4 * gs) {  // 4 independent 16-B loads in flight
            float4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = ld_stream_f4(p + 4ull * (q + u * gs));
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                visit(v[u].x);
                visit(v[u].y);
                visit(v[u].z);
                visit(v[u].w);
            }
        }
        for (; q < n4; q += gs) {
            const float4 v = ld_stream_f4(p + 4ull * q);
            visit(v.x);
            visit(v.y);
            visit(v.z);
            visit(v.w);
        }
        for (uint32_t i = 4 * n4 + gt; i < n; i += gs) visit(p[i]);
    } else {
        for (uint32_t i = gt; i < n; i += gs) visit(p[i]);
    }
    for (int d = 16; d; d >>= 1) {
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, d));
        fl |= __shfl_xor_sync(0xffffffffu, fl, d);
    }
    __shared__ uint32_t s_mx[8], s_fl[8];
    __shared__ bool s_last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        s_mx[warp] = mx;
        s_fl[warp] = fl;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
            mx = max(mx, s_mx[w]);
            fl |= s_fl[w];
        }
        maxpart[2 * blockIdx.x] = mx;
        maxpart[2 * blockIdx.x + 1] = fl;
        __threadfence();
        s_last = atomicAdd(&counters[kCtrDoneK1], 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    // last block: fold all partials into the scale word
    __threadfence();
    mx = 0;
    fl = 0;
    for (uint32_t b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
        mx = max(mx, __ldcg(&maxpart[2 * b]));
        fl |= __ldcg(&maxpart[2 * b + 1]);
    }
    for (int d = 16; d; d >>= 1) {
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, d));
        fl |= __shfl_xor_sync(0xffffffffu, fl, d);
    }
    __syncthreads();
    if (lane == 0) {
        s_mx[warp] = mx;
        s_fl[warp] = fl;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
            mx = max(mx, s_mx[w]);
            fl |= s_fl[w];
        }
        scale_word[0] = mx;
        scale_word[1] = fl;
        counters[kCtrDoneK1] = 0;  // reset-on-consume for the next build
    }
}

// Load VPT consecutive weights of this thread (blocked layout) with bounds.
template <int VPT>
__device__ __forceinline__ void load_tile(const float* __restrict__ p, uint32_t first, uint32_t n,
                                          bool vec, float (&x)[VPT]) {
    if (vec && first + VPT <= n) {
#pragma unroll
        for (int k = 0; k < VPT; k += 4) {
            const float4 v = ld_stream_f4(p + first + k);
            x[k] = v.x;
            x[k + 1] = v.y;
            x[k + 2] = v.z;
            x[k + 3] = v.w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < VPT; ++k) x[k] = (first + k < n) ? p[first + k] : 0.0f;
    }
}

// ============================================================== K2: tile totals + scan

// Pfx combine of consecutive runs is (sum, sum, max): the last positive index
// only grows along the array (-1 = none).
__device__ __forceinline__ Pfx shfl_xor_pfx(const Pfx& v, int d) {
    Pfx r;
    r.W = __shfl_xor_sync(0xffffffffu, v.W, d);
    r.cnt = __shfl_xor_sync(0xffffffffu, v.cnt, d);
    r.last = __shfl_xor_sync(0xffffffffu, v.last, d);
    return r;
}

// K2 works on super-tiles of kSubs K3 tiles (SUB = THREADS * VPT entries each):
// every thread keeps kSubs*VPT/4 float4 loads in flight (striped, coalesced).
// Each CTA writes its K3 tiles' aggregates; the last CTA to finish (completion
// counter) turns them into exclusive prefixes with one block scan.
template <int THREADS, int VPT>
__global__ void __launch_bounds__(THREADS)
    k_tile_totals(const float* __restrict__ p, uint32_t n, int B, const uint32_t* scale_word,
                  uint32_t* counters, Pfx* excl, rtf_header* hdr, uint32_t nst, uint32_t nt,
                  bool vec) {
    constexpr int NW = THREADS / 32;
    constexpr int SUB = THREADS * VPT;
    constexpr int SUPER = kSubs * SUB;
    constexpr int NF4 = SUPER / (4 * THREADS);
    constexpr int F4_PER_SUB = NF4 / kSubs;  // float4 k of every thread lies in sub-tile k / F4_PER_SUB
    static_assert(F4_PER_SUB >= 1 && VPT % 4 == 0, "bad tile shape");
    __shared__ uint64_t s_w[2 * NW];
    __shared__ uint32_t s_c[2 * NW];
    __shared__ int32_t s_l[2 * NW];
    __shared__ bool s_last;
    const uint32_t mx = scale_word[0], fl = scale_word[1];
    const uint32_t status = fl | (mx == 0 ? RTF_DATA_ALLZERO : 0u);
    if (status) {
        if (blockIdx.x == 0 && threadIdx.x == 0) hdr->status = status;
        return;
    }
    const int E = floor_log2_bits(mx);
    const int shift = B - E;
    const uint32_t st = blockIdx.x;
    const uint32_t base = st * SUPER;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    Pfx acc[kSubs];
#pragma unroll
    for (int q = 0; q < kSubs; ++q) acc[q] = Pfx{0ull, 0u, -1};
    if (vec && (uint64_t)base + SUPER <= n) {
        float4 v[NF4];
#pragma unroll
        for (int k = 0; k < NF4; ++k) v[k] = ld_stream_f4(p + base + 4 * (k * THREADS + threadIdx.x));
#pragma unroll
        for (int k = 0; k < NF4; ++k) {
            const int q = k / F4_PER_SUB;
            const int32_t e = (int32_t)(base + 4 * (k * THREADS + threadIdx.x));
            const float xs[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint64_t w = quantize(xs[u], shift);
                acc[q].W += w;
                acc[q].cnt += w != 0;
                if (w) acc[q].last = e + u;
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < NF4; ++k) {
            const int q = k / F4_PER_SUB;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint64_t e = (uint64_t)base + 4 * (k * THREADS + threadIdx.x) + u;
                if (e < n) {
                    const uint64_t w = quantize(p[e], shift);
                    acc[q].W += w;
                    acc[q].cnt += w != 0;
                    if (w) acc[q].last = (int32_t)e;
                }
            }
        }
    }
#pragma unroll
    for (int q = 0; q < kSubs; ++q) {
#pragma unroll
        for (int d = 16; d; d >>= 1) {
            const Pfx o = shfl_xor_pfx(acc[q], d);
            acc[q].W += o.W;
            acc[q].cnt += o.cnt;
            acc[q].last = max(acc[q].last, o.last);
        }
    }
    if (lane == 0) {
#pragma unroll
        for (int q = 0; q < kSubs; ++q) {
            s_w[q * NW + warp] = acc[q].W;
            s_c[q * NW + warp] = acc[q].cnt;
            s_l[q * NW + warp] = acc[q].last;
        }
    }
    __syncthreads();
    if (threadIdx.x < kSubs) {  // aggregate of K3 tile kSubs*st + q (a prefix after the scan)
        const int q = threadIdx.x;
        Pfx s{0ull, 0u, -1};
        for (int w = 0; w < NW; ++w) {
            s.W += s_w[q * NW + w];
            s.cnt += s_c[q * NW + w];
            s.last = max(s.last, s_l[q * NW + w]);
        }
        const uint32_t t3 = kSubs * st + q;
        if (t3 < nt) st_pfx(&excl[t3], s);
        __threadfence();
    }
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(&counters[kCtrDoneK2], 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;

    // ---- the last CTA: exclusive scan over all nt tile aggregates (in place)
    __threadfence();
    const uint32_t per = (nt + THREADS - 1) / THREADS;  // contiguous chunk per thread
    const uint32_t t0 = min(nt, threadIdx.x * per), t1 = min(nt, t0 + per);
    Pfx own{0ull, 0u, -1};
    for (uint32_t t = t0; t < t1; ++t) {
        const Pfx a = ld_pfx_cg(&excl[t]);
        own.W += a.W;
        own.cnt += a.cnt;
        own.last = max(own.last, a.last);
    }
    uint64_t w_ex, w_tot;
    uint32_t c_ex, c_tot;
    int32_t l_ex;
    block_scan3_excl<THREADS>(own.W, own.cnt, own.last, w_ex, c_ex, l_ex, w_tot, c_tot, s_w, s_c,
                              s_l);
    Pfx run{w_ex, c_ex, l_ex};
    for (uint32_t t = t0; t < t1; ++t) {
        const Pfx a = ld_pfx_cg(&excl[t]);
        st_pfx(&excl[t], run);
        run.W += a.W;
        run.cnt += a.cnt;
        run.last = max(run.last, a.last);
    }
    if (threadIdx.x == THREADS - 1) {  // whole-array totals -> header
        const uint64_t T = w_tot;
        rtf_header h;
        h.total = T;
        h.n_pos = c_tot;
        h.exponent = E;
        h.scale_bits = B;
        h.status = 0;
        h.reserved = 0;
        const uint32_t s = (uint32_t)__clzll((long long)T);  // T >= 1
        h.norm_shift = s;
        h.recip = reciprocal_of(T << s);
        *hdr = h;
        counters[kCtrDoneK2] = 0;  // reset-on-consume for the next build
    }
}

// ============================================================== K3: scan, normalise, phase-1 Alg. 1

struct BuildArgs {
    const float* p;
    uint32_t n, m;
    const Pfx* excl;    // exclusive prefix of every K3 tile (from K2)
    const rtf_header* hdr;
    rtf_node* nodes;
    int32_t* table;
    uint8_t* lam;       // global split levels (read by phase 2)
    int32_t* ob;        // global otherBounds, -1 when idle
    PendingLeaf* pend;  // 2 per tile
    RunChunk* queue;
    uint32_t* counters;
    uint32_t qcap;
    uint64_t* cdf;      // CDF mode only
    bool vec;
};

// Shared-memory arrays indexed by the local leaf index are padded with one slot
// every 8 entries: with blocked ownership (lane L works on leaves ~8L + r) and
// with strided access (consecutive leaves) both hit distinct banks.
__device__ __forceinline__ uint32_t pad8(uint32_t j) { return j + (j >> 3); }

template <int THREADS, int VPT>
__host__ __device__ constexpr size_t scan_build_padded() {
    return (size_t)THREADS * VPT + (size_t)THREADS * VPT / 8;
}

template <int THREADS, int VPT>
constexpr size_t scan_build_smem() {
    // p tile / otherBounds (i32), keys (u64), child0, child1 (i32), split levels (u8)
    return scan_build_padded<THREADS, VPT>() * (4 + 8 + 4 + 4) +
           ((scan_build_padded<THREADS, VPT>() + 15) & ~(size_t)15);
}

// Guide-table entries owed by leaf j (orig i) whose split level is a boundary:
// the anchor of the next non-empty cell and ~i for the empty cells between.
__device__ __noinline__ void table_runs(int32_t* __restrict__ table, uint32_t m,
                                        uint32_t* __restrict__ counters,
                                        RunChunk* __restrict__ queue, uint32_t qcap, uint32_t j,
                                        int32_t i, uint32_t cell, uint32_t cn) {
    if (cn < m) table[cn] = (int32_t)(j + 1);
    const uint32_t len = cn - cell - 1;
    if (!len) return;
    if (len <= kShortRun) {
        for (uint32_t g = cell + 1; g < cn; ++g) table[g] = ~i;
        return;
    }
    const uint32_t nch = (len + kChunk - 1) / kChunk;
    const uint32_t q = atomicAdd(&counters[kCtrQueue], nch);
    for (uint32_t c = 0; c < nch && q + c < qcap; ++c) {
        RunChunk rc;
        rc.start = cell + 1 + c * kChunk;
        rc.len = min(kChunk, len - c * kChunk);
        rc.value = ~i;
        rc.pad = 0;
        queue[q + c] = rc;
    }
}

// Persistent: each CTA walks tiles t = blockIdx.x, +gridDim.x, ...  The weights
// of a tile arrive in shared memory by a 1-D TMA bulk copy (issued as soon as
// the previous tile's otherBounds are flushed); two CTAs per SM overlap each
// other's copies and compute.  Each thread owns the compacted leaves of its VPT
// consecutive entries (blocked), so leaf references come from registers.
template <int THREADS, int VPT>
__global__ void __launch_bounds__(THREADS, 2) k_scan_build(BuildArgs A, uint32_t nt) {
    constexpr int TILE = THREADS * VPT;
    constexpr int NW = THREADS / 32;
    constexpr int P = (int)scan_build_padded<THREADS, VPT>();
    extern __shared__ __align__(128) unsigned char smem[];
    float* s_p = reinterpret_cast<float*>(smem);       // tile weights (TMA target)
    int32_t* s_ob = reinterpret_cast<int32_t*>(smem);  // ... then otherBounds
    uint64_t* s_key = reinterpret_cast<uint64_t*>(smem + 4 * P);
    int32_t* s_c0 = reinterpret_cast<int32_t*>(s_key + P);
    int32_t* s_c1 = s_c0 + P;
    uint8_t* s_lam = reinterpret_cast<uint8_t*>(s_c1 + P);
    __shared__ __align__(8) uint64_t s_bar;
    __shared__ uint64_t s_w[2 * NW];
    __shared__ uint32_t s_c[2 * NW];
    __shared__ int32_t s_l[2 * NW];
    __shared__ uint64_t s_key_after;

    const rtf_header* hdr = A.hdr;
    if (hdr->status) return;  // poisoned build: no-op
    const uint64_t T = hdr->total;
    Norm nm;
    nm.s = hdr->norm_shift;
    nm.d = T << nm.s;
    nm.v = hdr->recip;
    const int shift = hdr->scale_bits - hdr->exponent;
    const uint32_t m = A.m, n = A.n;
    const bool tma = A.vec;
    const uint32_t tid = threadIdx.x;
    auto tma_tile = [&](uint32_t t) { return tma && t < nt && (uint64_t)(t + 1) * TILE <= n; };
    if (tid == 0) {
        mbar_init(&s_bar, 1);
        fence_proxy_async_smem();
        if (tma_tile(blockIdx.x)) {
            mbar_arrive_expect_tx(&s_bar, TILE * 4);
            tma_load_1d(s_p, A.p + (size_t)blockIdx.x * TILE, TILE * 4, &s_bar);
        }
    }
    __syncthreads();

    Pfx pre_next = A.excl[blockIdx.x < nt ? blockIdx.x : 0];
    uint32_t phase = 0;
    for (uint32_t t = blockIdx.x; t < nt; t += gridDim.x) {
        const Pfx pre = pre_next;
        if (t + gridDim.x < nt) pre_next = A.excl[t + gridDim.x];
        const uint32_t first = t * TILE + tid * VPT;

        // ---- (0) weights of this thread's VPT consecutive entries
        float x[VPT];
        if (tma_tile(t)) {
            mbar_wait(&s_bar, phase);
            phase ^= 1u;
#pragma unroll
            for (int k = 0; k < VPT; k += 4) {
                const float4 v = *reinterpret_cast<const float4*>(s_p + tid * VPT + k);
                x[k] = v.x;
                x[k + 1] = v.y;
                x[k + 2] = v.z;
                x[k + 3] = v.w;
            }
        } else {
            load_tile<VPT>(A.p, first, n, A.vec, x);
        }
        uint64_t w[VPT];
        uint64_t tw = 0;
        uint32_t tc = 0, posmask = 0;
        int32_t tl = -1;
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
            w[k] = quantize(x[k], shift);
            tw += w[k];
            if (w[k]) {
                ++tc;
                posmask |= 1u << k;
                tl = (int32_t)(first + k);
            }
        }
        // ---- (1) block scan (its barriers also retire every read of s_p);
        // one exact division per positive entry
        uint64_t w_ex, w_tot;
        uint32_t c_ex, cnt;
        int32_t l_ex;
        block_scan3_excl<THREADS>(tw, tc, tl, w_ex, c_ex, l_ex, w_tot, cnt, s_w, s_c, s_l);
        const uint32_t j0 = pre.cnt;  // global index of the tile's first leaf
        {
            // Node records start as anchors: child0 = ~orig(j-1) (Fig. 6 caption
            // P:1276-1277; j = 0 -> ~orig(0)); internal nodes overwrite it in Alg. 1.
            int32_t prevo = l_ex >= 0 ? l_ex : (j0 ? pre.last : -1);
            uint64_t W = pre.W + w_ex;
            uint32_t jl = c_ex;
#pragma unroll
            for (int k = 0; k < VPT; ++k) {
                if (w[k]) {
                    const int32_t i = (int32_t)(first + k);
                    const uint32_t q = pad8(jl);
                    s_key[q] = fixed_point(W, nm);
                    s_c0[q] = ~(prevo >= 0 ? prevo : i);
                    s_c1[q] = INT32_MIN;
                    s_ob[q] = -1;
                    prevo = i;
                    ++jl;
                }
                W += w[k];
            }
        }
        // the tile's first and last leaf stay pending for phase 2 (K4)
        if (tc && c_ex == 0)
            A.pend[2 * t] = PendingLeaf{(int32_t)j0, ~(int32_t)(first + __ffs(posmask) - 1)};
        if (tc && c_ex + tc == cnt)
            A.pend[2 * t + 1] = cnt >= 2 ? PendingLeaf{(int32_t)(j0 + cnt - 1), ~tl}
                                         : PendingLeaf{-1, 0};
        if (cnt == 0 && tid == 0) A.pend[2 * t] = A.pend[2 * t + 1] = PendingLeaf{-1, 0};
        if (tid == THREADS - 1) {  // key of the first leaf after the tile (or "1")
            const uint64_t We = pre.W + w_tot;
            s_key_after = (We == T) ? kOne63 : fixed_point(We, nm);
        }
        __syncthreads();

        // ---- (2) own leaves: cell, split level, guide table
        {
            const uint64_t key_after = s_key_after;
            uint32_t jl = c_ex;
            uint64_t key = tc ? s_key[pad8(jl)] : 0ull;
            for (uint32_t mask = posmask; mask; mask &= mask - 1, ++jl) {
                const uint64_t kn = (jl + 1 < cnt) ? s_key[pad8(jl + 1)] : key_after;
                const uint32_t cell = cell_of(key, m);
                const uint32_t cn = (kn == kOne63) ? m : cell_of(kn, m);
                const uint32_t lam = (cn != cell) ? kLamBoundary : split_level(key, kn);
                s_lam[pad8(jl)] = (uint8_t)lam;
                const uint32_t j = j0 + jl;
                if (j == 0) A.table[0] = 0;
                if (lam == kLamBoundary)
                    table_runs(A.table, m, A.counters, A.queue, A.qcap, j,
                               (int32_t)(first + __ffs(mask) - 1), cell, cn);
                key = kn;
            }
        }
        __syncthreads();

        // ---- (3) phase 1: Alg. 1 for the tile's interior leaves 1..cnt-2 with
        // shared-memory atomicExch.  A range that would contain the pending
        // first/last leaf can never complete here, so every range stays in
        // [1, cnt-2] and every parent slot in [1, cnt-1] -- inside the tile.
        // Each lane walks its own leaves back to back; a merge re-reads only the
        // split level on the side that moved.  A cell root (both neighbours out
        // of cell, lambda = 64 on both sides) is the right child of its anchor
        // lo and needs no exchange.
        {
            uint32_t mask = posmask;
            uint32_t l = c_ex;
            bool active = false;
            int32_t lo = 0, hi = 0, node = 0;
            uint32_t lamL = 0, lamR = 0;
            while (true) {
                while (!active && mask) {
                    const uint32_t k = __ffs(mask) - 1;
                    mask &= mask - 1;
                    const uint32_t ll = l++;
                    if (ll >= 1 && ll + 1 < cnt) {
                        active = true;
                        lo = hi = (int32_t)ll;
                        node = ~(int32_t)(first + k);
                        lamL = s_lam[pad8(ll - 1)];
                        lamR = s_lam[pad8(ll)];
                    }
                }
                if (!__any_sync(0xffffffffu, active)) break;
                if (active) {
                    const bool right = lamL <= lamR;  // Alg. 1: child 1 unless left is farther
                    const bool root = (lamL & lamR & kLamBoundary) != 0;
                    const int32_t parent = right ? lo : hi + 1;
                    const uint32_t q = pad8((uint32_t)parent);
                    (right ? s_c1 : s_c0)[q] = node;
                    const int32_t other = root ? -1 : atomicExch(&s_ob[q], right ? hi : lo);
                    active = other >= 0;  // first to arrive (or a root): stop
                    if (active) {
                        s_ob[q] = -1;  // reset-on-consume
                        const uint32_t lv = s_lam[pad8(right ? other - 1 : other)];
                        if (right) {
                            lo = other;
                            lamL = lv;
                        } else {
                            hi = other;
                            lamR = lv;
                        }
                        node = (int32_t)(j0 + parent);
                    }
                }
            }
        }
        __syncthreads();

        // ---- (4) flush: leftover deposits first, then the next tile's TMA copy
        // can reuse the buffer while records (coalesced 16 B) and split levels go out
        for (uint32_t l = 1 + tid; l < cnt; l += THREADS) {
            const int32_t o = s_ob[pad8(l)];
            if (o >= 0) A.ob[j0 + l] = (int32_t)j0 + o;
        }
        __syncthreads();
        if (tid == 0 && tma_tile(t + gridDim.x)) {
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(&s_bar, TILE * 4);
            tma_load_1d(s_p, A.p + (size_t)(t + gridDim.x) * TILE, TILE * 4, &s_bar);
        }
        {
            uint4* gnode = reinterpret_cast<uint4*>(A.nodes + j0);
            for (uint32_t l = tid; l < cnt; l += THREADS) {
                const uint32_t q = pad8(l);
                const uint64_t key = s_key[q];
                gnode[l] = make_uint4((uint32_t)key, (uint32_t)(key >> 32), (uint32_t)s_c0[q],
                                      (uint32_t)s_c1[q]);
                A.lam[j0 + l] = s_lam[q];
            }
        }
        __syncthreads();  // keys, children and split levels are free for the next tile
    }
}

// Baseline CDF over all entries: K[i] = floor(W_i 2^63 / T) (zeros included).
template <int THREADS, int VPT>
__global__ void __launch_bounds__(THREADS) k_cdf(BuildArgs A) {
    __shared__ uint64_t s_w[2 * (THREADS / 32)];
    __shared__ uint32_t s_c[2 * (THREADS / 32)];
    const rtf_header* hdr = A.hdr;
    if (hdr->status) return;
    const uint64_t T = hdr->total;
    Norm nm;
    nm.s = hdr->norm_shift;
    nm.d = T << nm.s;
    nm.v = hdr->recip;
    const int shift = hdr->scale_bits - hdr->exponent;
    const uint32_t tile = blockIdx.x;
    const Pfx pre = A.excl[tile];
    const uint32_t first = tile * THREADS * VPT + threadIdx.x * VPT;
    float x[VPT];
    load_tile<VPT>(A.p, first, A.n, A.vec, x);
    uint64_t w[VPT];
    uint64_t tw = 0;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
        w[k] = quantize(x[k], shift);
        tw += w[k];
    }
    uint64_t w_ex, w_tot;
    uint32_t c_ex, cnt;
    block_scan_excl<THREADS>(tw, 0u, w_ex, c_ex, w_tot, cnt, s_w, s_c);
    uint64_t W = pre.W + w_ex;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
        if (first + k < A.n) A.cdf[first + k] = (W == T) ? kOne63 : fixed_point(W, nm);
        W += w[k];
    }
}

// ============================================================== K4: cross-tile Alg. 1 + long table runs

__global__ void __launch_bounds__(256) k_cross_tile(BuildArgs A, uint32_t npend,
                                                    uint32_t walker_blocks) {
    if (A.hdr->status) return;
    if (blockIdx.x < walker_blocks) {
        const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
        if (t >= npend) return;
        const PendingLeaf pl = A.pend[t];
        if (pl.j < 0) return;
        int32_t lo = pl.j, hi = pl.j, node = pl.ref;
        const uint8_t* __restrict__ lam = A.lam;  // read-only in this kernel
        uint32_t lamL = lo ? __ldg(lam + lo - 1) : kLamBoundary;
        uint32_t lamR = __ldg(lam + hi);
        while (true) {
            const bool right = lamL <= lamR;
            const int32_t parent = right ? lo : hi + 1;
            A.nodes[parent].child[right ? 1 : 0] = node;
            if (lamL & lamR & kLamBoundary) break;  // cell root: right child of its anchor
            const int32_t other = atomicExch(&A.ob[parent], right ? hi : lo);
            if (other < 0) break;
            A.ob[parent] = -1;
            // a sibling's bound always extends the range; anything else means an
            // uninitialised workspace -- stop instead of wandering
            if (right ? other >= lo : other <= hi) break;
            if (right) {
                lo = other;
                lamL = lo ? __ldg(lam + lo - 1) : kLamBoundary;
            } else {
                hi = other;
                lamR = __ldg(lam + hi);
            }
            node = parent;
        }
        return;
    }
    // long empty-cell runs of the guide table: one warp per chunk
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x - walker_blocks) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const uint32_t nwarps = (gridDim.x - walker_blocks) * (blockDim.x >> 5);
    const uint32_t nq = min(A.counters[kCtrQueue], A.qcap);
    for (uint32_t q = warp; q < nq; q += nwarps) {
        const RunChunk rc = A.queue[q];
        for (uint32_t g = lane; g < rc.len; g += 32) A.table[rc.start + g] = rc.value;
    }
}

// ============================================================== host-side launch

struct TileCfg {
    int threads, vpt;
};

static inline TileCfg tile_cfg(uint32_t flags) {
    return (flags & RTF_BUILD_SMALL_TILES) ? TileCfg{64, 4} : TileCfg{512, 8};
}

uint32_t build_tile_size(uint32_t flags) {
    const TileCfg c = tile_cfg(flags);
    return (uint32_t)(c.threads * c.vpt);
}

uint32_t build_queue_capacity(uint32_t m) { return m / 32u + m / kChunk + 64u; }

size_t build_workspace_layout(uint32_t n, uint32_t m, uint32_t flags, WsLayout* L) {
    const uint32_t tile = build_tile_size(flags);
    const uint32_t nt = (uint32_t)(((uint64_t)n + tile - 1) / tile);
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off += (bytes + 255) & ~(size_t)255;
        return o;
    };
    L->nt = nt;
    L->maxpart = take(sizeof(uint32_t) * 2 * kMaxScaleBlocks + 16);
    L->counters = take(64);
    L->excl = take(sizeof(Pfx) * (size_t)nt);
    L->pend = take(sizeof(PendingLeaf) * 2 * (size_t)nt);
    L->ob = take(sizeof(int32_t) * (size_t)n);
    L->lam = take((size_t)n);
    L->qcap = build_queue_capacity(m);
    L->queue = take(sizeof(RunChunk) * (size_t)L->qcap);
    L->total = off;
    return off;
}

static int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
            sms <= 0)
            sms = 148;
    }
    return sms;
}

template <int THREADS, int VPT>
static cudaError_t launch_pipeline(const float* p, uint32_t n, uint32_t m, rtf_header* hdr,
                                   rtf_node* nodes, int32_t* table, uint64_t* cdf,
                                   unsigned char* ws, const WsLayout& L, cudaStream_t st,
                                   int* launches) {
    const bool vec = ((uintptr_t)p & 15u) == 0;
    const int B = 62 - ceil_log2_u32(n);
    const uint32_t nt = L.nt, nst = (nt + kSubs - 1) / kSubs;
    uint32_t* maxpart = reinterpret_cast<uint32_t*>(ws + L.maxpart);
    uint32_t* scale_word = maxpart + 2 * kMaxScaleBlocks;
    uint32_t* counters = reinterpret_cast<uint32_t*>(ws + L.counters);
    Pfx* excl = reinterpret_cast<Pfx*>(ws + L.excl);

    // K1: 256-thread blocks, ~32 float4 per thread, at most 8 blocks per SM
    const uint32_t nb1 = (uint32_t)std::max<uint64_t>(
        1, std::min<uint64_t>(kMaxScaleBlocks, ((uint64_t)n + 32767) / 32768));
    k_scale<<<nb1, 256, 0, st>>>(p, n, maxpart, counters, scale_word, vec);
    ++*launches;
    // K2: super-tiles of kSubs K3 tiles
    k_tile_totals<THREADS, VPT><<<nst, THREADS, 0, st>>>(p, n, B, scale_word, counters, excl,
                                                         hdr, nst, nt, vec);
    ++*launches;
    BuildArgs A;
    A.p = p;
    A.n = n;
    A.m = m;
    A.excl = excl;
    A.hdr = hdr;
    A.nodes = nodes;
    A.table = table;
    A.lam = reinterpret_cast<uint8_t*>(ws + L.lam);
    A.ob = reinterpret_cast<int32_t*>(ws + L.ob);
    A.pend = reinterpret_cast<PendingLeaf*>(ws + L.pend);
    A.queue = reinterpret_cast<RunChunk*>(ws + L.queue);
    A.counters = counters;
    A.qcap = L.qcap;
    A.cdf = cdf;
    A.vec = vec;
    if (cdf) {
        k_cdf<THREADS, VPT><<<nt, THREADS, 0, st>>>(A);
        ++*launches;
        return cudaGetLastError();
    }
    // K3: persistent, 2 CTAs per SM
    const size_t smem = scan_build_smem<THREADS, VPT>();
    static bool attr_set = false;  // per instantiation
    if (!attr_set) {
        const cudaError_t e = cudaFuncSetAttribute(k_scan_build<THREADS, VPT>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   (int)smem);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    const uint32_t grid3 = std::min<uint32_t>(nt, 2u * (uint32_t)num_sms());
    k_scan_build<THREADS, VPT><<<grid3, THREADS, smem, st>>>(A, nt);
    ++*launches;
    // K4
    const uint32_t npend = 2 * nt;
    const uint32_t walker_blocks = (npend + 255) / 256;
    const uint32_t fill_blocks =
        std::max<uint32_t>(1u, std::min<uint32_t>(148u * 4u, m / 8192u + 1u));
    k_cross_tile<<<walker_blocks + fill_blocks, 256, 0, st>>>(A, npend, walker_blocks);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_build(const float* p, uint32_t n, uint32_t m, uint32_t flags, rtf_header* hdr,
                         rtf_node* nodes, int32_t* table, uint64_t* cdf, void* ws,
                         const WsLayout& L, cudaStream_t st, int* launches) {
    unsigned char* w = reinterpret_cast<unsigned char*>(ws);
    if (flags & RTF_BUILD_SMALL_TILES)
        return launch_pipeline<64, 4>(p, n, m, hdr, nodes, table, cdf, w, L, st, launches);
    return launch_pipeline<512, 8>(p, n, m, hdr, nodes, table, cdf, w, L, st, launches);
}

}  // namespace rtf
