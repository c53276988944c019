// rtf_build.cu -- the forest build: 4 kernels on the caller's stream.
//
//   K1 k_scale        read p once: max weight bits (for E), NaN/Inf/negative flags;
//                     resets the per-build look-back flags and counters.
//   K2 k_tile_totals  per tile: quantise (w), sum W, count positives, last
//                     positive index; decoupled look-back gives every tile its
//                     inclusive prefix (the parallel prefix sum of P:239);
//                     the last tile publishes T, n' and the reciprocal of T.
//   K3 k_scan_build   per tile: block scan + tile prefix -> W_j, compaction,
//                     key_j, cell, split level lambda_j; guide-table runs
//                     (P:1333-1335); Alg. 1 for every leaf of the
//                     tile except its first and last ("phase 1", shared-memory
//                     atomics); coalesced flush of the 16-B node records.
//   K4 k_cross_tile   "phase 2": the <= 2 pending edge leaves per tile continue
//                     Alg. 1 with global atomicExch, consuming the deposits the
//                     tiles flushed; plus the long empty-cell runs of the table.
// The result bytes do not depend on the schedule.
#include <cstdio>

#include "rtf_device.cuh"
#include "rtf_internal.h"

namespace rtf {

constexpr uint32_t kFlagAggregate = 1, kFlagInclusive = 2;
constexpr uint32_t kShortRun = 32;    // empty-cell runs up to this length: written in place
constexpr uint32_t kChunk = 2048;     // longer runs: queued in chunks of this many cells

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
                                               uint32_t* __restrict__ tile_flags, uint32_t nt,
                                               bool vec) {
    const uint32_t gt = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t gs = gridDim.x * blockDim.x;
    for (uint32_t t = gt; t < nt; t += gs) tile_flags[t] = 0;
    if (gt == 0) {
        counters[0] = 0;  // tile ticket
        counters[1] = 0;  // run-chunk queue length
    }
    uint32_t mx = 0, fl = 0;
    auto visit = [&](float x) {
        uint32_t b = __float_as_uint(x);
        if (x != x) fl |= RTF_DATA_NAN;
        else if (fabsf(x) == __int_as_float(0x7f800000)) fl |= RTF_DATA_INF;
        else if (x < 0.0f) fl |= RTF_DATA_NEG;
        else if (x > 0.0f) mx = max(mx, b);
    };
    if (vec) {
        const uint32_t n4 = n >> 2;
        for (uint32_t q = gt; q < n4; q += gs) {
            float4 v = ld_stream_f4(p + 4ull * q);
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
    }
}

// Reduce K1's per-block partials (every K2 block does this redundantly; <= 2 KB).
template <int THREADS>
__device__ __forceinline__ void reduce_partials(const uint32_t* maxpart, uint32_t nparts,
                                                uint32_t& mx, uint32_t& fl, uint32_t* s_red) {
    mx = 0;
    fl = 0;
    for (uint32_t i = threadIdx.x; i < nparts; i += THREADS) {
        mx = max(mx, maxpart[2 * i]);
        fl |= maxpart[2 * i + 1];
    }
    for (int d = 16; d; d >>= 1) {
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, d));
        fl |= __shfl_xor_sync(0xffffffffu, fl, d);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        s_red[2 * warp] = mx;
        s_red[2 * warp + 1] = fl;
    }
    __syncthreads();
    mx = 0;
    fl = 0;
    for (int w = 0; w < THREADS / 32; ++w) {
        mx = max(mx, s_red[2 * w]);
        fl |= s_red[2 * w + 1];
    }
}

// Load VPT consecutive weights of this thread (blocked layout) with bounds.
template <int VPT>
__device__ __forceinline__ void load_tile(const float* __restrict__ p, uint64_t first, uint32_t n,
                                          bool vec, float (&x)[VPT]) {
    if (vec && first + VPT <= n) {
#pragma unroll
        for (int k = 0; k < VPT; k += 4) {
            float4 v = ld_stream_f4(p + first + k);
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

// ============================================================== K2: tile totals + look-back

template <int THREADS, int VPT>
__global__ void __launch_bounds__(THREADS)
    k_tile_totals(const float* __restrict__ p, uint32_t n, int B, const uint32_t* maxpart,
                  uint32_t nparts, uint32_t* counters, uint32_t* tile_flags, Pfx* agg, Pfx* inc,
                  rtf_header* hdr, uint32_t nt, bool vec) {
    constexpr int TILE = THREADS * VPT;
    __shared__ uint32_t s_tile;
    __shared__ uint32_t s_red[2 * (THREADS / 32)];
    __shared__ uint64_t s_w[THREADS / 32];
    __shared__ uint32_t s_c[THREADS / 32];
    __shared__ int32_t s_l[THREADS / 32];
    if (threadIdx.x == 0) s_tile = atomicAdd(&counters[0], 1u);
    uint32_t mx, fl;
    reduce_partials<THREADS>(maxpart, nparts, mx, fl, s_red);  // contains __syncthreads
    const uint32_t tile = s_tile;
    uint32_t status = fl | (mx == 0 ? RTF_DATA_ALLZERO : 0u);
    if (status) {
        if (tile == 0 && threadIdx.x == 0) hdr->status = status;
        return;
    }
    const int E = floor_log2_bits(mx);
    const int shift = B - E;
    const uint64_t first = (uint64_t)tile * TILE + (uint64_t)threadIdx.x * VPT;
    float x[VPT];
    load_tile<VPT>(p, first, n, vec, x);
    uint64_t tw = 0;
    uint32_t tc = 0;
    int32_t tl = -1;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
        uint64_t w = quantize(x[k], shift);
        tw += w;
        tc += w != 0;
        if (w) tl = (int32_t)(first + k);
    }
    // block reduction (sum, sum, max)
    for (int d = 16; d; d >>= 1) {
        tw += __shfl_xor_sync(0xffffffffu, tw, d);
        tc += __shfl_xor_sync(0xffffffffu, tc, d);
        tl = max(tl, __shfl_xor_sync(0xffffffffu, tl, d));
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        s_w[warp] = tw;
        s_c[warp] = tc;
        s_l[warp] = tl;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    Pfx a{0ull, 0u, -1};
    for (int w = 0; w < THREADS / 32; ++w) {
        a.W += s_w[w];
        a.cnt += s_c[w];
        a.last = max(a.last, s_l[w]);
    }
    // decoupled look-back (single thread; tiles are ticketed in order, so every
    // predecessor is resident or finished)
    Pfx incl = a;
    if (tile == 0) {
        st_pfx(&inc[0], a);
        st_release_u32(&tile_flags[0], kFlagInclusive);
    } else {
        st_pfx(&agg[tile], a);
        st_release_u32(&tile_flags[tile], kFlagAggregate);
        Pfx acc{0ull, 0u, -1};
        int t = (int)tile - 1;
        while (true) {
            uint32_t f;
            while ((f = ld_acquire_u32(&tile_flags[t])) == 0) {
            }
            Pfx v = ld_pfx_cg(f == kFlagInclusive ? &inc[t] : &agg[t]);
            acc = combine(v, acc);
            if (f == kFlagInclusive) break;
            --t;
        }
        incl = combine(acc, a);
        st_pfx(&inc[tile], incl);
        st_release_u32(&tile_flags[tile], kFlagInclusive);
    }
    if (tile == nt - 1) {  // whole-array totals -> header
        const uint64_t T = incl.W;
        rtf_header h;
        h.total = T;
        h.n_pos = incl.cnt;
        h.exponent = E;
        h.scale_bits = B;
        h.status = 0;
        h.reserved = 0;
        const uint32_t s = (uint32_t)__clzll((long long)T);  // T >= 1
        h.norm_shift = s;
        h.recip = reciprocal_of(T << s);
        *hdr = h;
    }
}

// ============================================================== K3: scan, normalise, phase-1 Alg. 1

struct BuildArgs {
    const float* p;
    uint32_t n, m;
    const Pfx* inc;
    const rtf_header* hdr;
    rtf_node* nodes;
    int32_t* table;
    uint8_t* lam;         // global split levels (read by phase 2)
    int32_t* ob;          // global otherBounds, -1 when idle
    PendingLeaf* pend;    // 2 per tile
    RunChunk* queue;
    uint32_t* counters;
    uint32_t qcap;
    uint64_t* cdf;        // CDF mode only
    bool vec;
};

struct __align__(16) SRec {
    uint64_t key;
    int32_t c0, c1;
};

template <int THREADS, int VPT>
constexpr size_t scan_build_smem() {
    return (size_t)THREADS * VPT * (sizeof(SRec) + 4 + 4 + 1);
}

template <int THREADS, int VPT, bool CDF_MODE>
__global__ void __launch_bounds__(THREADS) k_scan_build(BuildArgs A) {
    constexpr int TILE = THREADS * VPT;
    extern __shared__ __align__(16) unsigned char smem[];
    SRec* s_rec = reinterpret_cast<SRec*>(smem);
    int32_t* s_orig = reinterpret_cast<int32_t*>(s_rec + TILE);
    int32_t* s_ob = s_orig + TILE;
    uint8_t* s_lam = reinterpret_cast<uint8_t*>(s_ob + TILE);
    __shared__ uint64_t s_w[2 * (THREADS / 32)];
    __shared__ uint32_t s_c[2 * (THREADS / 32)];

    const rtf_header* hdr = A.hdr;
    if (hdr->status) return;  // poisoned build: no-op
    const uint32_t tile = blockIdx.x;
    const uint64_t T = hdr->total;
    Norm nm;
    nm.s = hdr->norm_shift;
    nm.d = T << nm.s;
    nm.v = hdr->recip;
    const int shift = hdr->scale_bits - hdr->exponent;
    const uint32_t m = A.m;
    Pfx pre{0ull, 0u, -1};
    if (tile) pre = A.inc[tile - 1];

    const uint64_t first = (uint64_t)tile * TILE + (uint64_t)threadIdx.x * VPT;
    float x[VPT];
    load_tile<VPT>(A.p, first, A.n, A.vec, x);
    uint64_t w[VPT];
    uint64_t tw = 0;
    uint32_t tc = 0;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
        w[k] = quantize(x[k], shift);
        tw += w[k];
        tc += w[k] != 0;
    }
    uint64_t w_ex, w_tot;
    uint32_t c_ex, cnt;
    block_scan_excl<THREADS>(tw, tc, w_ex, c_ex, w_tot, cnt, s_w, s_c);
    uint64_t W = pre.W + w_ex;

    if (CDF_MODE) {  // baseline: K[i] = floor(W_i 2^63 / T) for every entry
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
            if (first + k < A.n) A.cdf[first + k] = (W == T) ? kOne63 : fixed_point(W, nm);
            W += w[k];
        }
        return;
    }

    const uint32_t j0 = pre.cnt;  // global index of the tile's first leaf
    uint32_t jl = c_ex;           // local compacted index
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
        if (!w[k]) continue;
        const int32_t i = (int32_t)(first + k);
        const uint32_t j = j0 + jl;
        const uint64_t key = fixed_point(W, nm);
        const uint64_t Wn = W + w[k];
        const bool last = (Wn == T);
        const uint64_t kn = last ? kOne63 : fixed_point(Wn, nm);
        const uint32_t cell = cell_of(key, m);
        const uint32_t cn = last ? m : cell_of(kn, m);
        const uint32_t lam = (cn != cell) ? kLamBoundary : split_level(key, kn);
        s_rec[jl].key = key;
        s_lam[jl] = (uint8_t)lam;
        s_orig[jl] = i;
        // guide table: anchors of non-empty cells, ~i for the
        // empty cells this interval overlaps entirely
        if (j == 0) A.table[0] = 0;
        if (lam == kLamBoundary) {
            if (cn < m) A.table[cn] = (int32_t)(j + 1);
            const uint32_t len = cn - cell - 1;
            if (len && len <= kShortRun) {
                for (uint32_t g = cell + 1; g < cn; ++g) A.table[g] = ~i;
            } else if (len) {
                const uint32_t nch = (len + kChunk - 1) / kChunk;
                const uint32_t q = atomicAdd(&A.counters[1], nch);
                for (uint32_t c = 0; c < nch && q + c < A.qcap; ++c) {
                    RunChunk rc;
                    rc.start = cell + 1 + c * kChunk;
                    rc.len = min(kChunk, len - c * kChunk);
                    rc.value = ~i;
                    rc.pad = 0;
                    A.queue[q + c] = rc;
                }
            }
        }
        W = Wn;
        ++jl;
    }
    __syncthreads();

    // node records start as anchors: child0 = ~orig(j-1) (Fig. 6 caption
    // P:1276-1277; j = 0 -> ~orig(0)); internal nodes overwrite it below.
    const int32_t prev_orig = j0 ? pre.last : s_orig[0];
    for (uint32_t l = threadIdx.x; l < cnt; l += THREADS) {
        s_rec[l].c0 = ~(l ? s_orig[l - 1] : prev_orig);
        s_rec[l].c1 = INT32_MIN;
        s_ob[l] = -1;
    }
    __syncthreads();

    // phase 1: Alg. 1 for the tile's interior leaves 1..cnt-2 with shared-memory
    // atomics.  A range that would contain the pending first/last leaf can never
    // complete here, so every range stays in [1, cnt-2] and every parent slot in
    // [1, cnt-1] -- all inside the tile.
    for (uint32_t l = 1 + threadIdx.x; l + 1 < cnt; l += THREADS) {
        int32_t lo = (int32_t)l, hi = (int32_t)l;
        int32_t node = ~s_orig[l];
        while (true) {
            const uint32_t lamL = s_lam[lo - 1], lamR = s_lam[hi];
            if (lamL == kLamBoundary && lamR == kLamBoundary) {  // cell root -> anchor lo
                s_rec[lo].c1 = node;
                break;
            }
            const int c = lamL > lamR ? 0 : 1;
            const int32_t parent = c ? lo : hi + 1;
            if (c) s_rec[parent].c1 = node;
            else s_rec[parent].c0 = node;
            const int32_t other = atomicExch(&s_ob[parent], c ? hi : lo);
            if (other < 0) break;  // first to arrive: the sibling continues
            s_ob[parent] = -1;     // reset-on-consume
            if (c) lo = other;
            else hi = other;
            node = (int32_t)(j0 + parent);
        }
    }
    __syncthreads();

    // flush: records (coalesced 16 B), split levels, pending deposits, edge leaves
    uint4* gnode = reinterpret_cast<uint4*>(A.nodes + j0);
    const uint4* snode = reinterpret_cast<const uint4*>(s_rec);
    for (uint32_t l = threadIdx.x; l < cnt; l += THREADS) {
        gnode[l] = snode[l];
        A.lam[j0 + l] = s_lam[l];
        if (l >= 1 && s_ob[l] >= 0) A.ob[j0 + l] = (int32_t)j0 + s_ob[l];
    }
    if (threadIdx.x == 0) {
        PendingLeaf a{-1, 0}, b{-1, 0};
        if (cnt >= 1) a = PendingLeaf{(int32_t)j0, ~s_orig[0]};
        if (cnt >= 2) b = PendingLeaf{(int32_t)(j0 + cnt - 1), ~s_orig[cnt - 1]};
        A.pend[2 * tile] = a;
        A.pend[2 * tile + 1] = b;
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
        const volatile uint8_t* lam = A.lam;
        while (true) {
            const uint32_t lamL = lo ? lam[lo - 1] : kLamBoundary;
            const uint32_t lamR = lam[hi];
            if (lamL == kLamBoundary && lamR == kLamBoundary) {
                A.nodes[lo].child[1] = node;
                break;
            }
            const int c = lamL > lamR ? 0 : 1;
            const int32_t parent = c ? lo : hi + 1;
            A.nodes[parent].child[c] = node;
            const int32_t other = atomicExch(&A.ob[parent], c ? hi : lo);
            if (other < 0) break;
            A.ob[parent] = -1;
            if (c) lo = other;
            else hi = other;
            node = parent;
        }
        return;
    }
    // long empty-cell runs of the guide table: one warp per chunk
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x - walker_blocks) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const uint32_t nwarps = (gridDim.x - walker_blocks) * (blockDim.x >> 5);
    const uint32_t nq = min(A.counters[1], A.qcap);
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
    return (flags & RTF_BUILD_SMALL_TILES) ? TileCfg{64, 2} : TileCfg{512, 8};
}

uint32_t build_tile_size(uint32_t flags) {
    TileCfg c = tile_cfg(flags);
    return (uint32_t)(c.threads * c.vpt);
}

uint32_t build_queue_capacity(uint32_t m) { return m / 32u + m / kChunk + 64u; }

size_t build_workspace_layout(uint32_t n, uint32_t m, uint32_t flags, WsLayout* L) {
    const uint32_t tile = build_tile_size(flags);
    const uint32_t nt = (uint32_t)(((uint64_t)n + tile - 1) / tile);
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += (bytes + 255) & ~(size_t)255;
        return o;
    };
    L->nt = nt;
    L->maxpart = take(sizeof(uint32_t) * 2 * kMaxScaleBlocks);
    L->counters = take(64);
    L->tile_flags = take(sizeof(uint32_t) * nt);
    L->agg = take(sizeof(Pfx) * nt);
    L->inc = take(sizeof(Pfx) * nt);
    L->pend = take(sizeof(PendingLeaf) * 2 * (size_t)nt);
    L->ob = take(sizeof(int32_t) * (size_t)n);
    L->lam = take((size_t)n);
    L->qcap = build_queue_capacity(m);
    L->queue = take(sizeof(RunChunk) * (size_t)L->qcap);
    L->total = off;
    return off;
}

template <int THREADS, int VPT>
static cudaError_t launch_pipeline(const float* p, uint32_t n, uint32_t m, rtf_header* hdr,
                                   rtf_node* nodes, int32_t* table, uint64_t* cdf,
                                   unsigned char* ws, const WsLayout& L, cudaStream_t st,
                                   int* launches) {
    const bool vec = ((uintptr_t)p & 15u) == 0;
    const int B = 62 - ceil_log2_u32(n);
    uint32_t* maxpart = reinterpret_cast<uint32_t*>(ws + L.maxpart);
    uint32_t* counters = reinterpret_cast<uint32_t*>(ws + L.counters);
    uint32_t* tile_flags = reinterpret_cast<uint32_t*>(ws + L.tile_flags);
    Pfx* agg = reinterpret_cast<Pfx*>(ws + L.agg);
    Pfx* inc = reinterpret_cast<Pfx*>(ws + L.inc);

    // K1
    const uint32_t nb1 = (uint32_t)std::min<uint64_t>(kMaxScaleBlocks, ((uint64_t)n + 4095) / 4096);
    k_scale<<<nb1, 256, 0, st>>>(p, n, maxpart, counters, tile_flags, L.nt, vec);
    ++*launches;
    // K2
    k_tile_totals<THREADS, VPT><<<L.nt, THREADS, 0, st>>>(p, n, B, maxpart, nb1, counters,
                                                          tile_flags, agg, inc, hdr, L.nt, vec);
    ++*launches;
    // K3
    BuildArgs A;
    A.p = p;
    A.n = n;
    A.m = m;
    A.inc = inc;
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
    const size_t smem = scan_build_smem<THREADS, VPT>();
    if (cdf) {
        k_scan_build<THREADS, VPT, true><<<L.nt, THREADS, 0, st>>>(A);
        ++*launches;
        return cudaGetLastError();
    }
    static bool attr_set = false;  // per instantiation
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(k_scan_build<THREADS, VPT, false>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    k_scan_build<THREADS, VPT, false><<<L.nt, THREADS, smem, st>>>(A);
    ++*launches;
    // K4
    const uint32_t npend = 2 * L.nt;
    const uint32_t walker_blocks = (npend + 255) / 256;
    const uint32_t fill_blocks = std::max<uint32_t>(1u, std::min<uint32_t>(148u * 4u, m / 8192u + 1u));
    k_cross_tile<<<walker_blocks + fill_blocks, 256, 0, st>>>(A, npend, walker_blocks);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_build(const float* p, uint32_t n, uint32_t m, uint32_t flags, rtf_header* hdr,
                         rtf_node* nodes, int32_t* table, uint64_t* cdf, void* ws,
                         const WsLayout& L, cudaStream_t st, int* launches) {
    unsigned char* w = reinterpret_cast<unsigned char*>(ws);
    if (flags & RTF_BUILD_SMALL_TILES)
        return launch_pipeline<64, 2>(p, n, m, hdr, nodes, table, cdf, w, L, st, launches);
    return launch_pipeline<512, 8>(p, n, m, hdr, nodes, table, cdf, w, L, st, launches);
}

}  // namespace rtf
