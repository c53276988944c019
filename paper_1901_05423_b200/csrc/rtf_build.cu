// rtf_build.cu -- the forest build: ONE persistent cooperative kernel (one CTA
// pair per SM) whose phases are separated by grid-wide barriers:
//
//   A  scale      read p once: max weight bits (for E), NaN/Inf/negative flags.
//   B  totals     per 4096-entry tile: quantise (w), sum W, count positives,
//                 last positive index (aggregates of the prefix sum).
//   C  spine      CTA 0 turns the tile aggregates into exclusive prefixes and
//                 publishes T, n' and the reciprocal of T (header).
//   D  tiles      per tile (TMA-fed): block scan + tile prefix -> W_j,
//                 compaction, one exact division per leaf (key_j); per owned
//                 leaf: cell, split level lambda_j, guide-table anchors and
//                 short runs; Alg. 1 for every leaf
//                 of the tile except its first and last ("phase 1", shared-
//                 memory atomicExch); coalesced flush of the 16-B records.
//   E  cross      "phase 2": the <= 2 pending edge leaves per tile continue
//                 Alg. 1 with global atomicExch, consuming the deposits the
//                 tiles flushed; then the long empty-cell runs of the table.
//
// A deposit in otherBounds carries the depositor's far bound AND the split
// level beyond it, so the sibling that continues never re-reads lambda.
// The result bytes do not depend on the schedule.

#include "rtf_device.cuh"
#include "rtf_internal.h"
#include <atomic>
#include <cstdlib>

namespace rtf {

constexpr uint32_t kShortRun = 32;  // empty-cell runs up to this length: written in place
constexpr uint32_t kChunk = 2048;   // longer runs: queued in chunks of this many cells
constexpr uint32_t kMaxGrid = 8192; // partials capacity (CTAs of the cooperative grid)

// workspace counters
enum : int { kCtrGridBar = 0, kCtrQueue = 1, kCtrTile = 2, kCtrRpre = 3 };

struct RunChunk {
    uint32_t start, len;
    int32_t value;
    uint32_t pad;
};

// What phase 1 leaves open in a tile, for the cross-tile links (phase E).
// The tile's split levels lambda_0..lambda_{cnt-1} (gap l lies between leaves
// l and l+1; the last one reaches the next tile's first leaf) have a left
// spine -- the strict prefix maxima -- and a right spine -- the strict suffix
// maxima.  Exactly the spine gaps (and the tile's first leaf) have a parent
// outside what phase 1 can see; every other node was linked in the tile.
// Along the left spine lambda increases, along the right spine it decreases,
// so each spine is a set of distinct split levels: a mask plus the local gap
// index per level.  lambda = 64 (a cell boundary) is a wall: it needs no parent.
struct TileSpine {
    unsigned long long mL, mR;  // split levels 0..63 on the left / right spine
    uint32_t j0, cnt;           // global index of the tile's first leaf; leaves
    uint32_t walls;             // bit 0: a wall on the left spine; bit 1: on the right
    int32_t c0_next;            // left child of the last gap, linked in the tile (kNoLink: none)
    int32_t ref0;               // ~orig of the tile's first leaf
    uint32_t pad[3];
    uint16_t iL[65], iR[65];    // local gap index per split level (where the mask is set)
    uint32_t pad2[3];
};
static_assert(sizeof(TileSpine) % 16 == 0, "TileSpine rows stay 16-B aligned");
constexpr int32_t kNoLink = INT32_MIN;

struct BuildArgs {
    const float* p;
    uint32_t n, m, nt;
    int B;              // 62 - ceil(log2 n_global)
    uint32_t phases;
    uint32_t index_base;       // global index of p[0] (sharded build), else 0
    uint32_t* scale_io;        // sharded: 4 words {max bits, nan, inf, neg} (MAX-reducible)
    const Pfx* shard_totals;   // sharded: every shard's total, shard_count entries
    uint32_t shard_rank, shard_count;
    Pfx* total_out;            // sharded: this shard's total
    TileSpine* spine;          // phase D: one row per tile of this call
    const TileSpine* spine_in; // phase E: the rows to link (a sharded finish: all shards')
    uint32_t nt_in;            // rows in spine_in
    uint8_t* tmax;             // phase E: per row, 1 + the largest split level (0: empty)
    uint32_t* bmax;            // phase E: per 64 rows, the maximum of tmax
    uint32_t* maxpart;  // 2 per CTA
    uint32_t* counters;
    Pfx* excl;          // per tile: exclusive prefix within its range (phase B)
    Pfx* rng;           // per range of tiles: total (phase B)
    Pfx* rpre;          // per range of tiles: exclusive prefix (phase C, CTA 0)
    uint32_t epoch;     // this launch's number: CTA 0 publishes rpre with it
    uint32_t mshift;    // m a power of two: cell = key >> mshift (63 - log2 m)
    uint32_t j_lo, j_hi;  // phase E writes only node slots in [j_lo, j_hi) (a ranged finish)
    // fused ranged sharding: records and table cells are stored straight into
    // the buffer of the rank owning their cell (cells [r cpo, (r + 1) cpo)),
    // over NVLink peer memory; jbound[k] receives the first leaf of cell k cpo
    rtf_node* const* peer_nodes;
    rtf_ref* const* peer_table;
    uint32_t npeer, cpo;
    uint32_t* jbound;
    rtf_header* hdr;
    rtf_node* nodes;
    rtf_ref* table;
    RunChunk* queue;
    uint32_t qcap;
    uint64_t* cdf;                // CDF mode only
    bool vec;
};

// ------------------------------------------------------------ grid barrier
// Sense-reversing (the cooperative-groups scheme): CTA 0 adds 2^31 - (G-1),
// the others add 1, so the top bit flips exactly when all G arrived and the
// word returns to its old low bits -- reusable across phases and launches.
__device__ __forceinline__ void grid_barrier(uint32_t* bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t nb = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1) : 1u;
        uint32_t old;
        asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;"
                     : "=r"(old)
                     : "l"(bar), "r"(nb)
                     : "memory");
        while (((ld_acquire_u32(bar) ^ old) & 0x80000000u) == 0) __nanosleep(20);
        __threadfence();  // also drops stale L1 lines of this SM
    }
    __syncthreads();
}

// ------------------------------------------------------------ block reductions

template <int THREADS>
__device__ __forceinline__ void block_max_or(uint32_t& mx, uint32_t& fl, uint32_t* s2) {
    for (int d = 16; d; d >>= 1) {
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, d));
        fl |= __shfl_xor_sync(0xffffffffu, fl, d);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) {
        s2[2 * warp] = mx;
        s2[2 * warp + 1] = fl;
    }
    __syncthreads();
    mx = 0;
    fl = 0;
    for (int w = 0; w < THREADS / 32; ++w) {
        mx = max(mx, s2[2 * w]);
        fl |= s2[2 * w + 1];
    }
}

// Pfx of consecutive runs combines as (sum, sum, max): the last positive index
// only grows along the array (-1 = none).
__device__ __forceinline__ void warp_sum_pfx(Pfx& a) {
    for (int d = 16; d; d >>= 1) {
        a.W += __shfl_xor_sync(0xffffffffu, a.W, d);
        a.cnt += __shfl_xor_sync(0xffffffffu, a.cnt, d);
        a.last = max(a.last, __shfl_xor_sync(0xffffffffu, a.last, d));
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

// Shared-memory arrays indexed by the local leaf index are padded with one slot
// every 8 entries: with blocked ownership (lane L works on leaves ~8L + r) and
// with strided access (consecutive leaves) both hit distinct banks.
__device__ __forceinline__ uint32_t pad8(uint32_t j) { return j + (j >> 3); }

template <int THREADS, int VPT>
__host__ __device__ constexpr size_t tile_padded() {
    return (size_t)THREADS * VPT + (size_t)THREADS * VPT / 8 + 4;  // + slot pad8(TILE)
}

template <int THREADS, int VPT>
constexpr size_t build_smem_bytes() {
    // p tile / otherBounds (i32), keys (u64), child0, child1 (i32), split levels (u8)
    return tile_padded<THREADS, VPT>() * (4 + 8 + 4 + 4) +
           ((tile_padded<THREADS, VPT>() + 15) & ~(size_t)15);
}

// A long run of empty cells after the cell of leaf orig i: ~i for each, queued
// in chunks for phase E (short runs are written in place).
__device__ __noinline__ void table_queue(uint32_t* __restrict__ counters,
                                         RunChunk* __restrict__ queue, uint32_t qcap, int32_t i,
                                         uint32_t cell, uint32_t len) {
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

// ------------------------------------------------------------ phase E helpers

// smallest split level above v on a spine (levels 0..63 in m, the wall 64 in
// wall); 0xff if none.  v in [0, 63].
__device__ __forceinline__ uint32_t spine_above(unsigned long long m, bool wall, uint32_t v) {
    const unsigned long long x = v >= 63 ? 0ull : (m & (~0ull << (v + 1)));
    return x ? (uint32_t)(__ffsll((long long)x) - 1) : (wall ? 64u : 0xffu);
}

// lowest split level on a spine: lambda of the tile's first gap (left spine)
// or of its last gap (right spine)
__device__ __forceinline__ uint32_t spine_lowest(unsigned long long m, bool wall) {
    return m ? (uint32_t)(__ffsll((long long)m) - 1) : (wall ? 64u : 0xffu);
}

// position of the k-th (0-based) set bit
__device__ __forceinline__ uint32_t nth_bit(unsigned long long m, uint32_t k) {
    for (uint32_t i = 0; i < k; ++i) m &= m - 1;
    return (uint32_t)(__ffsll((long long)m) - 1);
}

// the 64 rows of block bb whose tmax exceeds thr, as a bit mask
__device__ __forceinline__ unsigned long long block_rows_above(const uint8_t* tmax, uint32_t bb,
                                                               uint32_t thr) {
    const uint4* p4 = reinterpret_cast<const uint4*>(tmax + 64ull * bb);
    const uint32_t t4 = thr * 0x01010101u;
    unsigned long long mask = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint4 v = __ldcg(p4 + i);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {  // byte flags 0x80 -> one nibble
            const uint32_t c = __vcmpgtu4(w[k], t4) & 0x80808080u;
            mask |= (unsigned long long)((c * 0x00204081u) >> 28) << (16 * i + 4 * k);
        }
    }
    return mask;
}

// nearest row u < t (u > t) whose tmax exceeds thr; -1 if none
__device__ int32_t row_left(const uint8_t* tmax, const uint32_t* bmax, uint32_t t, uint32_t thr) {
    if (t == 0) return -1;
    if (__ldcg(tmax + t - 1) > thr) return (int32_t)t - 1;
    const uint32_t bb = t >> 6;
    const unsigned long long mk = block_rows_above(tmax, bb, thr) & ((1ull << (t & 63)) - 1);
    if (mk) return (int32_t)(64 * bb + 63 - __clzll((long long)mk));
    for (int32_t c = (int32_t)bb - 1; c >= 0; --c)
        if (__ldcg(bmax + c) > thr)
            return 64 * c + 63 - __clzll((long long)block_rows_above(tmax, (uint32_t)c, thr));
    return -1;
}

__device__ int32_t row_right(const uint8_t* tmax, const uint32_t* bmax, uint32_t nrows, uint32_t t,
                             uint32_t thr) {
    if (t + 1 >= nrows) return -1;
    if (__ldcg(tmax + t + 1) > thr) return (int32_t)t + 1;
    const uint32_t bb = t >> 6, sh = (t & 63) + 1;
    const unsigned long long mk = sh >= 64 ? 0ull : (block_rows_above(tmax, bb, thr) & (~0ull << sh));
    if (mk) return (int32_t)(64 * bb + __ffsll((long long)mk) - 1);
    const uint32_t nb = (nrows + 63) / 64;
    for (uint32_t c = bb + 1; c < nb; ++c)
        if (__ldcg(bmax + c) > thr)
            return (int32_t)(64 * c + __ffsll((long long)block_rows_above(tmax, c, thr)) - 1);
    return -1;
}

// ------------------------------------------------------------ phase timing (debug builds)
// Compiled only with -DRTF_PHASE_TIMING (tools/phase_timing.py): thread 0 of
// each CTA accumulates clock64() deltas per phase; read with
// rtf_debug_phase_cycles().  The product library has neither.
#ifdef RTF_PHASE_TIMING
__device__ unsigned long long g_phase_cycles[kMaxGrid][16];
#define RTF_TICK(slot)                                                       \
    do {                                                                     \
        if (threadIdx.x == 0) {                                              \
            const long long now_ = clock64();                                \
            g_phase_cycles[blockIdx.x][slot] += (unsigned long long)(now_ - t_tick_); \
            t_tick_ = now_;                                                  \
        }                                                                    \
    } while (0)
#else
#define RTF_TICK(slot) \
    do {               \
    } while (0)
#endif

// ============================================================== the build kernel

template <int THREADS, int VPT, bool CDF, int MINB = 2, bool POW2 = false, bool FUSED = false>
__global__ void __launch_bounds__(THREADS, MINB) k_build(BuildArgs A) {
    constexpr int TILE = THREADS * VPT;
    constexpr int NW = THREADS / 32;
    constexpr int P = (int)tile_padded<THREADS, VPT>();
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
    __shared__ uint32_t s_red[2 * NW];
    __shared__ __align__(16) Pfx s_rpre;  // the next tile's range prefix (issuer thread)
    __shared__ Pfx s_tot;
    __shared__ uint32_t s_next;
    __shared__ __align__(16) Pfx s_pin;  // TMA target: the next tile's prefix within its range
    __shared__ uint64_t s_recip;
    __shared__ unsigned long long s_mL, s_mR;  // this tile's spines (TileSpine)
    __shared__ uint32_t s_walls;
    __shared__ uint32_t s_fw, s_lw, s_mx;  // first / last wall, (max split level << 16 | gap)
    __shared__ int32_t s_ref0;
    __shared__ uint16_t s_iL[65], s_iR[65];

    const uint32_t G = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
    const uint32_t n = A.n, m = A.m, nt = A.nt;
    // the cell of a key (Alg. 1): a shift when m is a power of two
    auto cell_fn = [&](uint64_t key) -> uint32_t {
        return POW2 ? (uint32_t)(key >> A.mshift) : cell_of(key, m);
    };
    // where cell g's table entry lives (the owner rank's table when fused)
    auto table_at = [&](uint32_t g) -> rtf_ref* {
        return FUSED ? A.peer_table[g / A.cpo] : A.table;
    };
    const int lane = tid & 31, warp = tid >> 5;
    uint32_t* gbar = &A.counters[kCtrGridBar];

    const uint32_t ph = A.phases;
    const int32_t ib = (int32_t)A.index_base;  // original indices are global
#ifdef RTF_PHASE_TIMING
    long long t_tick_ = clock64();
#endif
    const bool sharded = A.shard_count > 0;

    // the tiles form NRG ranges of krng consecutive tiles (phases A and B)
    const uint32_t NRG = min(G, (uint32_t)THREADS);
    const uint32_t krng = (nt + NRG - 1) / NRG;

    // ---------------------------------------------------------- A: scale
    if (b == 0 && tid == 0 && (ph & kPhTiles)) {
        A.counters[kCtrQueue] = 0;
        A.counters[kCtrTile] = 0;  // phase D's tile dispenser (a grid barrier precedes D)
    }
    if (ph & kPhTiles) {  // row maxima for phase E: padding rows stay 0
        const uint32_t nb = (nt + 63) / 64;
        for (uint32_t i = b * THREADS + tid; i < 16 * nb; i += G * THREADS)
            reinterpret_cast<uint32_t*>(A.tmax)[i] = 0u;
        for (uint32_t i = b * THREADS + tid; i < nb; i += G * THREADS) A.bmax[i] = 0u;
    }
    if (ph & kPhScale) {
        // Fast path: two integer maxima of the raw bits.  As signed integers the
        // positive finite floats order like their values and stay below +Inf
        // (0x7f800000); as unsigned integers anything with the sign bit set
        // exceeds 0x80000000 (-0.0) -- so valid data (no NaN, Inf or negative
        // value) is exactly smax < 0x7f800000 and umax <= 0x80000000, and then
        // max(smax, 0) is the bit pattern of the largest weight.  A CTA whose
        // share is not valid rescans it classifying every value (error path).
        int32_t smax = 0;
        uint32_t umax = 0;
        auto visit = [&](float x) {
            smax = max(smax, __float_as_int(x));
            umax = max(umax, __float_as_uint(x));
        };
        auto classify = [&](float x, uint32_t& f) {
            if (x != x) f |= RTF_DATA_NAN;
            else if (fabsf(x) == __int_as_float(0x7f800000)) f |= RTF_DATA_INF;
            else if (x < 0.0f) f |= RTF_DATA_NEG;
        };
        // This CTA's share is the range of tiles it sums in phase B, so that
        // phase B re-reads what this SM just pulled into its die's L2.
        const uint32_t a_lo = (uint32_t)min((uint64_t)n, (uint64_t)b * krng * TILE);
        const uint32_t a_hi = (uint32_t)min((uint64_t)n, ((uint64_t)b + 1) * krng * TILE);
        if (A.vec) {
            const uint32_t lo4 = a_lo >> 2, hi4 = a_hi >> 2;  // a_lo is a multiple of TILE
            uint32_t q = lo4 + tid;
            for (; q + 7 * THREADS < hi4; q += 8 * THREADS) {  // 8 independent 16-B loads in flight
                float4 v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = ld_stream_f4(A.p + 4ull * (q + u * THREADS));
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    visit(v[u].x);
                    visit(v[u].y);
                    visit(v[u].z);
                    visit(v[u].w);
                }
            }
            for (; q < hi4; q += THREADS) {
                const float4 v = ld_stream_f4(A.p + 4ull * q);
                visit(v.x);
                visit(v.y);
                visit(v.z);
                visit(v.w);
            }
            for (uint32_t i = 4 * hi4 + tid; i < a_hi; i += THREADS) visit(A.p[i]);
        } else {
            for (uint32_t i = a_lo + tid; i < a_hi; i += THREADS) visit(A.p[i]);
        }
        uint32_t mx = (uint32_t)smax, fl = (smax >= 0x7f800000 || umax > 0x80000000u) ? 1u : 0u;
        block_max_or<THREADS>(mx, fl, s_red);
        if (fl) {  // invalid data somewhere in this CTA's share: exact flags
            fl = 0;
            for (uint32_t i = a_lo + tid; i < a_hi; i += THREADS) classify(A.p[i], fl);
            uint32_t dummy = 0;
            block_max_or<THREADS>(dummy, fl, s_red);
        }
        block_max_or<THREADS>(mx, fl, s_red);
        if (tid == 0) {
            A.maxpart[2 * b] = mx;
            A.maxpart[2 * b + 1] = fl;
        }
    }
    grid_barrier(gbar);
    RTF_TICK(0);
    uint32_t mx = 0, fl = 0;
    if (ph & kPhScale) {
        for (uint32_t i = tid; i < G; i += THREADS) {
            mx = max(mx, __ldcg(&A.maxpart[2 * i]));
            fl |= __ldcg(&A.maxpart[2 * i + 1]);
        }
        block_max_or<THREADS>(mx, fl, s_red);
        if (sharded && b == 0 && tid == 0) {  // this shard's word, MAX-reduced across shards
            A.scale_io[0] = mx;
            A.scale_io[1] = (fl & RTF_DATA_NAN) ? 1u : 0u;
            A.scale_io[2] = (fl & RTF_DATA_INF) ? 1u : 0u;
            A.scale_io[3] = (fl & RTF_DATA_NEG) ? 1u : 0u;
        }
        if (sharded) return;  // sharded: phase A runs alone
    } else {                  // sharded: the reduced word of all shards
        mx = __ldcg(&A.scale_io[0]);
        fl = (__ldcg(&A.scale_io[1]) ? RTF_DATA_NAN : 0u) |
             (__ldcg(&A.scale_io[2]) ? RTF_DATA_INF : 0u) |
             (__ldcg(&A.scale_io[3]) ? RTF_DATA_NEG : 0u);
    }
    const uint32_t status = fl | (mx == 0 ? RTF_DATA_ALLZERO : 0u);
    if (status) {  // poisoned build: report and stop (uniform across the grid)
        if (b == 0 && tid == 0 && A.hdr) A.hdr->status = status;
        return;
    }
    const int E = floor_log2_bits(mx);
    const QScale scale = qscale(A.B - E);

    // ---------------------------------------------------------- B: tile totals
    // The tiles form NRG ranges of krng consecutive tiles; CTA r < NRG sums
    // range r, one warp per tile (8 float4 loads in flight per lane, no block
    // barrier per tile), then writes each tile's exclusive prefix within its
    // range (excl) and the range total (rng).  Phase C scans only the NRG
    // range totals.
    if ((ph & kPhTotals) && b < NRG) {
        Pfx* s_tagg = reinterpret_cast<Pfx*>(s_key);  // free until phase D
        constexpr uint32_t CAP = (uint32_t)(tile_padded<THREADS, VPT>() * 8 / sizeof(Pfx));
        constexpr int F = TILE / 128;  // float4 per lane per tile
        constexpr int BATCH = F < 8 ? F : 8;
        const uint32_t t_beg = b * krng, t_end = min(nt, t_beg + krng);
        Pfx run{0ull, 0u, -1};  // thread 0: the range so far
        // short ranges (small n): up to F / BATCH warps share a tile, so every
        // warp keeps loads in flight
        constexpr uint32_t NCH = F / BATCH;
        const uint32_t WPT = krng >= NW ? 1u : min(NCH, NW / krng >= 4 ? 4u : NW / krng >= 2 ? 2u : 1u);
        const uint32_t CAPT = CAP / WPT;
        for (uint32_t c0 = t_beg; c0 < t_end; c0 += CAPT) {
            const uint32_t c1 = min(t_end, c0 + CAPT);
            for (uint32_t u = warp; u < (c1 - c0) * WPT; u += NW) {
                const uint32_t t = c0 + u / WPT, part = u % WPT;
                Pfx acc{0ull, 0u, -1};
                const uint32_t base = t * TILE;
                if (A.vec && base + TILE <= n) {
                    const int cb = (int)(part * (F / WPT)), ce = cb + (int)(F / WPT);
#pragma unroll 1
                    for (int c = cb; c < ce; c += BATCH) {
                        float4 v[BATCH];
#pragma unroll
                        for (int u = 0; u < BATCH; ++u)
                            v[u] = ld_stream_f4(A.p + base + 4 * ((c + u) * 32 + lane));
#pragma unroll
                        for (int u = 0; u < BATCH; ++u) {
                            const int32_t e0 = (int32_t)(base + 4 * ((c + u) * 32 + lane)) + ib;
                            const float xs[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                const uint64_t w = quantize(xs[q], scale);
                                acc.W += w;
                                acc.cnt += w != 0;
                                if (w) acc.last = e0 + q;
                            }
                        }
                    }
                } else if (part == 0) {
                    for (uint32_t e = base + lane; e < min(n, base + TILE); e += 32) {
                        const uint64_t w = quantize(A.p[e], scale);
                        acc.W += w;
                        acc.cnt += w != 0;
                        if (w) acc.last = (int32_t)e + ib;
                    }
                }
                warp_sum_pfx(acc);
                if (lane == 0) s_tagg[u] = acc;
            }
            __syncthreads();
            if (tid == 0)
                for (uint32_t t = c0; t < c1; ++t) {
                    st_pfx(&A.excl[t], run);
                    for (uint32_t part = 0; part < WPT; ++part)
                        run = combine(run, s_tagg[(t - c0) * WPT + part]);
                }
            __syncthreads();
        }
        if (tid == 0) st_pfx(&A.rng[b], run);
    }
    // the tile weights of phase D can stream in while the spine scan runs
    const bool tma = !CDF && A.vec && (ph & kPhTiles);
    auto tma_tile = [&](uint32_t t) { return tma && t < nt && (t + 1) * TILE <= n; };
    if (tma && tid == 0) {
        mbar_init(&s_bar, 1);
        fence_proxy_async_smem();
        if (tma_tile(b)) {
            mbar_arrive_expect_tx(&s_bar, TILE * 4);
            tma_load_1d(s_p, A.p + (size_t)b * TILE, TILE * 4, &s_bar);
        }
    }
    // sharded: this shard writes only the table cells its leaves own; the rest
    // stays INT32_MIN so a MAX-reduction across shards assembles the table
    if (sharded && (ph & kPhTiles) && !FUSED)  // fused: every cell is written once by its builder
        for (uint32_t g = b * THREADS + tid; g < m; g += G * THREADS) st_cell(A.table, g, 0u, INT32_MIN);
    grid_barrier(gbar);
    RTF_TICK(1);

    // ---------------------------------------------------------- C: spine (every CTA)
    // Each CTA scans the NRG range totals itself (a few KB from L2) for the
    // total; CTA 0 publishes the exclusive prefix of every range (rpre, then
    // the epoch flag).  A tile's prefix is its range's combined with its
    // exclusive prefix within the range.
    Pfx total{0ull, 0u, -1};
    Pfx gpre{0ull, 0u, -1};  // thread tid: the exclusive prefix of range tid
    if (ph & (kPhSpine | kPhTiles)) {
        const Pfx own = tid < NRG ? ld_pfx_cg(&A.rng[tid]) : Pfx{0ull, 0u, -1};
        uint64_t w_ex, w_tot;
        uint32_t c_ex, c_tot;
        int32_t l_ex;
        block_scan3_excl<THREADS>(own.W, own.cnt, own.last, w_ex, c_ex, l_ex, w_tot, c_tot, s_w,
                                  s_c, s_l);
        gpre = Pfx{w_ex, c_ex, l_ex};
        if (tid == THREADS - 1) {
            s_tot = Pfx{w_tot, c_tot, max(l_ex, own.last)};
            // sharded: this shard's total, for the cross-GPU scan of shard totals
            if (sharded && b == 0 && (ph & kPhSpine)) st_pfx(A.total_out, s_tot);
        }
        __syncthreads();
        total = s_tot;
    }
    if (sharded && !(ph & (kPhTiles | kPhCross))) return;  // totals launch ends here
    RTF_TICK(2);

    // sharded: the exclusive prefix of this shard and the grand total come from
    // the gathered shard totals (the cross-GPU scan, done redundantly per CTA)
    if (sharded && (ph & kPhTiles)) {
        Pfx tot{0ull, 0u, -1}, shard_pre{0ull, 0u, -1};
        for (uint32_t r = 0; r < A.shard_count; ++r) {
            const Pfx s = ld_pfx_cg(&A.shard_totals[r]);
            if (r == A.shard_rank) shard_pre = tot;
            tot = combine(tot, s);
        }
        total = tot;
        gpre = combine(shard_pre, gpre);  // range prefixes become global
    }
    if ((ph & kPhTiles) && b == 0) {  // publish the range prefixes (read in phase D)
        if (tid < NRG) st_pfx(&A.rpre[tid], gpre);
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            st_release_u32(&A.counters[kCtrRpre], A.epoch);
        }
    }
    // the range prefixes of CTA 0 are visible once the flag carries this epoch
    auto wait_rpre = [&]() {
        if (tid == 0)
            while (ld_acquire_u32(&A.counters[kCtrRpre]) != A.epoch) __nanosleep(32);
        __syncthreads();
    };
    // T and its reciprocal (one thread per CTA); CTA 0 publishes the header
    const uint64_t T = total.W;  // >= 1: the largest weight quantises to >= 2^B
    Norm nm;
    nm.s = (uint32_t)__clzll((long long)T);
    nm.d = T << nm.s;
    if (ph & kPhTiles) {
        if (tid == THREADS - 1) {
            s_recip = reciprocal_fast(nm.d);
            if (b == 0) {
                rtf_header h;
                h.total = T;
                h.n_pos = total.cnt;
                h.exponent = E;
                h.scale_bits = A.B;
                h.status = 0;
                h.reserved = 0;
                h.norm_shift = nm.s;
                h.recip = s_recip;
                *A.hdr = h;
            }
        }
        __syncthreads();
    }
    nm.v = s_recip;

    // exclusive prefix of tile t: its range's, then its own within the range
    auto tile_prefix = [&](uint32_t t) -> Pfx {
        return combine(ld_pfx_cg(&A.rpre[t / krng]), ld_pfx_cg(&A.excl[t]));
    };

    if (CDF) {  // baseline: K[i] = floor(W_i 2^63 / T) for every entry, zeros included
        wait_rpre();
        for (uint32_t t = b; t < nt; t += G) {
            const Pfx pre = tile_prefix(t);
            const uint32_t first = t * TILE + tid * VPT;
            float x[VPT];
            load_tile<VPT>(A.p, first, n, A.vec, x);
            uint64_t w[VPT];
            uint64_t tw = 0;
#pragma unroll
            for (int k = 0; k < VPT; ++k) {
                w[k] = quantize(x[k], scale);
                tw += w[k];
            }
            uint64_t w_ex, w_tot;
            uint32_t c_ex, cnt;
            block_scan_excl<THREADS>(tw, 0u, w_ex, c_ex, w_tot, cnt, s_w, s_c);
            uint64_t W = pre.W + w_ex;
#pragma unroll
            for (int k = 0; k < VPT; ++k) {
                if (first + k < n) A.cdf[first + k] = (W == T) ? kOne63 : fixed_point(W, nm);
                W += w[k];
            }
            __syncthreads();
        }
        return;
    }

    // ---------------------------------------------------------- D: tiles
    // Tiles are dealt dynamically (their cost varies with the zero fraction
    // and the tree shape): CTA b starts with tile b, then takes G + tickets.
    // Thread 0 draws each ticket one tile ahead, so the atomic's latency is
    // hidden; the TMA copy of the next tile's weights also brings its prefix
    // within its range (one mbarrier for both).
    uint32_t phase = 0;
    uint32_t ticket = 0;  // issuer thread: the tile after the next one
    if (tid == 0) {
        s_mL = s_mR = 0ull;
        s_walls = 0u;
        s_fw = 0xffffffffu;
        s_lw = 0u;
        s_mx = 0u;
    }
    constexpr uint32_t kIssuer = THREADS - 1;  // TMA and tickets: the last warp (light duty)
    if (tid == kIssuer) {
        fence_proxy_async_global();  // phase B's prefixes, read by TMA below
        if (ph & kPhTiles) ticket = G + atomicAdd(&A.counters[kCtrTile], 1u);
    }
    if (ph & kPhTiles) wait_rpre();
    for (uint32_t t = b; (ph & kPhTiles) && t < nt; t = s_next) {
        const uint32_t first = t * TILE + tid * VPT;  // local index into p (global: + ib)

        // (0) weights of this thread's VPT consecutive entries
        float x[VPT];
        Pfx pre;
        if (tma_tile(t)) {
            mbar_wait(&s_bar, phase);
            phase ^= 1u;
            pre = t == b ? tile_prefix(t) : combine(s_rpre, s_pin);
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
            pre = tile_prefix(t);
        }
        uint64_t w[VPT];
        uint64_t tw = 0;
        uint32_t tc = 0, posmask = 0;
        int32_t tl = -1;
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
            w[k] = quantize(x[k], scale);
            tw += w[k];
            if (w[k]) {
                ++tc;
                posmask |= 1u << k;
                tl = (int32_t)(first + k) + ib;
            }
        }
        // (1) block scan (its barriers also retire every read of s_p);
        // one exact division per positive entry
        uint64_t w_ex, w_tot;
        uint32_t c_ex, cnt;
        int32_t l_ex;
        block_scan3_excl<THREADS>(tw, tc, tl, w_ex, c_ex, l_ex, w_tot, cnt, s_w, s_c, s_l);
        const uint32_t j0 = pre.cnt;  // global index of the tile's first leaf
        {  // otherBounds start empty; the consumed weight tile becomes the array
            int4* ob4 = reinterpret_cast<int4*>(s_ob);
            for (uint32_t u = tid; u < (uint32_t)P / 4; u += THREADS)
                ob4[u] = make_int4(-1, -1, -1, -1);
        }
        {
            // Node records start as anchors: child0 = ~orig(j-1) (Fig. 6 caption
            // P:1276-1277; j = 0 -> ~orig(0)); internal nodes overwrite it in
            // Alg. 1.  child1 needs no initial value: every slot's right child
            // is set by phase 1 here or by phase 2 afterwards.
            int32_t prevo = l_ex >= 0 ? l_ex : (j0 ? pre.last : -1);
            uint64_t W = pre.W + w_ex;
            uint32_t jl = c_ex;
#pragma unroll
            for (int k = 0; k < VPT; ++k) {
                const uint64_t wk = w[k];
                if (wk) {
                    const int32_t i = (int32_t)(first + k) + ib;
                    const uint32_t q = pad8(jl);
                    w[k] = fixed_point(W, nm);  // w[k] holds key_j from here on
                    s_key[q] = w[k];
                    s_c0[q] = ~(prevo >= 0 ? prevo : i);
                    prevo = i;
                    ++jl;
                }
                W += wk;
            }
        }
        // the tile's first leaf is linked in phase E (its left split level
        // belongs to the previous tile); the slot after the last leaf collects
        // the left child of the last gap, if phase 1 links it
        if (tc && c_ex == 0) s_ref0 = ~((int32_t)(first + __ffs(posmask) - 1) + ib);
        if (tid == 0) s_c0[pad8(cnt)] = kNoLink;
        if (tid == THREADS - 1) {  // key of the first leaf after the tile (or "1")
            const uint64_t We = pre.W + w_tot;
            s_key_after = (We == T) ? kOne63 : fixed_point(We, nm);
        }
        __syncthreads();

        RTF_TICK(3);
        // (2) own leaves: cell, split level, guide table; the
        // thread's own split levels also stay in registers (byte r = rank r)
        // keys come from registers (w[k]); only the key after the thread's last
        // leaf is read back (its owner's, or the one after the tile)
        uint64_t lampack = 0;
        if (tc) {
            uint64_t kn = (c_ex + tc < cnt) ? s_key[pad8(c_ex + tc)] : s_key_after;
            uint32_t cn = POW2 ? 0u : ((kn == kOne63) ? m : cell_of(kn, m));
            if (j0 == 0 && c_ex == 0) st_cell(table_at(0), 0, 0u, 0);  // leaf 0 (key 0): cell 0's anchor
#pragma unroll
            for (int k = VPT - 1; k >= 0; --k) {
                if ((posmask >> k) & 1u) {
                    const uint64_t key = w[k];
                    const uint32_t r = __popc(posmask & ((1u << k) - 1u));  // rank
                    const uint32_t jl = c_ex + r;
                    uint32_t cell, lam;
                    if (POW2) {  // a cell boundary lies between iff the keys differ at or
                                 // above bit mshift (kn = 2^63 "1" differs at bit 63)
                        const uint32_t d = split_level(key, kn);
                        lam = d >= A.mshift ? kLamBoundary : d;
                        cell = (uint32_t)(key >> A.mshift);
                        cn = (uint32_t)(kn >> A.mshift);
                    } else {
                        cell = cell_of(key, m);
                        lam = (cn != cell) ? kLamBoundary : split_level(key, kn);
                    }
                    s_lam[pad8(jl)] = (uint8_t)lam;
                    lampack |= (uint64_t)lam << (8 * r);
                    if (lam == kLamBoundary) {  // the table entries this leaf owes
                        const int32_t i = (int32_t)(first + k) + ib;
                        // the next cell's anchor (a one-leaf cell gets its
                        // two-interval entry from the anchor's tile, below)
                        if (cn < m) st_cell(table_at(cn), cn, 0u, (int32_t)(j0 + jl + 1));
                        if (FUSED)  // the first leaf of every owner boundary k cpo in (cell, cn]
                            for (uint32_t k = cell / A.cpo + 1; k <= min(A.npeer, cn / A.cpo); ++k)
                                A.jbound[k] = j0 + jl + 1;
                        const uint32_t len = cn - cell - 1;
                        if (len <= kShortRun) {
                            for (uint32_t g = cell + 1; g < cn; ++g) st_cell(table_at(g), g, 0u, ~i);
                        } else {
                            table_queue(A.counters, A.queue, A.qcap, i, cell, len);
                        }
                    }
                    kn = key;
                    cn = cell;
                }
            }
        }
        if (tc) {  // first / last wall and the largest other split level (byte SIMD)
            const uint32_t h0 = (uint32_t)lampack, h1 = (uint32_t)(lampack >> 32);
            const uint32_t w0 = __vcmpeq4(h0, 0x40404040u), w1 = __vcmpeq4(h1, 0x40404040u);
            const uint32_t wm = (((w0 & 0x80808080u) * 0x00204081u) >> 28) |
                                ((((w1 & 0x80808080u) * 0x00204081u) >> 28) << 4);
            if (wm) {
                atomicMin(&s_fw, c_ex + __ffs(wm) - 1);
                atomicMax(&s_lw, c_ex + 31 - __clz(wm));
            }
            const uint32_t v0 = h0 & ~w0, v1 = h1 & ~w1;  // walls -> 0; bytes past tc are 0
            uint32_t mv = __vmaxu4(v0, v1);
            mv = __vmaxu4(mv, mv >> 16);
            mv = max(mv & 0xffu, (mv >> 8) & 0xffu);
            const uint32_t e0 = __vcmpeq4(v0, mv * 0x01010101u), e1 = __vcmpeq4(v1, mv * 0x01010101u);
            const uint32_t em = (((e0 & 0x80808080u) * 0x00204081u) >> 28) |
                                ((((e1 & 0x80808080u) * 0x00204081u) >> 28) << 4);
            atomicMax(&s_mx, (mv + 1) << 16 | (c_ex + __ffs(em) - 1));
        }
        __syncthreads();

        RTF_TICK(4);
        // (3) phase 1: Alg. 1 for the tile's leaves 1..cnt-1 with shared-memory
        // atomicExch.  A range containing leaf 0 (whose left split level is
        // the previous tile's) never completes here; a range ending at the
        // last leaf may still become the left child of the last gap, whose
        // slot is cnt.  Every parent slot is in [1, cnt].  What stays open
        // (first arrivals without a sibling in the tile) is exactly what the
        // spines describe; those deposits are dropped.  Each lane walks its
        // own leaves back to back.  A cell root (lambda = 64 on both sides) is
        // the right child of its anchor lo and needs no exchange.  A deposit
        // is (lambda beyond the bound) << 16 | bound.
        {
            // Stage A: the FIRST step of every own interior leaf, straight-line
            // (half of all merge steps, without loop or divergence overhead).
            // Leaf of rank r is l = c_ex + r; its split levels come from
            // registers (lambda[l-1] of rank 0 from the previous thread).
            const uint32_t lam_prev = c_ex ? (uint32_t)s_lam[pad8(c_ex - 1)] : kLamBoundary;
            uint32_t contw[VPT];  // second arrivals: the sibling's packed deposit
            uint32_t pend = 0, rightbits = 0;
            {
                uint32_t mask = posmask;
#pragma unroll
                for (int r = 0; r < VPT; ++r) {
                    contw[r] = 0;
                    if ((uint32_t)r < tc) {
                        const uint32_t k = __ffs(mask) - 1;
                        mask &= mask - 1;
                        const uint32_t l = c_ex + r;
                        if (l >= 1) {
                            const uint32_t lamL =
                                r ? (uint32_t)(lampack >> (8 * (r - 1))) & 0xffu : lam_prev;
                            const uint32_t lamR = (uint32_t)(lampack >> (8 * r)) & 0xffu;
                            const bool right = lamL <= lamR;
                            const bool root = (lamL & lamR & kLamBoundary) != 0;
                            const uint32_t q = pad8(right ? l : l + 1);
                            s_c0[q + (right ? P : 0)] = ~((int32_t)(first + k) + ib);
                            if (!root) {
                                const int32_t other = atomicExch(
                                    &s_ob[q], (int32_t)((right ? lamR : lamL) << 16 | l));
                                if (other >= 0) {
                                    s_ob[q] = -1;  // reset-on-consume
                                    contw[r] = (uint32_t)other;
                                    pend |= 1u << r;
                                    rightbits |= (right ? 1u : 0u) << r;
                                }
                            } else {
                                // a one-leaf cell: exactly two intervals overlap it
                                // (P:1335-1338); slot q = l holds its key and the
                                // anchor's left child ~orig(l-1)
                                const uint64_t key = s_key[q];
                                const int32_t a = (int32_t)(j0 + l);
                                const uint2 e =
                                    single_leaf_cell(key, (int32_t)(first + k) + ib, ~s_c0[q], a);
                                if ((int32_t)e.y != a)
                                    st_cell(table_at(cell_fn(key)), cell_fn(key), e.x,
                                            (int32_t)e.y);
                            }
                        }
                    }
                }
            }
            // Stage B: the second arrivals climb on, one walker per lane at a time.
            bool active = false;
            int32_t lo = 0, hi = 0, node = 0;
            uint32_t lamL = 0, lamR = 0;
            while (true) {
                if (!active && pend) {
                    const uint32_t r = __ffs(pend) - 1;
                    pend &= pend - 1;
                    // select contw[r] by the bits of r (a 3-level tree of selects;
                    // measured 1.5 % faster than a chain of compares)
                    uint32_t sel[VPT];
#pragma unroll
                    for (int u = 0; u < VPT; ++u) sel[u] = contw[u];
#pragma unroll
                    for (int w = VPT / 2, bit = 1; w >= 1; w /= 2, bit <<= 1)
#pragma unroll
                        for (int u = 0; u < w; ++u) sel[u] = (r & bit) ? sel[2 * u + 1] : sel[2 * u];
                    const uint32_t other = sel[0];
                    const uint32_t l = c_ex + r;
                    const uint32_t bound = other & 0xffffu, lv = other >> 16;
                    const uint32_t own_lo = r ? (uint32_t)(lampack >> (8 * (r - 1))) & 0xffu
                                              : lam_prev;
                    const uint32_t own_hi = (uint32_t)(lampack >> (8 * r)) & 0xffu;
                    active = true;
                    if ((rightbits >> r) & 1u) {  // merged as the right child of node l
                        lo = (int32_t)bound;
                        hi = (int32_t)l;
                        lamL = lv;
                        lamR = own_hi;
                        node = (int32_t)(j0 + l);
                    } else {  // merged as the left child of node l + 1
                        lo = (int32_t)l;
                        hi = (int32_t)bound;
                        lamL = own_lo;
                        lamR = lv;
                        node = (int32_t)(j0 + l + 1);
                    }
                }
                if (!__any_sync(0xffffffffu, active)) break;
                if (active) {
                    const bool right = lamL <= lamR;  // Alg. 1: child 1 unless left is farther
                    const bool root = (lamL & lamR & kLamBoundary) != 0;
                    const int32_t parent = right ? lo : hi + 1;
                    const uint32_t q = pad8((uint32_t)parent);
                    s_c0[q + (right ? P : 0)] = node;
                    const int32_t dep = right ? (int32_t)(lamR << 16 | (uint32_t)hi)
                                              : (int32_t)(lamL << 16 | (uint32_t)lo);
                    const int32_t other = root ? -1 : atomicExch(&s_ob[q], dep);
                    active = other >= 0;  // first to arrive (or a root): stop
                    if (active) {
                        s_ob[q] = -1;  // reset-on-consume
                        const int32_t bound = other & 0xffff;
                        const uint32_t lv = (uint32_t)other >> 16;
                        lo = right ? bound : lo;
                        hi = right ? hi : bound;
                        lamL = right ? lv : lamL;
                        lamR = right ? lamR : lv;
                        node = (int32_t)(j0 + parent);
                    }
                }
            }
        }
        __syncthreads();

        RTF_TICK(5);
        // (4) the spines of the tile (TileSpine).  Every spine gap except the
        // tile's maximum got exactly one arrival here that found no sibling:
        // from its right (bound >= slot) on the left spine, from its left on
        // the right spine -- so the leftover deposits name them.  The walls
        // (first / last cell boundary) and, in a tile without walls, the
        // maximum complete the two spines.
        {
            auto add = [&](bool left, uint32_t lv, uint32_t gap) {
                if (left) {
                    s_iL[lv] = (uint16_t)gap;
                    atomicOr(&s_mL, 1ull << lv);
                } else {
                    s_iR[lv] = (uint16_t)gap;
                    atomicOr(&s_mR, 1ull << lv);
                }
            };
            auto leftover = [&](uint32_t e, int32_t o) {
                if (o < 0) return;
                const uint32_t q = e - e / 9;  // slot (gap q - 1)
                add((uint32_t)(o & 0xffff) >= q, s_lam[pad8(q - 1)], q - 1);
            };
            const int4* ob4 = reinterpret_cast<const int4*>(s_ob);
            const uint32_t n4 = cnt ? pad8(cnt) / 4 + 1 : 0u;
            for (uint32_t u = tid; u < n4; u += THREADS) {
                const int4 v = ob4[u];
                if ((v.x & v.y & v.z & v.w) < 0) continue;  // four empty slots
                leftover(4 * u, v.x);
                leftover(4 * u + 1, v.y);
                leftover(4 * u + 2, v.z);
                leftover(4 * u + 3, v.w);
            }
            if (tid == THREADS - 33 && cnt) {  // another warp than the issuer's
                if (s_fw != 0xffffffffu) {
                    s_iL[64] = (uint16_t)s_fw;
                    s_iR[64] = (uint16_t)s_lw;
                    s_walls = 3u;
                } else {  // no wall: the maximum heads both spines
                    const uint32_t lv = (s_mx >> 16) - 1, gap = s_mx & 0xffffu;
                    add(true, lv, gap);
                    add(false, lv, gap);
                }
            }
        }
        // (5) the next tile's weights and prefix: TMA into the consumed weight
        // buffer once every thread is done reading otherBounds; s_pin was read
        // at step (0)
        __syncthreads();
        if (tid == kIssuer) {
            const uint32_t nx = ticket;
            s_next = nx;  // read after the barrier below
            if (tma_tile(nx)) {
                fence_proxy_async_smem();
                mbar_arrive_expect_tx(&s_bar, TILE * 4 + (uint32_t)sizeof(Pfx));
                tma_load_1d(s_p, A.p + (size_t)nx * TILE, TILE * 4, &s_bar);
                tma_load_1d(&s_pin, A.excl + nx, (uint32_t)sizeof(Pfx), &s_bar);
            }
            if (nx < nt) {
                s_rpre = ld_pfx_cg(&A.rpre[nx / krng]);  // read at the next tile's step (0)
                ticket = G + atomicAdd(&A.counters[kCtrTile], 1u);
            }
        }
        // (6) node records, coalesced 16 B
        {
            uint4* gnode = reinterpret_cast<uint4*>(A.nodes + j0);
            for (uint32_t l = tid; l < cnt; l += THREADS) {
                const uint32_t q = pad8(l);
                const uint64_t key = s_key[q];
                const uint4 rec = make_uint4((uint32_t)key, (uint32_t)(key >> 32),
                                             (uint32_t)s_c0[q], (uint32_t)s_c1[q]);
                if (FUSED)  // fused: to the rank owning the record's cell (peer memory)
                    reinterpret_cast<uint4*>(A.peer_nodes[cell_fn(key) / A.cpo] + j0)[l] = rec;
                else
                    gnode[l] = rec;
            }
        }
        __syncthreads();  // spines complete; keys and children are free
        {
            TileSpine* row = A.spine + t;
            for (uint32_t u = tid; u < 65; u += THREADS) {
                row->iL[u] = s_iL[u];
                row->iR[u] = s_iR[u];
            }
            if (tid == 0) {
                row->mL = s_mL;
                row->mR = s_mR;
                row->j0 = j0;
                row->cnt = cnt;
                row->walls = s_walls;
                row->c0_next = cnt ? s_c0[pad8(cnt)] : kNoLink;
                row->ref0 = cnt ? s_ref0 : 0;
                // phase E's row maxima: 1 + the largest split level, 0 if empty
                const uint32_t enc = !cnt ? 0u : s_walls ? 65u : (s_mx >> 16);
                A.tmax[t] = (uint8_t)enc;
                if (enc) atomicMax(&A.bmax[t >> 6], enc);
                s_mL = s_mR = 0ull;  // the next tile's atomics follow its scan barriers
                s_walls = 0u;
                s_fw = 0xffffffffu;
                s_lw = 0u;
                s_mx = 0u;
            }
        }
        // no barrier here: the next tile writes shared memory only after its scan
        RTF_TICK(6);
    }
    if (FUSED) __threadfence_system();  // peer stores visible before the next exchange
    grid_barrier(gbar);
    RTF_TICK(7);

    // ---------------------------------------------------------- E: cross-tile links
    // Phase 1 linked every node whose parent lies in its tile.  The rest --
    // the spine gaps and each tile's first leaf -- take the parent Alg. 1
    // gives them: of the nearest greater split levels on either
    // side, the smaller one (ties only between two walls: a cell root, the
    // right child of its anchor).  The tree is unique, so this is the forest
    // the bottom-up merge builds; the neighbours come from the rows' spines.
    if (ph & kPhCross) {
        const TileSpine* SP = A.spine_in;
        const uint32_t NR = A.nt_in, NB = (NR + 63) / 64;
        // E0 (gathered rows only; phase D records its own): per row 1 + its
        // largest split level (0: no leaves), per 64 rows the maximum
        const bool gathered = !(ph & kPhTiles);
        for (uint32_t bb = b * NW + warp; gathered && bb < NB; bb += G * NW) {
            uint32_t mx = 0;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint32_t u = 64 * bb + 32 * h + lane;
                uint32_t e = 0;
                if (u < NR && __ldcg(&SP[u].cnt))
                    e = (__ldcg(&SP[u].walls) & 1u)
                            ? 65u
                            : 64u - (uint32_t)__clzll((long long)__ldcg(&SP[u].mL));
                A.tmax[u] = (uint8_t)e;
                mx = max(mx, e);
            }
            mx = __reduce_max_sync(0xffffffffu, mx);
            if (lane == 0) A.bmax[bb] = mx;
        }
        if (gathered) grid_barrier(gbar);
        // a ranged finish (sharded.py, ranged=True) holds only the records of
        // its cell range [j_lo, j_hi): the other links are other ranks'
        auto local = [&](uint32_t slot) { return slot >= A.j_lo && slot < A.j_hi; };
        // E1: one warp per row; lane e links entry e
        auto far_left = [&](uint32_t t, uint32_t v, uint32_t& lam, int32_t& gap) {
            const int32_t u = row_left(A.tmax, A.bmax, t, v + 1);
            lam = 64u;
            gap = -1;  // the start of the array: a wall
            if (u >= 0) {
                const TileSpine* U = SP + u;
                lam = spine_above(__ldcg(&U->mR), __ldcg(&U->walls) & 2u, v);
                gap = (int32_t)(__ldcg(&U->j0) + __ldcg(&U->iR[lam]));
            }
        };
        auto far_right = [&](uint32_t t, uint32_t v, uint32_t& lam, int32_t& gap) {
            const int32_t u = row_right(A.tmax, A.bmax, NR, t, v + 1);
            lam = 0xffu;  // cannot happen: the last gap of the array is a wall
            gap = INT32_MAX;
            if (u >= 0) {
                const TileSpine* U = SP + u;
                lam = spine_above(__ldcg(&U->mL), __ldcg(&U->walls) & 1u, v);
                gap = (int32_t)(__ldcg(&U->j0) + __ldcg(&U->iL[lam]));
            }
        };
        for (uint32_t t = b * NW + warp; t < NR; t += G * NW) {
            const TileSpine* S = SP + t;
            const uint32_t cnt = __ldcg(&S->cnt);
            if (!cnt) continue;
            const uint32_t j0 = __ldcg(&S->j0), walls = __ldcg(&S->walls);
            const unsigned long long mL = __ldcg(&S->mL), mR = __ldcg(&S->mR);
            const bool wL = walls & 1u, wR = walls & 2u;
            // right-spine entries except the row maximum (linked as a left entry)
            const unsigned long long mRx =
                wR ? mR : (mR & ~(1ull << (63 - __clzll((long long)mR))));
            const uint32_t nL = __popcll(mL), nE = 2 + nL + __popcll(mRx);
            for (uint32_t e = lane; e < nE; e += 32) {
                if (e == 0) {  // the first leaf: right child of the gap before it, or
                               // left child of the gap after it
                    const uint32_t lam0 = spine_lowest(mL, wL);
                    const int32_t u = row_left(A.tmax, A.bmax, t, 0u);
                    uint32_t lamp = 64u;
                    if (u >= 0)
                        lamp = spine_lowest(__ldcg(&SP[u].mR), __ldcg(&SP[u].walls) & 2u);
                    const int32_t ref = __ldcg(&S->ref0);
                    if (lamp <= lam0) {
                        if (local(j0)) A.nodes[j0].child[1] = ref;
                    } else if (local(j0 + 1)) {
                        A.nodes[j0 + 1].child[0] = ref;
                    }
                    if ((lamp & lam0 & kLamBoundary) != 0 && local(j0)) {  // a one-leaf cell
                        const uint64_t key = __ldcg(&A.nodes[j0].key);
                        const uint2 e = single_leaf_cell(key, ~ref, ~__ldcg(&A.nodes[j0].child[0]),
                                                         (int32_t)j0);
                        if ((int32_t)e.y != (int32_t)j0)
                            st_cell(A.table, cell_fn(key), e.x, (int32_t)e.y);
                    }
                } else if (e == 1) {  // left child of the last gap, linked in the tile
                    const int32_t c = __ldcg(&S->c0_next);
                    if (c != kNoLink && local(j0 + cnt)) A.nodes[j0 + cnt].child[0] = c;
                } else {
                    const bool left = e - 2 < nL;
                    const uint32_t v = left ? nth_bit(mL, e - 2) : nth_bit(mRx, e - 2 - nL);
                    const uint32_t g = j0 + __ldcg(left ? &S->iL[v] : &S->iR[v]);
                    uint32_t lamL, lamR;
                    int32_t gL, gR;
                    if (left) {  // next left entry, else (the row maximum) beyond the row
                        const uint32_t a = spine_above(mL, wL, v);
                        if (a != 0xffu) {
                            lamR = a;
                            gR = (int32_t)(j0 + __ldcg(&S->iL[a]));
                        } else {
                            far_right(t, v, lamR, gR);
                        }
                        far_left(t, v, lamL, gL);
                    } else {  // previous right entry; beyond the row on the right
                        lamL = spine_above(mR, wR, v);
                        gL = (int32_t)(j0 + __ldcg(&S->iR[lamL]));
                        far_right(t, v, lamR, gR);
                    }
                    const int32_t node = (int32_t)(g + 1);
                    if (lamL <= lamR) {
                        if (local((uint32_t)(gL + 1))) A.nodes[gL + 1].child[1] = node;
                    } else if (local((uint32_t)(gR + 1))) {
                        A.nodes[gR + 1].child[0] = node;
                    }
                }
            }
        }
    }
    // long empty-cell runs of the guide table: one warp per chunk
    const uint32_t nq = (ph & kPhRuns) ? min(__ldcg(&A.counters[kCtrQueue]), A.qcap) : 0u;
    for (uint32_t q = b * NW + warp; q < nq; q += G * NW) {
        const RunChunk rc = A.queue[q];
        for (uint32_t g = lane; g < rc.len; g += 32)
            st_cell(table_at(rc.start + g), rc.start + g, 0u, rc.value);
    }
    __syncthreads();
    RTF_TICK(8);
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

size_t spine_row_bytes() { return sizeof(TileSpine); }

#ifdef RTF_PHASE_TIMING
extern "C" int rtf_debug_phase_cycles(unsigned long long* host, int rows, int reset) {
    cudaError_t e = cudaMemcpyFromSymbol(host, g_phase_cycles, sizeof(unsigned long long) * 16 * rows);
    if (reset && e == cudaSuccess) {
        static unsigned long long zeros[kMaxGrid][16];
        e = cudaMemcpyToSymbol(g_phase_cycles, zeros, sizeof(zeros));
    }
    return e == cudaSuccess ? 0 : 5;
}
#endif

// n: entries this call processes (a shard's, for sharded builds); n_global: the
// whole distribution (a sharded finish links all shards' tiles).
size_t build_workspace_layout(uint32_t n, uint32_t m, uint32_t flags, WsLayout* L,
                              uint32_t n_global) {
    if (n_global < n) n_global = n;
    const uint32_t tile = build_tile_size(flags);
    const uint32_t nt = (uint32_t)(((uint64_t)n + tile - 1) / tile);
    const bool sharded = n_global != n || (flags & kBuildShardedLayout);
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off += (bytes + 255) & ~(size_t)255;
        return o;
    };
    L->nt = nt;
    L->maxpart = take(sizeof(uint32_t) * 2 * kMaxGrid);
    L->counters = take(64);
    L->scale = take(16);
    L->total = take(16);
    L->excl = take(sizeof(Pfx) * (size_t)nt);
    L->rng = take(sizeof(Pfx) * 1024);  // <= THREADS ranges
    L->rpre = take(sizeof(Pfx) * 1024);
    // a sharded finish links count x nt_max rows; shards are 4096-entry aligned
    const uint32_t cap = sharded ? (uint32_t)(((uint64_t)n_global + tile - 1) / tile) +
                                       (4096u / tile) * kMaxShards
                                 : nt;
    L->nt_cap = std::max(cap, nt);
    L->spine = take(sizeof(TileSpine) * (size_t)nt);
    L->tmax = take(64 * (((size_t)L->nt_cap + 63) / 64));
    L->bmax = take(sizeof(uint32_t) * (((size_t)L->nt_cap + 63) / 64));
    L->qcap = build_queue_capacity(m);
    L->queue = take(sizeof(RunChunk) * (size_t)L->qcap);
    L->peers = take(2 * sizeof(void*) * kMaxShards);  // fused sharding: peer nodes, tables
    L->jbound = take(sizeof(uint32_t) * (kMaxShards + 1));
    L->bytes = off;
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

template <int THREADS, int VPT, bool CDF, int MINB = 2, bool POW2 = false, bool FUSED = false>
static cudaError_t launch_fused(BuildArgs& A, cudaStream_t st, int* launches) {
    auto kern = k_build<THREADS, VPT, CDF, MINB, POW2, FUSED>;
    const size_t smem = build_smem_bytes<THREADS, VPT>();  // phase B stages tile totals there
    // per instantiation and device: co-resident CTAs (the attribute is per device)
    static int max_grid_dev[kMaxDevices] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices)
        return cudaErrorInvalidDevice;
    int& max_grid = max_grid_dev[dev];
    if (!max_grid) {
        cudaError_t e = cudaSuccess;
        if (smem)
            e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        int per_sm = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, THREADS, smem);
        if (e != cudaSuccess) return e;
        if (per_sm < 1) return cudaErrorCooperativeLaunchTooLarge;
        max_grid = std::min<int>(per_sm * num_sms(), (int)kMaxGrid);
    }
    const uint32_t grid = std::max<uint32_t>(1u, std::min<uint32_t>(A.nt, (uint32_t)max_grid));
    void* args[] = {&A};
    const cudaError_t e =
        cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(THREADS), args, smem, st);
    ++*launches;
    return e;
}

cudaError_t launch_build(const float* p, uint32_t n, uint32_t m, uint32_t flags, rtf_header* hdr,
                         rtf_node* nodes, rtf_ref* table, uint64_t* cdf, void* ws,
                         const WsLayout& L, cudaStream_t st, int* launches,
                         const ShardCall* sc) {
    unsigned char* w = reinterpret_cast<unsigned char*>(ws);
    BuildArgs A;
    A.p = p;
    A.n = n;
    A.m = m;
    A.nt = L.nt;
    A.B = 62 - ceil_log2_u32(sc ? sc->n_global : n);
    A.phases = sc ? sc->phases : kPhFull;
    A.index_base = sc ? sc->index_base : 0;
    A.j_lo = sc ? sc->j_lo : 0u;
    A.j_hi = sc ? sc->j_hi : 0xffffffffu;
    A.npeer = sc ? sc->npeer : 0u;
    A.cpo = A.npeer ? m / A.npeer : 0u;
    A.peer_nodes = A.npeer ? reinterpret_cast<rtf_node* const*>(w + L.peers) : nullptr;
    A.peer_table = A.npeer ? reinterpret_cast<rtf_ref* const*>(w + L.peers) + kMaxShards : nullptr;
    A.jbound = reinterpret_cast<uint32_t*>(w + L.jbound);
    A.scale_io = reinterpret_cast<uint32_t*>(w + L.scale);
    A.shard_totals = sc ? reinterpret_cast<const Pfx*>(sc->totals) : nullptr;
    A.shard_rank = sc ? sc->rank : 0;
    A.shard_count = sc ? sc->count : 0;
    A.total_out = reinterpret_cast<Pfx*>(w + L.total);
    A.spine = reinterpret_cast<TileSpine*>(w + L.spine);
    const bool gathered = sc && sc->spine_in;
    A.spine_in = gathered ? reinterpret_cast<const TileSpine*>(sc->spine_in) : A.spine;
    A.nt_in = gathered ? sc->nt_in : L.nt;
    if (A.nt_in > L.nt_cap) return cudaErrorInvalidValue;
    A.tmax = reinterpret_cast<uint8_t*>(w + L.tmax);
    A.bmax = reinterpret_cast<uint32_t*>(w + L.bmax);
    A.maxpart = reinterpret_cast<uint32_t*>(w + L.maxpart);
    A.counters = reinterpret_cast<uint32_t*>(w + L.counters);
    A.excl = reinterpret_cast<Pfx*>(w + L.excl);
    A.rng = reinterpret_cast<Pfx*>(w + L.rng);
    A.rpre = reinterpret_cast<Pfx*>(w + L.rpre);
    static std::atomic<uint32_t> s_epoch{0};
    A.epoch = 1u + s_epoch.fetch_add(1u, std::memory_order_relaxed) % 0xfffffffeu;  // never 0
    A.hdr = hdr;
    A.nodes = nodes;
    A.table = table;
    A.queue = reinterpret_cast<RunChunk*>(w + L.queue);
    A.qcap = L.qcap;
    A.cdf = cdf;
    A.vec = ((uintptr_t)p & 15u) == 0;
    const bool small = flags & RTF_BUILD_SMALL_TILES;
    if (cdf)
        return small ? launch_fused<64, 4, true>(A, st, launches)
                     : launch_fused<512, 8, true>(A, st, launches);
    // 512 x 8 at 2 CTAs/SM measured best on B200 (vs 512x8 @1, 256x16 @2,
    // 1024x4 @1: 336 vs 399 / 352 / 403 us for config 3)
    // (2048-entry tiles at 4 or 3 CTAs/SM and 1024-entry tiles at 8 CTAs/SM
    // were measured again with the fused kernel: 293 / 315 / 399 us for c3)
    const bool pow2 = (m & (m - 1)) == 0;
    A.mshift = 63u - (uint32_t)ceil_log2_u32(m);
    if (A.npeer)  // fused ranged sharding (rtf_shard_build_peers)
        return small ? launch_fused<64, 4, false, 2, false, true>(A, st, launches)
                     : launch_fused<512, 8, false, 2, false, true>(A, st, launches);
    if (small)
        return pow2 ? launch_fused<64, 4, false, 2, true>(A, st, launches)
                    : launch_fused<64, 4, false>(A, st, launches);
    return pow2 ? launch_fused<512, 8, false, 2, true>(A, st, launches)
                : launch_fused<512, 8, false>(A, st, launches);
}

}  // namespace rtf
