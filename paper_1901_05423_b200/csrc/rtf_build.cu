// rtf_build.cu -- the forest build: ONE persistent cooperative kernel (one CTA
// pair per SM) whose phases are separated by grid-wide barriers:
//
//   A  scale      read p once: max weight bits (for E), NaN/Inf/negative flags.
//   B  totals     per 4096-entry tile: quantise (w), sum W, count positives,
//                 last positive index (aggregates of the prefix sum).
//   C  spine      CTA 0 turns the tile aggregates into exclusive prefixes and
//                 publishes T, n' and the reciprocal of T (header).
//   D  tiles      per tile (TMA-fed, dealt dynamically): block scan + tile
//                 prefix -> W_j, compaction, one exact division per leaf
//                 (key_j); per thread (8 entries): split levels lambda_j,
//                 cells and guide-table entries, the 16-B records
//                 {key_j, ~orig(j-1), ~orig(j)} staged in a 128-B-swizzled
//                 shared-memory tile; then the radix forest of the tile:
//                 every gap's parent is the nearer-in-level of its nearest
//                 greater split levels on either side (the node Alg. 1,
//                 P:1085-1121, merges it into), found in registers inside
//                 the thread's 8 gaps and across threads from per-thread
//                 spine summaries; one 4-B link per internal child into the
//                 staged records; TMA tensor stores write the records out.
//   E  cross      the links whose nearest greater split level lies in another
//                 tile (each tile's spines), then the long empty-cell runs.
//
// The result bytes do not depend on the schedule.

#include "rtf_device.cuh"
#include "rtf_internal.h"
#include <atomic>
#include <type_traits>
#include <cstdlib>
#include <cstring>
#include <cuda.h>
#include <cudaTypedefs.h>

namespace rtf {

#ifndef RTF_SHORT_RUN
#define RTF_SHORT_RUN 32
#endif
constexpr uint32_t kShortRun = RTF_SHORT_RUN;  // empty-cell runs up to this length: written in place
constexpr uint32_t kChunk = 2048;   // longer runs: queued in chunks of this many cells
constexpr uint32_t kMaxGrid = 8192; // partials capacity (CTAs of the cooperative grid)
#ifndef RTF_LOADS
#define RTF_LOADS 8  // phases A and B: 16-B loads in flight per thread
#endif
static_assert(RTF_LOADS == 4 || RTF_LOADS == 8 || RTF_LOADS == 16,
              "phase B's batches must divide a tile's 32 float4 per lane");

// workspace counters
enum : int {
    kCtrGridBar = 0,
    kCtrQueue = 1,
    kCtrTile = 2,
    kCtrRpre = 3,
};

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

// phase D's record stores: tensor maps of the node array with boxes of
// 64 << k records (k = 0..5)
constexpr int kNodeMaps = 6;
struct NodeMaps {
    CUtensorMap m[kNodeMaps];
};

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
    int32_t j_rank;       // >= 0: [j_lo, j_hi) = [jbound[j_rank], jbound[j_rank + 1]) (device)
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
    bool tma_store;               // records leave through the tensor maps (else plain stores)
    bool pack2;                   // two-leaf cells packed into the table (R20, pack2_possible(m))
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

// Dynamic shared memory of the build kernel (1024-B aligned base):
//   stage   (TILE + 64) records of 16 B: the tile's node records, record l at
//           row-swizzled position stage_pos(l + (j0 & 63)) (TMA SWIZZLE_128B)
//   p       TILE floats: the tile's weights (1-D TMA target)
//   per thread ("chunk" = its 8 entries): its packed split levels (u64, byte
//           r = gap r), first leaf, last positive entry, 1 + max split level
template <int THREADS, int VPT>
constexpr size_t build_smem_bytes() {
    return 1024 + (size_t)(THREADS * VPT + 64) * 16 + (size_t)THREADS * VPT * 4 +
           (size_t)THREADS * (8 + 4 + 4 + 1);
}

// the 128-B swizzle of a TMA tensor store with 128-B rows: 16-B chunk c of
// row r sits at chunk c ^ (r & 7).  A thread's 8 consecutive records then
// spread over all 32 banks across 8 lanes (blocked 16-B stores conflict-free).
__device__ __forceinline__ uint32_t stage_pos(uint32_t x) {
    return (x & ~7u) | ((x ^ (x >> 3)) & 7u);
}

// split level (byte) i of a thread's 8 packed split levels
__device__ __forceinline__ uint32_t lam_at(uint32_t lo, uint32_t hi, uint32_t i) {
    return __byte_perm(lo, hi, i) & 0xffu;
}

// first / last marked byte of a non-empty mask pair
__device__ __forceinline__ uint32_t byte_first(uint32_t glo, uint32_t ghi) {
    return glo ? (uint32_t)(__ffs(glo) - 1) >> 3 : 4u + ((uint32_t)(__ffs(ghi) - 1) >> 3);
}
__device__ __forceinline__ uint32_t byte_last(uint32_t glo, uint32_t ghi) {
    return ghi ? 4u + ((uint32_t)(31 - __clz(ghi)) >> 3) : (uint32_t)(31 - __clz(glo)) >> 3;
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
    // the block maxima 8 at a time (independent loads, one L2 round trip per
    // 8 blocks instead of one per block)
    for (int32_t c0 = (int32_t)bb - 1; c0 >= 0; c0 -= 8) {
        uint32_t v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = c0 - u >= 0 ? __ldcg(bmax + c0 - u) : 0u;
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (v[u] > thr) {
                const int32_t c = c0 - u;
                return 64 * c + 63 - __clzll((long long)block_rows_above(tmax, (uint32_t)c, thr));
            }
    }
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
    for (uint32_t c0 = bb + 1; c0 < nb; c0 += 8) {  // 8 block maxima per round trip
        uint32_t v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = c0 + u < nb ? __ldcg(bmax + c0 + u) : 0u;
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (v[u] > thr) {
                const uint32_t c = c0 + u;
                return (int32_t)(64 * c + __ffsll((long long)block_rows_above(tmax, c, thr)) - 1);
            }
    }
    return -1;
}

// ------------------------------------------------------------ slot-arrival check (debug builds)
// Compiled only with -DRTF_SLOT_CHECK (tools/slotcheck_target.py,
// tests/test_gpu_slotcheck.py): every link write of phases D and E also
// counts, per record child field, how often it was written, and per record,
// how often it was linked as an internal node.  A race between two writers of
// one field shows as a count of 2 even when the final bytes happen to agree;
// Alg. 1's invariant (every internal node gets exactly one
// parent) is a count of exactly 1 per non-anchor record.  The product library
// has neither.
// ------------------------------------------------------------ phase timing (debug builds)
// Compiled only with -DRTF_PHASE_TIMING (tools/phase_timing.py): thread 0 of
// each CTA accumulates clock64() deltas per phase; read with
// rtf_debug_phase_cycles().  The product library has neither.
#ifdef RTF_PHASE_TIMING
__device__ unsigned long long g_phase_cycles[kMaxGrid][16];
// per tile of phase D (the first 65536): globaltimer at its start and end, CTA
__device__ unsigned long long g_tile_ns[65536][3];
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// per block barrier of phase D: the spread of the warps' arrival times
// (last minus first, clock64 of lane 0 of each warp), accumulated in slots
// 11-13 of the CTA's row
__shared__ unsigned long long s_arr_lo[3], s_arr_hi[3];
__device__ unsigned long long g_last_warp[3][32];  // per barrier: how often warp w arrived last
#define RTF_ARRIVE(k)                                                        \
    do {                                                                     \
        if ((threadIdx.x & 31) == 0) {                                       \
            const unsigned long long c_ = (unsigned long long)clock64();     \
            atomicMin(&s_arr_lo[k], c_);                                     \
            atomicMax(&s_arr_hi[k], (c_ << 5) | (threadIdx.x >> 5));         \
        }                                                                    \
    } while (0)
#define RTF_SPREAD(k)                                                        \
    do {                                                                     \
        __syncthreads();                                                     \
        if (threadIdx.x == 0) {                                              \
            g_phase_cycles[blockIdx.x][11 + (k)] += (s_arr_hi[k] >> 5) - s_arr_lo[k]; \
            atomicAdd(&g_last_warp[k][s_arr_hi[k] & 31u], 1ull);            \
            s_arr_lo[k] = ~0ull;                                             \
            s_arr_hi[k] = 0ull;                                              \
        }                                                                    \
    } while (0)
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
#define RTF_ARRIVE(k) \
    do {              \
    } while (0)
#define RTF_SPREAD(k) \
    do {              \
    } while (0)
#endif

// ============================================================== the build kernel

template <int THREADS, int VPT, bool CDF, int MINB = 2, bool POW2 = false, bool FUSED = false>
__global__ void __launch_bounds__(THREADS, MINB)
    k_build(BuildArgs A, const __grid_constant__ NodeMaps tm) {
    constexpr int TILE = THREADS * VPT;
    constexpr int NW = THREADS / 32;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-B aligned (the TMA swizzle atom); derived from smem_raw so the
    // compiler keeps shared-memory accesses (LDS/STS, not generic LD/ST)
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    unsigned char* s_stage = smem;  // (TILE + 64) x 16-B staged records (swizzled)
    const uint32_t a_stage = smem_u32(s_stage);
    float* s_p = reinterpret_cast<float*>(smem + (size_t)(TILE + 64) * 16);  // TMA target
    unsigned long long* s_clp = reinterpret_cast<unsigned long long*>(s_p + TILE);
    uint32_t* s_ccex = reinterpret_cast<uint32_t*>(s_clp + THREADS);
    int32_t* s_clast = reinterpret_cast<int32_t*>(s_ccex + THREADS);
    uint8_t* s_cmax = reinterpret_cast<uint8_t*>(s_clast + THREADS);
    __shared__ __align__(8) uint64_t s_bar;
    __shared__ uint64_t s_w[2 * NW];
    __shared__ uint32_t s_c[2 * NW];
    __shared__ int32_t s_l[2 * NW];
    __shared__ uint32_t s_red[2 * NW];
    __shared__ uint32_t s_wmax[NW];  // per warp: max of its threads' 1 + max split level
    __shared__ uint32_t s_B[NW * 64];  // per warp and level v: its threads with a level > v
    __shared__ uint16_t s_task[NW * 256];  // per warp: its spine gaps (thread << 3 | gap)
    __shared__ __align__(16) Pfx s_rpre;  // TMA target: the next tile's range prefix
    __shared__ Pfx s_tot;
    __shared__ uint32_t s_next;
    __shared__ __align__(16) Pfx s_pin;  // TMA target: the next tile's prefix within its range
    __shared__ uint64_t s_recip;
    __shared__ Recip128 s_rc;
    __shared__ unsigned long long s_mL, s_mR;  // this tile's spines (TileSpine)
    __shared__ uint32_t s_fw, s_lw;            // first / last wall (lambda = 64) of the tile
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
    if (tid < 3) {
        s_arr_lo[tid] = ~0ull;
        s_arr_hi[tid] = 0ull;
    }
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
            // RTF_LOADS independent 16-B loads in flight per thread
            for (; q + (RTF_LOADS - 1) * THREADS < hi4; q += RTF_LOADS * THREADS) {
                float4 v[RTF_LOADS];
#pragma unroll
                for (int u = 0; u < RTF_LOADS; ++u) v[u] = ld_stream_f4(A.p + 4ull * (q + u * THREADS));
#pragma unroll
                for (int u = 0; u < RTF_LOADS; ++u) {
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
    Pfx* s_tagg = reinterpret_cast<Pfx*>(s_stage);  // phase B's tile totals; free until phase D
    constexpr uint32_t CAP = (uint32_t)(TILE + 64);
    constexpr int F = TILE / 128;  // float4 per lane per tile
    constexpr int BATCH = F < RTF_LOADS ? F : RTF_LOADS;
    // short ranges (small n): up to F / BATCH warps share a tile, so every
    // warp keeps loads in flight
    constexpr uint32_t NCH = F / BATCH;
    const uint32_t WPT = krng >= NW ? 1u : min(NCH, NW / krng >= 4 ? 4u : NW / krng >= 2 ? 2u : 1u);
    const uint32_t CAPT = CAP / WPT;
    if ((ph & kPhTotals) && b < NRG) {
        const uint32_t t_beg = b * krng, t_end = min(nt, t_beg + krng);
        Pfx run{0ull, 0u, -1};  // thread 0: the range so far
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
                            // positives as a 4-bit mask (w > 0 exactly when x > 0:
                            // the data is validated), counted once per float4
                            uint32_t pm = 0;
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                acc.W += quantize(xs[q], scale);
                                pm |= (xs[q] > 0.0f ? 1u : 0u) << q;
                            }
                            acc.cnt += __popc(pm);
                            if (pm) acc.last = e0 + 31 - __clz((int)pm);
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
    // the order tiles are dealt in: a dealing index maps to a tile (indices
    // >= nt stay out of range)
#ifdef RTF_TILE_INORDER
    auto tmap = [&](uint32_t x) -> uint32_t { return x; };
#else
    // the first wave in order (each CTA's first tile: its TMA load is issued
    // before phase C), then the rest from both ends inwards: x = G + 2k -> G
    // + k, x = G + 2k + 1 -> nt - 1 - k, so the middle of p is dealt last.
    // Skewed data is expensive at both ends of p (the deep trees of the first
    // cells, the table runs where p is large), and an expensive tile dealt
    // last leaves the other SMs idle (config 3: 262 vs 272 us in order).
    auto tmap = [&](uint32_t x) -> uint32_t {
        if (x < G || x >= nt) return x;
        const uint32_t y = x - G;
        return (y & 1u) ? nt - 1u - (y >> 1) : G + (y >> 1);
    };
#endif
    const uint32_t t_first = tmap(b);
    if (tma && tid == 0) {
        mbar_init(&s_bar, 1);
        fence_proxy_async_smem();
        if (tma_tile(t_first)) {
            mbar_arrive_expect_tx(&s_bar, TILE * 4);
            tma_load_1d(s_p, A.p + (size_t)t_first * TILE, TILE * 4, &s_bar);
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
        if (tid == 0) s_rc = recip128(T);  // the keys' reciprocal (fixed_point_r)
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
    const Recip128 rc = s_rc;

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
                if (first + k < n) A.cdf[first + k] = (W == T) ? kOne63 : fixed_point_r(W, rc, T);
                W += w[k];
            }
            __syncthreads();
        }
        return;
    }

    // ---------------------------------------------------------- D: tiles
    // Tiles are dealt dynamically (their cost varies with the zero fraction
    // and the tree shape): CTA b starts with tile b, then takes tmap(G +
    // ticket) -- both ends of p inwards.
    // The issuer thread draws each ticket one tile ahead, so the atomic's
    // latency is hidden; the TMA copy of the next tile's weights also brings
    // its prefix within its range (one mbarrier for both).  Three block
    // barriers per tile: (1) scan, (2) records + per-thread summaries written,
    // (3) every link written.
    if constexpr (!CDF) {
    static_assert(VPT == 8, "phase D packs a thread's 8 split levels into one 64-bit word");
    constexpr uint32_t kIssuer = THREADS - 1;  // TMA, tickets, stores: the last warp
    uint32_t phase = 0;
    // issuer: the dispenser's count for the tile after the next one; the
    // atomic's result is first used one tile later (tmap(G + ticket)), so its
    // latency hides behind a tile's work
    uint32_t ticket = 0;
    bool store_pending = false;  // issuer: a TMA store group may still read the stage
    auto draw = [&]() -> uint32_t { return atomicAdd(&A.counters[kCtrTile], 1u); };
    if (tid == 0) {
        s_mL = s_mR = 0ull;
        s_fw = 0xffffffffu;
        s_lw = 0u;
    }
    if (tid == kIssuer) {
        fence_proxy_async_global();  // phase B's prefixes, read by TMA below
        if (ph & kPhTiles) ticket = draw();
    }
    if (ph & kPhTiles) wait_rpre();
    if (tid == kIssuer) fence_proxy_async_global();  // the range prefixes, read by TMA below

    // Gaps above level v in a thread's packed split levels: byte + 127 - v
    // reaches bit 7 exactly when byte > v (bytes <= 64, so no carries).
    auto above = [](uint32_t lo, uint32_t hi, uint32_t v, uint32_t& glo, uint32_t& ghi) {
        const uint32_t c = __byte_perm(127u - v, 0u, 0u);  // 127 - v in every byte
        glo = (lo + c) & 0x80808080u;
        ghi = (hi + c) & 0x80808080u;
    };
    // the same flags as 8 bits (bit r: gap r above v)
    auto mask8 = [](uint32_t glo, uint32_t ghi) -> uint32_t {
        return ((glo * 0x00204081u) >> 28) | (((ghi * 0x00204081u) >> 28) << 4);
    };
    // The nearest greater split level of a gap at level v of thread c, to its
    // right / left outside the thread: the first / last gap above v of the
    // nearest thread whose largest level exceeds v (per-warp tables s_B).
    auto search_right = [&](uint32_t c, uint32_t v, uint32_t& gap, uint32_t& lev) -> bool {
        const uint32_t w = c >> 5, l = c & 31u;
        uint32_t mk = s_B[w * 64 + v] & ~((2u << l) - 1u);
        uint32_t u;
        if (mk) {
            u = (w << 5) + (uint32_t)__ffs(mk) - 1u;
        } else {
            uint32_t w2 = w + 1u;
            while (w2 < (uint32_t)NW && s_wmax[w2] <= v + 1u) ++w2;
            if (w2 >= (uint32_t)NW) return false;
            u = (w2 << 5) + (uint32_t)__ffs(s_B[w2 * 64 + v]) - 1u;
        }
        const unsigned long long lp = s_clp[u];
        uint32_t glo, ghi;
        above((uint32_t)lp, (uint32_t)(lp >> 32), v, glo, ghi);
        const uint32_t pos = (uint32_t)__ffs(mask8(glo, ghi)) - 1u;
        lev = lam_at((uint32_t)lp, (uint32_t)(lp >> 32), pos);
        gap = s_ccex[u] + pos;
        return true;
    };
    auto search_left = [&](uint32_t c, uint32_t v, uint32_t& gap, uint32_t& lev) -> bool {
        const uint32_t w = c >> 5, l = c & 31u;
        uint32_t mk = s_B[w * 64 + v] & ((1u << l) - 1u);
        uint32_t u;
        if (mk) {
            u = (w << 5) + 31u - (uint32_t)__clz(mk);
        } else {
            int32_t w2 = (int32_t)w - 1;
            while (w2 >= 0 && s_wmax[w2] <= v + 1u) --w2;
            if (w2 < 0) return false;
            u = ((uint32_t)w2 << 5) + 31u - (uint32_t)__clz(s_B[w2 * 64 + v]);
        }
        const unsigned long long lp = s_clp[u];
        uint32_t glo, ghi;
        above((uint32_t)lp, (uint32_t)(lp >> 32), v, glo, ghi);
        const uint32_t pos = 31u - (uint32_t)__clz(mask8(glo, ghi));
        lev = lam_at((uint32_t)lp, (uint32_t)(lp >> 32), pos);
        gap = s_ccex[u] + pos;
        return true;
    };

    for (uint32_t t = t_first; (ph & kPhTiles) && t < nt; t = s_next) {
#ifdef RTF_PHASE_TIMING
        if (tid == 0 && t < 65536) {
            g_tile_ns[t][0] = globaltimer_ns();
            g_tile_ns[t][2] = b;
        }
#endif
        const uint32_t first = t * TILE + tid * VPT;  // local index into p (global: + ib)

        // (0) weights of this thread's VPT consecutive entries
        float x[VPT];
        Pfx pre;
        if (tma_tile(t)) {
#ifdef RTF_PHASE_TIMING
            const long long tw1_ = clock64();
            mbar_wait(&s_bar, phase);
            if (tid == 0) g_phase_cycles[blockIdx.x][10] += (unsigned long long)(clock64() - tw1_);
#else
            mbar_wait(&s_bar, phase);
#endif
            phase ^= 1u;
            pre = t == t_first ? tile_prefix(t) : combine(s_rpre, s_pin);
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
        // (1) quantise; block scan of (W, positives) -- warp scans, one barrier,
        // then every warp scans the warp totals itself
        uint64_t w[VPT];
        uint64_t tw = 0;
        uint32_t posmask_in = 0;
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
            w[k] = quantize(x[k], scale);
            tw += w[k];
            posmask_in |= (x[k] > 0.0f ? 1u : 0u) << k;  // w > 0 exactly when x > 0
        }
        const uint32_t tc_in = __popc(posmask_in);
        s_clast[tid] = posmask_in ? 31 - __clz((int)posmask_in) : -1;
        uint64_t wi = tw;
        uint32_t ci = tc_in;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint64_t tw2 = shfl_up_u64(wi, d);
            const uint32_t tc2 = __shfl_up_sync(0xffffffffu, ci, d);
            if (lane >= d) {
                wi += tw2;
                ci += tc2;
            }
        }
        if (lane == 31) {
            s_w[warp] = wi;
            s_c[warp] = ci;
        }
        if (store_pending) {  // the previous tile's records have left the stage
#ifdef RTF_PHASE_TIMING
            const long long tw0_ = clock64();
            bulk_wait_read0();
            if (tid == kIssuer) g_phase_cycles[blockIdx.x][9] += (unsigned long long)(clock64() - tw0_);
#else
            bulk_wait_read0();
#endif
            store_pending = false;
        }
        RTF_ARRIVE(0);
        __syncthreads();
        RTF_SPREAD(0);
        RTF_TICK(3);
        if (tid == kIssuer) {  // every thread has its weights: the next tile can stream in
            const uint32_t nx = tmap(G + ticket);
            s_next = nx;  // read at the end of this tile
            if (tma_tile(nx)) {  // the weights, the prefix within the range and the range's prefix
                fence_proxy_async_smem();
                mbar_arrive_expect_tx(&s_bar, TILE * 4 + 2u * (uint32_t)sizeof(Pfx));
                tma_load_1d(s_p, A.p + (size_t)nx * TILE, TILE * 4, &s_bar);
                tma_load_1d(&s_pin, A.excl + nx, (uint32_t)sizeof(Pfx), &s_bar);
                tma_load_1d(&s_rpre, A.rpre + nx / krng, (uint32_t)sizeof(Pfx), &s_bar);
            }
            if (nx < nt) ticket = draw();
        }
        uint64_t w_ex;
        uint32_t c_ex_in, cnt;
        {
            uint64_t ww = lane < NW ? s_w[lane] : 0ull;
            uint32_t cc = lane < NW ? s_c[lane] : 0u;
#pragma unroll
            for (int d = 1; d < NW; d <<= 1) {
                const uint64_t tw2 = shfl_up_u64(ww, d);
                const uint32_t tc2 = __shfl_up_sync(0xffffffffu, cc, d);
                if (lane >= d) {
                    ww += tw2;
                    cc += tc2;
                }
            }
            const uint64_t wb = __shfl_sync(0xffffffffu, ww, warp ? warp - 1 : 0);
            const uint32_t cb = __shfl_sync(0xffffffffu, cc, warp ? warp - 1 : 0);
            cnt = __shfl_sync(0xffffffffu, cc, NW - 1);
            w_ex = (warp ? wb : 0ull) + wi - tw;
            c_ex_in = (warp ? cb : 0u) + ci - tc_in;
        }
        // The rest of the tile, specialised for tiles whose TILE entries are
        // all positive (ALLPOS: leaves = entries, every test on the positive
        // mask folds away) and for the general case; the choice is uniform
        // across the CTA (cnt), so the barriers inside stay CTA-wide.
        auto tile_body = [&](auto allpos) {
        constexpr bool ALLPOS = decltype(allpos)::value;
        const uint32_t posmask = ALLPOS ? 0xffu : posmask_in;
        const uint32_t tc = ALLPOS ? (uint32_t)VPT : tc_in;
        const uint32_t c_ex = ALLPOS ? tid * (uint32_t)VPT : c_ex_in;
        const uint32_t j0 = pre.cnt;      // global index of the tile's first leaf
        const uint32_t sh = j0 & 63u;     // record l is staged at stage_pos(l + sh)
        // the previous positive entry (the first own leaf's left neighbour)
        int32_t prevo = -1;
        if (ALLPOS) {
            prevo = tid ? (int32_t)(first - 1u) + ib : (j0 ? pre.last : -1);
        } else if (tc) {
            int32_t u = (int32_t)tid - 1;
            while (u >= 0 && s_clast[u] < 0) --u;
            prevo = u >= 0 ? (int32_t)(t * TILE + (uint32_t)u * VPT) + s_clast[u] + ib
                           : (j0 ? pre.last : -1);
        }

        // (2) one exact division per positive entry: w[k] holds key_j from here on;
        // kn = the key of the first leaf after this thread's entries ("1" at the end)
        uint64_t kn = kOne63;
        {
            uint64_t W = pre.W + w_ex;
#pragma unroll
            for (int k = 0; k < VPT; ++k) {
                const uint64_t wk = w[k];
                if (ALLPOS || wk) w[k] = fixed_point_r(W, rc, T);
                W += wk;
            }
            if (tc && W != T) kn = fixed_point_r(W, rc, T);
        }

        // (3) own gaps, last to first: split level lambda (byte r of lampack =
        // gap c_ex + r, between leaves c_ex + r and c_ex + r + 1); at a cell
        // boundary the guide-table entries the leaf owes: the
        // next cell's anchor -- or, when the next leaf is alone in its cell,
        // the two-interval entry (reading R18) -- and the empty cells between
        uint64_t lampack = 0;
        uint32_t lmax = 0;   // largest own split level
        uint64_t key_f = 0;  // the first own leaf: key, original index
        int32_t orig_f = 0;
        if (tc) {
            if (j0 == 0 && c_ex == 0) st_cell(table_at(0), 0, 0u, 0);  // leaf 0 (key 0) anchors cell 0
            uint64_t nxt = kn;
            uint32_t cn = POW2 ? (uint32_t)(kn >> A.mshift) : (kn == kOne63 ? m : cell_of(kn, m));
            uint32_t lam_nx = 0xffu;  // split level after the next leaf (0xff: another thread's)
            int32_t orig_nx = 0;
            uint32_t r = tc;
#pragma unroll
            for (int k = VPT - 1; k >= 0; --k) {
                if ((posmask >> k) & 1u) {
                    --r;
                    const uint64_t key = w[k];
                    const int32_t i = (int32_t)(first + k) + ib;
                    uint32_t cell, lam;
                    if (POW2) {  // a cell boundary lies between iff the keys differ at or
                                 // above bit mshift (kn = 2^63 "1" differs at bit 63)
                        const uint32_t d = split_level(key, nxt);
                        lam = d >= A.mshift ? kLamBoundary : d;
                        cell = (uint32_t)(key >> A.mshift);
                    } else {
                        cell = cell_of(key, m);
                        lam = (cn != cell) ? kLamBoundary : split_level(key, nxt);
                    }
                    lampack = (lampack << 8) | lam;
                    lmax = max(lmax, lam);
                    if (lam == kLamBoundary) {
                        const int32_t anchor = (int32_t)(j0 + c_ex + r + 1u);
                        if (cn < m) {
                            uint2 e = make_uint2(0u, (uint32_t)anchor);
                            if (lam_nx == kLamBoundary)  // the next leaf is alone in cell cn
                                e = single_leaf_cell(nxt, orig_nx, i, anchor);
                            st_cell(table_at(cn), cn, e.x, (int32_t)e.y);
                        }
                        if (FUSED)  // the first leaf of every owner boundary k cpo in (cell, cn]
                            for (uint32_t q = cell / A.cpo + 1; q <= min(A.npeer, cn / A.cpo); ++q)
                                A.jbound[q] = (uint32_t)anchor;
                        const uint32_t len = cn - cell - 1;
                        if (len <= kShortRun) {
                            if (FUSED) {  // the run may cross an owner's boundary
                                for (uint32_t g = cell + 1; g < cn; ++g) st_cell(table_at(g), g, 0u, ~i);
                            } else {
                                fill_run(A.table, cell + 1, cn, ~i);
                            }
                        } else {
                            table_queue(A.counters, A.queue, A.qcap, i, cell, len);
                        }
                    }
                    lam_nx = lam;
                    orig_nx = i;
                    nxt = key;
                    cn = cell;
                }
            }
            key_f = nxt;
            orig_f = orig_nx;
            if (c_ex == 0) s_ref0 = ~orig_f;  // the tile's first leaf: linked in phase E
        }
        const uint32_t lo32 = (uint32_t)lampack, hi32 = (uint32_t)(lampack >> 32);

        if (tid == 0) sts_u32(a_stage + 16u * stage_pos(cnt + sh) + 8u, (uint32_t)kNoLink);
        // (4) the staged records {key_j, ~orig(j-1), ~orig(j)}: the left child
        // of an anchor (Fig. 6 caption P:1276-1277) or of an internal node whose
        // left child is the leaf j-1, the right child of a node whose right
        // child is the leaf j.  Every other child is an internal node and is
        // linked over it in (6).
        {
            int32_t po = prevo;
            uint32_t l = c_ex + sh;
#pragma unroll
            for (int k = 0; k < VPT; ++k) {
                if ((posmask >> k) & 1u) {
                    const int32_t i = (int32_t)(first + k) + ib;
                    const uint64_t key = w[k];
                    sts_v4(a_stage + 16u * stage_pos(l),
                           make_uint4((uint32_t)key, (uint32_t)(key >> 32),
                                      (uint32_t)~(po >= 0 ? po : i), (uint32_t)~i));
                    po = i;
                    ++l;
                }
            }
        }

        // (5) this thread's summary (its packed split levels, first leaf, 1 +
        // its largest level) and the warp's level tables s_B[v] = the lanes
        // whose largest level exceeds v; the tile's first and last wall
        const uint32_t encmax = tc ? lmax + 1u : 0u;
        s_clp[tid] = lampack;
        s_ccex[tid] = c_ex;
        s_cmax[tid] = (uint8_t)encmax;
        {
            const uint32_t wm = __reduce_max_sync(0xffffffffu, encmax);
            if (lane == 0) s_wmax[warp] = wm;
#ifdef RTF_WALL_ATOMICS_PER_THREAD
            if (lmax == kLamBoundary && tc) {
                uint32_t glo, ghi;
                above(lo32, hi32, kLamBoundary - 1u, glo, ghi);  // the walls
                atomicMin(&s_fw, c_ex + byte_first(glo, ghi));
                atomicMax(&s_lw, c_ex + byte_last(glo, ghi));
            }
#else
            // the warp's first wall (its lowest lane with one) and last wall:
            // two shared atomics per warp, not two per thread
            const uint32_t wb = __ballot_sync(0xffffffffu, lmax == kLamBoundary && tc);
            if (wb) {
                const uint32_t lf = (uint32_t)__ffs(wb) - 1u, ll = 31u - (uint32_t)__clz(wb);
                if ((uint32_t)lane == lf || (uint32_t)lane == ll) {
                    uint32_t glo, ghi;
                    above(lo32, hi32, kLamBoundary - 1u, glo, ghi);  // the walls
                    if ((uint32_t)lane == lf) atomicMin(&s_fw, c_ex + byte_first(glo, ghi));
                    if ((uint32_t)lane == ll) atomicMax(&s_lw, c_ex + byte_last(glo, ghi));
                }
            }
#endif
            __syncwarp();
            // lane L: the tables of levels L and L + 32 from the warp's 32 maxima
            const uint4 m0 = *reinterpret_cast<const uint4*>(s_cmax + (warp << 5));
            const uint4 m1 = *reinterpret_cast<const uint4*>(s_cmax + (warp << 5) + 16);
            const uint32_t mw[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint32_t v = (uint32_t)lane + 32u * h;  // encodings > v + 1
                const uint32_t c = __byte_perm(126u - v, 0u, 0u);
                uint32_t bits = 0;
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    bits |= ((((mw[q] + c) & 0x80808080u) * 0x00204081u) >> 28) << (4 * q);
                s_B[warp * 64 + v] = bits;
            }
        }
        RTF_ARRIVE(1);
        __syncthreads();
        RTF_SPREAD(1);
        RTF_TICK(4);

        // (5b) cells holding exactly two leaves a, a+1 (reading R20) with
        // leaf a-1 in this tile (the rest: phase E): packed into the table by
        // the owner of leaf a+1, replacing the anchor written in (3), from
        // the walls (split level 64) after leaves a+1 and a-1 and none after
        // leaf a, and the staged records of leaves a, a+1 (keys; as prefilled,
        // ~orig(a-1) = the anchor's child0 and ~orig(a+1) = child1 of the
        // cell root)
        if (A.pack2 && tc) {
            uint32_t glo, ghi;
            above(lo32, hi32, kLamBoundary - 1u, glo, ghi);  // the walls
            const uint32_t wm = (((glo * 0x00204081u) >> 28) & 0xfu) | ((((ghi * 0x00204081u) >> 28) & 0xfu) << 4);
            // bit r + 2: a wall after own leaf r; bits 1, 0: after the two
            // leaves before own leaf 0 (earlier threads of the tile)
            uint32_t ext = wm << 2;
            if ((wm & 3u) && c_ex > 0) {
                int32_t u = (int32_t)tid - 1;
                while (s_cmax[u] == 0) --u;
                const unsigned long long lpu = s_clp[u];
                const uint32_t cu = c_ex - s_ccex[u];  // leaves of thread u
                ext |= (lam_at((uint32_t)lpu, (uint32_t)(lpu >> 32), cu - 1u) == kLamBoundary) ? 2u : 0u;
                uint32_t lb = 0xffu;
                if (cu >= 2) {
                    lb = lam_at((uint32_t)lpu, (uint32_t)(lpu >> 32), cu - 2u);
                } else {
                    int32_t u2 = u - 1;
                    while (u2 >= 0 && s_cmax[u2] == 0) --u2;
                    if (u2 >= 0) {
                        const unsigned long long lp2 = s_clp[u2];
                        lb = lam_at((uint32_t)lp2, (uint32_t)(lp2 >> 32), s_ccex[u] - s_ccex[u2] - 1u);
                    }
                }
                ext |= lb == kLamBoundary ? 1u : 0u;
            }
            // own leaf r ends a two-leaf cell: walls after r and r - 2, none after r - 1
            uint32_t pat = (ext >> 2) & ~(ext >> 1) & ext & ((1u << tc) - 1u);
            pat &= c_ex >= 2 ? 0xffu : (c_ex == 1 ? 0xfeu : 0xfcu);  // leaf a-1 in this tile
            while (pat) {
                const uint32_t q = c_ex + (uint32_t)__ffs(pat) - 1u;  // local index of leaf a+1
                pat &= pat - 1u;
                const uint4 ra = lds_v4(a_stage + 16u * stage_pos(q - 1u + sh));
                const uint4 rb = lds_v4(a_stage + 16u * stage_pos(q + sh));
                const uint64_t kb = (uint64_t)rb.x | ((uint64_t)rb.y << 32);
                const uint32_t g = cell_fn(kb);
                const uint2 e = pack2_cell(g, A.mshift - 31u, (uint64_t)ra.x | ((uint64_t)ra.y << 32),
                                           kb, ~(int32_t)ra.z, ~(int32_t)rb.w);
                if (e.x) st_cell(table_at(g), g, e.x, (int32_t)e.y);
            }
        }

        // (6) the forest.  A gap's node hangs under the nearer-in-level of its
        // nearest greater split levels on either side (Alg. 1's merge order,
        // P:1101-1113; equal levels only between walls: the right child of the
        // left wall's anchor) -- as the right child of the left one or the
        // left child of the right one.  Found inside the thread's 8 gaps by
        // byte arithmetic, otherwise from the other threads' summaries; a gap
        // whose nearest greater level lies outside the tile is a spine gap of
        // the tile (phase E).
        // The first own leaf may close a one-leaf cell whose left wall is the
        // previous thread's last gap (the two-interval entry, reading R18).
        if (tc && c_ex > 0 && (lo32 & 0xffu) == kLamBoundary) {
            int32_t u = (int32_t)tid - 1;
            while (s_cmax[u] == 0) --u;  // c_ex > 0: some earlier thread has a leaf
            const unsigned long long lpu = s_clp[u];
            const uint32_t lastu = s_ccex[tid] - s_ccex[u] - 1u;  // its last gap
            if (lam_at((uint32_t)lpu, (uint32_t)(lpu >> 32), lastu) == kLamBoundary) {
                const int32_t a = (int32_t)(j0 + c_ex);
                const uint2 e = single_leaf_cell(key_f, orig_f, prevo, a);
                if ((int32_t)e.y != a) st_cell(table_at(cell_fn(key_f)), cell_fn(key_f), e.x, (int32_t)e.y);
            }
        }
        {
            // gap g's node under its parent: the right child of the left
            // neighbour gl (slot gl + 1) if vl <= vr, else the left child of gr
            // (slot cnt, the next tile's first record, has a stage row too: only
            // its child0 -- the left child of the tile's last gap -- is written,
            // and it goes to the tile's spine row, not to the records)
            auto link = [&](uint32_t g, uint32_t gl, uint32_t vl, uint32_t gr, uint32_t vr) {
                const uint32_t node = j0 + g + 1u;
                const bool right = vl <= vr;
                const uint32_t slot = (right ? gl : gr) + 1u;
                sts_u32(a_stage + 16u * stage_pos(slot + sh) + (right ? 12u : 8u), node);
                RTF_SLOT(j0 + slot, right ? 1u : 0u, node);
            };
            // (a) both nearest greater levels inside the window of this thread
            // and its two neighbours (24 gaps; a neighbour without leaves has
            // no gaps): link now; the others become tasks (thread << 5 | r << 2
            // | 1), about a sixth of the gaps for random split levels
            const unsigned long long lpl = tid > 0 ? s_clp[tid - 1] : 0ull;
            const unsigned long long lpr = tid + 1 < (uint32_t)THREADS ? s_clp[tid + 1] : 0ull;
            const uint32_t llo = (uint32_t)lpl, lhi = (uint32_t)(lpl >> 32);
            const uint32_t rlo = (uint32_t)lpr, rhi = (uint32_t)(lpr >> 32);
            const uint32_t cel = tid > 0 ? s_ccex[tid - 1] : 0u, cer = c_ex + tc;
            uint32_t ntask = 0, tasks[VPT];
#pragma unroll
            for (int r = 0; r < VPT; ++r) {
                const uint32_t v = lam_at(lo32, hi32, (uint32_t)r);
                tasks[r] = 0;
                if ((uint32_t)r < tc && v < kLamBoundary) {
                    uint32_t glo, ghi;
                    above(lo32, hi32, v, glo, ghi);
                    const uint32_t m8 = mask8(glo, ghi);
                    const uint32_t ml = m8 & ((1u << r) - 1u), mr = m8 & (0xfeu << r);
                    uint32_t gl, vl, gr, vr;
                    bool ok = true;
                    if (ml) {
                        const uint32_t q = 31u - (uint32_t)__clz(ml);
                        gl = c_ex + q;
                        vl = lam_at(lo32, hi32, q);
                    } else {
                        above(llo, lhi, v, glo, ghi);
                        const uint32_t mm = mask8(glo, ghi);
                        const uint32_t q = 31u - (uint32_t)__clz(mm);
                        gl = cel + q;
                        vl = lam_at(llo, lhi, q);
                        ok = mm != 0u;
                    }
                    if (mr) {
                        const uint32_t q = (uint32_t)__ffs(mr) - 1u;
                        gr = c_ex + q;
                        vr = lam_at(lo32, hi32, q);
                    } else {
                        above(rlo, rhi, v, glo, ghi);
                        const uint32_t mm = mask8(glo, ghi);
                        const uint32_t q = (uint32_t)__ffs(mm) - 1u;
                        gr = cer + q;
                        vr = lam_at(rlo, rhi, q);
                        ok = ok && mm != 0u;
                    }
                    if (ok) {
                        link(c_ex + r, gl, vl, gr, vr);
                    } else {
                        tasks[r] = tid << 5 | (uint32_t)r << 2 | 1u;
                        ++ntask;
                    }
                }
            }
            // (b) the tasks, compacted per warp so that every lane searches
            uint32_t incl = ntask;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t t2 = __shfl_up_sync(0xffffffffu, incl, d);
                if (lane >= d) incl += t2;
            }
            const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
            uint16_t* q = s_task + warp * 256;
            uint32_t qi = incl - ntask;
#pragma unroll
            for (int r = 0; r < VPT; ++r)
                if (tasks[r]) q[qi++] = (uint16_t)tasks[r];
            __syncwarp();
            for (uint32_t k = lane; k < total; k += 32) {
                const uint32_t task = q[k], o = task >> 5, r = (task >> 2) & 7u;
                const unsigned long long lp = s_clp[o];
                const uint32_t lo = (uint32_t)lp, hi = (uint32_t)(lp >> 32), ce = s_ccex[o];
                const uint32_t v = lam_at(lo, hi, r), g = ce + r;
                uint32_t glo, ghi;
                above(lo, hi, v, glo, ghi);
                const uint32_t m8 = mask8(glo, ghi);
                // in-thread neighbours, else the search (which finds the
                // window's neighbour threads first; garbage on a searched side)
                const uint32_t ml = m8 & ((1u << r) - 1u), mr = m8 & (0xfeu << r);
                const uint32_t nl = 31u - (uint32_t)__clz(ml);
                const uint32_t nr = (uint32_t)__ffs(mr) - 1u;
                uint32_t gl = ce + nl, vl = lam_at(lo, hi, nl), gr = ce + nr, vr = lam_at(lo, hi, nr);
                bool hl = true, hr = true;
                if (!ml) hl = search_left(o, v, gl, vl);
                if (!mr) hr = search_right(o, v, gr, vr);
                if (hl && hr) {
                    link(g, gl, vl, gr, vr);
                } else {  // a spine gap of the tile: phase E links it
                    if (!hl) {
                        s_iL[v] = (uint16_t)g;
                        atomicOr(&s_mL, 1ull << v);
                    }
                    if (!hr) {
                        s_iR[v] = (uint16_t)g;
                        atomicOr(&s_mR, 1ull << v);
                    }
                }
            }
        }
        fence_proxy_async_smem();  // the staged records are read by the TMA store below
        RTF_ARRIVE(2);
        __syncthreads();
        RTF_SPREAD(2);
        RTF_TICK(5);

        // (7) records out: whole 64-record blocks (1024-B aligned in the stage)
        // by TMA tensor stores, the unaligned head and tail by the threads
        {
            const uint32_t e1 = j0 + cnt;
            uint32_t a0 = (j0 + 63u) & ~63u, a1 = e1 & ~63u;
            if (!A.tma_store || FUSED || a1 <= a0) a0 = a1 = e1;  // every record by the threads
            if (tid == kIssuer && a1 > a0) {
                const uint32_t base = j0 & ~63u;
                // the largest power-of-two box (2048 .. 64 records) that fits:
                // at most 6 store instructions for the aligned middle
                for (uint32_t a = a0; a < a1;) {
                    const uint32_t left = (a1 - a) >> 6;  // whole 64-record blocks
                    const int k = min(5, 31 - __clz((int)left));
                    tma_store_2d(&tm.m[k], 0, (int)(a >> 3), s_stage + 16u * (a - base));
                    a += 64u << k;
                }
                bulk_commit();
                store_pending = true;
            }
            const uint32_t nhead = a0 - j0, ntot = nhead + (e1 - a1);
            for (uint32_t q = tid; q < ntot; q += THREADS) {
                const uint32_t l = q < nhead ? q : a1 - j0 + (q - nhead);
                const uint4 rec = lds_v4(a_stage + 16u * stage_pos(l + sh));
                if (FUSED) {  // to the rank owning the record's cell (peer memory)
                    const uint64_t key = (uint64_t)rec.x | ((uint64_t)rec.y << 32);
                    reinterpret_cast<uint4*>(A.peer_nodes[cell_fn(key) / A.cpo] + j0)[l] = rec;
                } else {
                    reinterpret_cast<uint4*>(A.nodes + j0)[l] = rec;
                }
            }
        }
        // (8) the tile's spine row for phase E
        {
            TileSpine* row = A.spine + t;
            // by the middle warps: warp 0 starts the next tile's bookkeeping
            // and warp 15 holds the issuer
            constexpr uint32_t kRowT = THREADS >= 512 ? 256u : 0u;
            for (uint32_t u = tid - kRowT; u < 64; u += THREADS) {
                row->iL[u] = s_iL[u];
                row->iR[u] = s_iR[u];
            }
            if (tid == kRowT) {
                const uint32_t walls = s_fw != 0xffffffffu ? 3u : 0u;
                row->mL = s_mL;
                row->mR = s_mR;
                row->j0 = j0;
                row->cnt = cnt;
                row->walls = walls;
                row->iL[64] = walls ? (uint16_t)s_fw : (uint16_t)0;
                row->iR[64] = walls ? (uint16_t)s_lw : (uint16_t)0;
                row->c0_next = cnt ? (int32_t)lds_u32(a_stage + 16u * stage_pos(cnt + sh) + 8u) : kNoLink;
                row->ref0 = cnt ? s_ref0 : 0;
                // phase E's row maxima: 1 + the largest split level, 0 if empty
                const uint32_t enc = !cnt ? 0u
                                     : walls ? kLamBoundary + 1u
                                             : 64u - (uint32_t)__clzll((long long)s_mL);
                A.tmax[t] = (uint8_t)enc;
                if (enc) atomicMax(&A.bmax[t >> 6], enc);
                s_mL = s_mR = 0ull;  // the next tile's writers follow its barriers
                s_fw = 0xffffffffu;
                s_lw = 0u;
            }
        }
        };
        if (cnt == (uint32_t)TILE) tile_body(std::true_type{});
        else tile_body(std::false_type{});
        RTF_TICK(6);
#ifdef RTF_PHASE_TIMING
        if (tid == 0 && t < 65536) g_tile_ns[t][1] = globaltimer_ns();
#endif
    }
    if (store_pending) {  // every record written before the grid barrier
        bulk_wait0();
        fence_proxy_async_global();
    }
    }  // !CDF
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
        const uint32_t jlo = A.j_rank >= 0 ? __ldcg(&A.jbound[A.j_rank]) : A.j_lo;
        const uint32_t jhi = A.j_rank >= 0 ? __ldcg(&A.jbound[A.j_rank + 1]) : A.j_hi;
        auto local = [&](uint32_t slot) { return slot >= jlo && slot < jhi; };
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
                        if (local(j0)) {
                            A.nodes[j0].child[1] = ref;
                            RTF_SLOT(j0, 1u, -1);
                        }
                    } else if (local(j0 + 1)) {
                        A.nodes[j0 + 1].child[0] = ref;
                        RTF_SLOT(j0 + 1, 0u, -1);
                    }
                    if ((lamp & lam0 & kLamBoundary) != 0 && local(j0)) {  // a one-leaf cell
                        const uint64_t key = __ldcg(&A.nodes[j0].key);
                        const uint2 e = single_leaf_cell(key, ~ref, ~__ldcg(&A.nodes[j0].child[0]),
                                                         (int32_t)j0);
                        if ((int32_t)e.y != (int32_t)j0)
                            st_cell(A.table, cell_fn(key), e.x, (int32_t)e.y);
                    }
                    // two-leaf cells across the row boundary (R20; (5b) packs the rest):
                    // leaves {j0, j0+1} (the row's first gap inside the cell, its
                    // second a wall) or {j0-1, j0} (the previous row's last gap
                    // inside the cell, the one before it a wall); the records hold
                    // the keys and, as prefilled, ~orig(a-1) (anchor child0) and
                    // ~orig(a+1) (child1 of the cell root)
                    if (A.pack2) {
                        uint32_t a = 0xffffffffu;
                        if (lamp == kLamBoundary && lam0 < kLamBoundary && wL &&
                            __ldcg(&S->iL[64]) == 1u && j0 >= 1) {
                            a = j0;
                        } else if (lam0 == kLamBoundary && lamp < kLamBoundary && u >= 0 && j0 >= 2) {
                            const TileSpine* U = SP + u;
                            const uint32_t cu = __ldcg(&U->cnt);
                            bool wall2;  // the gap before leaf j0-1 is a wall
                            if (cu >= 2) {
                                wall2 = (__ldcg(&U->walls) & 2u) && __ldcg(&U->iR[64]) == cu - 2u;
                            } else {
                                const int32_t u2 = row_left(A.tmax, A.bmax, (uint32_t)u, 0u);
                                wall2 = u2 < 0 || spine_lowest(__ldcg(&SP[u2].mR),
                                                               __ldcg(&SP[u2].walls) & 2u) == kLamBoundary;
                            }
                            if (wall2) a = j0 - 1;
                        }
                        if (a != 0xffffffffu && local(a)) {
                            const uint64_t ka = __ldcg(&A.nodes[a].key), kb = __ldcg(&A.nodes[a + 1].key);
                            const uint32_t g = cell_fn(kb);
                            const uint2 e = pack2_cell(g, A.mshift - 31u, ka, kb,
                                                       ~__ldcg(&A.nodes[a].child[0]),
                                                       ~__ldcg(&A.nodes[a + 1].child[1]));
                            if (e.x) st_cell(A.table, g, e.x, (int32_t)e.y);
                        }
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
                        if (local((uint32_t)(gL + 1))) {
                            A.nodes[gL + 1].child[1] = node;
                            RTF_SLOT(gL + 1, 1u, node);
                        }
                    } else if (local((uint32_t)(gR + 1))) {
                        A.nodes[gR + 1].child[0] = node;
                        RTF_SLOT(gR + 1, 0u, node);
                    }
                }
            }
        }
    }
    RTF_TICK(14);
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

// threads per CTA of the production tile (8 entries each), CTAs per SM
#ifndef RTF_TILE_THREADS
#define RTF_TILE_THREADS 512
#endif
constexpr int kTT = RTF_TILE_THREADS;
#ifndef RTF_TILE_MINB
#define RTF_TILE_MINB (1024 / RTF_TILE_THREADS)
#endif
constexpr int kTB = RTF_TILE_MINB;

struct TileCfg {
    int threads, vpt;
};

static inline TileCfg tile_cfg(uint32_t flags) {
    return (flags & RTF_BUILD_SMALL_TILES) ? TileCfg{32, 8} : TileCfg{kTT, 8};
}

uint32_t build_tile_size(uint32_t flags) {
    const TileCfg c = tile_cfg(flags);
    return (uint32_t)(c.threads * c.vpt);
}

uint32_t build_queue_capacity(uint32_t m) { return m / (kShortRun + 1u) + m / kChunk + 64u; }

size_t spine_row_bytes() { return sizeof(TileSpine); }

// ------------------------------------------------------------ phase A per chunk
// Phase A of a build from host memory (rtf_build_host), run on each chunk as
// its host-to-device copy lands, so the scan for the largest weight overlaps
// the rest of the copy: the same two integer maxima of the raw float bits as
// phase A (exact flags when a chunk holds invalid data), MAX-reduced into the
// scale word {bits of max p, NaN, Inf, negative} the build then reads instead
// of running phase A (the scale word of a sharded build, kPhScale absent).
__global__ void __launch_bounds__(256) k_scale_chunk(const float* __restrict__ p, uint32_t n,
                                                     uint32_t* __restrict__ scale_io) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x, G = gridDim.x * blockDim.x;
    const bool vec = ((uintptr_t)p & 15u) == 0;
    const uint32_t n4 = vec ? n >> 2 : 0u;
    // every element this thread owns: float4 q = tid + k G, then the scalar tail
    auto each = [&](auto&& f) {
        for (uint32_t q = tid; q < n4; q += G) {
            const float4 v = ld_stream_f4(p + 4ull * q);
            f(v.x);
            f(v.y);
            f(v.z);
            f(v.w);
        }
        for (uint32_t i = 4 * n4 + tid; i < n; i += G) f(p[i]);
    };
    int32_t smax = 0;
    uint32_t umax = 0;
    each([&](float x) {
        smax = max(smax, __float_as_int(x));
        umax = max(umax, __float_as_uint(x));
    });
    uint32_t fl = 0;
    if (smax >= 0x7f800000 || umax > 0x80000000u)  // invalid data among this thread's: exact flags
        each([&](float x) {
            if (x != x) fl |= RTF_DATA_NAN;
            else if (fabsf(x) == __int_as_float(0x7f800000)) fl |= RTF_DATA_INF;
            else if (x < 0.0f) fl |= RTF_DATA_NEG;
        });
    const uint32_t mx = __reduce_max_sync(0xffffffffu, (uint32_t)smax);
    fl = __reduce_or_sync(0xffffffffu, fl);
    if ((threadIdx.x & 31) == 0) {
        atomicMax(&scale_io[0], mx);
        if (fl & RTF_DATA_NAN) atomicMax(&scale_io[1], 1u);
        if (fl & RTF_DATA_INF) atomicMax(&scale_io[2], 1u);
        if (fl & RTF_DATA_NEG) atomicMax(&scale_io[3], 1u);
    }
}

static int num_sms(int dev);

cudaError_t launch_scale_chunk(const float* p, uint32_t n, void* ws, const WsLayout& L,
                               cudaStream_t st, int* launches) {
    if (n == 0) return cudaSuccess;
    uint32_t* scale_io = reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(ws) + L.scale);
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return cudaErrorInvalidDevice;
    const uint32_t want = (n / 4 + 255) / 256;  // one float4 per thread, capped at 4 CTAs per SM
    const uint32_t grid = std::max(1u, std::min(want, (uint32_t)(4 * num_sms(dev))));
    k_scale_chunk<<<grid, 256, 0, st>>>(p, n, scale_io);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t clear_scale(void* ws, const WsLayout& L, cudaStream_t st) {
    return cudaMemsetAsync(reinterpret_cast<unsigned char*>(ws) + L.scale, 0, 16, st);
}

#ifdef RTF_SLOT_CHECK
// fields: 2 (n' + 1) zeroed u32, nodes: n' + 1 zeroed u32 (device; null: off)
int rows_slot_buffers(uint32_t* fields, uint32_t* nodes);  // rtf_rows.cu
extern "C" int rtf_debug_slot_buffers(uint32_t* fields, uint32_t* nodes) {
    cudaError_t e = cudaMemcpyToSymbol(g_slot_fields, &fields, sizeof(fields));
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_slot_nodes, &nodes, sizeof(nodes));
    if (e != cudaSuccess) return 5;
    return rows_slot_buffers(fields, nodes);
}
#endif

#ifdef RTF_PHASE_TIMING
extern "C" int rtf_debug_last_warp(unsigned long long* host) {
    return cudaMemcpyFromSymbol(host, g_last_warp, sizeof(g_last_warp)) == cudaSuccess ? 0 : 5;
}
extern "C" int rtf_debug_tile_ns(unsigned long long* host, int tiles) {
    return cudaMemcpyFromSymbol(host, g_tile_ns, sizeof(unsigned long long) * 3 * tiles) ==
                   cudaSuccess ? 0 : 5;
}
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

// SMs of device `dev` (queried per device: a process may drive several GPUs)
static int num_sms(int dev) {
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0)
        sms = 148;
    return sms;
}

// the node array as rows of 8 records (128 B) for the TMA tensor stores of
// phase D: boxes of 8 << k rows (64 << k records, k = 0..5), 128-B swizzle
// (the stage layout, stage_pos).  false: no tensor stores.
static bool node_tensor_maps(rtf_node* nodes, uint64_t records, NodeMaps* tm) {
    static std::atomic<PFN_cuTensorMapEncodeTiled_v12000> s_enc{nullptr};
    static std::atomic<int> s_tried{0};
    PFN_cuTensorMapEncodeTiled_v12000 enc = s_enc.load();
    if (!enc && !s_tried.exchange(1)) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            s_enc.store(reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn));
        enc = s_enc.load();
    }
    const uint64_t rows = records / 8;
    if (!enc || !nodes || rows == 0 || ((uintptr_t)nodes & 15u)) return false;
    cuuint64_t dims[2] = {32, rows};
    cuuint64_t strides[1] = {128};
    cuuint32_t es[2] = {1, 1};
    for (int k = 0; k < kNodeMaps; ++k) {
        cuuint32_t box[2] = {32, 8u << k};
        if (enc(&tm->m[k], CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, nodes, dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return false;
    }
    return true;
}

template <int THREADS, int VPT, bool CDF, int MINB = 2, bool POW2 = false, bool FUSED = false>
static cudaError_t launch_fused(BuildArgs& A, const NodeMaps* tm,
                                cudaStream_t st, int* launches) {
    auto kern = k_build<THREADS, VPT, CDF, MINB, POW2, FUSED>;
    const size_t smem = build_smem_bytes<THREADS, VPT>();  // phase B stages tile totals there
    // per instantiation and device: co-resident CTAs (the attribute is per device)
    // (atomic: host threads may launch on several devices concurrently)
    static std::atomic<int> max_grid_dev[kMaxDevices] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices)
        return cudaErrorInvalidDevice;
    int max_grid = max_grid_dev[dev].load(std::memory_order_relaxed);
    if (!max_grid) {
        cudaError_t e = cudaSuccess;
        if (smem)
            e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        int per_sm = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, THREADS, smem);
        if (e != cudaSuccess) return e;
        if (per_sm < 1) return cudaErrorCooperativeLaunchTooLarge;
        max_grid = std::min<int>(per_sm * num_sms(dev), (int)kMaxGrid);
        max_grid_dev[dev].store(max_grid, std::memory_order_relaxed);
    }
    const uint32_t grid = std::max<uint32_t>(1u, std::min<uint32_t>(A.nt, (uint32_t)max_grid));
    void* args[] = {&A, const_cast<NodeMaps*>(tm)};
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
    A.j_rank = sc ? sc->j_rank : -1;
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
    // phase D's record stores: tensor maps over the caller's node array
    // (sharded calls address the whole forest with global leaf indices)
    NodeMaps tm;
    std::memset(&tm, 0, sizeof(tm));
    A.mshift = 63u - (uint32_t)ceil_log2_u32(m);
#ifdef RTF_NO_PACK2
    A.pack2 = false;
#else
    A.pack2 = !cdf && pack2_possible(m);
#endif
    A.tma_store = !cdf && (A.phases & kPhTiles) &&
                  node_tensor_maps(nodes, sc ? sc->n_global : n, &tm);
    const bool small = flags & RTF_BUILD_SMALL_TILES;
    if (cdf)
        return small ? launch_fused<64, 4, true>(A, &tm, st, launches)
                     : launch_fused<kTT, 8, true, kTB>(A, &tm, st, launches);
    // 512 x 8 at 2 CTAs/SM (4096-entry tiles); RTF_BUILD_SMALL_TILES: 32 x 8
    // (256-entry tiles, most links cross tiles: a test schedule)
    const bool pow2 = (m & (m - 1)) == 0;
    A.mshift = 63u - (uint32_t)ceil_log2_u32(m);
    if (A.npeer)  // fused ranged sharding (rtf_shard_build_peers)
        return small ? launch_fused<32, 8, false, 2, false, true>(A, &tm, st, launches)
                     : launch_fused<kTT, 8, false, kTB, false, true>(A, &tm, st, launches);
    if (small)
        return pow2 ? launch_fused<32, 8, false, 2, true>(A, &tm, st, launches)
                    : launch_fused<32, 8, false>(A, &tm, st, launches);
    return pow2 ? launch_fused<kTT, 8, false, kTB, true>(A, &tm, st, launches)
                : launch_fused<kTT, 8, false, kTB>(A, &tm, st, launches);
}

}  // namespace rtf
