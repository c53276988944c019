// rtf_device.cuh -- device helpers of librtf (product path; shares nothing with oracle/).
//
// Fixed-point conventions (readings R4/R7/R11):
//   w_i   = max(1, floor(p_i 2^(B-E))) for p_i > 0, else 0
//   key_j = floor(W_j 2^63 / T)       (63 fractional bits, "1" = 2^63)
//   cell  = floor(key m / 2^63)       (Alg. 1, curCell = floor(data m))
//   lambda_j = 64 at a cell boundary / array end, else msb(key_j ^ key_{j+1})
//              (XOR distance P:1049-1055, "distance set to the maximum" P:1078-1079)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/rtf.h"

namespace rtf {

constexpr uint64_t kOne63 = 1ull << 63;
constexpr uint32_t kLamBoundary = 64;

// ------------------------------------------------------------ memory-model helpers

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// completion counter: the release orders this CTA's prior writes (ordered before
// the call by a barrier), the acquire lets the last arriver read everyone's
__device__ __forceinline__ uint32_t atom_add_acq_rel_u32(uint32_t* p, uint32_t v) {
    uint32_t old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;"
                 : "=r"(old)
                 : "l"(p), "r"(v)
                 : "memory");
    return old;
}

// streaming 16-byte load that does not allocate in L1 (read-once data)
__device__ __forceinline__ uint4 ld_stream_u4(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// L2 cache policies: streamed inputs leave L2 first, the forest stays
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint4 ld_stream_u4_pol(const void* p, uint64_t pol) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ ulonglong2 ld_nc_u64x2_pol(const void* p, uint64_t pol) {
    ulonglong2 r;
    asm volatile("ld.global.nc.L2::cache_hint.v2.u64 {%0,%1}, [%2], %3;"
                 : "=l"(r.x), "=l"(r.y)
                 : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ int32_t ld_nc_s32_pol(const int32_t* p, uint64_t pol) {
    int32_t r;
    asm volatile("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ void st_stream_s4_pol(void* p, int4 v, uint64_t pol) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.s32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p),
                 "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol)
                 : "memory");
}

__device__ __forceinline__ float4 ld_stream_f4(const float* p) {
    uint4 r = ld_stream_u4(p);
    return make_float4(__uint_as_float(r.x), __uint_as_float(r.y), __uint_as_float(r.z),
                       __uint_as_float(r.w));
}

__device__ __forceinline__ float4 ld_stream_f4_pol(const float* p, uint64_t pol) {
    uint4 r = ld_stream_u4_pol(p, pol);
    return make_float4(__uint_as_float(r.x), __uint_as_float(r.y), __uint_as_float(r.z),
                       __uint_as_float(r.w));
}

// ------------------------------------------------------------ TMA bulk copies + mbarrier

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

// order generic-proxy shared-memory accesses before later async-proxy (TMA) ones
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// generic-proxy writes to global memory (earlier phases) before TMA reads them
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

// 1-D bulk copy global -> shared (UBLKCP), completion counted on `bar`
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// the same with an L2 cache policy (e.g. evict_first for a last read)
__device__ __forceinline__ void tma_load_1d_pol(void* dst, const void* src, uint32_t bytes,
                                                uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

// 2-D TMA tensor store shared -> global (UTMASTG), tracked as a bulk async-group
__device__ __forceinline__ void tma_store_2d(const void* tmap, int c0, int c1, const void* src) {
    asm volatile(
        "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(tmap),
        "r"(c0), "r"(c1), "r"(smem_u32(src))
        : "memory");
}
__device__ __forceinline__ void bulk_commit() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// the committed stores have READ their shared-memory source (it may be reused)
__device__ __forceinline__ void bulk_wait_read0() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// the committed stores are complete (visible in global memory)
__device__ __forceinline__ void bulk_wait0() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// explicit shared-memory accesses on precomputed 32-bit addresses (keeps the
// compiler from re-deriving generic->shared windows inside hot loops)
__device__ __forceinline__ void sts_u32(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts_v4(uint32_t a, uint4 v) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ uint4 lds_v4(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(a)
                 : "memory");
    return v;
}
__device__ __forceinline__ int32_t atoms_exch(uint32_t a, int32_t v) {
    int32_t r;
    asm volatile("atom.shared.exch.b32 %0, [%1], %2;" : "=r"(r) : "r"(a), "r"(v) : "memory");
    return r;
}

// ------------------------------------------------------------ quantisation

// floor(log2(x)) of a positive finite float given its bits
__device__ __forceinline__ int floor_log2_bits(uint32_t b) {
    uint32_t be = b >> 23;
    if (be) return (int)be - 127;
    return (31 - __clz((int)b)) - 149;  // subnormal: frac * 2^-149
}

// w = max(1, floor(x 2^shift)) for x > 0, 0 for x = +-0 (the build rejects
// negative, NaN and Inf data before quantising).  Exact in FP32: shift lies in
// [-97, 211], so 2^shift = s1 s2 with s1 = 2^min(shift, 127) and s2 = 2^(shift
// - 127) or 1, both normal floats; multiplying by a power of two is exact
// unless the result leaves the normal range, and here the product overflows
// never (x 2^shift < 2^63) and underflows only below 2^-126, where floor = 0
// and the max with 1 decides anyway.  The round-toward-zero conversion is the
// floor.  (FMUL, FMUL, FSETP, FSEL, FMNMX, F2I.U64: no FP64 pipe.)
struct QScale {
    float s1, s2;
};

__device__ __forceinline__ QScale qscale(int shift) {
    const int a = shift > 127 ? 127 : shift;
    return QScale{__int_as_float((127 + a) << 23), __int_as_float((127 + shift - a) << 23)};
}

__device__ __forceinline__ uint64_t quantize(float x, QScale q) {
    const float y = fmaxf((x * q.s1) * q.s2, x > 0.0f ? 1.0f : 0.0f);
    return __float2ull_rz(y);
}

// ------------------------------------------------------------ exact normalisation
//
// key = floor(W 2^63 / T) for 0 <= W < T < 2^63 by division with a precomputed
// reciprocal of the normalised divisor d = T << s (Moller & Granlund 2011,
// "Improved division by invariant integers", Alg. 4): the numerator is
// (u1, u0) = (W << (s-1), 0) since W 2^63 2^s = (W 2^(s-1)) 2^64.

struct Norm {
    uint64_t d;  // T << s, msb set
    uint64_t v;  // floor((2^128 - 1) / d) - 2^64
    uint32_t s;  // clz(T) >= 1
};

// v for a normalised d: the 128/64 quotient of (~d, ~0) by d, bit by bit.
__device__ __forceinline__ uint64_t reciprocal_of(uint64_t d) {
    uint64_t rem = ~d, lo = ~0ull, q = 0;
    for (int i = 63; i >= 0; --i) {
        uint64_t carry = rem >> 63;
        rem = (rem << 1) | ((lo >> i) & 1ull);
        q <<= 1;
        if (carry || rem >= d) {
            rem -= d;
            q |= 1ull;
        }
    }
    return q;
}

// The same v without the 64-step loop: a float64 estimate of 2^128 / d (within
// a few 2^12 of v), then an exact correction from the signed remainder
// e = (2^128 - 1) - (2^64 + v) d, computed mod 2^128 (|e| < 2^80).
__device__ __forceinline__ uint64_t reciprocal_fast(uint64_t d) {
    typedef unsigned __int128 u128;
    typedef __int128 s128;
    const double t = __dadd_rn(__ddiv_rn(0x1p128, __ull2double_rn(d)), -0x1p64);
    uint64_t v = t >= 0x1p64 ? ~0ull : (t <= 0.0 ? 0ull : __double2ull_rz(t));
    const u128 D = d;
    s128 e = (s128)(~(u128)0 - (((u128)1 << 64) + v) * D);
    const double ed = __dadd_rn(__dmul_rn((double)(int64_t)(e >> 64), 0x1p64),
                                __ull2double_rn((uint64_t)e));
    const int64_t c = (int64_t)floor(__ddiv_rn(ed, __ull2double_rn(d)));
    v += (uint64_t)c;
    e -= (s128)c * (s128)D;
    while (e < 0) {
        --v;
        e += (s128)D;
    }
    while (e >= (s128)D) {
        ++v;
        e -= (s128)D;
    }
    return v;
}

__device__ __forceinline__ uint64_t fixed_point(uint64_t W, const Norm& nm) {
    uint64_t u1 = W << (nm.s - 1);
    uint64_t q0 = nm.v * u1;
    uint64_t q1 = __umul64hi(nm.v, u1) + u1 + 1ull;
    uint64_t r = 0ull - q1 * nm.d;  // u0 - q1 d (mod 2^64), u0 = 0
    if (r > q0) {
        q1 -= 1ull;
        r += nm.d;
    }
    if (r >= nm.d) q1 += 1ull;
    return q1;
}

// The same key with a 128-bit fixed-point reciprocal R = floor(2^127 / T)
// (hi = floor(2^63 / T), lo = the next 64 bits): q = floor(W R / 2^64) =
// W hi + umulhi(W, lo) is key or key - 1 (R is short of 2^127 / T by less
// than 1, so W R / 2^64 is short of W 2^63 / T by less than W / 2^64 < 1/2),
// and the remainder W 2^63 - q T, which lies in [0, 2T) < 2^64, is exact
// modulo 2^64: one comparison fixes q.  About 20 instructions against the
// Moller-Granlund step's 28.
struct Recip128 {
    uint64_t hi, lo;
};

// R for T >= 1: one 64-bit division, then 64 steps of long division (once per CTA)
__device__ __forceinline__ Recip128 recip128(uint64_t T) {
    Recip128 R;
    R.hi = (1ull << 63) / T;
    uint64_t r = (1ull << 63) - R.hi * T;  // < T
    uint64_t lo = 0;
    for (int i = 0; i < 64; ++i) {
        const uint64_t carry = r >> 63;
        r <<= 1;
        lo <<= 1;
        if (carry || r >= T) {
            r -= T;
            lo |= 1ull;
        }
    }
    R.lo = lo;
    return R;
}

__device__ __forceinline__ uint64_t fixed_point_r(uint64_t W, Recip128 R, uint64_t T) {
    const uint64_t q = W * R.hi + __umul64hi(W, R.lo);
    const uint64_t r = (W << 63) - q * T;  // W 2^63 - q T (mod 2^64), in [0, 2T)
    return r >= T ? q + 1ull : q;
}

// floor(key m / 2^63) for key < 2^63, m < 2^31: key m = hi 2^32 + lo with
// hi = key_hi m < 2^62, lo = key_lo m < 2^63, and the fraction of lo / 2^32
// cannot carry across a multiple of 2^31.
__device__ __forceinline__ uint32_t cell_of(uint64_t key, uint32_t m) {
    const uint64_t hi = (uint64_t)(uint32_t)(key >> 32) * m;
    const uint64_t lo = (uint64_t)(uint32_t)key * m;
    return (uint32_t)((hi + (lo >> 32)) >> 31);
}

__device__ __forceinline__ uint32_t split_level(uint64_t a, uint64_t b) {
    return 63u - (uint32_t)__clzll((long long)(a ^ b));  // msb(a ^ b)
}

// ------------------------------------------------------------ guide-table cells

// Guide-table cell of a cell holding exactly one leaf a (rtf_ref, the
// two-interval flag of P:1335-1338; reading R18): key32 = ceil(key_a / 2^31)
// splits the cell between intervals a-1 and a when their references are
// consecutive (no zero weight between them); key32 = 0 marks a cell inside a
// single interval; otherwise the anchor node a stays.
__device__ __forceinline__ uint2 single_leaf_cell(uint64_t key_a, int32_t orig_a,
                                                  int32_t orig_prev, int32_t anchor) {
    const uint64_t kc = (key_a + 0x7fffffffull) >> 31;  // key_a < 2^63: no overflow
    if (kc == 0) return make_uint2(0u, (uint32_t)~orig_a);           // a = 0
    if (kc == (1ull << 32)) return make_uint2(0u, (uint32_t)~orig_prev);  // a unreachable
    if (orig_a == orig_prev + 1) return make_uint2((uint32_t)kc, (uint32_t)~orig_a);
    return make_uint2(0u, (uint32_t)anchor);
}

// Packed three-interval cells (reading R20, oracle O16): a cell of a
// power-of-two table with m >= 2^17 (so a cell spans at most 2^15 xi values,
// its first xi being xi0 = g 2^32 / m) that holds exactly the two leaves a,
// a+1 -- overlapped by the intervals a-1, a, a+1 with orig(a+1) = orig(a-1) + 2
// and a >= 1 -- stores both split points as offsets from xi0 next to
// orig(a-1): key32 = s1 | s2 << 16 (s = ceil(key / 2^31) - xi0, s2 >= 1),
// ref = orig(a-1) >= 0.  "Further information could also be stored in the
// reference": no node is read for such a cell.
constexpr uint32_t kPackMinLog2M = 17;

__host__ __device__ __forceinline__ bool pack2_possible(uint32_t m) {
    return m >= (1u << kPackMinLog2M) && (m & (m - 1)) == 0;
}

// the packed entry of the two-leaf cell g (leaves a, a+1 with keys ka, kb and
// original indices orig(a-1) = op, orig(a+1) = oq), or {0, 0} when the three
// intervals are not consecutive (a zero weight between: the anchor stays).
// shift = 32 - log2 m.
__device__ __forceinline__ uint2 pack2_cell(uint32_t g, uint32_t shift, uint64_t ka, uint64_t kb,
                                            int32_t op, int32_t oq) {
    if (oq != op + 2) return make_uint2(0u, 0u);
    const uint64_t xi0 = (uint64_t)g << shift;
    const uint32_t s1 = (uint32_t)(((ka + 0x7fffffffull) >> 31) - xi0);
    const uint32_t s2 = (uint32_t)(((kb + 0x7fffffffull) >> 31) - xi0);
    return make_uint2(s1 | s2 << 16, (uint32_t)op);
}

// Alg. 2's first step on a guide-table cell e (rtf_ref as int2) for xi = x:
// a node reference (anchor: key32 = 0, ref >= 0), a packed three-interval
// cell (key32 != 0, ref >= 0; xoff = x mod (2^32 / m)), or a leaf that a
// two-interval cell (key32 != 0, ref < 0; reading R18) splits with one
// comparison (key32 = 0, ref < 0: one interval).  Returns a node index >= 0
// or ~leaf.
__device__ __forceinline__ int32_t table_step(int2 e, uint32_t x, uint32_t xoff) {
    // branch-free (selects): the samplers issue their next loads without waiting
    // on a divergent branch per sample
    const uint32_t s1 = (uint32_t)e.x & 0xffffu, s2 = (uint32_t)e.x >> 16;
    const int32_t packed = ~(e.y + (xoff >= s1 ? 1 : 0) + (xoff >= s2 ? 1 : 0));
    const int32_t plain = (e.y >= 0 || x >= (uint32_t)e.x) ? e.y : e.y + 1;
    return (e.y >= 0 && e.x != 0) ? packed : plain;
}

// x mod (2^32 / m) for a power-of-two m (the offset table_step needs), else 0
__host__ __device__ __forceinline__ uint32_t xoff_mask(uint32_t m) {
    if (m & (m - 1)) return 0u;
    uint32_t lg = 0;
    while ((1u << lg) < m) ++lg;
    return lg == 0 ? 0xffffffffu : ((1u << (32u - lg)) - 1u);
}

__device__ __forceinline__ void st_cell(rtf_ref* table, uint32_t g, uint32_t key32, int32_t ref) {
    *reinterpret_cast<uint2*>(table + g) = make_uint2(key32, (uint32_t)ref);
}

// Cells [g0, g1) of an empty run all get {0, ref}.  RTF_WIDE_RUNS: scalar up
// to a 4-cell (32-B) boundary, then one 256-bit store per 4 cells (the table
// is 256-B aligned) -- measured slower on configs 2 and 3 (280 vs 272 us,
// 76 vs 72 us: the runs there are a few cells long), so not the default.
__device__ __forceinline__ void fill_run(rtf_ref* table, uint32_t g0, uint32_t g1, int32_t ref) {
#ifndef RTF_WIDE_RUNS
    for (uint32_t g = g0; g < g1; ++g) st_cell(table, g, 0u, ref);
#else
    uint32_t g = g0;
    const uint32_t r = (uint32_t)ref;
    for (; g < g1 && (g & 3u); ++g) st_cell(table, g, 0u, ref);
    for (; g + 4u <= g1; g += 4u)
        asm volatile("st.global.v8.b32 [%0], {%1, %2, %1, %2, %1, %2, %1, %2};"
                     :: "l"(table + g), "r"(0u), "r"(r) : "memory");
    for (; g < g1; ++g) st_cell(table, g, 0u, ref);
#endif
}

// ------------------------------------------------------------ scan prefix payload

// Aggregate of a run of entries: sum of quantised weights, number of positive
// entries, original index of the last positive entry (-1 if none).
struct __align__(16) Pfx {
    uint64_t W;
    uint32_t cnt;
    int32_t last;
};

__device__ __forceinline__ Pfx combine(const Pfx& a, const Pfx& b) {  // a precedes b
    Pfx r;
    r.W = a.W + b.W;
    r.cnt = a.cnt + b.cnt;
    r.last = b.last >= 0 ? b.last : a.last;
    return r;
}

__device__ __forceinline__ Pfx ld_pfx_cg(const Pfx* p) {
    uint4 u = __ldcg(reinterpret_cast<const uint4*>(p));
    Pfx r;
    r.W = (uint64_t)u.x | ((uint64_t)u.y << 32);
    r.cnt = u.z;
    r.last = (int32_t)u.w;
    return r;
}

__device__ __forceinline__ void st_pfx(Pfx* p, const Pfx& v) {
    uint4 u = make_uint4((uint32_t)v.W, (uint32_t)(v.W >> 32), v.cnt, (uint32_t)v.last);
    *reinterpret_cast<uint4*>(p) = u;
}

// ------------------------------------------------------------ warp / block scans

__device__ __forceinline__ uint64_t shfl_up_u64(uint64_t v, int d) {
    return __shfl_up_sync(0xffffffffu, v, d);
}

// Block-wide exclusive scan of (u64, u32) pairs.  scratch: 2 * (THREADS/32) words of each.
template <int THREADS>
__device__ __forceinline__ void block_scan_excl(uint64_t w, uint32_t c, uint64_t& w_ex,
                                                uint32_t& c_ex, uint64_t& w_tot, uint32_t& c_tot,
                                                uint64_t* s_w, uint32_t* s_c) {
    constexpr int NW = THREADS / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t wi = w;
    uint32_t ci = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        uint64_t tw = shfl_up_u64(wi, d);
        uint32_t tc = __shfl_up_sync(0xffffffffu, ci, d);
        if (lane >= d) {
            wi += tw;
            ci += tc;
        }
    }
    if (lane == 31) {
        s_w[warp] = wi;
        s_c[warp] = ci;
    }
    __syncthreads();
    if (warp == 0) {
        uint64_t ww = lane < NW ? s_w[lane] : 0ull;
        uint32_t cc = lane < NW ? s_c[lane] : 0u;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            uint64_t tw = shfl_up_u64(ww, d);
            uint32_t tc = __shfl_up_sync(0xffffffffu, cc, d);
            if (lane >= d) {
                ww += tw;
                cc += tc;
            }
        }
        if (lane < NW) {
            s_w[NW + lane] = ww;  // inclusive warp prefixes
            s_c[NW + lane] = cc;
        }
    }
    __syncthreads();
    uint64_t wbase = warp ? s_w[NW + warp - 1] : 0ull;
    uint32_t cbase = warp ? s_c[NW + warp - 1] : 0u;
    w_ex = wbase + wi - w;
    c_ex = cbase + ci - c;
    w_tot = s_w[2 * NW - 1];
    c_tot = s_c[2 * NW - 1];
}

// Block-wide exclusive scan of (sum u64, count u32) plus an exclusive max of an
// i32 (the last positive index before each thread).  Scratch: 2*NW entries each.
template <int THREADS>
__device__ __forceinline__ void block_scan3_excl(uint64_t w, uint32_t c, int32_t l, uint64_t& w_ex,
                                                 uint32_t& c_ex, int32_t& l_ex, uint64_t& w_tot,
                                                 uint32_t& c_tot, uint64_t* s_w, uint32_t* s_c,
                                                 int32_t* s_l) {
    constexpr int NW = THREADS / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t wi = w;
    uint32_t ci = c;
    int32_t li = l;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint64_t tw = shfl_up_u64(wi, d);
        const uint32_t tc = __shfl_up_sync(0xffffffffu, ci, d);
        const int32_t tl = __shfl_up_sync(0xffffffffu, li, d);
        if (lane >= d) {
            wi += tw;
            ci += tc;
            li = max(li, tl);
        }
    }
    if (lane == 31) {
        s_w[warp] = wi;
        s_c[warp] = ci;
        s_l[warp] = li;
    }
    __syncthreads();
    if (warp == 0) {
        uint64_t ww = lane < NW ? s_w[lane] : 0ull;
        uint32_t cc = lane < NW ? s_c[lane] : 0u;
        int32_t ll = lane < NW ? s_l[lane] : -1;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint64_t tw = shfl_up_u64(ww, d);
            const uint32_t tc = __shfl_up_sync(0xffffffffu, cc, d);
            const int32_t tl = __shfl_up_sync(0xffffffffu, ll, d);
            if (lane >= d) {
                ww += tw;
                cc += tc;
                ll = max(ll, tl);
            }
        }
        if (lane < NW) {
            s_w[NW + lane] = ww;
            s_c[NW + lane] = cc;
            s_l[NW + lane] = ll;
        }
    }
    __syncthreads();
    const uint64_t wbase = warp ? s_w[NW + warp - 1] : 0ull;
    const uint32_t cbase = warp ? s_c[NW + warp - 1] : 0u;
    const int32_t lbase = warp ? s_l[NW + warp - 1] : -1;
    const int32_t lprev = __shfl_up_sync(0xffffffffu, li, 1);
    w_ex = wbase + wi - w;
    c_ex = cbase + ci - c;
    l_ex = max(lbase, lane ? lprev : -1);
    w_tot = s_w[2 * NW - 1];
    c_tot = s_c[2 * NW - 1];
}

}  // namespace rtf
