// rtf_rows.cu -- batched build of many small independent distributions (config 5:
// per-pixel / per-light tables; Sec.5 P:1531-1533 "adding yet another criterion
// to the extended check ... the index boundary of a row").
//
// One CTA per row; the whole pipeline of rtf_build (validate, quantise, scan,
// normalise, cells, split levels, guide table, Alg. 1) runs in shared memory and
// the row's records and table are written once, coalesced.  Each row has its
// own scale E, B and total T (reading R15).
#include "rtf_device.cuh"
#include "rtf_internal.h"

namespace rtf {

struct RowsArgs {
    const float* p;
    uint32_t rows, n_row, m_row;
    rtf_header* hdr;
    rtf_node* nodes;
    rtf_ref* table;
    int32_t* jmap;  // optional: row-local compacted leaf index per entry (-1: zero weight)
    bool vec;
};

// 1024-entry rows (256 x 4): at least 5 CTAs per SM (48 registers, shared carve-out at
// 100 %): measured 1.16 vs 1.18 ms for config 5 (6 CTAs: 40 registers with
// spills, 1.17 ms).  2048-entry rows (256 x 8): 3 CTAs per SM (80 registers, no
// spills; 96 registers allowed only 2): 1024 x 2048 rows in 44 vs 50 us.
template <int THREADS, int VPT>
constexpr int rows_min_blocks() { return (THREADS == 256 && VPT == 4) ? 5 : (THREADS == 256 && VPT == 8) ? 3 : 1; }

template <int THREADS, int VPT>
__host__ __device__ constexpr int rows_padded() { return THREADS * VPT + THREADS; }

template <int THREADS, int VPT>
__host__ __device__ constexpr size_t rows_smem() { return (size_t)rows_padded<THREADS, VPT>() * (8 + 5 * 4) + THREADS * VPT; }

template <int THREADS, int VPT>
__global__ void __launch_bounds__(THREADS, rows_min_blocks<THREADS, VPT>()) k_build_rows(RowsArgs A) {
    constexpr int NMAX = THREADS * VPT;
    constexpr int NP = rows_padded<THREADS, VPT>();
    // Structure of arrays with pad slots, so that both access patterns hit 32
    // distinct banks: blocked (a thread's VPT consecutive leaves or cells, VPT
    // slots apart from its lane neighbour's) and contiguous (one slot per
    // lane).  4-B arrays: one pad per 32 slots (Pd).  The 8-B keys: one pad per
    // VPT slots (PdK), an odd stride for the blocked stores.
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t* s_key = reinterpret_cast<uint64_t*>(smem);
    int32_t* s_c0 = reinterpret_cast<int32_t*>(s_key + NP);
    int32_t* s_c1 = s_c0 + NP;
    int32_t* s_orig = s_c1 + NP;
    int32_t* s_anc = s_orig + NP;   // [m_row] first leaf of the cell, -1 if empty
    int32_t* s_lst = s_anc + NP;    // [m_row] last leaf of the cell, -1 if empty
    int32_t* s_ob = s_anc;          // otherBounds (Alg. 1) replace the anchors after the table
    uint8_t* s_lam = reinterpret_cast<uint8_t*>(s_lst + NP);
    auto Pd = [](uint32_t j) { return j + j / 32; };    // 4-B arrays
    auto PdK = [](uint32_t j) { return j + j / VPT; };  // the 8-B keys
    __shared__ uint64_t s_w[2 * (THREADS / 32)];
    __shared__ uint32_t s_c[2 * (THREADS / 32)];
    __shared__ uint32_t s_red[2 * (THREADS / 32)];
    __shared__ uint64_t s_recip;

    const uint32_t r = blockIdx.x;
    const uint32_t n = A.n_row, m = A.m_row;
    const float* p = A.p + (size_t)r * n;
    const uint32_t first = threadIdx.x * VPT;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    float x[VPT];
    if (A.vec && first + VPT <= n) {
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
        for (int k = 0; k < VPT; ++k) x[k] = first + k < n ? p[first + k] : 0.0f;
    }
    // validate + max (K1 of the single-distribution pipeline)
    uint32_t mx = 0, fl = 0;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
        const float v = x[k];
        if (v != v) fl |= RTF_DATA_NAN;
        else if (fabsf(v) == __int_as_float(0x7f800000)) fl |= RTF_DATA_INF;
        else if (v < 0.0f) fl |= RTF_DATA_NEG;
        else if (v > 0.0f) mx = max(mx, __float_as_uint(v));
    }
    for (int d = 16; d; d >>= 1) {
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, d));
        fl |= __shfl_xor_sync(0xffffffffu, fl, d);
    }
    if (lane == 0) {
        s_red[2 * warp] = mx;
        s_red[2 * warp + 1] = fl;
    }
    for (uint32_t g = threadIdx.x; g < m; g += THREADS) {
        s_anc[Pd(g)] = -1;
        s_lst[Pd(g)] = -1;
    }
    __syncthreads();
    mx = 0;
    fl = 0;
    for (int w = 0; w < THREADS / 32; ++w) {
        mx = max(mx, s_red[2 * w]);
        fl |= s_red[2 * w + 1];
    }
    const uint32_t status = fl | (mx == 0 ? RTF_DATA_ALLZERO : 0u);
    if (status) {
        if (threadIdx.x == 0) {
            rtf_header h{};
            h.status = status;
            A.hdr[r] = h;
        }
        // a poisoned row's cells answer the leaf ~INT32_MIN = INT32_MAX (the
        // data-error output) without a header read in the sampler
        for (uint32_t g = threadIdx.x; g < m; g += THREADS)
            st_cell(A.table + (size_t)r * m, g, 0u, INT32_MIN);
        return;
    }
    const int E = floor_log2_bits(mx);
    const int B = 62 - (n > 1 ? 32 - __clz((int)(n - 1)) : 0);
    const QScale qs = qscale(B - E);
    uint64_t w[VPT];
    uint64_t tw = 0;
    uint32_t tc = 0, posmask = 0;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
        w[k] = quantize(x[k], qs);
        tw += w[k];
        if (w[k]) {
            ++tc;
            posmask |= 1u << k;
        }
    }
    uint64_t W, T;
    uint32_t c_ex, cnt;
    block_scan_excl<THREADS>(tw, tc, W, c_ex, T, cnt, s_w, s_c);
    Norm nm;
    nm.s = (uint32_t)__clzll((long long)T);
    nm.d = T << nm.s;
    if (threadIdx.x == 0) s_recip = reciprocal_fast(nm.d);
    __syncthreads();
    nm.v = s_recip;

    // keys (one exact division per positive entry; w[k] holds key_j from here on)
    {
        uint32_t jl = c_ex;
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
            if (!w[k]) {
                if (A.jmap && first + k < n) A.jmap[(size_t)r * n + first + k] = -1;
                continue;
            }
            if (A.jmap) A.jmap[(size_t)r * n + first + k] = (int32_t)jl;
            const uint64_t Wn = W + w[k];
            w[k] = fixed_point(W, nm);
            s_key[PdK(jl)] = w[k];
            s_orig[Pd(jl)] = (int32_t)(first + k);
            W = Wn;
            ++jl;
        }
    }
    if (threadIdx.x == 0 && cnt) s_anc[0] = 0;  // Pd(0) = 0
    __syncthreads();
    // cells and split levels of the own leaves (the row boundary is a wall);
    // the key after the thread's last leaf is its neighbour's (or "1")
    uint64_t lampack = 0;
    if (tc) {
        uint64_t kn = (c_ex + tc < cnt) ? s_key[PdK(c_ex + tc)] : kOne63;
        uint32_t cn = (kn == kOne63) ? m : cell_of(kn, m);
#pragma unroll
        for (int k = VPT - 1; k >= 0; --k) {
            if ((posmask >> k) & 1u) {
                const uint64_t key = w[k];
                const uint32_t rk = __popc(posmask & ((1u << k) - 1u));
                const uint32_t jl = c_ex + rk;
                const uint32_t cell = cell_of(key, m);
                const uint32_t lam = cn != cell ? kLamBoundary : split_level(key, kn);
                s_lam[jl] = (uint8_t)lam;
                lampack |= (uint64_t)lam << (8 * rk);
                if (lam == kLamBoundary) {
                    s_lst[Pd(cell)] = (int32_t)jl;
                    if (cn < m) s_anc[Pd(cn)] = (int32_t)(jl + 1);
                }
                kn = key;
                cn = cell;
            }
        }
    }
    __syncthreads();
    for (uint32_t l = threadIdx.x; l < cnt; l += THREADS) {
        s_c0[Pd(l)] = ~s_orig[Pd(l ? l - 1 : 0)];
        s_c1[Pd(l)] = INT32_MIN;
    }
    // guide table: exclusive max-scan of the last leaf per cell (cells blocked per thread)
    {
        constexpr int MPT = NMAX / THREADS;
        const uint32_t g0 = threadIdx.x * MPT;
        int32_t loc = -1;
#pragma unroll
        for (int k = 0; k < MPT; ++k)
            if (g0 + k < m) loc = max(loc, s_lst[Pd(g0 + k)]);
        int32_t inc = loc;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int32_t t = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= d) inc = max(inc, t);
        }
        __syncthreads();
        int32_t* s_wmax = reinterpret_cast<int32_t*>(s_c);  // reuse scan scratch
        if (lane == 31) s_wmax[warp] = inc;
        __syncthreads();
        int32_t before = -1;
        for (int w2 = 0; w2 < warp; ++w2) before = max(before, s_wmax[w2]);
        int32_t run = max(before, __shfl_up_sync(0xffffffffu, inc, 1));
        if (lane == 0) run = before;
        rtf_ref* tab = A.table + (size_t)r * m;
#pragma unroll
        for (int k = 0; k < MPT; ++k) {
            const uint32_t g = g0 + k;
            if (g < m) {
                const int32_t a = s_anc[Pd(g)];
                const int32_t lst = s_lst[Pd(g)];
                if (a < 0) {
                    st_cell(tab, g, 0u, ~s_orig[Pd(run)]);
                } else if (lst == a) {  // one leaf: two intervals
                    const uint2 e = single_leaf_cell(s_key[PdK(a)], s_orig[Pd(a)],
                                                     s_orig[Pd(a ? a - 1 : 0)], a);
                    st_cell(tab, g, e.x, (int32_t)e.y);
                } else {
                    st_cell(tab, g, 0u, a);
                }
                run = max(run, lst);
            }
            s_ob[Pd(g)] = -1;  // slot g's anchor is read (only by this thread)
        }
    }
    __syncthreads();
    // Alg. 1 over all leaves of the row (the row boundary is lambda = 64 at
    // both ends).  Stage A: the first step of every own leaf, straight-line;
    // stage B: the second arrivals climb on, one walker per lane at a time.
    // A deposit is (split level beyond the bound) << 16 | bound.
    {
        const uint32_t lam_prev = c_ex ? (uint32_t)s_lam[c_ex - 1] : kLamBoundary;
        uint32_t contw[VPT];
        uint32_t pend = 0, rightbits = 0;
        {
            uint32_t mask = posmask;
#pragma unroll
            for (int rk = 0; rk < VPT; ++rk) {
                contw[rk] = 0;
                if ((uint32_t)rk < tc) {
                    const uint32_t k = __ffs(mask) - 1;
                    mask &= mask - 1;
                    const uint32_t l = c_ex + rk;
                    const uint32_t lamL = rk ? (uint32_t)(lampack >> (8 * (rk - 1))) & 0xffu : lam_prev;
                    const uint32_t lamR = (uint32_t)(lampack >> (8 * rk)) & 0xffu;
                    const bool right = lamL <= lamR;
                    const int32_t leaf = ~(int32_t)(first + k);
                    if ((lamL & lamR & kLamBoundary) != 0) {  // a cell root
                        s_c1[Pd(l)] = leaf;
                        RTF_SLOT((uint64_t)r * n + l, 1u, -1);
                        continue;
                    }
                    const uint32_t q = right ? l : l + 1;
                    const uint32_t qp = Pd(q);
                    (right ? s_c1 : s_c0)[qp] = leaf;
                    RTF_SLOT((uint64_t)r * n + q, right ? 1u : 0u, -1);
                    const int32_t other = atomicExch(&s_ob[qp], (int32_t)((right ? lamR : lamL) << 16 | l));
                    if (other >= 0) {
                        s_ob[qp] = -1;
                        contw[rk] = (uint32_t)other;
                        pend |= 1u << rk;
                        rightbits |= (right ? 1u : 0u) << rk;
                    }
                }
            }
        }
        bool active = false;
        int32_t lo = 0, hi = 0, node = 0;
        uint32_t lamL = 0, lamR = 0;
        while (true) {
            if (!active && pend) {
                const uint32_t rk = __ffs(pend) - 1;
                pend &= pend - 1;
                uint32_t sel[VPT];
#pragma unroll
                for (int u = 0; u < VPT; ++u) sel[u] = contw[u];
#pragma unroll
                for (int wd = VPT / 2, bit = 1; wd >= 1; wd /= 2, bit <<= 1)
#pragma unroll
                    for (int u = 0; u < wd; ++u) sel[u] = (rk & bit) ? sel[2 * u + 1] : sel[2 * u];
                const uint32_t other = sel[0];
                const uint32_t l = c_ex + rk;
                const uint32_t bound = other & 0xffffu, lv = other >> 16;
                active = true;
                if ((rightbits >> rk) & 1u) {  // merged as the right child of node l
                    lo = (int32_t)bound;
                    hi = (int32_t)l;
                    lamL = lv;
                    lamR = (uint32_t)(lampack >> (8 * rk)) & 0xffu;
                    node = (int32_t)l;
                } else {  // merged as the left child of node l + 1
                    lo = (int32_t)l;
                    hi = (int32_t)bound;
                    lamL = rk ? (uint32_t)(lampack >> (8 * (rk - 1))) & 0xffu : lam_prev;
                    lamR = lv;
                    node = (int32_t)(l + 1);
                }
            }
            if (!__any_sync(0xffffffffu, active)) break;
            if (active) {
                if ((lamL & lamR & kLamBoundary) != 0) {  // a cell root: right child of its anchor
                    s_c1[Pd(lo)] = node;
                    RTF_SLOT((uint64_t)r * n + (uint32_t)lo, 1u, (uint64_t)r * n + (uint32_t)node);
                    active = false;
                    continue;
                }
                const bool right = lamL <= lamR;
                const int32_t parent = right ? lo : hi + 1;
                const uint32_t pp = Pd((uint32_t)parent);
                (right ? s_c1 : s_c0)[pp] = node;
                RTF_SLOT((uint64_t)r * n + (uint32_t)parent, right ? 1u : 0u, (uint64_t)r * n + (uint32_t)node);
                const int32_t dep = right ? (int32_t)(lamR << 16 | (uint32_t)hi)
                                          : (int32_t)(lamL << 16 | (uint32_t)lo);
                const int32_t other = atomicExch(&s_ob[pp], dep);
                active = other >= 0;
                if (active) {
                    s_ob[pp] = -1;
                    const int32_t bound = other & 0xffff;
                    const uint32_t lv = (uint32_t)other >> 16;
                    lo = right ? bound : lo;
                    hi = right ? hi : bound;
                    lamL = right ? lv : lamL;
                    lamR = right ? lamR : lv;
                    node = parent;
                }
            }
        }
    }
    __syncthreads();
    uint4* gnode = reinterpret_cast<uint4*>(A.nodes + (size_t)r * n);
    for (uint32_t l = threadIdx.x; l < cnt; l += THREADS) {
        const uint32_t q = Pd(l);
        const uint64_t key = s_key[PdK(l)];
        gnode[l] = make_uint4((uint32_t)key, (uint32_t)(key >> 32), (uint32_t)s_c0[q], (uint32_t)s_c1[q]);
    }
    // the free slot after the last leaf holds the key "1" (2^63), so the upper
    // bound of any leaf's interval is the next slot's key (the 2-D sampler)
    if (threadIdx.x == 0 && cnt < n) gnode[cnt] = make_uint4(0u, 0x80000000u, 0x80000000u, 0x80000000u);
    if (threadIdx.x == 0) {
        rtf_header h;
        h.total = T;
        h.recip = nm.v;
        h.n_pos = cnt;
        h.exponent = E;
        h.scale_bits = B;
        h.status = 0;
        h.norm_shift = nm.s;
        h.reserved = 0;
        A.hdr[r] = h;
    }
}

template <int THREADS, int VPT>
static cudaError_t launch_rows_t(const RowsArgs& A, cudaStream_t st) {
    const size_t smem = rows_smem<THREADS, VPT>();
    static bool attr_dev[kMaxDevices] = {};  // the attributes are per device
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices)
        return cudaErrorInvalidDevice;
    bool& attr = attr_dev[dev];
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k_build_rows<THREADS, VPT>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        // all of the unified L1 / shared storage as shared memory: more rows per SM
        e = cudaFuncSetAttribute(k_build_rows<THREADS, VPT>,
                                 cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    k_build_rows<THREADS, VPT><<<A.rows, THREADS, smem, st>>>(A);
    return cudaGetLastError();
}

cudaError_t launch_build_rows(const float* p, uint32_t rows, uint32_t n_row, uint32_t m_row,
                              rtf_header* hdr, rtf_node* nodes, rtf_ref* table, int32_t* jmap,
                              cudaStream_t st, int* launches) {
    RowsArgs A;
    A.p = p;
    A.rows = rows;
    A.n_row = n_row;
    A.m_row = m_row;
    A.hdr = hdr;
    A.nodes = nodes;
    A.table = table;
    A.jmap = jmap;
    A.vec = (((uintptr_t)p & 15u) == 0) && (n_row % 4 == 0);
    const uint32_t need = std::max(n_row, m_row);
    cudaError_t e;
    if (need <= 256) e = launch_rows_t<64, 4>(A, st);
    else if (need <= 1024) e = launch_rows_t<256, 4>(A, st);
    else if (need <= 2048) e = launch_rows_t<256, 8>(A, st);  // 65 KB, 80 registers: 3 CTAs per SM
    else e = launch_rows_t<512, 8>(A, st);
    ++*launches;
    return e;
}

#ifdef RTF_SLOT_CHECK
int rows_slot_buffers(uint32_t* fields, uint32_t* nodes) {
    cudaError_t e = cudaMemcpyToSymbol(g_slot_fields, &fields, sizeof(fields));
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_slot_nodes, &nodes, sizeof(nodes));
    return e == cudaSuccess ? 0 : 5;
}
#endif

}  // namespace rtf
