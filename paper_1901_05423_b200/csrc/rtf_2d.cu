// rtf_2d.cu -- 2-D distributions (Sec.6): the row weights of the
// marginal from the rows' build headers, and the component-wise sampler with
// the sub-pixel rescale.  Reading R19.
#include "rtf_device.cuh"
#include "rtf_internal.h"

namespace rtf {

constexpr int kRowWeightThreads = 1024;
constexpr int k2dThreads = 256;
constexpr int kMaxVisits2d = 64;

// q_y = float32(float64(T_y) 2^(E_y - B_y - K)), K = max over non-empty rows of
// E_y - B_y; an all-zero row gets 0, a row with NaN / Inf / negative data NaN
// (so the marginal build reports the data error).  dense: bit y set if row y
// has W positive weights (its index map is the identity).  One CTA.
__global__ void __launch_bounds__(kRowWeightThreads)
    k_row_weights(const rtf_header* __restrict__ hdr, uint32_t H, uint32_t W, float* __restrict__ q,
                  uint32_t* __restrict__ dense) {
    __shared__ int s_max[kRowWeightThreads / 32];
    int k = INT_MIN;
    for (uint32_t y = threadIdx.x; y < H; y += kRowWeightThreads)
        if (hdr[y].status == 0) k = max(k, hdr[y].exponent - hdr[y].scale_bits);
    k = __reduce_max_sync(0xffffffffu, k);
    if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = k;
    __syncthreads();
    int K = INT_MIN;
    for (int w = 0; w < kRowWeightThreads / 32; ++w) K = max(K, s_max[w]);
    for (uint32_t y0 = 0; y0 < H; y0 += kRowWeightThreads) {  // uniform trip count (ballot)
        const uint32_t y = y0 + threadIdx.x;
        const bool in = y < H;
        const rtf_header h = in ? hdr[y] : rtf_header{};
        const uint32_t bits = __ballot_sync(0xffffffffu, in && h.status == 0 && h.n_pos == W);
        if (in && (threadIdx.x & 31) == 0) dense[y >> 5] = bits;
        if (!in) continue;
        float v;
        if (h.status & (RTF_DATA_NAN | RTF_DATA_INF | RTF_DATA_NEG)) v = __int_as_float(0x7fc00000);
        else if (h.status) v = 0.0f;  // all-zero row
        else v = __double2float_rn(ldexp(__ull2double_rn(h.total), h.exponent - h.scale_bits - K));
        q[y] = v;
    }
}

// one Alg. 2 descent in a row forest (nodes + table of that row); returns ~leaf
__device__ __forceinline__ int32_t descend_row(const rtf_node* __restrict__ nodes,
                                               const rtf_ref* __restrict__ table, uint32_t m,
                                               uint32_t xmask, uint32_t x) {
    const int2 e = __ldg(reinterpret_cast<const int2*>(table) + (uint32_t)(((uint64_t)x * m) >> 32));
    int32_t j = table_step(e, x, x & xmask);
    const uint64_t x63 = (uint64_t)x << 31;
    for (int d = 0; j >= 0 && d < kMaxVisits2d; ++d) {
        const ulonglong2 r = __ldg(reinterpret_cast<const ulonglong2*>(nodes + j));
        j = (int32_t)(x63 < r.x ? (uint32_t)r.y : (uint32_t)(r.y >> 32));
    }
    return j;
}

// relative position of x inside the interval of leaf j; last: the entry is the
// row's last one (slot j + 1 is then past the row).  Otherwise slot j + 1 holds
// the next leaf's key, or the key "1" that the row build stores after the last
// leaf (no header read per sample).
__device__ __forceinline__ double rel_pos(const rtf_node* __restrict__ nodes, int32_t j,
                                          bool last, uint32_t x) {
    const uint64_t lo = __ldg(&nodes[j].key);
    const uint64_t hi = last ? kOne63 : __ldg(&nodes[j + 1].key);
    return __ddiv_rn(__ull2double_rn(((uint64_t)x << 31) - lo), __ull2double_rn(hi - lo));
}

__global__ void __launch_bounds__(k2dThreads, 8)  // 32 registers: 2048 threads per SM
    k_sample_2d(rtf_forest2d f, uint32_t xmask_x, uint32_t xmask_y, const uint32_t* __restrict__ xi1,
                const uint32_t* __restrict__ xi2, uint64_t count, int32_t* __restrict__ pixel,
                float* __restrict__ pos) {
    const uint64_t gs = (uint64_t)gridDim.x * blockDim.x;
    const bool bad = f.marginal.header->status != 0;
    const bool marg_dense = f.marginal.header->n_pos == f.H;  // every row weight positive
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count; k += gs) {
        const uint32_t a = xi1[k], b = xi2[k];
        int32_t out = INT32_MAX;
        float px = __int_as_float(0x7fc00000), py = px;
        if (!bad) {
            const int32_t jy = descend_row(f.marginal.nodes, f.marginal.table, f.my, xmask_y, a);
            const int32_t y = ~jy;
            const rtf_node* rn = f.rows.nodes + (size_t)y * f.W;
            const int32_t jx = descend_row(rn, f.rows.table + (size_t)y * f.mx, f.mx, xmask_x, b);
            const int32_t x = ~jx;
            if (jy >= 0 || jx >= 0) {
                out = INT32_MIN;  // corrupted forest (a descent did not end in a leaf)
            } else {
                out = y * (int32_t)f.W + x;
                if (pos) {
                    const int32_t jy_node = marg_dense ? y : __ldg(&f.marg_jmap[y]);
                    const double u = rel_pos(f.marginal.nodes, jy_node, (uint32_t)y + 1 == f.H, a);
                    const bool dense = (__ldg(&f.rows_dense[(uint32_t)y >> 5]) >> (y & 31)) & 1u;
                    const int32_t jx_node =
                        dense ? x : __ldg(&f.rows_jmap[(size_t)y * f.W + x]);
                    const double v = rel_pos(rn, jx_node, (uint32_t)x + 1 == f.W, b);
                    px = __double2float_rz(__ddiv_rn(__dadd_rn((double)x, v), (double)f.W));
                    py = __double2float_rz(__ddiv_rn(__dadd_rn((double)y, u), (double)f.H));
                }
            }
        }
        pixel[k] = out;
        if (pos) reinterpret_cast<float2*>(pos)[k] = make_float2(px, py);
    }
}

// Rows built by the cooperative kernel (wider than the row kernel's 4096
// entries, or a marginal of more than 4096 rows): the row-local compacted
// leaf index of every entry (-1 for a zero weight) by a block scan per row,
// and the key "1" after the row's last leaf when the row has zero weights
// (what the row kernel stores there; rel_pos reads it).  One CTA per row.
constexpr int kJmapThreads = 1024;
__global__ void __launch_bounds__(kJmapThreads)
    k_rows_jmap(const float* __restrict__ p, uint32_t W, const rtf_header* __restrict__ hdr,
                rtf_node* __restrict__ nodes, int32_t* __restrict__ jmap) {
    __shared__ uint32_t s_cnt[kJmapThreads / 32];
    const uint32_t y = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const float* row = p + (size_t)y * W;
    int32_t* jm = jmap + (size_t)y * W;
    uint32_t base = 0;
    for (uint32_t x0 = 0; x0 < W; x0 += kJmapThreads) {
        const uint32_t x = x0 + threadIdx.x;
        const bool pos = x < W && row[x] > 0.0f;
        const uint32_t bal = __ballot_sync(0xffffffffu, pos);
        if (lane == 0) s_cnt[warp] = __popc(bal);
        __syncthreads();
        uint32_t before = base, total = 0;
        for (uint32_t w = 0; w < kJmapThreads / 32; ++w) {
            if (w < warp) before += s_cnt[w];
            total += s_cnt[w];
        }
        if (x < W) jm[x] = pos ? (int32_t)(before + __popc(bal & ((1u << lane) - 1u))) : -1;
        base += total;
        __syncthreads();
    }
    if (threadIdx.x == 0 && hdr[y].status == 0 && hdr[y].n_pos < W)
        nodes[(size_t)y * W + hdr[y].n_pos].key = kOne63;
}

cudaError_t launch_rows_jmap(const float* p, uint32_t W, uint32_t H, const rtf_header* hdr,
                             rtf_node* nodes, int32_t* jmap, cudaStream_t st, int* launches) {
    k_rows_jmap<<<H, kJmapThreads, 0, st>>>(p, W, hdr, nodes, jmap);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_row_weights(const rtf_header* rows_hdr, uint32_t H, uint32_t W, float* q,
                               uint32_t* dense, cudaStream_t st, int* launches) {
    k_row_weights<<<1, kRowWeightThreads, 0, st>>>(rows_hdr, H, W, q, dense);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_sample_2d(const rtf_forest2d& f, const uint32_t* xi1, const uint32_t* xi2,
                             uint64_t count, int32_t* pixel, float* pos, cudaStream_t st,
                             int* launches) {
    if (count == 0) return cudaSuccess;
    const uint64_t want = (count + k2dThreads - 1) / k2dThreads;
    const uint32_t grid = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(want, (uint64_t)device_sms() * 32ull));
    k_sample_2d<<<grid, k2dThreads, 0, st>>>(f, xoff_mask(f.mx), xoff_mask(f.my), xi1, xi2, count,
                                             pixel, pos);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace rtf
