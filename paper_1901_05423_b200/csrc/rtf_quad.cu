// rtf_quad.cu -- 4-ary collapsed records for sampling (Sec.5: "Due to
// memory access granularity, it may be beneficial to construct 4-ary or even
// wider trees.  A higher branching factor simply results by just collapsing two
// (or more) levels of the binary trees.").
//
// Record j (32 B, one sector, one request: tools/gather_bench.cu) holds the
// decisions of binary node j AND of both its children:
//   k[0] = ceil(key_j / 2^31), k[1] / k[2] = the same for child 0 / child 1,
//   g[0..3] = the grandchildren (child 0's c0, c1; child 1's c0, c1); a child
//   that is a leaf appears as both of its "grandchildren" (k = 0: always right).
// For a 32-bit xi, xi 2^31 < key  <=>  xi < ceil(key / 2^31), so one comparison
// per level is exact; ceil(key / 2^31) = 2^32 does not fit 32 bits and is
// flagged (bit i of flags: "xi < k[i]" is always true).  A descent reads one
// record per two levels of Alg. 2 and ends on the same leaf.
#include "rtf_device.cuh"
#include "rtf_internal.h"

namespace rtf {

constexpr int kQuadThreads = 256;
constexpr int kMaxQuadVisits = 33;  // 64 binary visits, two per record

__device__ __forceinline__ void key_ceil32(uint64_t key, uint32_t& k, uint32_t& flag, int bit) {
    const uint64_t c = (key >> 31) + ((key & 0x7fffffffull) != 0);
    k = (uint32_t)c;  // c = 2^32 wraps to 0, flagged
    flag |= (c >> 32) ? (1u << bit) : 0u;
}

__global__ void __launch_bounds__(kQuadThreads)
    k_collapse4(const rtf_node* __restrict__ nodes, const rtf_header* __restrict__ hdr, uint32_t n,
                uint4* __restrict__ rec4) {
    const uint32_t n_pos = hdr->status ? 0u : hdr->n_pos;
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n_pos && j < n;
         j += gridDim.x * blockDim.x) {
        const ulonglong2 r = __ldg(reinterpret_cast<const ulonglong2*>(nodes + j));
        const int32_t c[2] = {(int32_t)(uint32_t)r.y, (int32_t)(uint32_t)(r.y >> 32)};
        uint32_t k[3], flags = 0;
        int32_t g[4];
        key_ceil32(r.x, k[0], flags, 0);
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            if (c[i] >= 0 && (uint32_t)c[i] < n) {  // bounded: a ranged shard's foreign slots are stale
                const ulonglong2 rc = __ldg(reinterpret_cast<const ulonglong2*>(nodes + c[i]));
                key_ceil32(rc.x, k[1 + i], flags, 1 + i);
                g[2 * i] = (int32_t)(uint32_t)rc.y;
                g[2 * i + 1] = (int32_t)(uint32_t)(rc.y >> 32);
            } else {
                k[1 + i] = 0;  // never below: the leaf itself, on both sides
                g[2 * i] = g[2 * i + 1] = c[i];
            }
        }
        uint4* o = rec4 + 2 * (size_t)j;
        o[0] = make_uint4(k[0], k[1], k[2], flags);
        o[1] = make_uint4((uint32_t)g[0], (uint32_t)g[1], (uint32_t)g[2], (uint32_t)g[3]);
    }
}

__device__ __forceinline__ int32_t quad_step(const uint4* __restrict__ rec4, int32_t j,
                                             uint32_t x) {
    uint32_t k0, k1, k2, fl, g0, g1, g2, g3;
    asm("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(k0), "=r"(k1), "=r"(k2), "=r"(fl), "=r"(g0), "=r"(g1), "=r"(g2), "=r"(g3)
        : "l"(rec4 + 2 * (size_t)j));
    const bool left = x < k0 || (fl & 1u);
    const uint32_t kc = left ? k1 : k2;
    const bool cl = x < kc || ((fl >> (left ? 1 : 2)) & 1u);
    return (int32_t)(left ? (cl ? g0 : g1) : (cl ? g2 : g3));
}

__device__ __forceinline__ int32_t cell_ref(const rtf_ref* __restrict__ table, uint32_t m,
                                            uint32_t xmask, uint32_t x) {
    const int2 e = __ldg(reinterpret_cast<const int2*>(table) + (uint32_t)(((uint64_t)x * m) >> 32));
    return table_step(e, x, x & xmask);
}

// four samples per thread in lock-step, as k_sample
__global__ void __launch_bounds__(kQuadThreads)
    k_sample4(const uint4* __restrict__ rec4, const rtf_ref* __restrict__ table,
              const rtf_header* __restrict__ hdr, uint32_t m, uint32_t xmask,
              const uint32_t* __restrict__ xi,
              uint64_t count, int32_t* __restrict__ out, bool vec) {
    const uint64_t gt = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t gs = (uint64_t)gridDim.x * blockDim.x;
    const bool bad = hdr->status != 0;
    uint64_t done = 0;
    if (vec) {
        const uint64_t nq = count >> 2;
        for (uint64_t q = gt; q < nq; q += gs) {
            const uint4 xv = ld_stream_u4(xi + 4 * q);
            const uint32_t x[4] = {xv.x, xv.y, xv.z, xv.w};
            int32_t j[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) j[k] = bad ? -1 : cell_ref(table, m, xmask, x[k]);
            for (int it = 0; (j[0] & j[1] & j[2] & j[3]) >= 0 && it < kMaxQuadVisits; ++it) {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (j[k] >= 0) j[k] = quad_step(rec4, j[k], x[k]);
            }
            int4 o;
            o.x = bad ? INT32_MAX : (j[0] >= 0 ? INT32_MIN : ~j[0]);
            o.y = bad ? INT32_MAX : (j[1] >= 0 ? INT32_MIN : ~j[1]);
            o.z = bad ? INT32_MAX : (j[2] >= 0 ? INT32_MIN : ~j[2]);
            o.w = bad ? INT32_MAX : (j[3] >= 0 ? INT32_MIN : ~j[3]);
            __stcs(reinterpret_cast<int4*>(out + 4 * q), o);
        }
        done = nq << 2;
    }
    for (uint64_t k = done + gt; k < count; k += gs) {
        const uint32_t x = xi[k];
        int32_t j = bad ? -1 : cell_ref(table, m, xmask, x);
        for (int it = 0; j >= 0 && it < kMaxQuadVisits; ++it) j = quad_step(rec4, j, x);
        out[k] = bad ? INT32_MAX : (j >= 0 ? INT32_MIN : ~j);
    }
}

static inline uint32_t quad_grid(uint64_t items) {
    const uint64_t want = (items + kQuadThreads - 1) / kQuadThreads;
    return (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(want, (uint64_t)device_sms() * 64ull));
}

cudaError_t launch_collapse4(const rtf_forest& f, void* rec4, cudaStream_t st, int* launches) {
    k_collapse4<<<quad_grid(f.n), kQuadThreads, 0, st>>>(f.nodes, f.header, f.n,
                                                           static_cast<uint4*>(rec4));
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_sample4(const rtf_forest& f, const void* rec4, const uint32_t* xi,
                           uint64_t count, int32_t* out, cudaStream_t st, int* launches) {
    if (count == 0) return cudaSuccess;
    const bool vec = (((uintptr_t)xi | (uintptr_t)out) & 15u) == 0;
    k_sample4<<<quad_grid(vec ? (count + 3) / 4 : count), kQuadThreads, 0, st>>>(
        static_cast<const uint4*>(rec4), f.table, f.header, f.m, xoff_mask(f.m), xi, count, out, vec);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace rtf
