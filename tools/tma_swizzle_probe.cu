// tma_swizzle_probe.cu -- does a TMA tensor store with SWIZZLE_128B and a
// 16-byte inner box dimension un-swizzle a shared-memory buffer in which the
// 16-B record j sits at chunk (j ^ ((j >> 3) & 7)) of its 128-B row?  (The
// build kernel stages its node records that way so that blocked per-thread
// record writes are bank-conflict free.)  Also times a 64 KB store.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>

__global__ void k_probe(const __grid_constant__ CUtensorMap tm, uint32_t start, int nbox, int swz, int inner) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const int R = 256 * nbox;
    for (int j = threadIdx.x; j < R; j += blockDim.x) {
        // swizzle span S = 16 << swz bytes: chunk bits [4, 4+swz) ^= bits [7, 7+swz)
        const uint32_t off = 16u * j;
        const uint32_t phys = (off ^ (((off >> 7) & ((1u << swz) - 1u)) << 4)) / 16u;
        uint4 v = make_uint4(j, j + 100000, j + 200000, j + 300000);
        *reinterpret_cast<uint4*>(smem + 16 * phys) = v;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int b = 0; b < nbox; ++b) {
            const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem + 4096 * b);
            const int rows = 256 * 4 / inner;
            asm volatile(
                "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&tm),
                "r"(0), "r"((int)start + rows * b), "r"(sa)
                : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

int main(int argc, char** argv) {
    const int swz = argc > 1 ? atoi(argv[1]) : 3;   // 0 none, 1 32B, 2 64B, 3 128B
    const int inner = argc > 2 ? atoi(argv[2]) : 4; // u32 elements per box row
    const CUtensorMapSwizzle SW[4] = {CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
                                      CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_SWIZZLE_128B};
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q) != cudaSuccess || !enc) {
        printf("no cuTensorMapEncodeTiled\n");
        return 1;
    }
    const uint64_t N = 1 << 20;
    uint4* d;
    cudaMalloc(&d, N * 16);
    for (uint32_t start : {0u, 3u, 1000u, 4097u}) {
        cudaMemset(d, 0xff, N * 16);
        CUtensorMap tm;
        cuuint64_t dims[2] = {4, N};
        cuuint64_t strides[1] = {16};
        cuuint32_t box[2] = {(cuuint32_t)inner, 256};
        if (inner != 4) { dims[0] = (cuuint64_t)inner; dims[1] = N * 4 / inner; strides[0] = 4 * inner; box[1] = 256 * 4 / inner; }
        cuuint32_t es[2] = {1, 1};
        CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, d, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, SW[swz],
                         CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
        const int nbox = 16;
        cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 4096 * nbox + 1024);
        if (inner != 4 && start % (inner / 4)) continue;
        k_probe<<<1, 512, 4096 * nbox + 1024>>>(tm, inner == 4 ? start : start / (inner / 4), nbox, swz, inner);
        cudaError_t e0 = cudaGetLastError();
        cudaError_t e = cudaDeviceSynchronize();
        printf("swz %d inner %d launch: %s\n", swz, inner, cudaGetErrorString(e0));
        std::vector<uint4> h(256 * nbox + 16);
        cudaMemcpy(h.data(), d + start, h.size() * 16, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int j = 0; j < 256 * nbox; ++j)
            if (h[j].x != (uint32_t)j || h[j].y != (uint32_t)j + 100000 || h[j].w != (uint32_t)j + 300000) {
                if (bad < 5) printf("  start %u rec %d = %u %u %u %u\n", start, j, h[j].x, h[j].y, h[j].z, h[j].w);
                ++bad;
            }
        const bool tail_ok = h[256 * nbox].x == 0xffffffffu;
        printf("start %u: err=%s bad=%d tail_untouched=%d\n", start, cudaGetErrorString(e), bad, (int)tail_ok);
        // timing: 64 KB store, 200 launches
        cudaEvent_t a, b;
        cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        for (int i = 0; i < 200; ++i) k_probe<<<1, 512, 4096 * nbox + 1024>>>(tm, inner == 4 ? start : start / (inner / 4), nbox, swz, inner);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("  %.2f us per launch (64 KB)\n", ms * 1000 / 200);
    }
    return 0;
}
