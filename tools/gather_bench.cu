// Random-gather microbenchmark (measurement aid for the sampler's record
// layout): per lane, one random 16-B load, one random 32-B load (a single
// 256-bit ld.global.nc.v4.u64), or two 16-B loads of the same 32-B sector, over
// an L2-resident (32 MB) and a DRAM-resident (4 GB) buffer.  Prints ns per
// gathered item and G items/s.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/gather_bench tools/gather_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

template <int MODE>
__global__ void __launch_bounds__(256) k_gather(const ulonglong2* __restrict__ buf, uint64_t mask32,
                                                uint64_t items, unsigned long long* sink) {
    unsigned long long acc = 0;
    const uint64_t gs = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < items; i += gs) {
        const uint64_t s = hash32((uint32_t)i * 2654435761u + (uint32_t)(i >> 32)) & mask32;  // 32-B slot
        if (MODE == 0) {  // one 16-B load
            const ulonglong2 a = __ldg(buf + 2 * s);
            acc += a.x ^ a.y;
        } else if (MODE == 1) {  // one 32-B load
            unsigned long long a, b, c, d;
            asm volatile("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];"
                         : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(buf + 2 * s));
            acc += a ^ b ^ c ^ d;
        } else {  // two 16-B loads of the same sector
            const ulonglong2 a = __ldg(buf + 2 * s), b = __ldg(buf + 2 * s + 1);
            acc += a.x ^ a.y ^ b.x ^ b.y;
        }
    }
    if (acc == 0x123456789ull) *sink = acc;
}

template <int MODE>
static float run(const ulonglong2* buf, uint64_t slots, uint64_t items, unsigned long long* sink) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int grid = 148 * 8;
    k_gather<MODE><<<grid, 256>>>(buf, slots - 1, items, sink);
    cudaEventRecord(a);
    k_gather<MODE><<<grid, 256>>>(buf, slots - 1, items, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

int main() {
    const uint64_t big = 4ull << 30, small = 32ull << 20;
    ulonglong2* buf;
    unsigned long long* sink;
    if (cudaMalloc(&buf, big) != cudaSuccess || cudaMalloc(&sink, 8) != cudaSuccess) return 1;
    cudaMemset(buf, 1, big);
    const uint64_t items = 1ull << 28;
    const char* names[3] = {"16-B load", "32-B load (v4.u64)", "2 x 16-B same sector"};
    for (uint64_t bytes : {small, big}) {
        const uint64_t slots = bytes / 32;
        for (int mode = 0; mode < 3; ++mode) {
            const float ms = mode == 0 ? run<0>(buf, slots, items, sink)
                           : mode == 1 ? run<1>(buf, slots, items, sink)
                                       : run<2>(buf, slots, items, sink);
            printf("{\"buffer_mb\": %llu, \"mode\": \"%s\", \"ms\": %.3f, \"g_items_per_s\": %.2f}\n",
                   (unsigned long long)(bytes >> 20), names[mode], ms, items / (ms * 1e-3) / 1e9);
        }
    }
    cudaFree(buf);
    return 0;
}
