// tools/microbench.cu -- calibration microbenchmarks (not product code).
// Times streaming reads of a 64 MiB float array in several shapes, and the
// per-element costs of the build's ingredients, with CUDA events.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/mb tools/microbench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ float4 ldnc(const float* p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    return r;
}

// grid-stride max, U float4 per iteration
template <int U>
__global__ void k_max(const float* p, uint32_t n4, uint32_t* out) {
    uint32_t gs = gridDim.x * blockDim.x, q = blockIdx.x * blockDim.x + threadIdx.x;
    float m = 0.f;
    for (; q + (U - 1) * gs < n4; q += U * gs) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ldnc(p + 4ull * (q + u * gs));
#pragma unroll
        for (int u = 0; u < U; ++u) m = fmaxf(m, fmaxf(fmaxf(v[u].x, v[u].y), fmaxf(v[u].z, v[u].w)));
    }
    for (; q < n4; q += gs) { float4 v = ldnc(p + 4ull * q); m = fmaxf(m, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w))); }
    if (m == 12345.f) out[0] = 1;
}

// one tile per CTA: THREADS x NF4 float4, block reduce (like K2)
template <int THREADS, int NF4, int MODE>
__global__ void k_tile(const float* p, uint32_t* out, double scale) {
    const uint32_t base = blockIdx.x * THREADS * NF4 * 4;
    float4 v[NF4];
#pragma unroll
    for (int k = 0; k < NF4; ++k) v[k] = ldnc(p + base + 4 * (k * THREADS + threadIdx.x));
    uint64_t acc = 0;
#pragma unroll
    for (int k = 0; k < NF4; ++k) {
        const float xs[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (MODE == 0) acc += __float_as_uint(xs[u]);
            else acc += xs[u] > 0.f ? __double2ull_rz((double)xs[u] * scale) : 0ull;
        }
    }
    for (int d = 16; d; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
    __shared__ uint64_t s[32];
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < THREADS / 32; ++w) acc += s[w];
        if (acc == 12345) out[0] = 1;
    }
}

template <typename F>
float timeit(F f, int reps = 20) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms * 1000.f / reps;
}

int main() {
    const uint32_t n = 1u << 24;
    float* p;
    uint32_t* out;
    CK(cudaMalloc(&p, 4ull * n));
    CK(cudaMalloc(&out, 64));
    // fill with positive values
    CK(cudaMemset(p, 0x3f, 4ull * n));
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    printf("SMs %d; 64 MiB read at 6.5 TB/s = %.1f us\n", sms, 4.0 * n / 6.5e12 * 1e6);
    for (int blocks : {sms * 2, sms * 4, sms * 8, 1024, 4096}) {
        printf("k_max<8>  grid %5d x 256: %7.2f us\n", blocks,
               timeit([&] { k_max<8><<<blocks, 256>>>(p, n / 4, out); }));
    }
    for (int blocks : {sms * 4, sms * 8}) {
        printf("k_max<4>  grid %5d x 256: %7.2f us\n", blocks,
               timeit([&] { k_max<4><<<blocks, 256>>>(p, n / 4, out); }));
        printf("k_max<16> grid %5d x 256: %7.2f us\n", blocks,
               timeit([&] { k_max<16><<<blocks, 256>>>(p, n / 4, out); }));
    }
    printf("k_tile<512,4,sum>  %4u CTAs: %7.2f us\n", n / 8192, timeit([&] { k_tile<512, 4, 0><<<n / 8192, 512>>>(p, out, 1.0); }));
    printf("k_tile<512,4,q64>  %4u CTAs: %7.2f us\n", n / 8192, timeit([&] { k_tile<512, 4, 1><<<n / 8192, 512>>>(p, out, 1.0); }));
    printf("k_tile<256,8,sum>  %4u CTAs: %7.2f us\n", n / 8192, timeit([&] { k_tile<256, 8, 0><<<n / 8192, 256>>>(p, out, 1.0); }));
    printf("k_tile<256,8,q64>  %4u CTAs: %7.2f us\n", n / 8192, timeit([&] { k_tile<256, 8, 1><<<n / 8192, 256>>>(p, out, 1.0); }));
    printf("k_tile<512,8,q64>  %4u CTAs: %7.2f us\n", n / 16384, timeit([&] { k_tile<512, 8, 1><<<n / 16384, 512>>>(p, out, 1.0); }));
    printf("k_tile<1024,4,q64> %4u CTAs: %7.2f us\n", n / 16384, timeit([&] { k_tile<1024, 4, 1><<<n / 16384, 1024>>>(p, out, 1.0); }));
    // empty launch overhead
    printf("empty launch x1:   %7.2f us\n", timeit([&] { k_tile<32, 1, 0><<<1, 32>>>(p, out, 1.0); }));
    return 0;
}
