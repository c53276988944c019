#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k_empty(int* p) { extern __shared__ int s[]; if (threadIdx.x == 9999) p[0] = s[0]; }
__device__ __forceinline__ void gbar(unsigned* bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned nb = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1) : 1u, old;
        asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(bar), "r"(nb) : "memory");
        unsigned v;
        do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory"); } while (((v ^ old) & 0x80000000u) == 0);
    }
    __syncthreads();
}
__global__ void k_bar(unsigned* bar, int nb) { extern __shared__ int s[]; for (int i = 0; i < nb; ++i) gbar(bar); }
int main() {
    int* p; cudaMalloc(&p, 64); unsigned* bar; cudaMalloc(&bar, 64); cudaMemset(bar, 0, 64);
    size_t smem = 98 * 1024;
    cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_bar, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int mode = 0; mode < 5; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            for (int i = 0; i < 100; ++i) {
                if (mode == 0) k_empty<<<296, 512, smem>>>(p);
                else if (mode == 1) { void* args[] = {&p}; cudaLaunchCooperativeKernel((void*)k_empty, 296, 512, args, smem, 0); }
                else { int nb = mode == 2 ? 1 : (mode == 3 ? 4 : 16); void* args[] = {&bar, &nb}; cudaLaunchCooperativeKernel((void*)k_bar, 296, 512, args, smem, 0); }
            }
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (rep) printf("mode %d: %.2f us per launch (%s)\n", mode, ms * 10, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
