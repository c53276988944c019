#include <cstdio>
#include <cstdint>
#include "../paper_1901_05423_b200/csrc/rtf_device.cuh"
__global__ void k(const uint64_t* d, uint64_t n, unsigned long long* bad) {
    for (uint64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint64_t a = rtf::reciprocal_of(d[i]), b = rtf::reciprocal_fast(d[i]);
        if (a != b) atomicAdd(bad, 1ull);
    }
}
int main() {
    const uint64_t n = 1 << 22;
    uint64_t* h = (uint64_t*)malloc(n * 8);
    uint64_t s = 88172645463325252ull;
    for (uint64_t i = 0; i < n; ++i) {
        s ^= s << 13; s ^= s >> 7; s ^= s << 17;
        uint64_t v = s | (1ull << 63);
        if (i < 64) v = (1ull << 63) + i;                // smallest d
        else if (i < 128) v = ~0ull - (i - 64);         // largest d
        else if (i < 4096) v = (1ull << 63) | (s >> (i % 60)) | ((1ull << (i % 63)));
        h[i] = v;
    }
    uint64_t* d; unsigned long long* bad; cudaMalloc(&d, n * 8); cudaMalloc(&bad, 8);
    cudaMemcpy(d, h, n * 8, cudaMemcpyHostToDevice); cudaMemset(bad, 0, 8);
    k<<<1184, 256>>>(d, n, bad);
    unsigned long long hb = 0; cudaMemcpy(&hb, bad, 8, cudaMemcpyDeviceToHost);
    printf("mismatches %llu of %llu (%s)\n", hb, (unsigned long long)n, cudaGetErrorString(cudaGetLastError()));
    return hb != 0;
}
