/* rtf_demo.c -- using librtf.so from plain C (no Python, no PyTorch): the C ABI
 * of include/rtf.h is the whole interface.  Builds the forest of the
 * triangular distribution p_i = i + 1 (n = 1000, m = 256), samples a
 * stratified set of 2^20 points and checks every bucket count against N p_i
 * (a stratified set places N p_i points in interval i, up to rounding).
 *
 *   gcc -O2 -o rtf_demo examples/rtf_demo.c -Iinclude -I/usr/local/cuda/include \
 *       -Lpaper_1901_05423_b200 -lrtf -L/usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_1901_05423_b200
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime.h>

#include "rtf.h"

#define CHECK(x)                                                                  \
    do {                                                                          \
        int s_ = (int)(x);                                                        \
        if (s_) {                                                                 \
            fprintf(stderr, "%s failed: %d (%s)\n", #x, s_, rtf_status_string(s_)); \
            return 1;                                                             \
        }                                                                         \
    } while (0)

int main(void) {
    const uint32_t n = 1000, m = 256;
    const uint64_t N = 1u << 20;
    float *p_host = malloc(sizeof(float) * n);
    double total = 0.0;
    for (uint32_t i = 0; i < n; ++i) total += (p_host[i] = (float)(i + 1));
    uint32_t *xi_host = malloc(sizeof(uint32_t) * N);
    for (uint64_t k = 0; k < N; ++k) xi_host[k] = (uint32_t)(k << 12);  /* k / N */

    float *p;
    uint32_t *xi;
    int32_t *out;
    void *forest_buf, *ws;
    const size_t fb = rtf_forest_bytes(n, m, 1), wb = rtf_workspace_bytes(n, m, 0);
    if (cudaMalloc((void **)&p, sizeof(float) * n) || cudaMalloc((void **)&xi, 4 * N) ||
        cudaMalloc((void **)&out, 4 * N) || cudaMalloc(&forest_buf, fb) || cudaMalloc(&ws, wb)) {
        fprintf(stderr, "cudaMalloc failed\n");
        return 1;
    }
    cudaMemcpy(p, p_host, sizeof(float) * n, cudaMemcpyHostToDevice);
    cudaMemcpy(xi, xi_host, 4 * N, cudaMemcpyHostToDevice);

    rtf_forest f;
    CHECK(rtf_workspace_init(ws, wb, n, m, 0, NULL));
    CHECK(rtf_build(p, n, m, 0, forest_buf, fb, ws, wb, NULL, &f));
    CHECK(rtf_sample(&f, xi, N, out, NULL));
    rtf_header h;
    CHECK(rtf_forest_status(&f, NULL, &h));

    int32_t *out_host = malloc(4 * N);
    cudaMemcpy(out_host, out, 4 * N, cudaMemcpyDeviceToHost);
    uint64_t *count = calloc(n, sizeof(uint64_t));
    for (uint64_t k = 0; k < N; ++k) {
        if (out_host[k] < 0 || (uint32_t)out_host[k] >= n) {
            fprintf(stderr, "bad index %d\n", out_host[k]);
            return 1;
        }
        if (k && out_host[k] < out_host[k - 1]) {
            fprintf(stderr, "not monotone at %llu\n", (unsigned long long)k);
            return 1;
        }
        ++count[out_host[k]];
    }
    double worst = 0.0;
    for (uint32_t i = 0; i < n; ++i) {
        const double d = fabs((double)count[i] - (double)N * p_host[i] / total);
        if (d > worst) worst = d;
    }
    printf("n=%u m=%u n'=%u T=%llu, %llu stratified samples, worst |count - N p| = %.3f\n", n, m,
           h.n_pos, (unsigned long long)h.total, (unsigned long long)N, worst);
    if (worst > 1.0) {
        fprintf(stderr, "histogram off\n");
        return 1;
    }
    printf("ok (%llu librtf kernels)\n", (unsigned long long)rtf_launch_count());
    return 0;
}
