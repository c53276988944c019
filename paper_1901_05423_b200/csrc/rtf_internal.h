// rtf_internal.h -- declarations shared between librtf translation units (not installed).
#pragma once
#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/rtf.h"

namespace rtf {

constexpr uint32_t kMaxScaleBlocks = 148 * 8;  // K1 grid cap (multiple of the SM count)
constexpr uint32_t kRowsMax = 4096;            // rtf_build_rows: n_row, m_row limit

inline int ceil_log2_u32(uint32_t n) {
    int c = 0;
    while ((1ull << c) < (uint64_t)n) ++c;
    return c;
}

struct WsLayout {
    uint32_t nt;  // tiles
    uint32_t qcap;
    size_t maxpart, counters, excl, pend, ob, lam, queue, total;
};

uint32_t build_tile_size(uint32_t flags);
size_t build_workspace_layout(uint32_t n, uint32_t m, uint32_t flags, WsLayout* L);

cudaError_t launch_build(const float* p, uint32_t n, uint32_t m, uint32_t flags, rtf_header* hdr,
                         rtf_node* nodes, int32_t* table, uint64_t* cdf, void* ws,
                         const WsLayout& L, cudaStream_t st, int* launches);

cudaError_t launch_build_rows(const float* p, uint32_t rows, uint32_t n_row, uint32_t m_row,
                              rtf_header* hdr, rtf_node* nodes, int32_t* table, cudaStream_t st,
                              int* launches);

cudaError_t launch_sample(const rtf_forest& f, const uint32_t* row, const uint32_t* xi,
                          uint64_t count, int32_t* out, cudaStream_t st, int* launches);

cudaError_t launch_sample_loads(const rtf_forest& f, const uint32_t* xi, uint64_t count,
                                int32_t* loads, cudaStream_t st, int* launches);

cudaError_t launch_bsearch(const uint64_t* cdf, uint32_t n, const rtf_header* hdr,
                           const uint32_t* xi, uint64_t count, int32_t* out, cudaStream_t st,
                           int* launches);

cudaError_t launch_philox(uint64_t seed, uint64_t start, uint64_t count, uint32_t* out,
                          cudaStream_t st, int* launches);

}  // namespace rtf
