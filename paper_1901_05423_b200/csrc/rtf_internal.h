// rtf_internal.h -- declarations shared between librtf translation units (not installed).
#pragma once
#include <algorithm>
#include <atomic>
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/rtf.h"

namespace rtf {

constexpr uint32_t kRowsMax = 4096;  // rtf_build_rows: n_row, m_row limit
constexpr int kMaxDevices = 64;     // per-device launch attributes cached by the launchers

// phases of the build kernel (bitmask); a single-GPU build runs kPhFull
enum : uint32_t {
    kPhScale = 1,     // A: max weight, data flags
    kPhTotals = 2,    // B: tile aggregates
    kPhSpine = 4,     // C: exclusive tile prefixes (+ header or shard total)
    kPhTiles = 8,     // D: keys, split levels, table, in-tile Alg. 1, records
    kPhRuns = 16,     // E: long empty-cell runs of the table
    kPhCross = 32,    // E: cross-tile links from the tiles' spines
    kPhFull = kPhScale | kPhTotals | kPhSpine | kPhTiles | kPhRuns | kPhCross,
};
constexpr uint32_t kBuildShardedLayout = 0x100;  // internal flag: room for all shards' rows
constexpr uint32_t kMaxShards = 1024;

// SM count of the current device, cached per device (grid-stride launchers
// size their grids in multiples of it)
inline int device_sms() {
    static std::atomic<int> cache[kMaxDevices] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return 148;
    int s = cache[dev].load(std::memory_order_relaxed);
    if (!s) {
        if (cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || s <= 0)
            s = 148;
        cache[dev].store(s, std::memory_order_relaxed);
    }
    return s;
}

inline int ceil_log2_u32(uint32_t n) {
    int c = 0;
    while ((1ull << c) < (uint64_t)n) ++c;
    return c;
}

struct WsLayout {
    uint32_t nt;  // tiles
    uint32_t qcap;
    uint32_t nt_cap;  // rows phase E can link (a sharded finish: all shards' tiles)
    size_t maxpart, counters, scale, total, excl, rng, rpre, spine, tmax, bmax, queue, peers,
        jbound, bytes;
};

// one call of a sharded build (config 4); see rtf_shard_* in include/rtf.h
struct ShardCall {
    uint32_t phases, n_global, index_base, rank, count, nt_in;
    const void* totals;        // device: count shard totals (16 B each)
    const void* spine_in;      // device: finish -- all shards' tile spines (nt_in rows)
    uint32_t j_lo = 0, j_hi = 0xffffffffu;  // finish: node slots this rank holds
    uint32_t npeer = 0;  // fused ranged build: peer pointers already in the workspace
    int32_t j_rank = -1;  // >= 0: finish reads [j_lo, j_hi) = jbound[j_rank .. j_rank + 1]
};

// phase A of a host-buffer build, one chunk of p at a time (rtf_build_host):
// MAX-reduces into the workspace's scale word (cleared first by clear_scale)
cudaError_t launch_scale_chunk(const float* p, uint32_t n, void* ws, const WsLayout& L,
                               cudaStream_t st, int* launches);
cudaError_t clear_scale(void* ws, const WsLayout& L, cudaStream_t st);

// leaves of nodes[j0, j0 + cnt) whose cell is below bound[k]: counts[k], k < nb
cudaError_t launch_count_cells(const rtf_node* nodes, uint32_t j0, uint32_t cnt, uint32_t m,
                               const uint32_t* bounds, uint32_t nb, uint32_t* counts,
                               cudaStream_t st, int* launches);

uint32_t build_rows(uint32_t n, uint32_t flags);  // warp ranges (spine rows) of a build
size_t build_workspace_layout(uint32_t n, uint32_t m, uint32_t flags, WsLayout* L,
                              uint32_t n_global = 0);
size_t spine_row_bytes();       // bytes of one tile-spine row

cudaError_t launch_build(const float* p, uint32_t n, uint32_t m, uint32_t flags, rtf_header* hdr,
                         rtf_node* nodes, rtf_ref* table, uint64_t* cdf, void* ws,
                         const WsLayout& L, cudaStream_t st, int* launches,
                         const ShardCall* sc = nullptr);

cudaError_t launch_build_rows(const float* p, uint32_t rows, uint32_t n_row, uint32_t m_row,
                              rtf_header* hdr, rtf_node* nodes, rtf_ref* table, int32_t* jmap,
                              cudaStream_t st, int* launches);

// 2-D (Sec.6): row weights from the rows' headers, and the component-wise sampler
cudaError_t launch_rows_jmap(const float* p, uint32_t W, uint32_t H, const rtf_header* hdr,
                             rtf_node* nodes, int32_t* jmap, cudaStream_t st, int* launches);
cudaError_t launch_row_weights(const rtf_header* rows_hdr, uint32_t H, uint32_t W, float* q,
                               uint32_t* dense, cudaStream_t st, int* launches);
cudaError_t launch_sample_2d(const rtf_forest2d& f, const uint32_t* xi1, const uint32_t* xi2,
                             uint64_t count, int32_t* pixel, float* pos, cudaStream_t st,
                             int* launches);

cudaError_t launch_sample(const rtf_forest& f, const uint32_t* row, const uint32_t* xi,
                          uint64_t count, int32_t* out, cudaStream_t st, int* launches);

cudaError_t launch_sample_f32(const rtf_forest& f, const float* xi, uint64_t count, int32_t* out,
                              cudaStream_t st, int* launches);

cudaError_t launch_sample_loads(const rtf_forest& f, const uint32_t* xi, uint64_t count,
                                int32_t* loads, int32_t* loads_plain, cudaStream_t st,
                                int* launches);
cudaError_t launch_fallback(const rtf_forest& f, uint32_t* depth, uint32_t* last, cudaStream_t st,
                            int* launches);
// 4-ary collapsed records (rtf_quad.cu)
cudaError_t launch_collapse4(const rtf_forest& f, void* rec4, cudaStream_t st, int* launches);
cudaError_t launch_sample4(const rtf_forest& f, const void* rec4, const uint32_t* xi,
                           uint64_t count, int32_t* out, cudaStream_t st, int* launches);

cudaError_t launch_bsearch(const uint64_t* cdf, uint32_t n, const rtf_header* hdr,
                           const uint32_t* xi, uint64_t count, int32_t* out, cudaStream_t st,
                           int* launches);

cudaError_t launch_eytzinger_build(const uint64_t* cdf, uint32_t n, uint64_t* eyt,
                                   cudaStream_t st, int* launches);
cudaError_t launch_eytzinger(const uint64_t* eyt, uint32_t n, const rtf_header* hdr,
                             const uint32_t* xi, uint64_t count, int32_t* out, cudaStream_t st,
                             int* launches);

cudaError_t launch_alias_2d(const uint2* marg, uint32_t ky, const uint2* rows, uint32_t kx,
                            uint32_t W, const uint32_t* xi1, const uint32_t* xi2, uint64_t count,
                            int32_t* pixel, cudaStream_t st, int* launches);
cudaError_t launch_alias(const uint2* tab, uint32_t k, const uint32_t* xi, uint64_t count,
                         int32_t* out, cudaStream_t st, int* launches);
cudaError_t launch_cutpoint_build(const uint64_t* cdf, uint32_t n, uint32_t m, uint32_t* cut,
                                  cudaStream_t st, int* launches);

cudaError_t launch_cutpoint(const uint64_t* cdf, uint32_t n, const rtf_header* hdr,
                            const uint32_t* cut, uint32_t m, bool binary, const uint32_t* xi,
                            uint64_t count, int32_t* out, cudaStream_t st, int* launches);

cudaError_t launch_philox(uint64_t seed, uint64_t start, uint64_t count, uint32_t* out,
                          cudaStream_t st, int* launches);

// Slot-arrival check (debug builds only, -DRTF_SLOT_CHECK; rtf_debug_slot_buffers,
// tools/slotcheck_target.py): every link write also counts, per record child
// field, how often it was written, and per record, how often it was linked as
// an internal node (node < 0: a leaf reference, not counted).  A race between
// two writers of one field shows as a count of 2 even when the bytes agree;
// Alg. 1's invariant (every internal node gets exactly one
// parent) is a count of exactly 1 per non-anchor record.  Each translation
// unit has its own copy of the two pointers (set by rtf_debug_slot_buffers).
#ifdef RTF_SLOT_CHECK
static __device__ uint32_t* g_slot_fields;  // 2 per record (+ 1 spare record)
static __device__ uint32_t* g_slot_nodes;   // per record
#define RTF_SLOT(rec, side, node)                                                         \
    do {                                                                                  \
        if (g_slot_fields) atomicAdd(g_slot_fields + 2ull * (uint64_t)(rec) + (side), 1u); \
        if (g_slot_nodes && (int64_t)(node) >= 0) atomicAdd(g_slot_nodes + (uint64_t)(node), 1u); \
    } while (0)
#else
#define RTF_SLOT(rec, side, node) \
    do {                          \
    } while (0)
#endif

}  // namespace rtf
