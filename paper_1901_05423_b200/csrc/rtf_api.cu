// rtf_api.cu -- the C ABI of librtf (include/rtf.h): argument checks, buffer
// carve-up and launches on the caller's stream.  No device allocation, no CPU
// fallback: every result is computed by the kernels in rtf_build.cu,
// rtf_rows.cu and rtf_sample.cu.
#include <atomic>
#include <cstring>

#include "rtf_internal.h"

namespace {

std::atomic<uint64_t> g_launches{0};

constexpr size_t kAlign = 256;

inline size_t align_up(size_t x) { return (x + kAlign - 1) & ~(kAlign - 1); }

struct ForestLayout {
    size_t header, nodes, table, total;
};

ForestLayout forest_layout(uint32_t n, uint32_t m, uint32_t rows) {
    ForestLayout L;
    size_t off = 0;
    L.header = off;
    off += align_up(sizeof(rtf_header) * (size_t)rows);
    L.nodes = off;
    off += align_up(sizeof(rtf_node) * (size_t)n * rows);
    L.table = off;
    off += align_up(sizeof(rtf_ref) * (size_t)m * rows);
    L.total = off;
    return L;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline int check_nm(uint32_t n, uint32_t m) {
    if (n == 0 || m == 0) return RTF_EINVAL;
    if (n >= 0x80000000u || m >= 0x80000000u) return RTF_ETOOLARGE;
    return RTF_OK;
}

inline int finish(cudaError_t e, int launches) {
    g_launches.fetch_add((uint64_t)launches, std::memory_order_relaxed);
    return e == cudaSuccess ? RTF_OK : RTF_ECUDA;
}

}  // namespace

extern "C" {

const char* rtf_version(void) { return "rtf-b200 0.1 (sm_100a)"; }

const char* rtf_status_string(int s) {
    switch (s) {
        case RTF_OK: return "RTF_OK";
        case RTF_EINVAL: return "RTF_EINVAL";
        case RTF_EALLZERO: return "RTF_EALLZERO";
        case RTF_ETOOLARGE: return "RTF_ETOOLARGE";
        case RTF_ENOSPACE: return "RTF_ENOSPACE";
        case RTF_ECUDA: return "RTF_ECUDA";
        case RTF_EDATA: return "RTF_EDATA";
        default: return "RTF_UNKNOWN";
    }
}

uint64_t rtf_launch_count(void) { return g_launches.load(); }

size_t rtf_forest_bytes(uint32_t n, uint32_t m, uint32_t rows) {
    if (rows == 0) rows = 1;
    return forest_layout(n, m, rows).total;
}

size_t rtf_workspace_bytes(uint32_t n, uint32_t m, uint32_t flags) {
    rtf::WsLayout L;
    return rtf::build_workspace_layout(n ? n : 1, m ? m : 1, flags, &L);
}

int rtf_workspace_init(void* ws, size_t ws_bytes, uint32_t n, uint32_t m, uint32_t flags,
                       void* stream) {
    if (!ws) return RTF_EINVAL;
    if (int s = check_nm(n, m)) return s;
    rtf::WsLayout L;
    if (ws_bytes < rtf::build_workspace_layout(n, m, flags, &L)) return RTF_ENOSPACE;
    cudaStream_t st = as_stream(stream);
    unsigned char* w = static_cast<unsigned char*>(ws);
    // partials, counters (the grid barrier word must start at 0), prefixes;
    // the rest is written by every build before it is read
    const cudaError_t e = cudaMemsetAsync(w, 0, L.spine, st);
    return e == cudaSuccess ? RTF_OK : RTF_ECUDA;
}

int rtf_forest_view(void* buf, size_t bytes, uint32_t n, uint32_t m, uint32_t rows,
                    rtf_forest* out) {
    if (!buf || !out || rows == 0) return RTF_EINVAL;
    if (int s = check_nm(n, m)) return s;
    if (((uintptr_t)buf & (kAlign - 1)) != 0) return RTF_EINVAL;
    const ForestLayout L = forest_layout(n, m, rows);
    if (bytes < L.total) return RTF_ENOSPACE;
    unsigned char* b = static_cast<unsigned char*>(buf);
    out->n = n;
    out->m = m;
    out->rows = rows;
    out->flags = 0;
    out->header = reinterpret_cast<rtf_header*>(b + L.header);
    out->nodes = reinterpret_cast<rtf_node*>(b + L.nodes);
    out->table = reinterpret_cast<rtf_ref*>(b + L.table);
    return RTF_OK;
}

int rtf_build(const float* p, uint32_t n, uint32_t m, uint32_t flags, void* forest_buf,
              size_t forest_bytes, void* ws, size_t ws_bytes, void* stream, rtf_forest* out) {
    if (!p || !ws || !out) return RTF_EINVAL;
    if (flags & ~RTF_BUILD_SMALL_TILES) return RTF_EINVAL;
    if (((uintptr_t)p & 3u) != 0) return RTF_EINVAL;
    if (int s = rtf_forest_view(forest_buf, forest_bytes, n, m, 1, out)) return s;
    out->flags = flags;
    rtf::WsLayout L;
    if (ws_bytes < rtf::build_workspace_layout(n, m, flags, &L)) return RTF_ENOSPACE;
    if (((uintptr_t)ws & (kAlign - 1)) != 0) return RTF_EINVAL;
    int launches = 0;
    cudaError_t e;
    if (!(flags & RTF_BUILD_SMALL_TILES) && n <= rtf::kRowsMax && m <= rtf::kRowsMax)
        // one tile's worth: the row kernel builds the whole forest in one CTA's
        // shared memory (the same layout and bytes as a one-row batched forest),
        // without the cooperative kernel's grid barriers
        e = rtf::launch_build_rows(p, 1, n, m, out->header, out->nodes, out->table, nullptr,
                                   as_stream(stream), &launches);
    else
        e = rtf::launch_build(p, n, m, flags, out->header, out->nodes, out->table, nullptr, ws,
                              L, as_stream(stream), &launches);
    return finish(e, launches);
}

int rtf_build_rows(const float* p, uint32_t rows, uint32_t n_row, uint32_t m_row,
                   void* forest_buf, size_t forest_bytes, void* stream, rtf_forest* out) {
    if (!p || !out || rows == 0) return RTF_EINVAL;
    if (((uintptr_t)p & 3u) != 0) return RTF_EINVAL;
    if (int s = check_nm(n_row, m_row)) return s;
    if (n_row > rtf::kRowsMax || m_row > rtf::kRowsMax) return RTF_ETOOLARGE;
    if (int s = rtf_forest_view(forest_buf, forest_bytes, n_row, m_row, rows, out)) return s;
    int launches = 0;
    cudaError_t e = rtf::launch_build_rows(p, rows, n_row, m_row, out->header, out->nodes,
                                           out->table, nullptr, as_stream(stream), &launches);
    return finish(e, launches);
}

int rtf_forest_status(const rtf_forest* f, void* stream, rtf_header* headers_host) {
    if (!f || !f->header || f->rows == 0) return RTF_EINVAL;
    cudaStream_t st = as_stream(stream);
    rtf_header one;
    rtf_header* dst = headers_host ? headers_host : nullptr;
    int worst = RTF_OK;
    const size_t bytes = sizeof(rtf_header) * (size_t)f->rows;
    rtf_header* tmp = dst;
    bool owned = false;
    if (!tmp) {
        if (f->rows == 1) tmp = &one;
        else {
            tmp = new rtf_header[f->rows];
            owned = true;
        }
    }
    cudaError_t e = cudaMemcpyAsync(tmp, f->header, bytes, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) worst = RTF_ECUDA;
    else
        for (uint32_t r = 0; r < f->rows; ++r) {
            const uint32_t s = tmp[r].status;
            if (s & (RTF_DATA_NAN | RTF_DATA_INF | RTF_DATA_NEG)) worst = RTF_EDATA;
            else if ((s & RTF_DATA_ALLZERO) && worst == RTF_OK) worst = RTF_EALLZERO;
        }
    if (owned) delete[] tmp;
    return worst;
}

int rtf_sample(const rtf_forest* f, const uint32_t* xi, uint64_t count, int32_t* out,
               void* stream) {
    if (!f || !f->nodes || !f->table || !f->header || f->rows != 1) return RTF_EINVAL;
    if (count && (!xi || !out)) return RTF_EINVAL;
    if ((((uintptr_t)xi | (uintptr_t)out) & 3u) != 0) return RTF_EINVAL;
    int launches = 0;
    cudaError_t e = rtf::launch_sample(*f, nullptr, xi, count, out, as_stream(stream), &launches);
    return finish(e, launches);
}

size_t rtf_quad_bytes(uint32_t n) { return 32 * (size_t)(n ? n : 1); }

int rtf_build_quad(const rtf_forest* f, void* rec4, size_t rec4_bytes, void* stream) {
    if (!f || !f->nodes || !f->header || f->rows != 1 || !rec4) return RTF_EINVAL;
    if (((uintptr_t)rec4 & 31u) != 0) return RTF_EINVAL;
    if (rec4_bytes < rtf_quad_bytes(f->n)) return RTF_ENOSPACE;
    int launches = 0;
    cudaError_t e = rtf::launch_collapse4(*f, rec4, as_stream(stream), &launches);
    return finish(e, launches);
}

int rtf_sample_quad(const rtf_forest* f, const void* rec4, const uint32_t* xi, uint64_t count,
                    int32_t* out, void* stream) {
    if (!f || !f->table || !f->header || f->rows != 1 || !rec4) return RTF_EINVAL;
    if (f->flags & RTF_FOREST_MARKED) return RTF_EINVAL;  // the quad sampler does not bisect
    if (((uintptr_t)rec4 & 31u) != 0) return RTF_EINVAL;
    if (count && (!xi || !out)) return RTF_EINVAL;
    if ((((uintptr_t)xi | (uintptr_t)out) & 3u) != 0) return RTF_EINVAL;
    int launches = 0;
    cudaError_t e = rtf::launch_sample4(*f, rec4, xi, count, out, as_stream(stream), &launches);
    return finish(e, launches);
}

int rtf_sample_f32(const rtf_forest* f, const float* xi, uint64_t count, int32_t* out,
                   void* stream) {
    if (!f || !f->nodes || !f->table || !f->header || f->rows != 1) return RTF_EINVAL;
    if (count && (!xi || !out)) return RTF_EINVAL;
    if ((((uintptr_t)xi | (uintptr_t)out) & 3u) != 0) return RTF_EINVAL;
    int launches = 0;
    cudaError_t e = rtf::launch_sample_f32(*f, xi, count, out, as_stream(stream), &launches);
    return finish(e, launches);
}

int rtf_sample_loads(const rtf_forest* f, const uint32_t* xi, uint64_t count, int32_t* loads,
                     int32_t* loads_plain, void* stream) {
    if (!f || !f->nodes || !f->table || !f->header || f->rows != 1) return RTF_EINVAL;
    if (count && (!xi || !loads)) return RTF_EINVAL;
    if ((((uintptr_t)xi | (uintptr_t)loads | (uintptr_t)loads_plain) & 3u) != 0)
        return RTF_EINVAL;
    int launches = 0;
    cudaError_t e = rtf::launch_sample_loads(*f, xi, count, loads, loads_plain,
                                             as_stream(stream), &launches);
    return finish(e, launches);
}

int rtf_sample_rows(const rtf_forest* f, const uint32_t* row, const uint32_t* xi, uint64_t count,
                    int32_t* out, void* stream) {
    if (!f || !f->nodes || !f->table || !f->header || f->rows == 0) return RTF_EINVAL;
    if (count && (!xi || !out || !row)) return RTF_EINVAL;
    if ((((uintptr_t)xi | (uintptr_t)out | (uintptr_t)row) & 3u) != 0) return RTF_EINVAL;
    int launches = 0;
    cudaError_t e = rtf::launch_sample(*f, row, xi, count, out, as_stream(stream), &launches);
    return finish(e, launches);
}

// ------------------------------------------------------------------ 2-D (Sec.6)

namespace {
struct Layout2d {
    size_t rows, marginal, rows_jmap, marg_jmap, weights, dense, ws, ws_bytes, total;
};
// rows wider than the row kernel's 4096 entries (or with more than 4096
// cells), and a marginal of more than 4096 rows, are built one distribution at
// a time by the cooperative kernel, which needs a build workspace
bool rows_big(uint32_t W, uint32_t mx) { return W > rtf::kRowsMax || mx > rtf::kRowsMax; }
Layout2d layout_2d(uint32_t W, uint32_t H, uint32_t mx, uint32_t my) {
    Layout2d L;
    size_t off = 0;
    L.rows = off;
    off += align_up(rtf_forest_bytes(W, mx, H));
    L.marginal = off;
    off += align_up(rtf_forest_bytes(H, my, 1));
    L.rows_jmap = off;
    off += align_up(sizeof(int32_t) * (size_t)W * H);
    L.marg_jmap = off;
    off += align_up(sizeof(int32_t) * (size_t)H);
    L.weights = off;
    off += align_up(sizeof(float) * (size_t)H);
    L.dense = off;
    off += align_up(sizeof(uint32_t) * (((size_t)H + 31) / 32));
    L.ws = off;
    L.ws_bytes = 0;
    if (rows_big(W, mx) || rows_big(H, my)) {
        rtf::WsLayout wl;
        L.ws_bytes = std::max(rows_big(W, mx) ? rtf::build_workspace_layout(W, mx, 0, &wl) : 0,
                              rows_big(H, my) ? rtf::build_workspace_layout(H, my, 0, &wl) : 0);
        off += align_up(L.ws_bytes);
    }
    L.total = off;
    return L;
}
int check_2d(uint32_t W, uint32_t H, uint32_t mx, uint32_t my) {
    if (W == 0 || H == 0 || mx == 0 || my == 0) return RTF_EINVAL;
    if ((uint64_t)W * H > 0x7fffffffull) return RTF_ETOOLARGE;  // pixel indices are int32
    if (int s = check_nm(W, mx)) return s;
    return check_nm(H, my);
}
}  // namespace

size_t rtf_forest2d_bytes(uint32_t W, uint32_t H, uint32_t mx, uint32_t my) {
    return layout_2d(W ? W : 1, H ? H : 1, mx ? mx : 1, my ? my : 1).total;
}

int rtf_build_2d(const float* p, uint32_t W, uint32_t H, uint32_t mx, uint32_t my, void* buf,
                 size_t bytes, void* stream, rtf_forest2d* out) {
    if (!p || !buf || !out || ((uintptr_t)p & 3u)) return RTF_EINVAL;
    if (int s = check_2d(W, H, mx, my)) return s;
    if (((uintptr_t)buf & (kAlign - 1)) != 0) return RTF_EINVAL;
    const Layout2d L = layout_2d(W, H, mx, my);
    if (bytes < L.total) return RTF_ENOSPACE;
    unsigned char* b = static_cast<unsigned char*>(buf);
    out->W = W;
    out->H = H;
    out->mx = mx;
    out->my = my;
    if (int s = rtf_forest_view(b + L.rows, L.marginal - L.rows, W, mx, H, &out->rows)) return s;
    if (int s = rtf_forest_view(b + L.marginal, L.rows_jmap - L.marginal, H, my, 1, &out->marginal))
        return s;
    out->rows_jmap = reinterpret_cast<int32_t*>(b + L.rows_jmap);
    out->marg_jmap = reinterpret_cast<int32_t*>(b + L.marg_jmap);
    out->weights = reinterpret_cast<float*>(b + L.weights);
    out->rows_dense = reinterpret_cast<uint32_t*>(b + L.dense);
    cudaStream_t st = as_stream(stream);
    int launches = 0;
    // one distribution of n entries and m cells per row of `rows` (the row
    // kernel, or one cooperative build per row, then the index maps)
    auto build = [&](const float* q, uint32_t rows, uint32_t n, uint32_t m, rtf_forest& f,
                     int32_t* jmap) -> cudaError_t {
        if (!rows_big(n, m))
            return rtf::launch_build_rows(q, rows, n, m, f.header, f.nodes, f.table, jmap, st,
                                          &launches);
        rtf::WsLayout wl;
        rtf::build_workspace_layout(n, m, 0, &wl);
        void* ws = b + L.ws;
        cudaError_t e = cudaMemsetAsync(ws, 0, wl.spine, st);  // rtf_workspace_init
        for (uint32_t y = 0; y < rows && e == cudaSuccess; ++y)
            e = rtf::launch_build(q + (size_t)y * n, n, m, 0, f.header + y, f.nodes + (size_t)y * n,
                                  f.table + (size_t)y * m, nullptr, ws, wl, st, &launches);
        if (e == cudaSuccess) e = rtf::launch_rows_jmap(q, n, rows, f.header, f.nodes, jmap, st, &launches);
        return e;
    };
    cudaError_t e = build(p, H, W, mx, out->rows, out->rows_jmap);
    if (e == cudaSuccess)
        e = rtf::launch_row_weights(out->rows.header, H, W, out->weights, out->rows_dense, st,
                                    &launches);
    if (e == cudaSuccess) e = build(out->weights, 1, H, my, out->marginal, out->marg_jmap);
    return finish(e, launches);
}

int rtf_forest2d_status(const rtf_forest2d* f, void* stream) {
    if (!f) return RTF_EINVAL;
    return rtf_forest_status(&f->marginal, stream, nullptr);
}

int rtf_sample_2d(const rtf_forest2d* f, const uint32_t* xi1, const uint32_t* xi2, uint64_t count,
                  int32_t* pixel, float* pos, void* stream) {
    if (!f || !f->rows.nodes || !f->marginal.nodes || !f->rows_jmap || !f->marg_jmap ||
        !f->rows_dense)
        return RTF_EINVAL;
    if (count && (!xi1 || !xi2 || !pixel)) return RTF_EINVAL;
    if ((((uintptr_t)xi1 | (uintptr_t)xi2 | (uintptr_t)pixel) & 3u) || ((uintptr_t)pos & 7u))
        return RTF_EINVAL;
    int launches = 0;
    cudaError_t e = rtf::launch_sample_2d(*f, xi1, xi2, count, pixel, pos, as_stream(stream),
                                          &launches);
    return finish(e, launches);
}

int rtf_build_cdf(const float* p, uint32_t n, uint64_t* cdf, rtf_header* header, void* ws,
                  size_t ws_bytes, void* stream) {
    if (!p || !cdf || !header || !ws) return RTF_EINVAL;
    if (int s = check_nm(n, 1)) return s;
    if ((((uintptr_t)p & 3u) | ((uintptr_t)cdf & 7u) | ((uintptr_t)header & 7u)) != 0)
        return RTF_EINVAL;
    rtf::WsLayout L;
    if (ws_bytes < rtf::build_workspace_layout(n, 1, 0, &L)) return RTF_ENOSPACE;
    int launches = 0;
    cudaError_t e = rtf::launch_build(p, n, 1, 0, header, nullptr, nullptr, cdf, ws, L,
                                      as_stream(stream), &launches);
    return finish(e, launches);
}

int rtf_sample_bsearch(const uint64_t* cdf, uint32_t n, const rtf_header* header,
                       const uint32_t* xi, uint64_t count, int32_t* out, void* stream) {
    if (!cdf || !header) return RTF_EINVAL;
    if (int s = check_nm(n, 1)) return s;
    if (count && (!xi || !out)) return RTF_EINVAL;
    if ((((uintptr_t)xi | (uintptr_t)out) & 3u) != 0) return RTF_EINVAL;
    int launches = 0;
    cudaError_t e = rtf::launch_bsearch(cdf, n, header, xi, count, out, as_stream(stream),
                                        &launches);
    return finish(e, launches);
}

size_t rtf_fallback_bytes(uint32_t m) { return 2 * sizeof(uint32_t) * (size_t)(m ? m : 1); }

int rtf_build_fallback(rtf_forest* f, void* ws, size_t ws_bytes, void* stream) {
    if (!f || !f->nodes || !f->table || !f->header || f->rows != 1 || !ws) return RTF_EINVAL;
    if (((uintptr_t)ws & 3u) != 0) return RTF_EINVAL;
    if (ws_bytes < rtf_fallback_bytes(f->m)) return RTF_ENOSPACE;
    uint32_t* depth = static_cast<uint32_t*>(ws);
    int launches = 0;
    cudaError_t e = rtf::launch_fallback(*f, depth, depth + f->m, as_stream(stream), &launches);
    if (e == cudaSuccess) f->flags |= RTF_FOREST_MARKED;
    return finish(e, launches);
}

uint64_t rtf_eytzinger_slots(uint32_t n) { return 1ull << rtf::ceil_log2_u32(n); }

int rtf_build_eytzinger(const uint64_t* cdf, uint32_t n, uint64_t* eyt, void* stream) {
    if (!cdf || !eyt) return RTF_EINVAL;
    if (int s = check_nm(n, 1)) return s;
    if ((((uintptr_t)cdf | (uintptr_t)eyt) & 7u) != 0) return RTF_EINVAL;
    int launches = 0;
    cudaError_t e = rtf::launch_eytzinger_build(cdf, n, eyt, as_stream(stream), &launches);
    return finish(e, launches);
}

int rtf_sample_eytzinger(const uint64_t* eyt, uint32_t n, const rtf_header* header,
                         const uint32_t* xi, uint64_t count, int32_t* out, void* stream) {
    if (!eyt || !header) return RTF_EINVAL;
    if (int s = check_nm(n, 1)) return s;
    if (count && (!xi || !out)) return RTF_EINVAL;
    if ((((uintptr_t)xi | (uintptr_t)out) & 3u) != 0 || ((uintptr_t)eyt & 7u) != 0)
        return RTF_EINVAL;
    int launches = 0;
    cudaError_t e = rtf::launch_eytzinger(eyt, n, header, xi, count, out, as_stream(stream),
                                          &launches);
    return finish(e, launches);
}

int rtf_sample_alias(const void* table, uint32_t k, const uint32_t* xi, uint64_t count,
                     int32_t* out, void* stream) {
    if (!table || k < 1 || k > 31) return RTF_EINVAL;
    if (count && (!xi || !out)) return RTF_EINVAL;
    if ((((uintptr_t)xi | (uintptr_t)out) & 3u) != 0 || ((uintptr_t)table & 7u) != 0)
        return RTF_EINVAL;
    int launches = 0;
    cudaError_t e = rtf::launch_alias(static_cast<const uint2*>(table), k, xi, count, out,
                                      as_stream(stream), &launches);
    return finish(e, launches);
}

int rtf_sample_alias_2d(const void* marg, uint32_t ky, const void* rows, uint32_t kx,
                        uint32_t W, uint32_t H, const uint32_t* xi1, const uint32_t* xi2,
                        uint64_t count, int32_t* pixel, void* stream) {
    if (!marg || !rows || ky < 1 || ky > 31 || kx < 1 || kx > 31) return RTF_EINVAL;
    if (W == 0 || H == 0 || W > (1u << kx) || H > (1u << ky)) return RTF_EINVAL;
    if ((uint64_t)W * H > 0x7fffffffull) return RTF_ETOOLARGE;
    if (count && (!xi1 || !xi2 || !pixel)) return RTF_EINVAL;
    if ((((uintptr_t)xi1 | (uintptr_t)xi2 | (uintptr_t)pixel) & 3u) != 0 ||
        (((uintptr_t)marg | (uintptr_t)rows) & 7u) != 0)
        return RTF_EINVAL;
    int launches = 0;
    cudaError_t e = rtf::launch_alias_2d(static_cast<const uint2*>(marg), ky,
                                         static_cast<const uint2*>(rows), kx, W, xi1, xi2, count,
                                         pixel, as_stream(stream), &launches);
    return finish(e, launches);
}

int rtf_build_cutpoint(const uint64_t* cdf, uint32_t n, uint32_t m, uint32_t* cut, void* stream) {
    if (!cdf || !cut) return RTF_EINVAL;
    if (int s = check_nm(n, m)) return s;
    if (m == 0xffffffffu) return RTF_ETOOLARGE;
    int launches = 0;
    cudaError_t e = rtf::launch_cutpoint_build(cdf, n, m, cut, as_stream(stream), &launches);
    return finish(e, launches);
}

int rtf_sample_cutpoint(const uint64_t* cdf, uint32_t n, const rtf_header* header,
                        const uint32_t* cut, uint32_t m, int binary, const uint32_t* xi,
                        uint64_t count, int32_t* out, void* stream) {
    if (!cdf || !header || !cut) return RTF_EINVAL;
    if (int s = check_nm(n, m)) return s;
    if (count && (!xi || !out)) return RTF_EINVAL;
    if ((((uintptr_t)xi | (uintptr_t)out) & 3u) != 0) return RTF_EINVAL;
    int launches = 0;
    cudaError_t e = rtf::launch_cutpoint(cdf, n, header, cut, m, binary != 0, xi, count, out,
                                         as_stream(stream), &launches);
    return finish(e, launches);
}

int rtf_build_host(const float* p_host, uint32_t n, uint32_t m, uint32_t flags, float* p_dev,
                   void* forest_buf, size_t forest_bytes, void* ws, size_t ws_bytes, void* stream,
                   rtf_forest* out, rtf_header* header_host) {
    if (!p_host || !p_dev) return RTF_EINVAL;
    if (int s = check_nm(n, m)) return s;
    cudaStream_t st = as_stream(stream);
    rtf::WsLayout L;
    const bool rows_kernel = !(flags & RTF_BUILD_SMALL_TILES) && n <= rtf::kRowsMax && m <= rtf::kRowsMax;
    if (rows_kernel || !ws || ((uintptr_t)ws & (kAlign - 1)) != 0 || ((uintptr_t)p_dev & 3u) != 0 ||
        (flags & ~RTF_BUILD_SMALL_TILES) || ws_bytes < rtf::build_workspace_layout(n, m, flags, &L)) {
        // one copy, then the build (which validates its arguments itself)
        if (cudaMemcpyAsync(p_dev, p_host, sizeof(float) * (size_t)n, cudaMemcpyHostToDevice, st) !=
            cudaSuccess)
            return RTF_ECUDA;
        int s = rtf_build(p_dev, n, m, flags, forest_buf, forest_bytes, ws, ws_bytes, stream, out);
        if (s != RTF_OK) return s;
        return rtf_forest_status(out, stream, header_host);
    }
    if (int s = rtf_forest_view(forest_buf, forest_bytes, n, m, 1, out)) return s;
    out->flags = flags;
    // The copy goes in chunks on a copy stream; phase A (the largest weight,
    // the data flags) runs on each chunk on the caller's stream as soon as it
    // has landed, overlapping the next chunks' copies; the build then skips
    // phase A and reads the scale word (the sharded build's kPhScale-less
    // call, here with one shard).
    constexpr uint32_t kChunks = 8;
    const uint32_t chunk = ((n + kChunks - 1) / kChunks + 1023u) & ~1023u;  // 4-KB aligned chunks
    cudaStream_t s_cp = nullptr;
    cudaEvent_t ev_user = nullptr, ev[kChunks] = {};
    cudaError_t e = cudaStreamCreateWithFlags(&s_cp, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_user, cudaEventDisableTiming);
    for (uint32_t c = 0; c < kChunks && e == cudaSuccess; ++c)
        e = cudaEventCreateWithFlags(&ev[c], cudaEventDisableTiming);
    int launches = 0;
    if (e == cudaSuccess) e = rtf::clear_scale(ws, L, st);
    // the copy starts after everything already on the caller's stream (an
    // earlier build may still read p_dev)
    if (e == cudaSuccess) e = cudaEventRecord(ev_user, st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s_cp, ev_user, 0);
    for (uint32_t c = 0, off = 0; c < kChunks && off < n && e == cudaSuccess; ++c, off += chunk) {
        const uint32_t len = std::min(chunk, n - off);
        e = cudaMemcpyAsync(p_dev + off, p_host + off, sizeof(float) * (size_t)len,
                            cudaMemcpyHostToDevice, s_cp);
        if (e == cudaSuccess) e = cudaEventRecord(ev[c], s_cp);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(st, ev[c], 0);
        if (e == cudaSuccess) e = rtf::launch_scale_chunk(p_dev + off, len, ws, L, st, &launches);
    }
    if (e == cudaSuccess) {
        rtf::ShardCall sc{rtf::kPhFull & ~rtf::kPhScale, n, 0, 0, 0, 0, nullptr, nullptr};
        e = rtf::launch_build(p_dev, n, m, flags, out->header, out->nodes, out->table, nullptr, ws,
                              L, st, &launches, &sc);
    }
    if (s_cp) cudaStreamDestroy(s_cp);  // released once its work is done
    if (ev_user) cudaEventDestroy(ev_user);
    for (uint32_t c = 0; c < kChunks; ++c)
        if (ev[c]) cudaEventDestroy(ev[c]);
    const int s = finish(e, launches);
    if (s != RTF_OK) return s;
    return rtf_forest_status(out, stream, header_host);
}

int rtf_sample_host(const rtf_forest* f, const uint32_t* xi_host, uint64_t count, int32_t* out_host,
                    uint32_t* xi_dev, int32_t* out_dev, uint64_t chunk, void* stream) {
    if (!f || f->rows != 1 || (count && (!xi_host || !out_host || !xi_dev || !out_dev)))
        return RTF_EINVAL;
    if (count == 0) return RTF_OK;
    if (chunk == 0) return RTF_EINVAL;
    // The staging buffers hold 2 * chunk entries (rtf.h).  Round the chunk DOWN
    // to a multiple of 4 (16-B aligned halves for the sampler's vector path);
    // a chunk below 4 stays as given (launch_sample then uses scalar accesses).
    if (chunk >= 4) chunk &= ~3ull;
    cudaStream_t user = as_stream(stream);
    // three stages on three streams: H2D, sample, D2H; double-buffered staging.
    // Every handle starts null and every exit goes through the cleanup below,
    // which destroys only what was created.
    cudaStream_t s_in = nullptr, s_run = nullptr, s_out = nullptr;
    cudaEvent_t ev_in[2] = {}, ev_run[2] = {}, ev_out[2] = {}, ev_user = nullptr;
    cudaError_t e = cudaStreamCreateWithFlags(&s_in, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s_run, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s_out, cudaStreamNonBlocking);
    for (int b = 0; b < 2 && e == cudaSuccess; ++b) {
        e = cudaEventCreateWithFlags(&ev_in[b], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_run[b], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_out[b], cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_user, cudaEventDisableTiming);
    int launches = 0;
    if (e == cudaSuccess) {
        // order after everything already enqueued on the caller's stream (the build)
        e = cudaEventRecord(ev_user, user);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s_in, ev_user, 0);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s_run, ev_user, 0);
        uint64_t k = 0;
        for (uint64_t c = 0; k < count && e == cudaSuccess; ++c) {
            const int b = (int)(c & 1);
            const uint64_t len = std::min<uint64_t>(chunk, count - k);
            uint32_t* xd = xi_dev + (size_t)b * chunk;
            int32_t* od = out_dev + (size_t)b * chunk;
            if (c >= 2) cudaStreamWaitEvent(s_in, ev_run[b], 0);  // xi buffer b free
            e = cudaMemcpyAsync(xd, xi_host + k, len * 4, cudaMemcpyHostToDevice, s_in);
            cudaEventRecord(ev_in[b], s_in);
            cudaStreamWaitEvent(s_run, ev_in[b], 0);
            if (c >= 2) cudaStreamWaitEvent(s_run, ev_out[b], 0);  // out buffer b drained
            if (e == cudaSuccess) e = rtf::launch_sample(*f, nullptr, xd, len, od, s_run, &launches);
            cudaEventRecord(ev_run[b], s_run);
            cudaStreamWaitEvent(s_out, ev_run[b], 0);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(out_host + k, od, len * 4, cudaMemcpyDeviceToHost, s_out);
            cudaEventRecord(ev_out[b], s_out);
            k += len;
        }
    }
    for (cudaStream_t s : {s_out, s_run, s_in}) {
        if (!s) continue;
        const cudaError_t e2 = cudaStreamSynchronize(s);
        if (e == cudaSuccess) e = e2;
    }
    for (int b = 0; b < 2; ++b)
        for (cudaEvent_t ev : {ev_in[b], ev_run[b], ev_out[b]})
            if (ev) cudaEventDestroy(ev);
    if (ev_user) cudaEventDestroy(ev_user);
    for (cudaStream_t s : {s_in, s_run, s_out})
        if (s) cudaStreamDestroy(s);
    return finish(e, launches);
}

int rtf_philox_u32(uint64_t seed, uint64_t start, uint64_t count, uint32_t* out, void* stream) {
    if (count && !out) return RTF_EINVAL;
    int launches = 0;
    cudaError_t e = rtf::launch_philox(seed, start, count, out, as_stream(stream), &launches);
    return finish(e, launches);
}

// ------------------------------------------------------------------ sharded build (config 4)

size_t rtf_shard_workspace_bytes(uint32_t n_local, uint32_t n_global, uint32_t m) {
    rtf::WsLayout L;
    return rtf::build_workspace_layout(n_local ? n_local : 1, m ? m : 1, rtf::kBuildShardedLayout,
                                       &L, n_global);
}

static int shard_layout(void* ws, size_t ws_bytes, uint32_t n_local, uint32_t n_global, uint32_t m,
                        rtf::WsLayout* L) {
    if (!ws) return RTF_EINVAL;
    if (n_local == 0 || n_local > n_global) return RTF_EINVAL;
    if (int s = check_nm(n_global, m)) return s;
    if (((uintptr_t)ws & (kAlign - 1)) != 0) return RTF_EINVAL;
    if (ws_bytes < rtf::build_workspace_layout(n_local, m, rtf::kBuildShardedLayout, L, n_global))
        return RTF_ENOSPACE;
    return RTF_OK;
}

int rtf_shard_workspace_init(void* ws, size_t ws_bytes, uint32_t n_local, uint32_t n_global,
                             uint32_t m, void* stream) {
    rtf::WsLayout L;
    if (int s = shard_layout(ws, ws_bytes, n_local, n_global, m, &L)) return s;
    unsigned char* w = static_cast<unsigned char*>(ws);
    cudaStream_t st = as_stream(stream);
    const cudaError_t e = cudaMemsetAsync(w, 0, L.spine, st);
    return e == cudaSuccess ? RTF_OK : RTF_ECUDA;
}

int rtf_shard_get_view(void* ws, size_t ws_bytes, uint32_t n_local, uint32_t n_global, uint32_t m,
                       rtf_shard_view* out) {
    rtf::WsLayout L;
    if (!out) return RTF_EINVAL;
    if (int s = shard_layout(ws, ws_bytes, n_local, n_global, m, &L)) return s;
    unsigned char* w = static_cast<unsigned char*>(ws);
    out->spine = w + L.spine;
    out->scale = reinterpret_cast<uint32_t*>(w + L.scale);
    out->total = w + L.total;
    out->nt_local = L.nt;
    out->spine_row_bytes = (uint32_t)rtf::spine_row_bytes();
    out->nt_cap = L.nt_cap;
    out->reserved = 0;
    out->jbound = reinterpret_cast<uint32_t*>(w + L.jbound);
    return RTF_OK;
}

int rtf_shard_scale(const float* p, uint32_t n_local, uint32_t n_global, uint32_t m, void* ws,
                    size_t ws_bytes, void* stream) {
    rtf::WsLayout L;
    if (!p || ((uintptr_t)p & 3u)) return RTF_EINVAL;
    if (int s = shard_layout(ws, ws_bytes, n_local, n_global, m, &L)) return s;
    rtf::ShardCall sc{rtf::kPhScale, n_global, 0, 0, 1, 0, nullptr, nullptr};
    int launches = 0;
    cudaError_t e = rtf::launch_build(p, n_local, m, rtf::kBuildShardedLayout, nullptr, nullptr,
                                      nullptr, nullptr, ws, L, as_stream(stream), &launches, &sc);
    return finish(e, launches);
}

int rtf_shard_totals(const float* p, uint32_t n_local, uint32_t n_global, uint32_t m,
                     uint32_t index_base, void* ws, size_t ws_bytes, void* stream) {
    rtf::WsLayout L;
    if (!p || ((uintptr_t)p & 3u)) return RTF_EINVAL;
    if (int s = shard_layout(ws, ws_bytes, n_local, n_global, m, &L)) return s;
    if ((uint64_t)index_base + n_local > n_global) return RTF_EINVAL;
    rtf::ShardCall sc{rtf::kPhTotals | rtf::kPhSpine, n_global, index_base, 0, 1, 0,
                      nullptr, nullptr};
    int launches = 0;
    cudaError_t e = rtf::launch_build(p, n_local, m, rtf::kBuildShardedLayout, nullptr, nullptr,
                                      nullptr, nullptr, ws, L, as_stream(stream), &launches, &sc);
    return finish(e, launches);
}

int rtf_shard_build(const float* p, uint32_t n_local, uint32_t n_global, uint32_t m,
                    uint32_t index_base, uint32_t rank, uint32_t count, const void* totals,
                    void* forest_buf, size_t forest_bytes, void* ws, size_t ws_bytes, void* stream,
                    rtf_forest* out) {
    rtf::WsLayout L;
    if (!p || !totals || ((uintptr_t)p & 3u) || count == 0 || rank >= count) return RTF_EINVAL;
    if (int s = shard_layout(ws, ws_bytes, n_local, n_global, m, &L)) return s;
    if ((uint64_t)index_base + n_local > n_global) return RTF_EINVAL;
    if (int s = rtf_forest_view(forest_buf, forest_bytes, n_global, m, 1, out)) return s;
    rtf::ShardCall sc{rtf::kPhTiles | rtf::kPhRuns, n_global, index_base, rank, count, 0,
                      totals, nullptr};
    int launches = 0;
    cudaError_t e =
        rtf::launch_build(p, n_local, m, rtf::kBuildShardedLayout, out->header, out->nodes,
                          out->table, nullptr, ws, L, as_stream(stream), &launches, &sc);
    return finish(e, launches);
}

int rtf_shard_build_peers(const float* p, uint32_t n_local, uint32_t n_global, uint32_t m,
                          uint32_t index_base, uint32_t rank, uint32_t count, const void* totals,
                          void* const* peer_forest_bufs, uint32_t npeer, void* forest_buf,
                          size_t forest_bytes, void* ws, size_t ws_bytes, void* stream,
                          rtf_forest* out) {
    rtf::WsLayout L;
    if (!p || !totals || ((uintptr_t)p & 3u) || count == 0 || rank >= count) return RTF_EINVAL;
    if (npeer == 0 || npeer > rtf::kMaxShards || m % npeer) return RTF_EINVAL;
    if (int s = shard_layout(ws, ws_bytes, n_local, n_global, m, &L)) return s;
    if ((uint64_t)index_base + n_local > n_global) return RTF_EINVAL;
    if (int s = rtf_forest_view(forest_buf, forest_bytes, n_global, m, 1, out)) return s;
    unsigned char* w = static_cast<unsigned char*>(ws);
    cudaStream_t st = as_stream(stream);
    if (peer_forest_bufs) {  // upload now (else: rtf_shard_set_peers stored them)
        if (int s = rtf_shard_set_peers(ws, ws_bytes, n_local, n_global, m, peer_forest_bufs,
                                        npeer, forest_bytes, stream))
            return s;
    }
    if (cudaMemsetAsync(w + L.jbound, 0, sizeof(uint32_t) * (rtf::kMaxShards + 1), st))
        return RTF_ECUDA;
    rtf::ShardCall sc{rtf::kPhTiles | rtf::kPhRuns, n_global, index_base, rank, count, 0,
                      totals, nullptr};
    sc.npeer = npeer;
    int launches = 0;
    cudaError_t e =
        rtf::launch_build(p, n_local, m, rtf::kBuildShardedLayout, out->header, out->nodes,
                          out->table, nullptr, ws, L, st, &launches, &sc);
    return finish(e, launches);
}

int rtf_shard_set_peers(void* ws, size_t ws_bytes, uint32_t n_local, uint32_t n_global,
                        uint32_t m, void* const* peer_forest_bufs, uint32_t npeer,
                        size_t forest_bytes, void* stream) {
    rtf::WsLayout L;
    if (!peer_forest_bufs || npeer == 0 || npeer > rtf::kMaxShards || m % npeer) return RTF_EINVAL;
    if (int s = shard_layout(ws, ws_bytes, n_local, n_global, m, &L)) return s;
    // the peers' record and table sections (every forest buffer has this layout)
    void* ptrs[2 * rtf::kMaxShards];
    for (uint32_t r = 0; r < npeer; ++r) {
        rtf_forest f;
        if (int s = rtf_forest_view(peer_forest_bufs[r], forest_bytes, n_global, m, 1, &f)) return s;
        ptrs[r] = f.nodes;
        ptrs[rtf::kMaxShards + r] = f.table;
    }
    unsigned char* w = static_cast<unsigned char*>(ws);
    cudaStream_t st = as_stream(stream);
    if (cudaMemcpyAsync(w + L.peers, ptrs, sizeof(void*) * npeer, cudaMemcpyHostToDevice, st) ||
        cudaMemcpyAsync(w + L.peers + sizeof(void*) * rtf::kMaxShards, ptrs + rtf::kMaxShards,
                        sizeof(void*) * npeer, cudaMemcpyHostToDevice, st))
        return RTF_ECUDA;
    // the host pointer array is a stack buffer: wait for the copies
    return cudaStreamSynchronize(st) == cudaSuccess ? RTF_OK : RTF_ECUDA;
}

int rtf_shard_finish_own(uint32_t n_local, uint32_t n_global, uint32_t m, const void* spine_all,
                         uint32_t nt_all, uint32_t rank, void* forest_buf, size_t forest_bytes,
                         void* ws, size_t ws_bytes, void* stream, rtf_forest* out) {
    rtf::WsLayout L;
    if (!spine_all || ((uintptr_t)spine_all & 15u) || rank >= rtf::kMaxShards) return RTF_EINVAL;
    if (int s = shard_layout(ws, ws_bytes, n_local, n_global, m, &L)) return s;
    if (nt_all > L.nt_cap) return RTF_EINVAL;
    if (int s = rtf_forest_view(forest_buf, forest_bytes, n_global, m, 1, out)) return s;
    rtf::ShardCall sc{rtf::kPhCross, n_global, 0, 0, 1, nt_all, nullptr, spine_all};
    sc.j_rank = (int32_t)rank;
    int launches = 0;
    const float* dummy = reinterpret_cast<const float*>(ws);  // phases A-D do not run
    cudaError_t e =
        rtf::launch_build(dummy, n_local, m, rtf::kBuildShardedLayout, out->header, out->nodes,
                          out->table, nullptr, ws, L, as_stream(stream), &launches, &sc);
    return finish(e, launches);
}

int rtf_shard_finish_range(uint32_t n_local, uint32_t n_global, uint32_t m,
                           const void* spine_all, uint32_t nt_all, uint32_t j_lo, uint32_t j_hi,
                           void* forest_buf, size_t forest_bytes, void* ws, size_t ws_bytes,
                           void* stream, rtf_forest* out) {
    rtf::WsLayout L;
    if (!spine_all || ((uintptr_t)spine_all & 15u) || j_lo > j_hi) return RTF_EINVAL;
    if (int s = shard_layout(ws, ws_bytes, n_local, n_global, m, &L)) return s;
    if (nt_all > L.nt_cap) return RTF_EINVAL;
    if (int s = rtf_forest_view(forest_buf, forest_bytes, n_global, m, 1, out)) return s;
    rtf::ShardCall sc{rtf::kPhCross, n_global, 0, 0, 1, nt_all, nullptr, spine_all};
    sc.j_lo = j_lo;
    sc.j_hi = j_hi;
    int launches = 0;
    // any valid p pointer is fine: phases A-D do not run
    const float* dummy = reinterpret_cast<const float*>(ws);
    cudaError_t e =
        rtf::launch_build(dummy, n_local, m, rtf::kBuildShardedLayout, out->header, out->nodes,
                          out->table, nullptr, ws, L, as_stream(stream), &launches, &sc);
    return finish(e, launches);
}

int rtf_shard_finish(uint32_t n_local, uint32_t n_global, uint32_t m, const void* spine_all,
                     uint32_t nt_all, void* forest_buf, size_t forest_bytes, void* ws,
                     size_t ws_bytes, void* stream, rtf_forest* out) {
    return rtf_shard_finish_range(n_local, n_global, m, spine_all, nt_all, 0u, 0xffffffffu,
                                  forest_buf, forest_bytes, ws, ws_bytes, stream, out);
}

int rtf_shard_count_cells(const void* forest_buf, size_t forest_bytes, uint32_t n_global,
                          uint32_t m, uint32_t j0, uint32_t cnt, const uint32_t* bounds,
                          uint32_t nb, uint32_t* counts, void* stream) {
    rtf_forest f;
    if (!bounds || !counts || nb == 0) return RTF_EINVAL;
    if (int s = rtf_forest_view(const_cast<void*>(forest_buf), forest_bytes, n_global, m, 1, &f))
        return s;
    if ((uint64_t)j0 + cnt > n_global) return RTF_EINVAL;
    int launches = 0;
    cudaError_t e = rtf::launch_count_cells(f.nodes, j0, cnt, m, bounds, nb, counts,
                                            as_stream(stream), &launches);
    return finish(e, launches);
}

}  // extern "C"
