/*
 * rtf.h -- C ABI of librtf.so, the B200 (sm_100a) radix-tree-forest sampler.
 *
 * Implements the data-parallel hot path of Binder & Keller, arXiv 1901.05423:
 *   rtf_build:  p  ->  fixed-point CDF, guide table and radix-tree forest
 *               (prefix sum Sec.1, Alg. 1, guide-table
 *               encoding Sec.3.2);
 *   rtf_sample: xi -> i with P_{i-1} <= xi < P_i (Alg. 2).
 * "P:<line>" cites /root/reference/PAPER.md (not needed at run time).
 *
 * Conventions for every call
 *   - Pointers are DEVICE pointers unless the parameter name ends in _host.
 *   - The library never allocates device memory: the caller owns p, xi, out,
 *     the forest buffer and the workspace (sizes from the *_bytes calls).
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *     stream).  All device work is enqueued on it; calls return after
 *     enqueueing unless documented as synchronous.
 *   - Argument errors are detected on the host BEFORE any launch and returned
 *     as an rtf_status; nothing is enqueued then.
 *   - Data errors (NaN, +-Inf, negative or all-zero weights) are detected on
 *     the device: they set rtf_header.status, every later kernel of the build
 *     becomes a no-op and every rtf_sample output is INT32_MAX.  Read them
 *     with rtf_forest_status (synchronous).
 *   - Indices are 0-based (reading R1).  Sampled indices are ORIGINAL input
 *     indices; entries with p_i == 0 are never returned (reading R8).
 *   - Limits: 1 <= n < 2^31, 1 <= m < 2^31 (leaf references use the sign bit,
 *     P:1334 / reading R3).
 *   - Fixed point (reading R4, R7): weights are quantised to integers
 *     w_i = max(1, floor(p_i 2^(B-E))) for p_i > 0 (E = floor(log2 max p),
 *     B = 62 - ceil(log2 n)), T = sum w < 2^63, and the CDF boundaries are
 *     key_j = floor(W_j 2^63 / T) over the compacted positive entries; the
 *     implicit key_{n'} = 2^63 is "1".  xi is u32 fixed point xi/2^32 (R11).
 */
#ifndef RTF_H
#define RTF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ types */

typedef enum rtf_status {
    RTF_OK = 0,
    RTF_EINVAL = 1,    /* null pointer, n == 0, m == 0, bad flags, misaligned buffer */
    RTF_EALLZERO = 2,  /* (data) no strictly positive weight                          */
    RTF_ETOOLARGE = 3, /* n or m >= 2^31, or a batched row larger than supported      */
    RTF_ENOSPACE = 4,  /* caller buffer smaller than the *_bytes() requirement        */
    RTF_ECUDA = 5,     /* a CUDA runtime call failed (launch error, bad stream ...)   */
    RTF_EDATA = 6      /* (data) NaN / Inf / negative weight (see rtf_header.status)  */
} rtf_status;

/* rtf_header.status bits (device-side data errors) */
#define RTF_DATA_NAN 1u
#define RTF_DATA_INF 2u
#define RTF_DATA_NEG 4u
#define RTF_DATA_ALLZERO 8u

/* One node record, 16 bytes: the CDF boundary of node j interleaved with its
 * two children (Sec.3.2).  child >= 0: node index; child < 0:
 * leaf reference ~i of ORIGINAL interval i (Alg.2). */
typedef struct rtf_node {
    uint64_t key;      /* key_j = floor(W_j 2^63 / T), strictly increasing in j */
    int32_t child[2];  /* [0]: taken if xi 2^31 < key, [1]: otherwise          */
} rtf_node;

/* One guide-table cell, 8 bytes (Sec.3.2, reading R18):
 *   ref >= 0: the anchor node of the cell; Alg. 2 descends from nodes[ref].
 *   ref <  0: a leaf reference.  The cell is overlapped by one interval
 *             (key32 == 0: the leaf is ~ref) or by exactly two intervals
 *             ("a flag that there are exactly two intervals ... only one
 *             comparison must be performed and there is no need to
 *             explicitly store a node"): key32 = ceil(key_a /
 *             2^31) of the cell's only leaf a, and xi < key32 selects interval
 *             a-1, whose reference is ref + 1 (orig(a) = orig(a-1) + 1).
 * A cell whose single leaf a follows a zero weight keeps its anchor. */
typedef struct rtf_ref {
    uint32_t key32;  /* 0, or the two-interval split ceil(key_a / 2^31) */
    int32_t ref;     /* anchor node (>= 0) or leaf reference ~i (< 0)   */
} rtf_ref;

/* Device-resident build summary (one per row for batched forests). */
typedef struct rtf_header {
    uint64_t total;      /* T = sum of quantised weights, 0 < T < 2^63            */
    uint64_t recip;      /* internal: reciprocal of T << norm_shift                */
    uint32_t n_pos;      /* n' = number of strictly positive weights = #nodes     */
    int32_t exponent;    /* E = floor(log2(max p))                                 */
    int32_t scale_bits;  /* B = 62 - ceil(log2 n)                                  */
    uint32_t status;     /* 0 or RTF_DATA_* bits                                   */
    uint32_t norm_shift; /* internal                                               */
    uint32_t reserved;
} rtf_header; /* 40 bytes */

/* Host-side view of a forest living in a caller-owned device buffer. */
typedef struct rtf_forest {
    uint32_t n;      /* entries per row                                   */
    uint32_t m;      /* guide-table cells per row                         */
    uint32_t rows;   /* 1, or the number of independent rows (batched)    */
    uint32_t flags;  /* build flags; RTF_FOREST_MARKED after rtf_build_fallback */
    rtf_node *nodes; /* rows * n records (the first n_pos of each row valid;
                        rows_build: slot n_pos < n holds key 2^63, "1")   */
    rtf_ref *table;  /* rows * m guide-table cells (rtf_ref)              */
    rtf_header *header; /* rows headers                                  */
} rtf_forest;

/* rtf_build flags */
#define RTF_BUILD_DEFAULT 0u
#define RTF_FOREST_MARKED 0x100u /* set in rtf_forest.flags by rtf_build_fallback */
#define RTF_BUILD_SMALL_TILES 1u /* 256-entry tiles: a test/debug schedule that moves most
                                    links into the cross-tile phase; same result bytes */

/* ------------------------------------------------------------- sizing */

/* Bytes of the forest buffer for `rows` rows of n entries and m cells
 * (header + nodes + table, 256-byte aligned sections).  Host only. */
size_t rtf_forest_bytes(uint32_t n, uint32_t m, uint32_t rows);

/* Bytes of scratch workspace rtf_build needs for (n, m, flags).  Host only. */
size_t rtf_workspace_bytes(uint32_t n, uint32_t m, uint32_t flags);

/* Initialise a workspace once after allocating it (enqueues a memset of its
 * counters; Alg. 1's synchronisation array otherBounds, lives in shared
 * memory per tile).  Every rtf_build leaves it reusable, so this is needed
 * only once. */
int rtf_workspace_init(void *ws, size_t ws_bytes, uint32_t n, uint32_t m, uint32_t flags,
                       void *stream);

/* --------------------------------------------------------------- build */

/* Build the guide table and radix-tree forest of p[0..n) with m cells.
 *   p:      n float32 weights (device), >= 0, finite, not all zero; need not
 *           be normalised.  16-byte alignment gives vectorised loads.
 *   forest_buf / forest_bytes: >= rtf_forest_bytes(n, m, 1), 256-B aligned.
 *   ws / ws_bytes: >= rtf_workspace_bytes(n, m, flags), initialised once.
 *   out (host): receives the view of the forest.
 * Asynchronous: ONE cooperative kernel on `stream` whose phases are separated
 * by grid barriers (scale; tile totals; tiles: scan + exact normalisation +
 * cells/split levels/table + Alg. 1 in shared memory; cross-tile links from
 * the tiles' spines + long table runs).  With n <= 4096 and m <= 4096 (and no
 * RTF_BUILD_SMALL_TILES) the row kernel of rtf_build_rows builds it instead,
 * in one CTA without grid barriers.  The records [0, n_pos), the table and
 * the header are independent of the schedule, of the kernel and of `flags`.
 * Errors in the data (NaN, Inf, negative, all zero) are reported in
 * header->status (rtf_forest_status), not here. */
int rtf_build(const float *p, uint32_t n, uint32_t m, uint32_t flags, void *forest_buf,
              size_t forest_bytes, void *ws, size_t ws_bytes, void *stream, rtf_forest *out);

/* Batched build of `rows` independent distributions of n_row entries each
 * (p is row-major rows x n_row), m_row cells per row, one CTA per row entirely
 * in shared memory (Sec.5: the row boundary is one more partition
 * criterion).  Each row is normalised independently (reading R15).
 * Requires n_row <= 4096 and m_row <= 4096 (else RTF_ETOOLARGE).  No workspace. */
int rtf_build_rows(const float *p, uint32_t rows, uint32_t n_row, uint32_t m_row,
                   void *forest_buf, size_t forest_bytes, void *stream, rtf_forest *out);

/* Re-create a view of an existing forest buffer (no device work). */
int rtf_forest_view(void *forest_buf, size_t forest_bytes, uint32_t n, uint32_t m,
                    uint32_t rows, rtf_forest *out);

/* Synchronous: waits for `stream`, copies the f->rows device headers into
 * headers_host (may be NULL) and returns RTF_OK, RTF_EALLZERO or RTF_EDATA
 * (the worst row for batched forests). */
int rtf_forest_status(const rtf_forest *f, void *stream, rtf_header *headers_host);

/* ------------------------------------------------------------ sampling */

/* Alg. 2 for count samples: out[k] = the ORIGINAL index i with
 * key_i <= xi[k] 2^31 < key_next (guide-table lookup g = floor(xi m / 2^32);
 * a leaf cell answers at once, a two-interval cell with its one comparison;
 * else descent while the reference is a node).  Read-only on the forest, so
 * concurrent calls on one forest are safe.  xi / out need 4-byte alignment
 * (16-byte alignment enables vector access). */
int rtf_sample(const rtf_forest *f, const uint32_t *xi, uint64_t count, int32_t *out,
               void *stream);

/* rtf_sample for float xi in [0, 1): xi is first mapped exactly to the u32
 * fixed point floor(xi 2^32) (reading R11); values outside [0, 1) saturate to
 * 0 or 2^32 - 1 (NaN -> 0). */
int rtf_sample_f32(const rtf_forest *f, const float *xi, uint64_t count, int32_t *out,
                   void *stream);

/* Measurement aid: loads[k] = number of memory loads rtf_sample performs for
 * xi[k] (1 guide-table entry + 1 per node visited), the load-count convention
 * of Table 1; gives E[visits], the maximum and average_32.
 * loads_plain (may be NULL) receives the count without the two-interval flag
 * (a flagged cell would cost its anchor visit: 2 loads), i.e. the paper's own
 * structure. */
int rtf_sample_loads(const rtf_forest *f, const uint32_t *xi, uint64_t count, int32_t *loads,
                     int32_t *loads_plain, void *stream);

/* ------------------------------------ 4-ary collapsed records (Sec.5) */
/*
 * "Due to memory access granularity, it may be beneficial to construct 4-ary or
 * even wider trees.  A higher branching factor simply results by just
 * collapsing two (or more) levels of the binary trees."
 * rtf_build_quad writes, for every node j < n_pos of a built single forest, a
 * 32-B record {k0, k1, k2, flags, g0, g1, g2, g3}: k0 = ceil(key_j / 2^31),
 * k1 / k2 the same for node j's children, g the four grandchildren (a leaf
 * child stands for both of its slots), flags bit i: k_i = 2^32.  One 32-B load
 * then decides two levels of Alg. 2.  rec4: device, 32-B aligned, >=
 * rtf_quad_bytes(n) bytes, owned by the caller; valid until the forest is
 * rebuilt.  rtf_sample_quad returns exactly rtf_sample's indices, reading the
 * guide table and the quad records only.  On a ranged shard (rtf_shard_finish_range)
 * only the records of the rank's own slots are valid, so only its own xi
 * stratum may be sampled this way (child references are bounds-checked, never
 * followed outside the forest).  Errors: RTF_EINVAL (NULL, rows != 1,
 * misaligned), RTF_ENOSPACE (rec4 too small), RTF_ECUDA. */
size_t rtf_quad_bytes(uint32_t n); /* host only */
int rtf_build_quad(const rtf_forest *f, void *rec4, size_t rec4_bytes, void *stream);
int rtf_sample_quad(const rtf_forest *f, const void *rec4, const uint32_t *xi, uint64_t count,
                    int32_t *out, void *stream);

/* Batched: sample k uses row[k] (< f->rows); out is row-local. */
int rtf_sample_rows(const rtf_forest *f, const uint32_t *row, const uint32_t *xi,
                    uint64_t count, int32_t *out, void *stream);

/* ------------------------------------------- 2-D distributions (Sec.6) */
/*
 * "A multi-dimensional inversion method proceeds component by component"
 * (P:1523-1529): a marginal forest over the image rows selects y with xi1, the
 * forest of row y selects x with xi2, and the relative positions inside the
 * two chosen intervals give the sub-pixel position.  Rows are
 * built by the batched build (the row index boundary is the partition
 * criterion); the row weights are the rows' quantised masses
 * (reading R19).  Limits: W, H, mx, my <= 4096 (rtf_build_rows).
 */
typedef struct rtf_forest2d {
    uint32_t W, H;       /* columns, rows                                          */
    uint32_t mx, my;     /* cells per row / of the marginal                         */
    rtf_forest rows;     /* H rows of W entries: the conditional forests            */
    rtf_forest marginal; /* 1 row of H entries: the forest of the row weights       */
    int32_t *rows_jmap;  /* H*W: row-local node index of entry (y, x), -1 for p = 0 */
    int32_t *marg_jmap;  /* H:   node index of row y in the marginal, -1 if q_y = 0 */
    float *weights;      /* H:   the row weights q_y (reading R19)                   */
    uint32_t *rows_dense; /* H bits: bit y set if row y has no zero weight, so its
                             rows_jmap is the identity (the sampler skips it)       */
} rtf_forest2d;

/* Bytes of a 2-D forest buffer (both forests, index maps, weights).  Host only. */
size_t rtf_forest2d_bytes(uint32_t W, uint32_t H, uint32_t mx, uint32_t my);

/* Build from p (H x W float32, row-major, device; >= 0, finite).  Three
 * launches on `stream` (rows, row weights, marginal); asynchronous.  A NaN /
 * Inf / negative weight poisons the marginal (rtf_forest2d_status -> EDATA);
 * an all-zero row is legal (weight 0, never chosen). */
int rtf_build_2d(const float *p, uint32_t W, uint32_t H, uint32_t mx, uint32_t my, void *buf,
                 size_t bytes, void *stream, rtf_forest2d *out);

/* Synchronous: RTF_OK, RTF_EDATA (invalid data anywhere) or RTF_EALLZERO (no
 * positive weight at all). */
int rtf_forest2d_status(const rtf_forest2d *f, void *stream);

/* pixel[k] = y W + x for the pair (xi1[k], xi2[k]) (u32 fixed point);
 * pos (may be NULL): 2 floats per sample, ((x + v) / W, (y + u) / H) with u, v
 * the relative positions inside the chosen intervals, computed in float64 and
 * rounded toward zero (reading R19).  A poisoned forest gives INT32_MAX. */
int rtf_sample_2d(const rtf_forest2d *f, const uint32_t *xi1, const uint32_t *xi2,
                  uint64_t count, int32_t *pixel, float *pos, void *stream);

/* ----------------------------------------------- baselines (same CDF) */

/* The full fixed-point CDF over all n entries, zeros included:
 * cdf[i] = floor(W_i 2^63 / T), W_i = sum_{k<i} w_k (u64[n], device), and a
 * device header.  This is the array a plain binary search (Sec.2.2
 * P:114-127) searches.  Uses the same workspace as rtf_build. */
int rtf_build_cdf(const float *p, uint32_t n, uint64_t *cdf, rtf_header *header, void *ws,
                  size_t ws_bytes, void *stream);

/* Binary search baseline: out[k] = last i with cdf[i] <= xi[k] 2^31
 * (identical results to rtf_sample on the same p). */
int rtf_sample_bsearch(const uint64_t *cdf, uint32_t n, const rtf_header *header,
                       const uint32_t *xi, uint64_t count, int32_t *out, void *stream);

/* Degenerate-cell fallback (reading R21; "for degenerate hierarchical
 * structures the worst case may increase ... a fallback method constructs such
 * a structure upon detection to guarantee logarithmic complexity", Sec.3
 * P:983-984; criterion Sec.4).  Marks in f's guide table every
 * anchor cell holding k < 2^30 leaves whose radix tree makes some 32-bit xi
 * read more than ceil(log2(k + 1)) + 4 node records: key32 = 3 << 30 | k,
 * ref = the cell's first leaf (a packed cell never has both top bits set).  rtf_sample and rtf_sample_loads then search
 * such cells by bisection of their index interval (the implicit balanced tree
 * of Sec.6): at most ceil(log2(k + 1)) reads.  Sampled indices are
 * unchanged.  ws: >= rtf_fallback_bytes(m) bytes of device scratch; afterwards
 * it holds per cell the radix depth (u32[m]) and the cell's last leaf (u32[m]).
 * Sets RTF_FOREST_MARKED in f->flags (rtf_sample then launches its
 * bisecting variant; the unmarked sampler carries no code for it).
 * Asynchronous on `stream`; run it after rtf_build (a rebuild clears the
 * marks and the flag); rtf_sample_quad does not read marked tables
 * (RTF_EINVAL).  RTF_EINVAL for a rows forest or NULL pointers. */
size_t rtf_fallback_bytes(uint32_t m);
int rtf_build_fallback(rtf_forest *f, void *ws, size_t ws_bytes, void *stream);

/* Eytzinger binary-search baseline (Sec.2.2 P:114-127 laid out for a GPU):
 * rtf_build_eytzinger writes the keys cdf[1..n-1] as a complete binary
 * search tree in breadth-first order, eyt[k] for 1 <= k < 2^H,
 * H = ceil(log2 n) (u64[2^H], device, caller-owned; rtf_eytzinger_slots(n)
 * = 2^H entries; missing ranks hold UINT64_MAX).  rtf_sample_eytzinger:
 * out[k] as rtf_sample_bsearch (identical results), descending H levels, the
 * top 13 from a shared-memory copy per CTA.  Asynchronous on `stream`;
 * RTF_EINVAL on NULL or misaligned pointers. */
uint64_t rtf_eytzinger_slots(uint32_t n);
int rtf_build_eytzinger(const uint64_t *cdf, uint32_t n, uint64_t *eyt, void *stream);
int rtf_sample_eytzinger(const uint64_t *eyt, uint32_t n, const rtf_header *header,
                         const uint32_t *xi, uint64_t count, int32_t *out, void *stream);

/* Alias-method baseline (Walker / Vose, Sec.2.6; a comparison
 * system of the paper): table = 2^k entries {u32 prob, i32 alias} (device,
 * 8-B aligned, built on the host by baselines/alias.c over the same 32-bit
 * xi grid, so item i receives exactly the xi count the inverse mapping gives
 * it); out[i] = b if (xi mod 2^(32-k)) < prob[b] else alias[b], b = xi >>
 * (32-k).  Not monotone in xi (the property the forest keeps).  1 <= k <= 31;
 * RTF_EINVAL otherwise or on NULL / misaligned pointers. */
int rtf_sample_alias(const void *table, uint32_t k, const uint32_t *xi, uint64_t count,
                     int32_t *out, void *stream);

/* 2-D alias baseline (the alias-method curve of the paper's convergence
 * figure): marg = 2^ky entries {u32 prob, i32 alias} over the H
 * rows, rows = H x 2^kx entries (row y's table at rows + y 2^kx) over its W
 * columns, all built on the host (baselines.alias_2d) from the same exact
 * 32-bit xi counts the 2-D forest realises.  pixel[i] = y W + x with y =
 * alias(marg, xi1[i]), x = alias(row y, xi2[i]) (rule of rtf_sample_alias).
 * RTF_EINVAL on NULL / misaligned pointers, k outside [1, 31], W > 2^kx or H
 * > 2^ky; RTF_ETOOLARGE if W H >= 2^31. */
int rtf_sample_alias_2d(const void *marg, uint32_t ky, const void *rows, uint32_t kx,
                        uint32_t W, uint32_t H, const uint32_t *xi1, const uint32_t *xi2,
                        uint64_t count, int32_t *pixel, void *stream);

/* Cutpoint baselines (guide table of the classic cutpoint method, Sec.2.3
 * P:168-232; the "cutpoint + linear / binary" rows of Table 1) on
 * the same full CDF.  rtf_build_cutpoint: cut[g] (u32[m + 1], device) = the
 * index the smallest xi of cell g maps to (cut[m] = n - 1), one binary search
 * per cell.  rtf_sample_cutpoint: out[k] as rtf_sample_bsearch, by a linear
 * scan upwards from cut[g] (binary = 0; unbounded on skewed inputs -- the
 * degenerate case the paper sets out to avoid) or a binary search in
 * [cut[g], cut[g + 1]] (binary = 1).  Asynchronous on `stream`. */
int rtf_build_cutpoint(const uint64_t *cdf, uint32_t n, uint32_t m, uint32_t *cut, void *stream);
int rtf_sample_cutpoint(const uint64_t *cdf, uint32_t n, const rtf_header *header,
                        const uint32_t *cut, uint32_t m, int binary, const uint32_t *xi,
                        uint64_t count, int32_t *out, void *stream);

/* ------------------------------------------- host-buffer entry points */

/* End-to-end build from HOST weights: copies p_host (pinned for full speed)
 * into p_dev (n floats, device scratch), builds, and reads the header back.
 * The copy runs in 8 chunks on an internal copy stream; the scan for the
 * largest weight and the data flags (phase A) runs on each chunk as soon as
 * it lands, overlapping the rest of the copy, and the build then starts at
 * the tile totals (n or m above 4096, or RTF_BUILD_SMALL_TILES; otherwise one
 * copy, then rtf_build).  Ordered after the work already on `stream`.
 * Synchronous; returns the build status (data errors included). */
int rtf_build_host(const float *p_host, uint32_t n, uint32_t m, uint32_t flags, float *p_dev,
                   void *forest_buf, size_t forest_bytes, void *ws, size_t ws_bytes,
                   void *stream, rtf_forest *out, rtf_header *header_host);

/* End-to-end sampling from HOST xi to HOST out: chunks of `chunk` samples
 * are copied in, sampled and copied out on three internal streams so copies
 * overlap the kernel.  xi_dev / out_dev: device staging of 2*chunk entries
 * each.  Synchronous. */
int rtf_sample_host(const rtf_forest *f, const uint32_t *xi_host, uint64_t count,
                    int32_t *out_host, uint32_t *xi_dev, int32_t *out_dev, uint64_t chunk,
                    void *stream);

/* ---------------------------------------- sharded build across GPUs (config 4) */
/*
 * The distribution p[0..n_global) is split into contiguous shards; shard r
 * holds p[index_base_r .. index_base_r + n_local_r).  The build needs two tiny
 * exchanges between the calls below and one replication step; the library
 * does no communication itself (the caller runs NCCL, see
 * paper_1901_05423_b200/sharded.py):
 *   1. rtf_shard_scale            -> view.scale (4 words); MAX-reduce across shards
 *   2. rtf_shard_totals           -> view.total (16 B);    gather all shards' totals
 *      (the cross-GPU scan of per-shard totals: every shard derives its prefix
 *       and the grand total T from the gathered totals, on the device)
 *   3. rtf_shard_build            -> this shard's node records [J_r, J_r + n'_r),
 *      guide-table cells (others {0, INT32_MIN}) and one spine row per tile
 *      (view.spine: nt_local rows of view.spine_row_bytes)
 *   4. replicate records (broadcast from each owner), MAX-reduce the table as
 *      int64 words (ref in the high half),
 *      gather the spine rows of all shards, shard r's at rows
 *      [r * nt_max, r * nt_max + nt_local_r) (nt_max = the largest nt_local;
 *      pad with zero bytes: a row with zero leaves is skipped)
 *   5. rtf_shard_finish           -> the cross-tile links over all rows;
 *      every shard then holds the identical full forest (byte-equal to rtf_build).
 * Each shard owns a forest buffer sized for (n_global, m) and a shard workspace.
 */
typedef struct rtf_shard_view {  /* device pointers into a shard workspace */
    void *spine;              /* nt_local rows of spine_row_bytes (opaque)             */
    uint32_t *scale;          /* 4 words {max float bits, nan, inf, negative}           */
    void *total;              /* 16 B {u64 W, u32 n', i32 last positive index}         */
    uint32_t nt_local;        /* tiles (spine rows) of this shard                      */
    uint32_t spine_row_bytes; /* bytes per spine row (a multiple of 16)                */
    uint32_t nt_cap;          /* most rows rtf_shard_finish accepts                    */
    uint32_t reserved;
    uint32_t *jbound;         /* rtf_shard_build_peers: N + 1 words, J_k where this
                                 shard saw the boundary (0 elsewhere; MAX-reduce)      */
} rtf_shard_view;

size_t rtf_shard_workspace_bytes(uint32_t n_local, uint32_t n_global, uint32_t m);
int rtf_shard_workspace_init(void *ws, size_t ws_bytes, uint32_t n_local, uint32_t n_global,
                             uint32_t m, void *stream);
int rtf_shard_get_view(void *ws, size_t ws_bytes, uint32_t n_local, uint32_t n_global,
                       uint32_t m, rtf_shard_view *out);
int rtf_shard_scale(const float *p, uint32_t n_local, uint32_t n_global, uint32_t m, void *ws,
                    size_t ws_bytes, void *stream);
int rtf_shard_totals(const float *p, uint32_t n_local, uint32_t n_global, uint32_t m,
                     uint32_t index_base, void *ws, size_t ws_bytes, void *stream);
int rtf_shard_build(const float *p, uint32_t n_local, uint32_t n_global, uint32_t m,
                    uint32_t index_base, uint32_t rank, uint32_t count, const void *totals,
                    void *forest_buf, size_t forest_bytes, void *ws, size_t ws_bytes,
                    void *stream, rtf_forest *out);
/* spine_all: the gathered rows (device, 16-B aligned), nt_all of them
 * (<= view.nt_cap).  Writes the cross-tile links into this shard's full forest. */
int rtf_shard_finish(uint32_t n_local, uint32_t n_global, uint32_t m, const void *spine_all,
                     uint32_t nt_all, void *forest_buf, size_t forest_bytes, void *ws,
                     size_t ws_bytes, void *stream, rtf_forest *out);

/* Ranged sharding (the north star's "per-shard build over contiguous cell
 * ranges"): instead of replicating the whole forest, rank r keeps the cells
 * [g_r, g_{r+1}) (g_r = r m / N) -- a contiguous xi range -- and samples only
 * xi in it.  Its node slots are the leaves of those cells, [J_r, J_{r+1});
 * J_k = sum over shards of rtf_shard_count_cells(.., bounds = g, ..).  After
 * step 3, the records move to the rank of their cells (an all-to-all of
 * contiguous slices), the table is MAX-reduce-scattered by cell slice, the
 * spine rows are gathered, and rtf_shard_finish_range links only the slots
 * in [j_lo, j_hi) = [J_r, J_{r+1}).  Its records and table slice are then
 * byte-equal to the single build's. */
int rtf_shard_count_cells(const void *forest_buf, size_t forest_bytes, uint32_t n_global,
                          uint32_t m, uint32_t j0, uint32_t cnt, const uint32_t *bounds,
                          uint32_t nb, uint32_t *counts, void *stream);
int rtf_shard_finish_range(uint32_t n_local, uint32_t n_global, uint32_t m,
                           const void *spine_all, uint32_t nt_all, uint32_t j_lo, uint32_t j_hi,
                           void *forest_buf, size_t forest_bytes, void *ws, size_t ws_bytes,
                           void *stream, rtf_forest *out);
/* Fused ranged build (step 3 with the move folded in): the tile flush stores
 * each record, and every table write goes, straight into the forest buffer of
 * the rank owning its cell (peer_forest_bufs[r]: npeer device pointers valid
 * in this process -- NVLink peer memory across GPUs, e.g. CUDA symmetric
 * memory; plain device buffers for virtual shards; all laid out for
 * (n_global, m); m % npeer == 0).  The rank whose leaves straddle an owner
 * boundary k m / npeer writes J_k into view.jbound[k] (others 0), so a
 * MAX-reduce of jbound gives every rank its slots [J_r, J_{r+1}).  After the
 * spine rows are gathered (which also orders every rank's peer stores before
 * the finish), rtf_shard_finish_range completes each rank's cells.  Blocks
 * the host until the pointer upload is done -- unless peer_forest_bufs is
 * NULL: then the pointers rtf_shard_set_peers stored in the workspace are
 * used and the call only enqueues work (no host synchronisation). */
int rtf_shard_build_peers(const float *p, uint32_t n_local, uint32_t n_global, uint32_t m,
                          uint32_t index_base, uint32_t rank, uint32_t count, const void *totals,
                          void *const *peer_forest_bufs, uint32_t npeer, void *forest_buf,
                          size_t forest_bytes, void *ws, size_t ws_bytes, void *stream,
                          rtf_forest *out);

/* Set-up for repeated fused builds: stores the npeer peer forest pointers in
 * this shard's workspace once (blocks the host until the upload is done), so
 * that rtf_shard_build_peers(.., peer_forest_bufs = NULL, npeer, ..) needs no
 * host round trip.  Valid until the workspace is re-initialised. */
int rtf_shard_set_peers(void *ws, size_t ws_bytes, uint32_t n_local, uint32_t n_global,
                        uint32_t m, void *const *peer_forest_bufs, uint32_t npeer,
                        size_t forest_bytes, void *stream);
/* rtf_shard_finish_range with the slot range read on the device: after the
 * MAX-reduce of view.jbound, [J_rank, J_{rank+1}) = [jbound[rank],
 * jbound[rank + 1]) -- no copy of J to the host between build and finish. */
int rtf_shard_finish_own(uint32_t n_local, uint32_t n_global, uint32_t m, const void *spine_all,
                         uint32_t nt_all, uint32_t rank, void *forest_buf, size_t forest_bytes,
                         void *ws, size_t ws_bytes, void *stream, rtf_forest *out);

/* ---------------------------------------------------------- utilities */

/* Input generator (not part of the method): Philox4x32-10 u32 stream,
 * out[k] = word (start+k) mod 4 of philox(counter = ((start+k)/4 lo, hi, 0, 0),
 * key = seed).  Identical to workloads.philox_xi. */
int rtf_philox_u32(uint64_t seed, uint64_t start, uint64_t count, uint32_t *out, void *stream);

/* Number of kernels this process has launched through librtf (monotonic). */
uint64_t rtf_launch_count(void);

/* Human-readable status name. */
const char *rtf_status_string(int status);

/* Library version string. */
const char *rtf_version(void);

#ifdef __cplusplus
}
#endif
#endif /* RTF_H */
