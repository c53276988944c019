/*
 * rtf_oracle.c -- CPU ORACLE for the radix-tree-forest sampler of
 * Binder & Keller, "Massively Parallel Construction of Radix Tree Forests for
 * the Efficient Sampling of Discrete or Piecewise Constant Probability
 * Distributions" (arXiv 1901.05423).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_1901_05423_b200/) never links, imports or calls it,
 * and this file shares no code, header, table or constant generator with the
 * CUDA path.
 *
 * Plain, serial, slow and obviously correct: every step is the definition
 * written out (exact 128-bit integer arithmetic via unsigned __int128, a
 * top-down recursive radix split, a sequential descent).  Citations:
 * "P:<line>" = PAPER.md line, with section / equation / algorithm named;
 * readings R1..R17 are listed in DESIGN.md section 3.
 *
 * Steps ("oracle"):
 *   O1 validate            P:52-54 (p_i positive, sum 1); readings R7, R8
 *   O2 scale               reading R7 (E = floor(log2 max p), B = 62 - ceil(log2 n))
 *   O3 quantise            reading R7 (w_i = max(1, floor(p_i 2^(B-E))) for p_i > 0)
 *   O4 compaction          P:1018-1020 (indirection i' -> i); reading R8
 *   O5 exclusive scan      Sec.1 P:55-58 (partial sums P_k)
 *   O6 fixed point         P:57 (0 = P_0 < ... < P_n = 1); reading R4 ("1" = 2^63)
 *   O7 cells               Alg.1 P:1094 (curCell = floor(data[i] m))
 *   O8 split levels        Sec.3.1 P:1049-1055 (XOR distance), Sec.3.2
 *                          (distance set to the maximum at a partition boundary)
 *   O9 per-cell radix tree Sec.3.1 P:1039-1047 (node index = lowest leaf index
 *                          of its right subtree), Fig.6 caption P:1276-1279
 *                          (roots only have a right child; left child set to
 *                          the left neighbour)
 *   O10 guide table        Sec.3.2 P:1333-1335 (cell overlapped by a single
 *                          interval stores the complement of its index)
 *   O12 sampling           Alg.2
 * Parity status of every function is stated in DESIGN.md section 3.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

#define ORC_OK 0
#define ORC_EINVAL 1    /* n==0, m==0, NaN / Inf / negative weight */
#define ORC_EALLZERO 2  /* no strictly positive weight            */
#define ORC_ETOOLARGE 3 /* n or m >= 2^31 (leaf refs need the msb)  */

#define ORC_ONE ((uint64_t)1 << 63) /* fixed-point "1.0" (reading R4) */

/* ---------- O2 helpers: exact decomposition of an IEEE-754 binary32 ---------- */

/* x = mant * 2^exp2 exactly, for finite x > 0. */
static void f32_decompose(float x, uint64_t *mant, int *exp2) {
    uint32_t bits;
    memcpy(&bits, &x, 4);
    uint32_t biased = (bits >> 23) & 0xffu;
    uint32_t frac = bits & 0x7fffffu;
    if (biased == 0) { /* subnormal: frac * 2^-149 */
        *mant = frac;
        *exp2 = -149;
    } else { /* normal: (2^23 + frac) * 2^(biased - 150) */
        *mant = (uint64_t)frac | ((uint64_t)1 << 23);
        *exp2 = (int)biased - 150;
    }
}

/* floor(log2(x)) for finite x > 0. */
static int f32_floor_log2(float x) {
    uint64_t mant;
    int e;
    f32_decompose(x, &mant, &e);
    int msb = 63;
    while (!((mant >> msb) & 1u)) msb--;
    return msb + e;
}

static int ceil_log2_u32(uint32_t n) {
    int c = 0;
    while (((uint64_t)1 << c) < (uint64_t)n) c++;
    return c;
}

/* ---------- O1..O3: validate, scale, quantise ---------- */

/* w[i] = 0 for p_i == 0; else max(1, floor(p_i * 2^(B-E))).
 * Returns status; on success writes E, B. */
int orc_quantize(const float *p, uint32_t n, uint64_t *w, int *E_out, int *B_out) {
    if (n == 0) return ORC_EINVAL;
    if (n >= 0x80000000u) return ORC_ETOOLARGE;
    float pmax = 0.0f;
    for (uint32_t i = 0; i < n; i++) {
        float x = p[i];
        if (x != x) return ORC_EINVAL;                        /* NaN  */
        if (x > 3.4028235e38f || x < -3.4028235e38f) return ORC_EINVAL; /* +-Inf */
        if (x < 0.0f) return ORC_EINVAL;                      /* negative (-0.0 is zero) */
        if (x > pmax) pmax = x;
    }
    if (!(pmax > 0.0f)) return ORC_EALLZERO;
    int E = f32_floor_log2(pmax);
    int B = 62 - ceil_log2_u32(n);
    for (uint32_t i = 0; i < n; i++) {
        float x = p[i];
        if (!(x > 0.0f)) { w[i] = 0; continue; }
        uint64_t mant;
        int e;
        f32_decompose(x, &mant, &e);
        int sh = e + B - E; /* w = floor(mant * 2^sh) */
        uint64_t v;
        if (sh >= 0) v = mant << sh; /* mant*2^sh = p*2^(B-E) < 2^(B+1) <= 2^63 */
        else if (sh <= -64) v = 0;
        else v = mant >> (-sh);
        w[i] = v > 0 ? v : 1;
    }
    *E_out = E;
    *B_out = B;
    return ORC_OK;
}

/* ---------- O4..O6: compaction, exclusive scan, fixed point ---------- */

/* key = floor(W * 2^63 / T), 0 <= W <= T, 0 < T < 2^63. */
static uint64_t fixed_point(uint64_t W, uint64_t T) {
    return (uint64_t)(((u128)W << 63) / (u128)T);
}

/* Fixed-point CDF over ALL n entries (zeros included): K[i] = floor(W_i 2^63 / T)
 * with W_i = sum_{k<i} w_k.  This is the array the binary-search baseline
 * searches (Sec.2.2).  Returns status; T_out = T. */
int orc_cdf_all(const float *p, uint32_t n, uint64_t *K, uint64_t *T_out) {
    uint64_t *w = (uint64_t *)malloc(sizeof(uint64_t) * (n ? n : 1));
    int E, B;
    int st = orc_quantize(p, n, w, &E, &B);
    if (st != ORC_OK) { free(w); return st; }
    uint64_t T = 0;
    for (uint32_t i = 0; i < n; i++) T += w[i];
    uint64_t W = 0;
    for (uint32_t i = 0; i < n; i++) {
        K[i] = fixed_point(W, T);
        W += w[i];
    }
    *T_out = T;
    free(w);
    return ORC_OK;
}

/* ---------- O9: explicit top-down radix tree of one cell ---------- */

typedef struct {
    const uint8_t *lambda;
    const int32_t *orig;
    int32_t *child0;
    int32_t *child1;
} tree_ctx;

/* R(lo, hi): the radix tree over leaves lo..hi (all in one cell).  A single
 * leaf is the reference ~orig(lo) (reading R3: bitwise NOT).  Otherwise
 * the node is s = the position of the highest differing bit inside the range,
 * i.e. argmax_{s in (lo,hi]} lambda[s-1] (unique for distinct keys), which is
 * the lowest leaf index of its right subtree.  Left subtree
 * lo..s-1, right subtree s..hi; traversal goes left iff xi < key_s (Alg.2). */
static int32_t radix_subtree(const tree_ctx *c, uint32_t lo, uint32_t hi) {
    if (lo == hi) return ~c->orig[lo];
    uint32_t s = lo + 1;
    for (uint32_t t = lo + 2; t <= hi; t++)
        if (c->lambda[t - 1] > c->lambda[s - 1]) s = t;
    c->child0[s] = radix_subtree(c, lo, s - 1);
    c->child1[s] = radix_subtree(c, s, hi);
    return (int32_t)s;
}

/*
 * orc_build: O1..O11 for one distribution.
 * Outputs (arrays sized n; the first n_pos entries are meaningful):
 *   key[j], orig[j], cell[j], lambda[j], child0[j], child1[j]  for j < n_pos
 *   table[g] for g < m
 * Returns status; on success writes *T_out, *npos_out.
 */
int orc_build(const float *p, uint32_t n, uint32_t m, uint64_t *key, int32_t *orig,
              uint32_t *cell, uint8_t *lambda, int32_t *child0, int32_t *child1,
              int32_t *table, uint64_t *T_out, uint32_t *npos_out) {
    if (m == 0) return ORC_EINVAL;
    if (m >= 0x80000000u) return ORC_ETOOLARGE;
    uint64_t *w = (uint64_t *)malloc(sizeof(uint64_t) * (n ? n : 1));
    int E, B;
    int st = orc_quantize(p, n, w, &E, &B);
    if (st != ORC_OK) { free(w); return st; }

    /* O4 compaction + O5 serial exclusive scan */
    uint64_t *Wj = (uint64_t *)malloc(sizeof(uint64_t) * n);
    uint32_t npos = 0;
    uint64_t run = 0;
    for (uint32_t i = 0; i < n; i++) {
        if (w[i] == 0) continue;
        orig[npos] = (int32_t)i;
        Wj[npos] = run;
        run += w[i];
        npos++;
    }
    uint64_t T = run;

    /* O6 fixed point and O7 cells */
    for (uint32_t j = 0; j < npos; j++) {
        key[j] = fixed_point(Wj[j], T);
        cell[j] = (uint32_t)(((u128)key[j] * m) >> 63);
    }

    /* O8 split levels: lambda_j describes the pair (j, j+1). */
    for (uint32_t j = 0; j < npos; j++) {
        if (j + 1 == npos || cell[j + 1] != cell[j]) {
            lambda[j] = 64; /* partition boundary / array end: maximal distance */
        } else {
            uint64_t x = key[j] ^ key[j + 1];
            int msb = 63;
            while (!((x >> msb) & 1u)) msb--;
            lambda[j] = (uint8_t)msb;
        }
    }

    /* O9: one explicit radix tree per non-empty cell, rooted at the anchor. */
    tree_ctx c = {lambda, orig, child0, child1};
    uint32_t a = 0;
    while (a < npos) {
        uint32_t b = a;
        while (b + 1 < npos && cell[b + 1] == cell[a]) b++;
        child0[a] = ~orig[a > 0 ? a - 1 : 0]; /* Fig.6 caption P:1276-1277 */
        child1[a] = radix_subtree(&c, a, b);  /* root is the anchor's right child */
        a = b + 1;
    }

    /* O10 guide table: anchor of a non-empty cell, else ~orig of the interval
     * that overlaps the whole cell, i.e. the last leaf of an earlier cell. */
    uint32_t j = 0;        /* first leaf with cell >= g */
    int32_t last_before = -1; /* last leaf with cell < g */
    for (uint32_t g = 0; g < m; g++) {
        while (j < npos && cell[j] < g) { last_before = (int32_t)j; j++; }
        if (j < npos && cell[j] == g) table[g] = (int32_t)j;
        else table[g] = ~orig[last_before]; /* cell 0 always holds leaf 0 (key_0 = 0) */
    }

    *T_out = T;
    *npos_out = npos;
    free(Wj);
    free(w);
    return ORC_OK;
}

/* ---------- O12: Alg.2 sequential descent ---------- */

/* xi is u32 fixed point xi/2^32 (reading R11).  Returns the ORIGINAL index;
 * if loads != NULL stores the number of memory loads (1 per table entry,
 * 1 per node visited, the convention of Table 1). */
static int32_t sample_one(const uint64_t *key, const int32_t *child0, const int32_t *child1,
                          const int32_t *table, uint32_t m, uint32_t xi, uint32_t *loads) {
    uint32_t g = (uint32_t)(((uint64_t)xi * m) >> 32);
    int32_t j = table[g];
    uint32_t l = 1;
    uint64_t x63 = (uint64_t)xi << 31;
    while (j >= 0) { /* msb(j) != 1 */
        l++;
        j = (x63 < key[j]) ? child0[j] : child1[j];
    }
    if (loads) *loads = l;
    return ~j;
}

void orc_sample(const uint64_t *key, const int32_t *child0, const int32_t *child1,
                const int32_t *table, uint32_t m, const uint32_t *xi, uint64_t count,
                int32_t *out, uint32_t *loads) {
    for (uint64_t k = 0; k < count; k++)
        out[k] = sample_one(key, child0, child1, table, m, xi[k], loads ? &loads[k] : NULL);
}

/* Binary search over the full fixed-point CDF (Sec.2.2): the last i
 * with K[i] <= xi*2^31.  Zero-weight entries share the key of their successor,
 * so they are never returned. */
void orc_sample_bsearch(const uint64_t *K, uint32_t n, const uint32_t *xi, uint64_t count,
                        int32_t *out) {
    for (uint64_t k = 0; k < count; k++) {
        uint64_t x63 = (uint64_t)xi[k] << 31;
        uint32_t lo = 0, hi = n; /* first index with K > x63 */
        while (lo < hi) {
            uint32_t mid = lo + (hi - lo) / 2;
            if (K[mid] <= x63) lo = mid + 1;
            else hi = mid;
        }
        out[k] = (int32_t)lo - 1;
    }
}

/* Batched rows (Sec.5, reading R15): each row is an independent
 * distribution with its own scale and total.  Per-row status in row_status. */
int orc_build_rows(const float *p, uint32_t rows, uint32_t n_row, uint32_t m_row,
                   uint64_t *key, int32_t *orig, uint32_t *cell, uint8_t *lambda,
                   int32_t *child0, int32_t *child1, int32_t *table,
                   uint64_t *T_out, uint32_t *npos_out, int32_t *row_status) {
    int worst = ORC_OK;
    for (uint32_t r = 0; r < rows; r++) {
        size_t o = (size_t)r * n_row, t = (size_t)r * m_row;
        int st = orc_build(p + o, n_row, m_row, key + o, orig + o, cell + o, lambda + o,
                           child0 + o, child1 + o, table + t, &T_out[r], &npos_out[r]);
        row_status[r] = st;
        if (st != ORC_OK) worst = st;
    }
    return worst;
}
