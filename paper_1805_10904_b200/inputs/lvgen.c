/*
 * lvgen.c — seeded synthetic inputs for the Louvain hot path (see include/lvgen.h).
 *
 * Holds none of the method's arithmetic: it only draws undirected COO records.  All
 * randomness is Philox4x32-10 keyed by (seed, stream) and indexed by the record /
 * document / draw number, so the bytes produced do not depend on the thread count.
 * The recipes (sizes, distributions, seeds) are stated in DESIGN.md §4.
 */
#include "lvgen.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ Philox */
#define PH_M0 0xD2511F53u
#define PH_M1 0xCD9E8D57u
#define PH_W0 0x9E3779B9u
#define PH_W1 0xBB67AE85u

void lvgen_philox(uint32_t k0, uint32_t k1, uint32_t c0, uint32_t c1, uint32_t c2,
                  uint32_t c3, uint32_t out[4]) {
    for (int r = 0; r < 10; ++r) {
        uint64_t p0 = (uint64_t)PH_M0 * c0, p1 = (uint64_t)PH_M1 * c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += PH_W0; k1 += PH_W1;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static inline void ph(uint64_t seed, uint32_t stream, uint64_t idx, uint32_t sub, uint32_t o[4]) {
    lvgen_philox((uint32_t)seed, (uint32_t)(seed >> 32) ^ (stream * 0x85EBCA6Bu),
                 (uint32_t)idx, (uint32_t)(idx >> 32), sub, stream, o);
}

/* uniform integer in [0,r) for r < 2^32 (multiply-high) */
static inline uint32_t uni32(uint32_t x, uint64_t r) { return (uint32_t)(((uint64_t)x * r) >> 32); }
/* uniform double in [0,1) from 53 bits */
static inline double uni53(uint32_t a, uint32_t b) {
    return (double)(((uint64_t)a << 21) ^ (uint64_t)(b >> 11)) * (1.0 / 9007199254740992.0);
}

void lvgen_set_threads(int32_t t) {
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
#else
    (void)t;
#endif
}

/* ------------------------------------------------------------ permutation */
int lvgen_permutation(int64_t n, uint64_t seed, uint32_t stream, int32_t *perm) {
    if (n <= 0 || n > 0x7fffffffLL) return 1;
    for (int64_t i = 0; i < n; ++i) perm[i] = (int32_t)i;
    uint32_t o[4];
    for (int64_t i = n - 1; i > 0; --i) {
        ph(seed, stream, (uint64_t)i, 0, o);
        int64_t j = uni32(o[0], (uint64_t)(i + 1));
        int32_t t = perm[i]; perm[i] = perm[j]; perm[j] = t;
    }
    return 0;
}

/* ------------------------------------------------------------------ karate */
/* Zachary (1977) karate club, 0-based in networkx order. */
static const int8_t KARATE[78][2] = {
    {0,1},{0,2},{0,3},{0,4},{0,5},{0,6},{0,7},{0,8},{0,10},{0,11},{0,12},{0,13},{0,17},{0,19},{0,21},{0,31},
    {1,2},{1,3},{1,7},{1,13},{1,17},{1,19},{1,21},{1,30},{2,3},{2,7},{2,8},{2,9},{2,13},{2,27},{2,28},{2,32},
    {3,7},{3,12},{3,13},{4,6},{4,10},{5,6},{5,10},{5,16},{6,16},{8,30},{8,32},{8,33},{9,33},{13,33},{14,32},
    {14,33},{15,32},{15,33},{18,32},{18,33},{19,33},{20,32},{20,33},{22,32},{22,33},{23,25},{23,27},{23,29},
    {23,32},{23,33},{24,25},{24,27},{24,31},{25,31},{26,29},{26,33},{27,33},{28,31},{28,33},{29,32},{29,33},
    {30,32},{30,33},{31,32},{31,33},{32,33}};

int lvgen_karate(int32_t *src, int32_t *dst) {
    for (int k = 0; k < 78; ++k) { src[k] = KARATE[k][0]; dst[k] = KARATE[k][1]; }
    return 0;
}

/* --------------------------------------------------------- ring of cliques */
int64_t lvgen_ring_of_cliques_m(int32_t k, int32_t c) {
    if (k < 3 || c < 3) return -1;
    return (int64_t)k * c * (c - 1) / 2 + k;
}

int lvgen_ring_of_cliques(int32_t k, int32_t c, int32_t *src, int32_t *dst) {
    if (k < 3 || c < 3) return 1;
    int64_t e = 0;
    for (int32_t t = 0; t < k; ++t) {
        int32_t base = t * c;
        for (int32_t a = 0; a < c; ++a)
            for (int32_t b = a + 1; b < c; ++b) { src[e] = base + a; dst[e] = base + b; ++e; }
    }
    for (int32_t t = 0; t < k; ++t) { src[e] = t * c; dst[e] = ((t + 1) % k) * c; ++e; }
    return 0;
}

/* --------------------------------------------------------------------- SBM */
typedef struct { uint64_t *key; uint64_t mask; } hset_t;

static int hset_init(hset_t *h, int64_t want) {
    uint64_t cap = 1024;
    while (cap < (uint64_t)(2 * want)) cap <<= 1;
    h->key = (uint64_t *)malloc(cap * sizeof(uint64_t));
    if (!h->key) return 1;
    memset(h->key, 0xff, cap * sizeof(uint64_t));
    h->mask = cap - 1;
    return 0;
}

/* returns 1 if inserted (new), 0 if present */
static int hset_insert(hset_t *h, uint64_t k) {
    uint64_t s = (k * 0x9E3779B97F4A7C15ull) >> 20;
    for (;; ++s) {
        uint64_t *p = &h->key[s & h->mask];
        if (*p == ~0ull) { *p = k; return 1; }
        if (*p == k) return 0;
    }
}

int lvgen_sbm(int64_t n, int64_t blocks, int64_t avg_deg, double mu, uint64_t seed,
              int32_t *src, int32_t *dst, int32_t *truth) {
    if (n <= 1 || blocks <= 0 || n % blocks || avg_deg <= 0 || mu < 0 || mu > 1) return 1;
    int64_t bs = n / blocks;
    int64_t m = n * avg_deg / 2;
    int64_t m_out = (int64_t)llround(mu * (double)m);
    int64_t m_in = m - m_out;
    if (bs < 2 && m_in > 0) return 1;
    hset_t hs;
    if (hset_init(&hs, m)) return 1;
    int64_t e = 0;
    uint32_t o[4];
    /* intra-block pairs (stream 1), rejection of loops and duplicates, in draw order */
    for (uint64_t k = 0; e < m_in; ++k) {
        ph(seed, 1, k, 0, o);
        int64_t b = uni32(o[0], (uint64_t)blocks);
        int64_t u = b * bs + uni32(o[1], (uint64_t)bs), v = b * bs + uni32(o[2], (uint64_t)bs);
        if (u == v) continue;
        uint64_t lo = u < v ? (uint64_t)u : (uint64_t)v, hi = u < v ? (uint64_t)v : (uint64_t)u;
        if (!hset_insert(&hs, (lo << 32) | hi)) continue;
        src[e] = (int32_t)lo; dst[e] = (int32_t)hi; ++e;
    }
    /* inter-block pairs (stream 2) */
    for (uint64_t k = 0; e < m; ++k) {
        ph(seed, 2, k, 0, o);
        int64_t u = uni32(o[0], (uint64_t)n), v = uni32(o[1], (uint64_t)n);
        if (u / bs == v / bs) continue;
        uint64_t lo = u < v ? (uint64_t)u : (uint64_t)v, hi = u < v ? (uint64_t)v : (uint64_t)u;
        if (!hset_insert(&hs, (lo << 32) | hi)) continue;
        src[e] = (int32_t)lo; dst[e] = (int32_t)hi; ++e;
    }
    free(hs.key);
    int32_t *perm = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    if (!perm) return 1;
    lvgen_permutation(n, seed, 3, perm);
    for (int64_t k = 0; k < m; ++k) { src[k] = perm[src[k]]; dst[k] = perm[dst[k]]; }
    if (truth)
        for (int64_t v = 0; v < n; ++v) truth[perm[v]] = (int32_t)(v / bs);
    free(perm);
    return 0;
}

/* ------------------------------------------------------------ co-occurrence */
typedef struct {
    int64_t topics, tsz, docs;
    int32_t max_size;
    double p_in;
    uint64_t seed;
    double *size_cdf;   /* P(size <= 2+j), j = 0..max_size-2 */
    double *pop_cdf;    /* popularity CDF over ranks          */
    int32_t *perm;
} cooc_t;

static int cooc_init(cooc_t *q, int64_t topics, int64_t tsz, int64_t docs, double zipf_s,
                     int32_t max_size, double p_in, double pop_exp, uint64_t seed, int need_perm) {
    if (topics <= 0 || tsz <= 0 || docs < 0 || max_size < 2 || max_size > 64 || zipf_s <= 1.0 ||
        topics * tsz > 0x7fffffffLL)
        return 1;
    q->topics = topics; q->tsz = tsz; q->docs = docs; q->max_size = max_size;
    q->p_in = p_in; q->seed = seed; q->perm = NULL;
    /* size = min(1 + Z, max_size), Z ~ Zipf(s) on k >= 1 */
    double zeta = 0.0;
    for (int64_t k = 1; k <= 2000000; ++k) zeta += pow((double)k, -zipf_s);
    zeta += pow(2000000.0, 1.0 - zipf_s) / (zipf_s - 1.0);
    q->size_cdf = (double *)malloc((size_t)max_size * sizeof(double));
    double acc = 0.0;
    for (int32_t j = 0; j < max_size - 2; ++j) { acc += pow((double)(j + 1), -zipf_s) / zeta; q->size_cdf[j] = acc; }
    q->size_cdf[max_size - 2] = 2.0;   /* everything else caps at max_size */
    q->pop_cdf = (double *)malloc((size_t)tsz * sizeof(double));
    double tot = 0.0;
    for (int64_t r = 0; r < tsz; ++r) tot += pow((double)(r + 1), -pop_exp);
    acc = 0.0;
    for (int64_t r = 0; r < tsz; ++r) { acc += pow((double)(r + 1), -pop_exp) / tot; q->pop_cdf[r] = acc; }
    q->pop_cdf[tsz - 1] = 2.0;
    if (need_perm) {
        q->perm = (int32_t *)malloc((size_t)(topics * tsz) * sizeof(int32_t));
        lvgen_permutation(topics * tsz, seed, 7, q->perm);
    }
    return 0;
}

static void cooc_free(cooc_t *q) { free(q->size_cdf); free(q->pop_cdf); free(q->perm); }

static int64_t cdf_find(const double *cdf, int64_t len, double u) {
    int64_t lo = 0, hi = len - 1;
    while (lo < hi) { int64_t mid = (lo + hi) / 2; if (cdf[mid] > u) hi = mid; else lo = mid + 1; }
    return lo;
}

/* members of document d, sorted and unique; returns count */
static int cooc_doc(const cooc_t *q, int64_t d, int32_t *mem) {
    uint32_t o[4];
    ph(q->seed, 5, (uint64_t)d, 0, o);
    int64_t topic = uni32(o[0], (uint64_t)q->topics);
    int32_t s = 2 + (int32_t)cdf_find(q->size_cdf, q->max_size - 1, uni53(o[1], o[2]));
    int cnt = 0;
    for (int32_t t = 0; t < s; ++t) {
        ph(q->seed, 6, (uint64_t)d, (uint32_t)(t + 1), o);
        int64_t tp = o[0] < (uint32_t)(q->p_in * 4294967296.0) ? topic : (int64_t)uni32(o[1], (uint64_t)q->topics);
        int64_t r = cdf_find(q->pop_cdf, q->tsz, uni53(o[2], o[3]));
        int32_t id = (int32_t)(tp * q->tsz + r);
        /* insertion into sorted unique list */
        int pos = cnt;
        while (pos > 0 && mem[pos - 1] > id) --pos;
        if (pos > 0 && mem[pos - 1] == id) continue;
        memmove(mem + pos + 1, mem + pos, (size_t)(cnt - pos) * sizeof(int32_t));
        mem[pos] = id;
        ++cnt;
    }
    return cnt;
}

int64_t lvgen_cooc_count(int64_t topics, int64_t topic_size, int64_t docs, double zipf_s,
                         int32_t max_size, double p_in, double pop_exp, uint64_t seed) {
    cooc_t q;
    if (cooc_init(&q, topics, topic_size, docs, zipf_s, max_size, p_in, pop_exp, seed, 0)) return -1;
    int64_t total = 0;
#pragma omp parallel for schedule(static, 4096) reduction(+ : total)
    for (int64_t d = 0; d < docs; ++d) {
        int32_t mem[64];
        int64_t c = cooc_doc(&q, d, mem);
        total += c * (c - 1) / 2;
    }
    cooc_free(&q);
    return total;
}

int lvgen_cooc_fill(int64_t topics, int64_t topic_size, int64_t docs, double zipf_s,
                    int32_t max_size, double p_in, double pop_exp, uint64_t seed,
                    int32_t *src, int32_t *dst) {
    cooc_t q;
    if (cooc_init(&q, topics, topic_size, docs, zipf_s, max_size, p_in, pop_exp, seed, 1)) return 1;
    int64_t *off = (int64_t *)malloc((size_t)(docs + 1) * sizeof(int64_t));
    if (!off) { cooc_free(&q); return 1; }
#pragma omp parallel for schedule(static, 4096)
    for (int64_t d = 0; d < docs; ++d) {
        int32_t mem[64];
        int64_t c = cooc_doc(&q, d, mem);
        off[d + 1] = c * (c - 1) / 2;
    }
    off[0] = 0;
    for (int64_t d = 0; d < docs; ++d) off[d + 1] += off[d];
#pragma omp parallel for schedule(static, 4096)
    for (int64_t d = 0; d < docs; ++d) {
        int32_t mem[64];
        int c = cooc_doc(&q, d, mem);
        int64_t e = off[d];
        for (int a = 0; a < c; ++a)
            for (int b = a + 1; b < c; ++b) { src[e] = q.perm[mem[a]]; dst[e] = q.perm[mem[b]]; ++e; }
    }
    free(off);
    cooc_free(&q);
    return 0;
}

/* ------------------------------------------------------------------- R-MAT */
int lvgen_rmat(int32_t scale, int64_t edge_factor, double a, double b, double c,
               int32_t wmax, uint64_t seed, int32_t *src, int32_t *dst, int32_t *w) {
    if (scale < 1 || scale > 30 || edge_factor <= 0 || a < 0 || b < 0 || c < 0 || a + b + c > 1.0 || wmax < 0)
        return 1;
    int64_t n = (int64_t)1 << scale;
    int64_t m = edge_factor * n;
    uint32_t ta = (uint32_t)llround(a * 65536.0);
    uint32_t tb = ta + (uint32_t)llround(b * 65536.0);
    uint32_t tc = tb + (uint32_t)llround(c * 65536.0);
    int32_t *perm = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    if (!perm) return 1;
    lvgen_permutation(n, seed, 9, perm);
#pragma omp parallel for schedule(static, 65536)
    for (int64_t k = 0; k < m; ++k) {
        uint32_t o[4];
        uint32_t u = 0, v = 0;
        for (int32_t lev = 0; lev < scale; ++lev) {
            if ((lev & 7) == 0) ph(seed, 8, (uint64_t)k, (uint32_t)(lev >> 3), o);
            uint32_t word = o[(lev & 7) >> 1];
            uint32_t r = (lev & 1) ? (word >> 16) : (word & 0xffffu);
            uint32_t bu = 0, bv = 0;
            if (r < ta) { bu = 0; bv = 0; }
            else if (r < tb) { bu = 0; bv = 1; }
            else if (r < tc) { bu = 1; bv = 0; }
            else { bu = 1; bv = 1; }
            u = (u << 1) | bu;
            v = (v << 1) | bv;
        }
        src[k] = perm[u];
        dst[k] = perm[v];
        if (w) {
            if (wmax > 0) { ph(seed, 8, (uint64_t)k, 15u, o); w[k] = 1 + (int32_t)uni32(o[0], (uint64_t)wmax); }
            else w[k] = 1;
        }
    }
    free(perm);
    return 0;
}
