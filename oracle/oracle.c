/*
 * oracle.c — plain, slow CPU oracle (TEST INFRASTRUCTURE ONLY).
 *
 * Follows Forster, arXiv 1805.10904 (/root/reference/PAPER.md, cited "P:Lnn") step by
 * step, with the readings D1..D29 of DESIGN.md §3 wherever the paper is silent, garbled
 * or inconsistent.  No blocking, fusion or reordering: each function is the paper's
 * definition or algorithm written out.  Library primitives used as steps: qsort.
 *
 * Threads (OpenMP: "optionally OpenMP over the scoring loop, which is
 * still bit-identical under Jacobi").  Only loops whose result cannot depend on the
 * schedule are parallel:
 *   - the Jacobi vertex loop of a sweep (every decision reads only the snapshot; each
 *     thread has its own Eq. 1 scratch),
 *   - the exact integer sums of Eq. 3 (int64 / int128 addition is associative),
 *   - the per-row sort of the CSR build and of graph rebuilding (rows are disjoint).
 * og_set_threads(1) gives the single-threaded oracle; tests/test_oracle_pins.py checks
 * that 1 and several threads agree bit for bit.
 *
 * Sorting by (source, target) (P:L271 sort_by_key) is done as a counting sort
 * on the source (bucket each record into its row) followed by a qsort of each row on
 * the target — the same order as one global sort on the pair.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline, --impl reference)
 * may load this file's library.  It shares nothing with paper_1805_10904_b200/.
 *
 * Parity pins: see tests/test_oracle_*.py (Eq. 3 brute force + networkx, gain
 * consistency vs Eq. 3 differences, exhaustive optimum bound, ring of cliques,
 * karate band and exact values, SPEC examples, Theorem 1 invariant, weight
 * conservation, thread-count invariance).
 * Build: gcc -O2 -std=c11 -fopenmp -ffp-contract=off -fno-fast-math -shared -fPIC.
 */
#include "oracle.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

typedef __int128 i128;

/* ---------------------------------------------------------------- utilities */

/* D22 (as refined in DESIGN.md §3): pinned int128 → fp64 conversion on the magnitude,
 * d(x) = sign(x) · fl(fl(hi)·2^64 + fl(lo)) with (hi,lo) the 64-bit words of |x|.
 * (A two's-complement split fl(hi)·2^64 + fl(lo) cancels catastrophically for small
 * negative x, e.g. d(−2) = 0; tests/test_oracle_pins.py::test_modularity_closed_forms.) */
static double d128(i128 x) {
    int neg = x < 0;
    unsigned __int128 m = neg ? (unsigned __int128)(-x) : (unsigned __int128)x;
    uint64_t hi = (uint64_t)(m >> 64), lo = (uint64_t)m;
    double d = (double)hi * 18446744073709551616.0 + (double)lo;
    return neg ? -d : d;
}

void og_config_default(og_config *c) {
    c->theta = 1e-6;          /* D16 */
    c->big_theta = 1e-6;      /* D16 */
    c->max_sweeps = 100;      /* D12 */
    c->max_levels = 64;       /* D27 */
    c->stop_rule = 0;         /* D10: Alg. 1 literal */
    c->merge_isolated = 1;    /* D14 */
    c->theta_schedule = NULL; /* D21 */
    c->theta_schedule_len = 0;
    c->coloring = 0;          /* D29: off (the paper's pure Jacobi sweeps) */
    c->color_classes = 32;    /* D29: colours >= 31 share the last class ... */
    c->color_cap_min_n = 65536; /* ... on level graphs of more than 65536 vertices */
}

/* ------------------------------------------------------- graph construction */

void og_set_threads(int32_t t) { omp_set_num_threads(t > 0 ? t : 1); }
int32_t og_get_threads(void) { return (int32_t)omp_get_max_threads(); }

typedef struct { int32_t v; int64_t w; } ent_t;

static int ent_cmp(const void *a, const void *b) {
    const ent_t *x = (const ent_t *)a, *y = (const ent_t *)b;
    return x->v < y->v ? -1 : x->v > y->v ? 1 : 0;
}

static og_graph *graph_alloc(int64_t n) {
    og_graph *g = (og_graph *)calloc(1, sizeof(og_graph));
    if (!g) return NULL;
    g->n = n;
    g->row_ptr = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    g->loop = (int64_t *)calloc((size_t)n, sizeof(int64_t));
    g->delta = (int64_t *)calloc((size_t)n, sizeof(int64_t));
    if (!g->row_ptr || !g->loop || !g->delta) { og_graph_free(g); return NULL; }
    return g;
}

void og_graph_free(og_graph *g) {
    if (!g) return;
    free(g->row_ptr); free(g->col); free(g->w); free(g->loop); free(g->delta);
    free(g);
}

/* The CSR of directed records that were bucketed by source: row u holds its records
 * (col[k], w[k]) for k in [row_ptr[u], row_ptr[u+1]) in arbitrary order.  Sort each row
 * by target and merge duplicates by summing (P:L271 sort_by_key + reduce_by_key; D25),
 * compact, then δ_i = Σ_{j∈Γ(i)} ω(i,j) with a loop counted twice (D2). */
static int finish_csr(og_graph *g) {
    const int64_t n = g->n;
    int64_t maxlen = 0;
    for (int64_t u = 0; u < n; ++u)
        if (g->row_ptr[u + 1] - g->row_ptr[u] > maxlen) maxlen = g->row_ptr[u + 1] - g->row_ptr[u];
    int64_t *len = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    if (!len) return OG_ENOMEM;
    int err = 0;
#pragma omp parallel
    {
        ent_t *buf = (ent_t *)malloc((size_t)(maxlen > 0 ? maxlen : 1) * sizeof(ent_t));
        if (!buf) {
#pragma omp atomic write
            err = 1;
        }
#pragma omp for schedule(dynamic, 1024)
        for (int64_t u = 0; u < n; ++u) {
            if (!buf) { len[u] = 0; continue; }
            const int64_t b = g->row_ptr[u], e = g->row_ptr[u + 1];
            for (int64_t k = b; k < e; ++k) { buf[k - b].v = g->col[k]; buf[k - b].w = g->w[k]; }
            qsort(buf, (size_t)(e - b), sizeof(ent_t), ent_cmp);
            int64_t out = 0;
            for (int64_t k = 0; k < e - b; ++k) {
                if (out > 0 && buf[out - 1].v == buf[k].v) buf[out - 1].w += buf[k].w;
                else buf[out++] = buf[k];
            }
            for (int64_t k = 0; k < out; ++k) { g->col[b + k] = buf[k].v; g->w[b + k] = buf[k].w; }
            len[u] = out;
        }
        free(buf);
    }
    if (err) { free(len); return OG_ENOMEM; }
    /* compact (new offsets never exceed the old ones, so an in-place forward move) */
    int64_t o = 0;
    for (int64_t u = 0; u < n; ++u) {
        const int64_t b = g->row_ptr[u];
        g->row_ptr[u] = o;
        if (o != b) {
            memmove(g->col + o, g->col + b, (size_t)len[u] * sizeof(int32_t));
            memmove(g->w + o, g->w + b, (size_t)len[u] * sizeof(int64_t));
        }
        o += len[u];
    }
    g->row_ptr[n] = o;
    g->nnz = o;
    free(len);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        int64_t s = 2 * g->loop[i];
        for (int64_t e = g->row_ptr[i]; e < g->row_ptr[i + 1]; ++e) s += g->w[e];
        g->delta[i] = s;
    }
    return OG_OK;
}

/* Bucket directed records by source: row_ptr = exclusive scan of the per-row counts
 * (already in row_ptr[u+1]); allocates col/w with `cnt` entries; returns a cursor array
 * (next free slot of each row) or NULL. */
static int64_t *bucket_alloc(og_graph *g, int64_t cnt) {
    for (int64_t u = 0; u < g->n; ++u) g->row_ptr[u + 1] += g->row_ptr[u];
    g->col = (int32_t *)malloc((size_t)(cnt > 0 ? cnt : 1) * sizeof(int32_t));
    g->w = (int64_t *)malloc((size_t)(cnt > 0 ? cnt : 1) * sizeof(int64_t));
    int64_t *cur = (int64_t *)malloc((size_t)(g->n > 0 ? g->n : 1) * sizeof(int64_t));
    if (!g->col || !g->w || !cur) { free(cur); return NULL; }
    memcpy(cur, g->row_ptr, (size_t)g->n * sizeof(int64_t));
    return cur;
}

/* §5.1.2 "Neighbor computation": mirror every non-loop record, sort by
 * (source,target), merge, offsets by exclusive scan.  Loops go to loop[] (D2). */
int og_graph_build(int64_t n, int64_t m, const int32_t *src, const int32_t *dst,
                   const int64_t *w, og_graph **out) {
    *out = NULL;
    if (n <= 0 || m < 0) return OG_EINVAL;
    og_graph *g = graph_alloc(n);
    if (!g) return OG_ENOMEM;
    int64_t cnt = 0, W = 0;
    for (int64_t k = 0; k < m; ++k) {
        int32_t u = src[k], v = dst[k];
        int64_t wk = w ? w[k] : 1;                 /* D1: unweighted ⇒ 1 */
        if (u < 0 || v < 0 || u >= n || v >= n || wk <= 0) { og_graph_free(g); return OG_EGRAPH; }
        W += wk;                                    /* D3: W = Σ weights, loops once */
        if (u == v) { g->loop[u] += wk; continue; }
        g->row_ptr[u + 1]++; g->row_ptr[v + 1]++;   /* both orientations */
        cnt += 2;
    }
    int64_t *cur = bucket_alloc(g, cnt);
    if (!cur) { og_graph_free(g); return OG_ENOMEM; }
    for (int64_t k = 0; k < m; ++k) {
        int32_t u = src[k], v = dst[k];
        int64_t wk = w ? w[k] : 1;
        if (u == v) continue;
        g->col[cur[u]] = v; g->w[cur[u]++] = wk;
        g->col[cur[v]] = u; g->w[cur[v]++] = wk;
    }
    free(cur);
    int rc = finish_csr(g);
    if (rc) { og_graph_free(g); return rc; }
    g->W = W;
    *out = g;
    return W > 0 ? OG_OK : OG_EZEROW;
}

/* ------------------------------------------------ real weights (F1, reading D28) */

/* rint(ω · 2^s): ldexp is exact whenever the result is >= 2^-1022 (a power-of-two
 * scaling), and anything smaller rounds to 0 either way; rint rounds half to even in
 * the default rounding mode. */
static double fixed_of(double w, int32_t s) { return rint(ldexp(w, s)); }

int64_t og_fixed_sum(int64_t m, const double *w, int32_t s) {
    const double cap = 4611686018427387904.0;   /* 2^62 */
    __int128 t = 0;
    for (int64_t k = 0; k < m; ++k) {
        double x = fixed_of(w[k], s);
        if (!(x < cap)) return (int64_t)cap;      /* also catches inf */
        t += (__int128)(int64_t)x;
        if (t >= (__int128)(int64_t)cap) return (int64_t)cap;
    }
    return (int64_t)t;
}

int og_graph_build_real(int64_t n, int64_t m, const int32_t *src, const int32_t *dst,
                        const double *w, int32_t *s_out, og_graph **out) {
    *out = NULL;
    if (n <= 0 || m < 0 || !w || !s_out) return OG_EINVAL;
    for (int64_t k = 0; k < m; ++k)
        if (!(w[k] > 0.0) || !isfinite(w[k])) return OG_EGRAPH;      /* P:L43 positive */
    const int64_t lim = (int64_t)1 << 52;
    /* T(s) is non-decreasing in s: binary search the largest s with T(s) <= 2^52 over
     * [-1100, 1100] (T(-1100) = 0; T(1100) saturates for any ω > 0 when m > 0). */
    int32_t lo = -1100, hi = 1100;              /* invariant: T(lo) <= lim < T(hi) */
    if (m == 0) hi = lo;                        /* W = 0 below anyway */
    while (hi - lo > 1) {
        int32_t mid = lo + (hi - lo) / 2;
        if (og_fixed_sum(m, w, mid) <= lim) lo = mid; else hi = mid;
    }
    const int32_t s = lo;
    int64_t *wi = (int64_t *)malloc((size_t)(m > 0 ? m : 1) * sizeof(int64_t));
    if (!wi) return OG_ENOMEM;
    for (int64_t k = 0; k < m; ++k) {
        wi[k] = (int64_t)fixed_of(w[k], s);
        if (wi[k] <= 0) { free(wi); return OG_EGRAPH; }   /* ω~ = 0: range beyond 52 bits */
    }
    *s_out = s;
    int rc = og_graph_build(n, m, src, dst, wi, out);
    free(wi);
    return rc;
}

/* ----------------------------------------------------------- community state */

/* Eq. 1 scratch of one thread: e_{i→c} per label, and the list of touched labels */
typedef struct {
    int64_t *e;          /* e_{i→c} accumulator (Eq. 1)                */
    int32_t *touched;    /* list of touched labels                     */
} scratch_t;

static int scratch_init(scratch_t *s, int64_t n) {
    s->e = (int64_t *)calloc((size_t)n, sizeof(int64_t));
    s->touched = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    return s->e && s->touched;
}
static void scratch_free(scratch_t *s) { free(s->e); free(s->touched); s->e = NULL; s->touched = NULL; }

struct og_state {
    const og_graph *g;
    const int32_t *C;    /* snapshot labels (borrowed)                 */
    int64_t *deg;        /* deg_C (Eq. 2), indexed by label            */
    int64_t *size;       /* |C|, indexed by label                      */
    scratch_t s;         /* scratch of og_decide (single-vertex calls)  */
};

/* Eq. 2: deg_C = Σ_{i∈C} δ_i (and |C|), indexed by label.  Integer sums: the parallel
 * loop with atomic adds gives the same result as the sequential one. */
static void community_sums(int64_t n, const int32_t *labels, const int64_t *delta, int64_t *deg, int64_t *size) {
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < n; ++c) { deg[c] = 0; if (size) size[c] = 0; }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
#pragma omp atomic
        deg[labels[i]] += delta[i];
        if (size) {
#pragma omp atomic
            size[labels[i]] += 1;
        }
    }
}

og_state *og_state_new(const og_graph *g, const int32_t *labels) {
    og_state *st = (og_state *)calloc(1, sizeof(og_state));
    if (!st) return NULL;
    int64_t n = g->n;
    st->g = g;
    st->C = labels;
    st->deg = (int64_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    st->size = (int64_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    if (!st->deg || !st->size) { og_state_free(st); return NULL; }
    community_sums(n, labels, g->delta, st->deg, st->size);
    return st;
}

void og_state_free(og_state *st) {
    if (!st) return;
    free(st->deg); free(st->size); scratch_free(&st->s);
    free(st);
}

/* The decision of vertex i against the snapshot (Algorithm 1 body).
 *  mode 0 (local move):
 *   N_i = {C(i)} ∪ {C(j) : j ∈ Γ(i)}, loops excluded (D5)
 *   e_{i→c} per Eq. 1; gain of moving to c relative to staying, Eq. 4 read as D4:
 *     S(c)   = 2W·e_{i→c} − δ_i·deg_c                   (c ≠ C(i))
 *     S_own  = 2W·e_{i→C(i)} − δ_i·(deg_{C(i)} − δ_i)   (C(i)\{i})
 *     ΔQ_{i→c} = (S(c) − S_own) / (2W²)
 *   target = argmax ΔQ, ties → minimum label (Eq. 5, §3.1.2; D7)
 *   move iff ΔQ_{i→target} > 0 (D6 strict)
 *   singlet rule: singlet → singlet only if l(target) < l(C(i)) (§3.1.1; D8: else stay)
 *  mode 1 (isolated merge; D14): a singlet whose neighbours lie in exactly one
 *   community T moves to T (singlet rule applies). */
static int32_t decide(const og_state *st, scratch_t *sc, int64_t i, int32_t mode) {
    const og_graph *g = st->g;
    const int32_t *C = st->C;
    int32_t own = C[i];
    int64_t b = g->row_ptr[i], eend = g->row_ptr[i + 1];
    if (b == eend) return own;                       /* no non-loop neighbours */
    if (mode == 1 && st->size[own] != 1) return own; /* D14: singlets only     */
    int64_t nt = 0;
    for (int64_t k = b; k < eend; ++k) {             /* Eq. 1 */
        int32_t c = C[g->col[k]];
        if (sc->e[c] == 0) sc->touched[nt++] = c;    /* weights are > 0: e = 0 iff untouched */
        sc->e[c] += g->w[k];
    }
    int32_t result = own;
    if (mode == 0) {
        i128 twoW = (i128)2 * g->W;
        i128 di = g->delta[i];
        int64_t e_own = sc->e[own];
        i128 S_own = twoW * e_own - di * ((i128)st->deg[own] - di);
        int32_t best = -1;
        i128 S_best = 0;
        for (int64_t t = 0; t < nt; ++t) {
            int32_t c = sc->touched[t];
            if (c == own) continue;
            i128 S = twoW * sc->e[c] - di * (i128)st->deg[c];
            if (best < 0 || S > S_best || (S == S_best && c < best)) { best = c; S_best = S; }
        }
        if (best >= 0 && S_best > S_own) {
            if (st->size[own] == 1 && st->size[best] == 1 && best > own) result = own;
            else result = best;
        }
    } else {
        int32_t T = -1;
        int64_t distinct = 0;
        for (int64_t t = 0; t < nt; ++t)
            if (sc->touched[t] != own) { ++distinct; T = sc->touched[t]; }
        if (distinct == 1) {
            if (st->size[T] == 1 && T > own) result = own;
            else result = T;
        }
    }
    for (int64_t t = 0; t < nt; ++t) sc->e[sc->touched[t]] = 0;
    return result;
}

int32_t og_decide(og_state *st, int64_t i, int32_t mode) {
    if (!st->s.e && !scratch_init(&st->s, st->g->n)) return -1;
    return decide(st, &st->s, i, mode);
}

/* Per-thread Eq. 1 scratch, kept across sweeps (decide() leaves it all-zero), so a
 * sweep does not re-allocate and re-fault n-length arrays per thread.  Grown on demand. */
static __thread scratch_t tl_scratch;
static __thread int64_t tl_scratch_n = 0;
static scratch_t *thread_scratch(int64_t n) {
    if (tl_scratch_n < n) {
        if (tl_scratch_n) scratch_free(&tl_scratch);
        tl_scratch_n = 0;
        if (!scratch_init(&tl_scratch, n)) { scratch_free(&tl_scratch); return NULL; }
        tl_scratch_n = n;
    }
    return &tl_scratch;
}

int64_t og_sweep(const og_graph *g, const int32_t *labels_in, int32_t *labels_out, int32_t mode) {
    og_state *st = og_state_new(g, labels_in);
    if (!st) return -1;
    int64_t moved = 0;
    int err = 0;
    /* Jacobi: every decision reads only the snapshot (D9), so the vertices are
     * independent and the loop may run on any number of threads. */
#pragma omp parallel reduction(+ : moved)
    {
        scratch_t *sc = thread_scratch(g->n);
        if (!sc) {
#pragma omp atomic write
            err = 1;
        }
#pragma omp for schedule(dynamic, 256)
        for (int64_t i = 0; i < g->n; ++i) {
            if (!sc) continue;
            labels_out[i] = decide(st, sc, i, mode);
            moved += labels_out[i] != labels_in[i];
        }
    }
    og_state_free(st);
    return err ? -1 : moved;
}

/* ------------------------------------------------- colouring heuristic (F2, D29) */

uint64_t og_color_priority(int64_t v) {
    uint64_t k = (uint64_t)v ^ 0x9E3779B97F4A7C15ull;
    k ^= k >> 33; k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33; k *= 0xc4ceb9fe1a85ec53ull;
    k ^= k >> 33;
    return k;
}

typedef struct { uint64_t p; int32_t v; } prio_t;
static int prio_desc(const void *a, const void *b) {
    uint64_t x = ((const prio_t *)a)->p, y = ((const prio_t *)b)->p;
    return x < y ? 1 : x > y ? -1 : 0;
}

int32_t og_color(const og_graph *g, int32_t *color) {
    int64_t n = g->n;
    prio_t *ord = (prio_t *)malloc((size_t)n * sizeof(prio_t));
    uint8_t *used = (uint8_t *)calloc((size_t)n + 1, 1);
    if (!ord || !used) { free(ord); free(used); return -1; }
    for (int64_t v = 0; v < n; ++v) { ord[v].p = og_color_priority(v); ord[v].v = (int32_t)v; color[v] = -1; }
    qsort(ord, (size_t)n, sizeof(prio_t), prio_desc);
    int32_t K = 0;
    for (int64_t t = 0; t < n; ++t) {
        int32_t v = ord[t].v;
        for (int64_t e = g->row_ptr[v]; e < g->row_ptr[v + 1]; ++e)      /* mark */
            if (color[g->col[e]] >= 0) used[color[g->col[e]]] = 1;
        int32_t c = 0;
        while (used[c]) ++c;                                              /* smallest free */
        color[v] = c;
        if (c + 1 > K) K = c + 1;
        for (int64_t e = g->row_ptr[v]; e < g->row_ptr[v + 1]; ++e)      /* unmark */
            if (color[g->col[e]] >= 0) used[color[g->col[e]]] = 0;
        used[c] = 0;
    }
    free(ord); free(used);
    return K;
}

int64_t og_sweep_colored(const og_graph *g, const int32_t *color, int32_t ncolors,
                         const int32_t *labels_in, int32_t *labels_out) {
    int64_t n = g->n, moved = 0;
    int32_t *cur = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    if (!cur) return -1;
    memcpy(cur, labels_in, (size_t)n * sizeof(int32_t));
    memcpy(labels_out, labels_in, (size_t)n * sizeof(int32_t));
    for (int32_t c = 0; c < ncolors; ++c) {
        og_state *st = og_state_new(g, cur);              /* state after class c-1 */
        if (!st) { free(cur); return -1; }
        int err = 0;
#pragma omp parallel
        {
            scratch_t sc;
            int ok = scratch_init(&sc, n);
            if (!ok) {
#pragma omp atomic write
                err = 1;
            }
#pragma omp for schedule(dynamic, 256)
            for (int64_t i = 0; i < n; ++i)      /* Jacobi within the class */
                if (ok && color[i] == c) labels_out[i] = decide(st, &sc, i, 0);
            scratch_free(&sc);
        }
        og_state_free(st);
        if (err) { free(cur); return -1; }
        memcpy(cur, labels_out, (size_t)n * sizeof(int32_t));   /* commit class c */
    }
    for (int64_t i = 0; i < n; ++i) moved += labels_out[i] != labels_in[i];
    free(cur);
    return moved;
}

/* ---------------------------------------------------------------- modularity */

/* Eq. 3: Q = (1/2W) Σ_i e_{i→C(i)} − Σ_C (deg_C/2W)², with e_{i→C(i)} counting a loop
 * twice (D2, D24).  Exact numerator 2W·I2 − S2 over 4W². */
static void modularity_num(const og_graph *g, const int32_t *C, const int64_t *deg,
                           int64_t *I2, i128 *S2) {
    int64_t s = 0;
#pragma omp parallel for schedule(dynamic, 1024) reduction(+ : s)
    for (int64_t i = 0; i < g->n; ++i) {
        s += 2 * g->loop[i];
        for (int64_t k = g->row_ptr[i]; k < g->row_ptr[i + 1]; ++k)
            if (C[g->col[k]] == C[i]) s += g->w[k];
    }
    i128 q = 0;   /* exact: int128 addition is associative (partials per thread) */
#pragma omp parallel
    {
        i128 qt = 0;
#pragma omp for schedule(static)
        for (int64_t c = 0; c < g->n; ++c) qt += (i128)deg[c] * deg[c];
#pragma omp critical
        q += qt;
    }
    *I2 = s;
    *S2 = q;
}

static double q_from_num(int64_t W, int64_t I2, i128 S2) {
    i128 num = (i128)2 * W * I2 - S2;
    i128 den = (i128)4 * W * W;
    return d128(num) / d128(den);
}

int og_modularity(const og_graph *g, const int32_t *labels, int64_t *I2,
                  int64_t *S2_hi, uint64_t *S2_lo, double *Q) {
    if (g->W <= 0) return OG_EZEROW;
    int64_t *deg = (int64_t *)calloc((size_t)g->n, sizeof(int64_t));
    if (!deg) return OG_ENOMEM;
    for (int64_t i = 0; i < g->n; ++i) {
        if (labels[i] < 0 || labels[i] >= g->n) { free(deg); return OG_EINVAL; }
        deg[labels[i]] += g->delta[i];
    }
    int64_t i2; i128 s2;
    modularity_num(g, labels, deg, &i2, &s2);
    free(deg);
    *I2 = i2;
    *S2_hi = (int64_t)(s2 >> 64);
    *S2_lo = (uint64_t)s2;
    *Q = q_from_num(g->W, i2, s2);
    return OG_OK;
}

/* ------------------------------------------------------- renumber and induce */

/* "Renumbering nodes": sort the cluster ids, unique, map each to its
 * rank — i.e. an order-preserving dense relabel (D18). */
int64_t og_renumber(int64_t n, const int32_t *in, int32_t *outl) {
    int32_t *id = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    uint8_t *used = (uint8_t *)calloc((size_t)n, 1);
    for (int64_t i = 0; i < n; ++i) used[in[i]] = 1;
    int64_t k = 0;
    for (int64_t c = 0; c < n; ++c) id[c] = used[c] ? (int32_t)k++ : -1;
    for (int64_t i = 0; i < n; ++i) outl[i] = id[in[i]];
    free(id); free(used);
    return k;
}

/* Graph rebuilding (D19): each community becomes a vertex; an
 * intra-community edge adds its weight to the meta-vertex loop (old loops once);
 * inter-community weights are summed per community pair. */
int og_induce(const og_graph *g, const int32_t *C, int64_t k, og_graph **out) {
    *out = NULL;
    og_graph *h = graph_alloc(k);
    int64_t *intra2 = (int64_t *)calloc((size_t)(k > 0 ? k : 1), sizeof(int64_t));
    if (!h || !intra2) { og_graph_free(h); free(intra2); return OG_ENOMEM; }
    int64_t cnt = 0;
    for (int64_t u = 0; u < g->n; ++u) {               /* count inter entries per C(u) */
        int32_t cu = C[u];
        for (int64_t e = g->row_ptr[u]; e < g->row_ptr[u + 1]; ++e)
            if (C[g->col[e]] != cu) { h->row_ptr[cu + 1]++; ++cnt; }
    }
    int64_t *cur = bucket_alloc(h, cnt);
    if (!cur) { og_graph_free(h); free(intra2); return OG_ENOMEM; }
    for (int64_t u = 0; u < g->n; ++u) {
        int32_t cu = C[u];
        h->loop[cu] += g->loop[u];
        for (int64_t e = g->row_ptr[u]; e < g->row_ptr[u + 1]; ++e) {
            int32_t cv = C[g->col[e]];
            if (cv == cu) intra2[cu] += g->w[e];     /* each undirected edge seen twice */
            else { h->col[cur[cu]] = cv; h->w[cur[cu]++] = g->w[e]; }
        }
    }
    free(cur);
    for (int64_t c = 0; c < k; ++c) h->loop[c] += intra2[c] / 2;
    free(intra2);
    int rc = finish_csr(h);                          /* sort by (C(u), C(v)), sum */
    if (rc) { og_graph_free(h); return rc; }
    h->W = g->W;
    *out = h;
    /* W' = W (weight conservation): Σ directed inter weights / 2 + Σ loops */
    int64_t und = 0, lp = 0;
    for (int64_t e = 0; e < h->nnz; ++e) und += h->w[e];
    for (int64_t c = 0; c < k; ++c) lp += h->loop[c];
    if (und % 2 != 0 || und / 2 + lp != g->W) return OG_EGRAPH;
    return OG_OK;
}

/* -------------------------------------------------------------- Algorithm 1/2 */

typedef struct {
    int64_t n;
    int32_t *labels;
    double q;
    int32_t sweeps;
    int32_t trace_len;
    int64_t *moved;
    double *qs;
} og_level;

struct og_result {
    int32_t nlev;
    og_level *lev;
    int64_t n0;
    int64_t edge_visits;
};

/* D10/D11 stop test, identical expression on both sides (compiled without FMA). */
static int stop_test(int rule, double Q, double Qp, double theta) {
    if (rule == 0) {
        if (fabs(Qp) >= 1e-12) return fabs((Q - Qp) / Qp) < theta;
        return fabs(Q - Qp) < theta;
    }
    if (fabs(Qp) >= 1e-12) return (Q - Qp) / fabs(Qp) < theta;
    return (Q - Qp) < theta;
}

/* Algorithm 1 for one level: returns the committed labels in C (not
 * renumbered), the number of sweeps, and the per-sweep trace. */
static int one_level(const og_graph *g, const og_config *cfg, double theta, int32_t *C,
                     og_level *L, int64_t *visits) {
    int64_t n = g->n;
    int32_t *next = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    int64_t *deg = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    L->moved = (int64_t *)malloc((size_t)(cfg->max_sweeps + 1) * sizeof(int64_t));
    L->qs = (double *)malloc((size_t)(cfg->max_sweeps + 1) * sizeof(double));
    if (!next || !deg || !L->moved || !L->qs) { free(next); free(deg); return OG_ENOMEM; }
    for (int64_t i = 0; i < n; ++i) C[i] = (int32_t)i;   /* initStatus: singletons */
    int32_t *color = NULL, K = 0;
    if (cfg->coloring) {                                  /* D29: colour the level graph */
        color = (int32_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(int32_t));
        if (!color || (K = og_color(g, color)) < 0) { free(color); free(next); free(deg); return OG_ENOMEM; }
        if (cfg->color_classes > 0 && K > cfg->color_classes && n > cfg->color_cap_min_n) {   /* D29 cap */
            K = cfg->color_classes;
            for (int64_t i = 0; i < n; ++i) if (color[i] > K - 1) color[i] = K - 1;
        }
    }
    int first = 1;                                        /* Q_prev ← −∞ (D11) */
    double Qp = 0.0;
    int32_t s;
    L->trace_len = 0;
    for (s = 1; s <= cfg->max_sweeps; ++s) {              /* D12 cap */
        int64_t moved = cfg->coloring ? og_sweep_colored(g, color, K, C, next)   /* D29 */
                                      : og_sweep(g, C, next, 0);   /* decisions from the snapshot */
        if (moved < 0) { free(color); free(next); free(deg); return OG_ENOMEM; }
        *visits += g->nnz;
        memcpy(C, next, (size_t)n * sizeof(int32_t));     /* commit (D13) */
        community_sums(n, C, g->delta, deg, NULL);
        int64_t I2; i128 S2;
        modularity_num(g, C, deg, &I2, &S2);              /* "Compute new modularity" */
        double Q = q_from_num(g->W, I2, S2);
        L->moved[L->trace_len] = moved;
        L->qs[L->trace_len] = Q;
        L->trace_len++;
        int stop = !first && stop_test(cfg->stop_rule, Q, Qp, theta);
        first = 0;
        Qp = Q;
        if (stop || moved == 0) break;
    }
    L->sweeps = s > cfg->max_sweeps ? cfg->max_sweeps : s;
    if (cfg->merge_isolated) {
        og_sweep(g, C, next, 1);
        memcpy(C, next, (size_t)n * sizeof(int32_t));
    }
    free(color); free(next); free(deg);
    return OG_OK;
}

int og_run(const og_graph *g0, const og_config *cfg, og_result **out) {
    *out = NULL;
    if (g0->W <= 0) return OG_EZEROW;
    og_result *r = (og_result *)calloc(1, sizeof(og_result));
    r->lev = (og_level *)calloc((size_t)(cfg->max_levels > 0 ? cfg->max_levels : 1), sizeof(og_level));
    r->n0 = g0->n;
    const og_graph *g = g0;
    og_graph *owned = NULL;
    double mod_curr = 0.0;
    int rc = OG_OK;
    for (int32_t l = 0; l < cfg->max_levels; ++l) {
        double theta = cfg->theta;
        if (cfg->theta_schedule && cfg->theta_schedule_len > 0)      /* D21 */
            theta = cfg->theta_schedule[l % cfg->theta_schedule_len];
        og_level L;
        memset(&L, 0, sizeof(L));
        L.n = g->n;
        int32_t *C = (int32_t *)malloc((size_t)g->n * sizeof(int32_t));
        rc = one_level(g, cfg, theta, C, &L, &r->edge_visits);
        if (rc) { free(C); free(L.moved); free(L.qs); break; }
        int64_t k = og_renumber(g->n, C, C);
        int64_t I2, S2h; uint64_t S2l; double Ql;
        og_modularity(g, C, &I2, &S2h, &S2l, &Ql);       /* "modularity is recomputed" (D15) */
        L.labels = C;
        L.q = Ql;
        if (l == 0 || !(Ql - mod_curr < cfg->big_theta)) {   /* Alg. 2 (D17) */
            r->lev[r->nlev++] = L;
            mod_curr = Ql;
        } else {
            free(C); free(L.moved); free(L.qs);
            break;
        }
        if (l + 1 == cfg->max_levels) break;
        og_graph *h = NULL;
        rc = og_induce(g, C, k, &h);                      /* "Compute new input graph" */
        if (rc) { og_graph_free(h); break; }
        og_graph_free(owned);
        owned = h;
        g = h;
    }
    og_graph_free(owned);
    *out = r;
    return rc;
}

void og_result_free(og_result *r) {
    if (!r) return;
    for (int32_t l = 0; l < r->nlev; ++l) { free(r->lev[l].labels); free(r->lev[l].moved); free(r->lev[l].qs); }
    free(r->lev);
    free(r);
}

int32_t og_result_levels(const og_result *r) { return r->nlev; }
int64_t og_result_level_n(const og_result *r, int32_t l) { return r->lev[l].n; }
void og_result_level_labels(const og_result *r, int32_t l, int32_t *out) {
    memcpy(out, r->lev[l].labels, (size_t)r->lev[l].n * sizeof(int32_t));
}
double og_result_level_q(const og_result *r, int32_t l) { return r->lev[l].q; }
int32_t og_result_level_sweeps(const og_result *r, int32_t l) { return r->lev[l].sweeps; }
double og_result_final_q(const og_result *r) { return r->nlev ? r->lev[r->nlev - 1].q : 0.0; }
int32_t og_result_trace_len(const og_result *r, int32_t l) { return r->lev[l].trace_len; }
void og_result_trace(const og_result *r, int32_t l, int64_t *moved, double *q) {
    memcpy(moved, r->lev[l].moved, (size_t)r->lev[l].trace_len * sizeof(int64_t));
    memcpy(q, r->lev[l].qs, (size_t)r->lev[l].trace_len * sizeof(double));
}
int64_t og_result_edge_visits(const og_result *r) { return r->edge_visits; }

/* final partition: p[v] = L_last(…L_1(L_0[v])) (composition of the dendrogram) */
void og_result_final(const og_result *r, int32_t *out) {
    for (int64_t v = 0; v < r->n0; ++v) {
        int32_t c = (int32_t)v;
        for (int32_t l = 0; l < r->nlev; ++l) c = r->lev[l].labels[c];
        out[v] = c;
    }
}
