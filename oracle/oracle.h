/*
 * oracle.h — plain, slow, single-threaded CPU oracle for the GPU Louvain hot path of
 * Forster, "Parallel Louvain Community Detection Optimized for GPUs" (arXiv 1805.10904).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_1805_10904_b200/) never imports, links or executes anything under oracle/,
 * and shares no code, header, table or helper with it.
 *
 * Citations: "P:Lnn" = /root/reference/PAPER.md line nn; readings D1..D27 are the
 * resolutions listed in DESIGN.md §3 (taken from SURVEY.md §8(c)).
 *
 * Every function follows the paper's definitions / algorithms step by step:
 *   og_graph_build   — §2 graph model + §5.1.2 "Neighbor computation"
 *   og_modularity    — Eq. 3
 *   og_decide        — Eq. 1, 2, 4, 5 + §3.1.1/§3.1.2 heuristics
 *   og_sweep         — Algorithm 1 inner "for each i in V_k in parallel"
 *   og_merge_pass    — isolated-node merge
 *   og_renumber      — "Renumbering nodes"
 *   og_induce        — graph rebuilding / "Inducing new graph"
 *   og_run           — Algorithm 2 around Algorithm 1
 *
 * Integer weights only (all five BASELINE configs are integer-weighted).  All
 * aggregates are exact int64; move scores are exact int128 (reading D4, D22).
 */
#ifndef LOUVAIN_ORACLE_H
#define LOUVAIN_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int64_t  n;        /* vertices                                        */
    int64_t  nnz;      /* directed non-loop adjacency entries             */
    int64_t *row_ptr;  /* n+1                                             */
    int32_t *col;      /* nnz, sorted ascending within each row           */
    int64_t *w;        /* nnz                                             */
    int64_t *loop;     /* n   : loop weight ω(i,i) (D2)                   */
    int64_t *delta;    /* n   : δ_i = Σ_adj w + 2·loop_i (D2)             */
    int64_t  W;        /* Σ of undirected edge weights, loops once (D3)  */
} og_graph;

typedef struct {
    double  theta;            /* Alg. 1 θ; D16 default 1e-6          */
    double  big_theta;        /* Alg. 2 Θ; D16 default 1e-6          */
    int32_t max_sweeps;       /* D12 default 100                              */
    int32_t max_levels;       /* D27 default 64                               */
    int32_t stop_rule;        /* D10: 0 = Alg.1 |ΔQ/Qp|<θ, 1 = signed         */
    int32_t merge_isolated;   /* D14 default 1                                */
    const double *theta_schedule; /* D21 threshold cycling; NULL = constant θ */
    int32_t theta_schedule_len;
    int32_t coloring;         /* F2 / D29: 1 = sweep colour classes in turn         */
    int32_t color_classes;    /* D29: classes = min(colour, color_classes-1); 0 = all */
    int64_t color_cap_min_n;  /* D29: the cap applies to level graphs of > this many vertices */
} og_config;

/* error codes (0 = ok) */
enum { OG_OK = 0, OG_EINVAL = 1, OG_EGRAPH = 2, OG_EZEROW = 3, OG_ENOMEM = 4 };

/* §2 / "Neighbor computation": undirected records (src[k],dst[k],w[k]); loops allowed;
 * duplicate unordered pairs are summed (D25).  w == NULL means every weight is 1 (D1). */
int  og_graph_build(int64_t n, int64_t m, const int32_t *src, const int32_t *dst,
                    const int64_t *w, og_graph **out);
void og_graph_free(og_graph *g);

/* SURVEY §8(f) F1, reading D28: real weights ω (the paper stores float
 * weights; any finite ω > 0, given here as binary64 — binary32 inputs convert
 * exactly) are mapped to the fixed-point integers
 *     ω~_k = rint(ω_k · 2^s)     (round half to even; ω·2^s is exact in binary64)
 * with s the LARGEST integer such that Σ_k ω~_k <= 2^52 (so W~ <= 2^52 and every
 * aggregate is an exact integer, also exactly representable in fp64).  The graph of the
 * ω~ then runs the integer method unchanged.  Returns OG_EGRAPH if an ω is not finite or
 * <= 0, or if some ω~_k = 0 at that s (dynamic range beyond 52 bits); *s_out = s. */
int  og_graph_build_real(int64_t n, int64_t m, const int32_t *src, const int32_t *dst,
                         const double *w, int32_t *s_out, og_graph **out);
/* T(s) = Σ_k rint(ω_k · 2^s) as an exact integer, saturated at 2^62 (helper of the above;
 * exported for the pins). */
int64_t og_fixed_sum(int64_t m, const double *w, int32_t s);

/* Eq. 3 on partition `labels` (any int32 labels in [0,n)).  Outputs the exact
 * numerators I2 = Σ_i e_{i→C(i)} + 2Σloop, S2 = Σ_C deg_C² (as hi/lo words) and
 * Q = d(2W·I2 − S2) / d(4W²) (D22, D24). */
int  og_modularity(const og_graph *g, const int32_t *labels, int64_t *I2,
                   int64_t *S2_hi, uint64_t *S2_lo, double *Q);

/* Community state derived from a label vector: deg[c] (Eq. 2) and size[c]. */
typedef struct og_state og_state;
og_state *og_state_new(const og_graph *g, const int32_t *labels);
void      og_state_free(og_state *st);
/* Decision of one vertex against the snapshot `st` (Eq. 5 + heuristics).
 * mode 0 = local-move decision, mode 1 = isolated-merge decision. */
int32_t   og_decide(og_state *st, int64_t i, int32_t mode);   /* -1: out of memory */

/* One Jacobi sweep (mode 0) or one merge batch (mode 1) over all vertices from the
 * snapshot labels_in; writes labels_out; returns the number of vertices that moved. */
int64_t og_sweep(const og_graph *g, const int32_t *labels_in, int32_t *labels_out, int32_t mode);

/* SURVEY §8(f) F2, reading D29 — Lu et al.'s distance-1 colouring heuristic (the
 * "other heuristics" of P:L89 / P:L441).
 * og_color_priority: π(v) = fmix64(v XOR 0x9E3779B97F4A7C15) (MurmurHash3 finaliser, a
 *   bijection on 64-bit words, so priorities are distinct).
 * og_color: greedy colouring in order of decreasing π: colour(v) = the smallest c >= 0
 *   not used by an already coloured neighbour (loops ignored) — the colouring Jones-
 *   Plassmann rounds produce with these priorities.  Returns the number of colours.
 * og_sweep_colored: one sweep = the colour classes 0..K-1 in turn; the vertices of a
 *   class decide in parallel (og_decide, Jacobi within the class — no two of them are
 *   adjacent) against the state left by the previous class, whose moves are committed
 *   before the next class starts.  Returns the number of vertices that moved. */
uint64_t og_color_priority(int64_t v);
int32_t  og_color(const og_graph *g, int32_t *color);
int64_t  og_sweep_colored(const og_graph *g, const int32_t *color, int32_t ncolors,
                          const int32_t *labels_in, int32_t *labels_out);

/* Order-preserving dense renumbering (D18).  Returns k. */
int64_t og_renumber(int64_t n, const int32_t *labels_in, int32_t *labels_out);

/* Graph rebuilding (D19).  labels dense in [0,k). */
int  og_induce(const og_graph *g, const int32_t *labels, int64_t k, og_graph **out);

/* Algorithm 2 around Algorithm 1. */
typedef struct og_result og_result;
int  og_run(const og_graph *g, const og_config *cfg, og_result **out);
void og_result_free(og_result *r);
int32_t og_result_levels(const og_result *r);
int64_t og_result_level_n(const og_result *r, int32_t l);
void    og_result_level_labels(const og_result *r, int32_t l, int32_t *out);
double  og_result_level_q(const og_result *r, int32_t l);
int32_t og_result_level_sweeps(const og_result *r, int32_t l);
void    og_result_final(const og_result *r, int32_t *out);
double  og_result_final_q(const og_result *r);
/* per-sweep trace of level l: moved count and Q after each committed sweep */
int32_t og_result_trace_len(const og_result *r, int32_t l);
void    og_result_trace(const og_result *r, int32_t l, int64_t *moved, double *q);
/* total directed-edge visits in local-move sweeps (for the cpu_baseline rate) */
int64_t og_result_edge_visits(const og_result *r);

void og_config_default(og_config *cfg);

/* OpenMP threads of the schedule-independent loops (see oracle.c's header); 1 = the
 * single-threaded oracle.  Results do not depend on it. */
void    og_set_threads(int32_t t);
int32_t og_get_threads(void);

#ifdef __cplusplus
}
#endif
#endif
