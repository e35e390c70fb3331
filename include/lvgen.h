/*
 * lvgen.h — seeded synthetic-graph generators and text loaders (C ABI).
 *
 * This module produces INPUTS only (undirected COO records).  It holds none of the
 * Louvain method's arithmetic and is the one piece of code that both the CUDA path
 * (through its callers: tests, bench.py) and the CPU oracle's tests consume
 * (DESIGN.md §4 "input recipe").  Every generator is counter-based (Philox4x32-10,
 * keyed by (seed, stream)), so its output bytes are independent of thread count.
 *
 * Output convention: records (src[k], dst[k], w[k]) of an undirected graph on
 * vertices [0,n).  Loops (u==u) may appear; duplicate unordered pairs may appear
 * unless stated (the library sums them, paper P:L43 "multiple edges ... should not be
 * present" -> reading D25).  w == NULL in a signature means "unweighted" (weight 1,
 * reading D1).  All buffers are caller-owned host memory.  Functions return 0 on
 * success, nonzero on bad arguments.
 */
#ifndef LVGEN_H
#define LVGEN_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* Philox4x32-10 block: out[0..3] = Philox(key = (k0,k1), counter = (c0,c1,c2,c3)). */
void lvgen_philox(uint32_t k0, uint32_t k1, uint32_t c0, uint32_t c1, uint32_t c2,
                  uint32_t c3, uint32_t out[4]);

/* Zachary karate club, 34 vertices, 78 unit edges, networkx vertex order (C1). */
int lvgen_karate(int32_t *src, int32_t *dst);   /* 78 records */

/* Ring of k cliques of c vertices: n = k*c, m = k*c*(c-1)/2 + k. */
int64_t lvgen_ring_of_cliques_m(int32_t k, int32_t c);
int lvgen_ring_of_cliques(int32_t k, int32_t c, int32_t *src, int32_t *dst);

/* Planted-partition SBM (C2): n vertices in `blocks` equal blocks, m = n*avg_deg/2
 * distinct non-loop unit edges, a fraction mu of them between blocks; ids permuted by
 * a seeded permutation; truth[v] = planted block of (permuted) vertex v. */
int lvgen_sbm(int64_t n, int64_t blocks, int64_t avg_deg, double mu, uint64_t seed,
              int32_t *src, int32_t *dst, int32_t *truth);

/* Collaboration-Spotting-shaped co-occurrence graph (C3).  n = topics*topic_size
 * entities; `docs` documents, each with a uniform topic and size
 * min(1+Zipf(zipf_s), max_size); each member is drawn from the document's topic with
 * probability p_in (else from a uniform topic) with within-topic popularity
 * proportional to (rank+1)^-pop_exp; every unordered pair of distinct members of a
 * document is one unit record (duplicates across documents sum to co-occurrence
 * counts).  Two calls: _count returns the number of records, _fill writes them. */
int64_t lvgen_cooc_count(int64_t topics, int64_t topic_size, int64_t docs, double zipf_s,
                         int32_t max_size, double p_in, double pop_exp, uint64_t seed);
int lvgen_cooc_fill(int64_t topics, int64_t topic_size, int64_t docs, double zipf_s,
                    int32_t max_size, double p_in, double pop_exp, uint64_t seed,
                    int32_t *src, int32_t *dst);

/* Graph500-style R-MAT (C4/C5): m = edge_factor * 2^scale draws with quadrant
 * probabilities (a,b,c,1-a-b-c), no noise; weight per draw uniform in {1..wmax}
 * (wmax == 0 -> unweighted, w may be NULL); ids permuted by a seeded permutation. */
int lvgen_rmat(int32_t scale, int64_t edge_factor, double a, double b, double c,
               int32_t wmax, uint64_t seed, int32_t *src, int32_t *dst, int32_t *w);

/* Seeded permutation of [0,n) (Fisher-Yates over Philox draws). */
int lvgen_permutation(int64_t n, uint64_t seed, uint32_t stream, int32_t *perm);

/* Threads used by the OpenMP loops (0 = runtime default). */
void lvgen_set_threads(int32_t t);

#ifdef __cplusplus
}
#endif
#endif
