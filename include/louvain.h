/*
 * louvain.h — C ABI of the B200-native (sm_100a) GPU Louvain hot path.
 *
 * Method: Forster, "Parallel Louvain Community Detection Optimized for GPUs",
 * arXiv 1805.10904 (/root/reference/PAPER.md, cited "P:Lnn").  The library runs
 * Algorithm 2 around Algorithm 1 on one GPU (or one
 * sweep-sharded group of GPUs): the local-move phase (Eq. 1, 2, 4, 5 + the singlet and
 * generalized minimum-label heuristics), the deg_C / size update,
 * the modularity reduction (Eq. 3), the isolated-node merge,
 * renumbering and graph contraction.  Readings of the
 * paper where it is silent or garbled are D1..D27 in DESIGN.md §3; the library and the
 * CPU oracle (oracle/, test-only) implement the same readings independently.
 *
 * Arithmetic (reading D22): all aggregates are exact 64-bit integers and move scores
 * exact 128-bit integers, so partitions are a mathematical function of the input
 * (independent of thread count, schedule and GPU count).  Real (float) weights are mapped
 * to exact fixed point first (reading D28, louvain_weight_scale).
 *
 * Conventions for every function:
 *  - Return value: LV_OK (0) or an error code; nothing throws across the ABI.  After an
 *    error, louvain_last_error(handle) (or louvain_last_error(NULL) for a failed
 *    create) returns a NUL-terminated message owned by the library.
 *  - Pointers flagged `on_device` are CUDA device pointers on the handle's device;
 *    otherwise host pointers.  Input buffers are borrowed only for the duration of the
 *    call; output buffers are caller-owned and must hold `cap` elements.
 *  - All GPU work is ordered on the handle's stream; every call returns after that
 *    stream has been synchronised (results are complete).
 *  - One host thread per handle at a time; distinct handles are independent.
 */
#ifndef LOUVAIN_H
#define LOUVAIN_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LOUVAIN_ABI_VERSION 1

typedef struct louvain_ctx *louvain_t; /* opaque; owns all device memory it allocates */

typedef enum {
    LV_OK = 0,
    LV_EINVAL = 1,  /* bad argument (NULL pointer, bad config value, bad level)       */
    LV_EGRAPH = 2,  /* vertex id outside [0,n), weight <= 0 ("positive weight") */
    LV_EZEROW = 3,  /* W = 0: modularity undefined (Eq. 3 divides by 2W; reading D1)   */
    LV_ENOMEM = 4,  /* device or host allocation failed                                 */
    LV_ECUDA = 5,   /* CUDA runtime error (message in last_error)                       */
    LV_ENCCL = 6,   /* NCCL error in the sharded path                                   */
    LV_ESTATE = 7,  /* call out of order (e.g. get_partition before run)                */
    LV_ERANGE = 8   /* level index out of range                                         */
} louvain_status;

typedef enum {
    LV_W_NONE = 0, /* unweighted: every weight is 1 (reading D1; P:L43 says "0")        */
    LV_W_I32 = 1,  /* int32 weights, each > 0                                           */
    LV_W_I64 = 2,  /* int64 weights, each > 0                                           */
    LV_W_F32 = 3,  /* real weights (P:L247 stores floats), each finite and > 0; mapped to  */
    LV_W_F64 = 4   /* fixed point w~ = rint(w * 2^s), s max with sum w~ <= 2^52 (D28)       */
} louvain_wtype;

/* Undirected graph G(V,E,ω) as COO records, each undirected edge once; loops
 * (i,i) allowed; duplicate unordered pairs are summed (reading D25).  Vertex ids must
 * be dense in [0,n).  Layout: three parallel arrays of length m. */
typedef struct {
    int64_t n;            /* |V| >= 1 (vertices without edges are kept, reading D20)   */
    int64_t m;            /* number of records                                          */
    const int32_t *src;   /* m                                                          */
    const int32_t *dst;   /* m                                                          */
    const void *w;        /* m values of `wtype`, or NULL iff wtype == LV_W_NONE        */
    int32_t wtype;        /* louvain_wtype                                              */
    int32_t on_device;    /* 1: src/dst/w are device pointers; 0: host pointers         */
} louvain_graph;

/* Device-memory hooks (optional).  The Python binding routes them to PyTorch's
 * caching allocator; NULL means cudaMallocAsync/cudaFreeAsync on the handle stream. */
typedef void *(*louvain_alloc_fn)(void *ctx, size_t bytes, void *stream);
typedef void (*louvain_free_fn)(void *ctx, void *ptr, size_t bytes, void *stream);

typedef struct {
    double theta;            /* Alg. 1 θ; default 1e-6 (reading D16)          */
    double big_theta;        /* Alg. 2 Θ; default 1e-6 (reading D16)          */
    int32_t max_sweeps;      /* iteration cap per level (reading D12); default 100     */
    int32_t max_levels;      /* level cap (reading D27); default 64                    */
    int32_t stop_rule;       /* 0: Alg. 1 literal |(Q−Qp)/Qp| < θ; 1: signed (D10)     */
    int32_t merge_isolated;  /* isolated-node merge post-pass (D14); default 1 */
    const double *theta_schedule; /* threshold cycling (D21): level ℓ uses θ_s[ℓ mod L]  */
    int32_t theta_schedule_len;   /* 0: constant θ                                       */
    int32_t device;          /* CUDA device ordinal; default 0                          */
    void *stream;            /* cudaStream_t to run on; NULL = a library-owned stream   */
    louvain_alloc_fn alloc;  /* optional allocator hook (see above)                     */
    louvain_free_fn free;
    void *alloc_ctx;
    void *nccl_comm;         /* ncclComm_t for the sweep-sharded path; NULL = 1 GPU.
                                Every rank then holds the whole (replicated) level graph
                                and state, sweeps its edge-balanced vertex range, and
                                computes its row part of the CSR build and of each
                                contraction; louvain_create and louvain_run are
                                COLLECTIVE over the communicator (every rank calls them with
                                the same graph and configuration, on its own device).  Results
                                equal the 1-GPU run.                                      */
    int32_t rank, world;     /* this process's rank / world size in nccl_comm           */
    int32_t profile;         /* 1: time every sweep kernel with CUDA events during run   */
    int32_t coloring;        /* SURVEY F2, reading D29 (Lu et al.'s colouring heuristic,
                                P:L89 / P:L441 "other heuristics"): 1 = colour each level
                                (distance-1, greedy by fmix64 priority) and sweep the colour
                                classes in turn, each against the state the previous class
                                committed; default 0 (the paper's synchronous sweeps).
                                Not available in the sweep-sharded mode (LV_EINVAL).       */
    int32_t color_classes;   /* D29: colours >= color_classes-1 share the last class
                                (swept synchronously); 0 = one class per colour; default 32 */
    int64_t color_cap_min_n; /* D29: the class cap applies only to level graphs of more than
                                this many vertices (small dense levels keep every colour, so
                                no synchronous class oscillates there); default 65536     */
    int32_t reorder;         /* SURVEY F3 ("divergence ... could be reduced by ordering
                                the vertices by degree"): 1 = relabel the vertices before the
                                CSR build, in decreasing degree class — new id = position in
                                the stable order of key(v) = clz(d(v)) (d(v) = non-loop records
                                incident to v, duplicates counted; d = 0 -> key 32), i.e. by
                                floor(log2 d) descending, ascending old id within a class.  The
                                method then runs on the relabelled graph (the minimum-label
                                rule sees the new ids, so partitions equal the oracle's on the
                                same relabelled graph, not on the original one); partitions
                                of level 0 and of level -1 are returned indexed by the
                                ORIGINAL vertex ids; community ids, levels >= 1 and the
                                step-level entry points (louvain_sweep, louvain_get_csr, ...)
                                use the relabelled ids.  Default 0.                        */
} louvain_config;

/* Fill `cfg` with the defaults above. */
louvain_status louvain_config_default(louvain_config *cfg);

/* Validate G, copy it to the device and build the CSR (§5.1.2 "Neighbor computation",
 * P:L270-271): loops to loop[], mirror non-loop records, merge duplicates, row offsets
 * by prefix sum, δ_i = Σ w + 2·loop_i, W = Σ record weights.
 * Errors: LV_EINVAL (NULL/neg sizes), LV_EGRAPH (bad id / weight), LV_EZEROW (W = 0),
 * LV_ENOMEM, LV_ECUDA.  On error *out is NULL. */
louvain_status louvain_create(const louvain_graph *g, const louvain_config *cfg, louvain_t *out);

/* Run Algorithm 2 to completion (blocking).  May be called again to re-run. */
louvain_status louvain_run(louvain_t h);

/* Fixed-point scale s of a real-weighted graph (LV_W_F32/F64; reading D28, SURVEY §8(f)
 * F1): the library runs on w~ = rint(w * 2^s), the largest s with sum w~ <= 2^52, so
 * every sum and score stays exact; Q is that of the fixed-point graph (within m * 2^-s
 * relative of the real-weight Q).  0 for integer inputs.  Errors: LV_EINVAL.  (Create
 * fails with LV_EGRAPH if a real weight is not finite and > 0, or rounds to 0 at s.) */
louvain_status louvain_weight_scale(louvain_t h, int32_t *s);

/* Number of recorded dendrogram levels (>= 1 after run). */
louvain_status louvain_num_levels(louvain_t h, int32_t *levels);

/* Vertex count of level `level`'s graph (level 0 = n). */
louvain_status louvain_level_size(louvain_t h, int32_t level, int64_t *n);

/* Copy a partition: level in [0, levels) gives that level's dense labels (length
 * n_level, values in [0, n_{level+1})); level = -1 gives the final composed partition of
 * the input vertices (length n).  `cap` = capacity of `out` in elements.
 * Errors: LV_ESTATE before run, LV_ERANGE bad level, LV_EINVAL cap too small. */
louvain_status louvain_get_partition(louvain_t h, int32_t level, int32_t *out, int64_t cap,
                                     int32_t on_device);

/* Modularity (Eq. 3) of a level's partition (level = -1: final). */
louvain_status louvain_modularity(louvain_t h, int32_t level, double *q);

/* Per-level statistics: sweeps run, and times in ms of the paper's processes
 * (P:L267-313): [0] neighbour (CSR build, level 0 only), [1] init, [2] onelevel
 * (all sweeps + commits + merge), [3] renumber, [4] induce.  `times` may be NULL. */
louvain_status louvain_level_stats(louvain_t h, int32_t level, int32_t *sweeps, double *times);

/* directed-edge visits of all local-move sweeps of the last run, and the number of
 * kernel launches the handle issued since louvain_create (CSR build + every run). */
louvain_status louvain_run_stats(louvain_t h, int64_t *edge_visits, int64_t *launches);

/* Colouring heuristic (cfg.coloring, D29) statistics of a recorded level: number of
 * colours of the level graph (before the color_classes cap) and Jones–Plassmann rounds.
 * Both 0 when colouring was off.  Errors: LV_ESTATE before run, LV_ERANGE bad level. */
louvain_status louvain_level_colors(louvain_t h, int32_t level, int32_t *colors, int32_t *rounds);

/* ---- step-level entry points (tests, benchmarks).  Each operates on level 0 of the
 * handle's graph and leaves louvain_run's results untouched. ---- */

/* One local-move sweep (mode 0) or one isolated-merge batch (mode 1) from the snapshot
 * `labels_in` (length n, values in [0,n)): writes the decisions to labels_out and the
 * exact Eq. 3 numerators of the SNAPSHOT state: i2 = Σ_i e_{i→C(i)} + 2Σloop and
 * s2 = Σ_C deg_C² (hi/lo words).  `moved` = #vertices with labels_out != labels_in. */
louvain_status louvain_sweep(louvain_t h, const int32_t *labels_in, int32_t *labels_out,
                             int32_t mode, int32_t on_device, int64_t *moved, int64_t *i2,
                             int64_t *s2_hi, uint64_t *s2_lo);

/* Distance-1 colouring of the level-0 graph (D29): colors[v] (length n, host or device)
 * = the greedy colour in decreasing fmix64(v ^ 0x9E3779B97F4A7C15) order, computed by
 * Jones–Plassmann rounds; *ncolors = number of colours.  Errors: LV_EINVAL. */
louvain_status louvain_color(louvain_t h, int32_t *colors, int32_t on_device, int32_t *ncolors);

/* Time `reps` consecutive level-0 sweeps (each: all bin kernels + commit) from the
 * all-singleton state after `warm` untimed ones, with CUDA events on the handle stream.
 * Writes a NUL-terminated JSON object into `json` (capacity `cap` bytes):
 *   {"ms_sweep": mean ms per sweep, "alg_bytes_sweep": algorithmic bytes per sweep,
 *    "edges": directed edges per sweep, "kernels": [{"name", "ms", "alg_bytes",
 *    "launches"} per kernel, per sweep]}
 * Algorithmic bytes follow DESIGN.md §6.  Errors: LV_EINVAL if cap is too small. */
louvain_status louvain_time_sweeps(louvain_t h, int32_t warm, int32_t reps, char *json, int64_t cap);

/* Per-kernel profile of the last run (requires cfg.profile = 1): NUL-terminated JSON
 *   {"kernels": [{"name", "ms", "alg_bytes", "launches"}], "edge_visits": ...}
 * with total CUDA-event time and algorithmic bytes per kernel name,
 * accumulated over every sweep of every level.  Errors: LV_ESTATE (profiling off or no
 * run), LV_EINVAL (cap too small). */
louvain_status louvain_profile_json(louvain_t h, char *json, int64_t cap);

/* Level-0 CSR as built on the device (for parity tests): row_ptr (n+1), col (nnz),
 * w (nnz, int64), loop (n), delta (n); host buffers, any may be NULL. */
louvain_status louvain_get_csr(louvain_t h, int64_t *nnz, int64_t *row_ptr, int32_t *col,
                               int64_t *w, int64_t *loop, int64_t *delta, int64_t *W);

/* Contract level 0 by a dense partition (labels in [0,k)), like the induce step
 * (P:L306-313), and return the contracted graph's CSR through louvain_get_csr-style
 * host buffers (row_ptr k+1, col/w nnz_out).  Call once with col == NULL to get
 * *nnz_out, then again with buffers.  labels: host, n entries; a label outside [0,k)
 * returns LV_EINVAL before anything is contracted. */
louvain_status louvain_contract(louvain_t h, const int32_t *labels, int64_t k, int64_t *nnz_out,
                                int64_t *row_ptr, int32_t *col, int64_t *w, int64_t *loop,
                                int64_t *delta);

const char *louvain_last_error(louvain_t h);
void louvain_destroy(louvain_t h);

/* NCCL bootstrap helpers for the sweep-sharded path (thin wrappers around NCCL so
 * callers need no NCCL headers): get a unique id (128 bytes) on rank 0, broadcast it
 * out of band, then init on every rank. */
louvain_status louvain_nccl_unique_id(uint8_t id[128]);
louvain_status louvain_nccl_init(const uint8_t id[128], int32_t world, int32_t rank, int32_t device,
                                 void **comm_out);
louvain_status louvain_nccl_destroy(void *comm);

/* Sweep sharding (host helper, no GPU): contiguous edge-balanced vertex ranges of a CSR,
 * bounds[p] = first vertex v with row_ptr[v] >= p*nnz/world (bounds[0] = 0,
 * bounds[world] = n), the same rule the library applies on the device per level.
 * row_ptr: host, n+1 entries; bounds: host, world+1 entries. */
louvain_status louvain_shard_bounds(const int64_t *row_ptr, int64_t n, int32_t world, int64_t *bounds);

#ifdef __cplusplus
}
#endif
#endif
