// lv_agg.cuh — the hot path: per-row hash aggregation of (key -> Σ weight) with three
// epilogues.
//
//   M_SWEEP : the local-move decision of Algorithm 1.  For vertex i with
//             snapshot label own = C(i): e_{i->C} = Σ_{j∈Γ(i)} ω(i,j) per C = C(j)
//             (Eq. 1, loops excluded as in P:L279), then with deg_C (Eq. 2)
//                 S(C)  = 2W·e_{i->C} − δ_i·deg_C            (C ≠ own)
//                 S_own = 2W·e_{i->own} − δ_i·(deg_own − δ_i)
//             (Eq. 4 scaled by 2W², reading D4), best = argmax by (S desc, label asc)
//             (Eq. 5 + generalized minimum label, D7), move iff
//             S(best) > S_own (D6), singlet rule (D8).  A move is recorded
//             in the next-state deg/size.  It also emits e_{i->own} and deg[i]²
//             for the exact Eq. 3 numerators of the snapshot.
//   M_MERGE : isolated-node merge (D14): a singlet whose neighbours lie in
//             exactly one community T moves to T (singlet rule applies).
//   M_EMIT  : distinct (key, Σw) per row, for duplicate merging in "Neighbor
//             computation" (P:L271 reduce_by_key) and for graph contraction (P:L306-313:
//             sort_by_key + reduce_by_key).  Entries whose key equals the row id are
//             summed separately (intra-community weight -> the meta-vertex loop).
//
// Rows are binned by length (P:L438 motivates grouping by degree): bins of
// G ∈ {4,8,16,32} lanes per row with per-group shared-memory open-addressing tables,
// CTA-per-row bins with shared tables up to 8192 slots, and a hub path for rows longer
// than 4096 (radix-partitioned by a second key hash; see "hub path").  All sums are
// exact integers, so the result is independent of insertion order and schedule.
#pragma once
#include "lv_common.cuh"

namespace lv {

enum { M_SWEEP = 0, M_MERGE = 1, M_EMIT = 2 };
enum { WT_NONE = 0, WT_U32 = 1, WT_U64 = 2 };

struct WNone {
  static constexpr int id = WT_NONE;
  static constexpr int bytes = 0;
  __device__ __forceinline__ static u64 get(const void *, i64) { return 1ull; }
  __device__ __forceinline__ static u64 get(const void *, i64, u64) { return 1ull; }
};
struct WU32 {
  static constexpr int id = WT_U32;
  static constexpr int bytes = 4;
  __device__ __forceinline__ static u64 get(const void *w, i64 e) { return __ldg((const uint32_t *)w + e); }
  __device__ __forceinline__ static u64 get(const void *w, i64 e, u64 pol) { return ld_stream((const uint32_t *)w + e, pol); }
};
struct WU64 {
  static constexpr int id = WT_U64;
  static constexpr int bytes = 8;
  __device__ __forceinline__ static u64 get(const void *w, i64 e) { return __ldg((const u64 *)w + e); }
  __device__ __forceinline__ static u64 get(const void *w, i64 e, u64 pol) { return ld_stream((const u64 *)w + e, pol); }
};

struct Chunk {
  i64 beg, end;
  int32_t h, pad;
};

// Packed per-row header of a bin (built once per level): one 16-byte load per row
// instead of rows[] -> row_ptr[] -> row_ptr[+1].
struct RowHdr {
  i64 beg;
  int32_t r, len;
};

struct AggArgs {
  const i64 *ptr;          // row offsets: row r = [ptr[r], ptr[r+1])
  const RowHdr *hdr;       // headers of this bin's rows (smem bins)
  const int32_t *rows;     // rows of this bin
  i64 nrows;
  const int32_t *keys;     // SWEEP/MERGE: col[] (key = packed entry of col); EMIT: key directly
  const void *w;           // weights (WT)
  const u64 *ldeg;         // SWEEP/MERGE: packed snapshot entry per vertex v (see "packed
                           //   entries" below): lo = C(v) | singlet bit, hi = deg_C(v) (31-bit sat.)
  const uint32_t *cpk;     // per community c: singlet bit | min(deg_c, 2^31-1)
  int32_t *label_next;     // decisions
  const i64 *deg;          // deg_C, indexed by label (snapshot; read when the 31-bit copy saturates)
  i64 *deg_next;           // SWEEP/MERGE: copy of deg receiving this pass's moves
  int32_t *size_next;      //   (P:L291 remove/insert; exact int64 atomics, order-free)
  const i64 *delta;        // δ_i
  i64 twoW;                // 2W
  const i64 *out_base;     // EMIT: output offset of row r (NULL -> ptr)
  int32_t *out_key;        // EMIT outputs (NULL -> count only)
  void *out_w;             // weights of the emitted entries: u64, or uint32 when out_w32
  int out_w32;             // 1: out_w holds uint32 (the destination CSR's weight type)
  int out_wnone;           // 1: the destination CSR is unweighted (weights not written)
  i64 *out_cnt;            // distinct keys ≠ row id
  u64 *out_self;           // Σ w with key == row id (may be NULL)
  u64 *out_sum;            // Σ w over the row (may be NULL)
  u64 *counters;           // SWEEP/MERGE: [0] I2 [1] moved [2] S2 lo [3] S2 hi [4] cand
  const Chunk *chunks;     // hub path: HUB_CHUNK-edge chunks of the hub rows
  int hint;                // bit0: evict_first on streams; bit1: evict_last on gathers
  int coloring;            // 1: a colour-class pass (D29): counters [0] Σ e_own and [2,3]
                           //   Σ 2W·e_best over the MOVED vertices (ΔI2 of the class)
};

__device__ __forceinline__ void store_w(const AggArgs &a, i64 o, u64 v) {
  if (a.out_wnone) return;
  if (a.out_w32) ((uint32_t *)a.out_w)[o] = (uint32_t)v;
  else ((u64 *)a.out_w)[o] = v;
}

// ---- packed entries.  Once per pass every vertex v gets one 8-byte entry
//   ldeg[v] = { lo: C(v) | (|C(v)| == 1) << 31,  hi: min(deg_C(v), 2^31 - 1) }
// so the one gather an edge (i, j) makes yields the candidate community, its deg_C (Eq. 2)
// and its singlet flag — no per-candidate deg/size gathers.  The packed key
// (label | singlet bit) is what the tables hash: it is a bijection of the label within a
// pass, so distinct keys are distinct communities.  Labels are < n <= 2^31 - 1, so no
// packed key equals the empty marker -1 (0xFFFFFFFF).  A saturated deg (2^31 - 1) reads
// the exact 64-bit deg_C instead (at most 2W / 2^31 communities can saturate).
constexpr int32_t EMPTY = -1;
constexpr uint32_t SG_BIT = 0x80000000u;
constexpr uint32_t DEG_SAT = 0x7FFFFFFFu;
__device__ __forceinline__ int32_t key_label(int32_t k) { return k & 0x7FFFFFFF; }
__device__ __forceinline__ int key_sg(int32_t k) { return (int)((uint32_t)k >> 31); }
__device__ __forceinline__ i64 deg_of(const AggArgs &a, uint32_t d31, int32_t label) {
  return d31 != DEG_SAT ? (i64)d31 : __ldg(&a.deg[label]);
}
// deg_C of community c through the 31-bit copy
__device__ __forceinline__ i64 load_deg(const AggArgs &a, int32_t c) {
  return deg_of(a, __ldg(&a.cpk[c]) & DEG_SAT, c);
}
__device__ __forceinline__ u64 ld_entry(const AggArgs &a, int32_t v, u64 pol) {
  return (a.hint & 2) ? (u64)ld_keep((const i64 *)&a.ldeg[v], pol) : __ldg(&a.ldeg[v]);
}

__device__ __forceinline__ unsigned hslot(int32_t k, int lg) {
  return ((uint32_t)k * 0x9E3779B1u) >> (32 - lg);
}

// Exact 64-bit add (mod 2^64) with native 32-bit atomics: sm_100 has no native 64-bit
// shared-memory add (it compiles to a CAS loop, which collapses under the same-key
// contention of later sweeps); the low word's returned old value gives the carry.
__device__ __forceinline__ void add_u64_split(uint32_t q, u64 v) {
  const uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
  const uint32_t old = atom_add_s32(q, lo);
  const uint32_t carry = ((uint32_t)(old + lo) < old) ? 1u : 0u;
  if (hi + carry) red_add_s32(q + 4, hi + carry);
}

// Open-addressing insert into a shared-memory table (keys at shared address kb, values
// at vb) with linear probing; key -1 = empty.  Returns the slot.  VT = table value type:
// uint32_t when the caller has proved every row sum < 2^32 (native 32-bit atomics), else
// u64 (split 32-bit atomics).
template <class VT>
__device__ __forceinline__ unsigned tab_insert(uint32_t kb, uint32_t vb, unsigned mask, int lg, int32_t k, u64 v,
                                               bool *claimed = nullptr) {
  // CAS-first probing: one shared atomic per probe resolves all three cases — the slot is
  // empty (claimed), holds k (found) or holds another key (next slot) — where a load
  // followed by a CAS needed two operations and a nested branch (fewer instructions per
  // probe in the warp-divergent probe loop)
  unsigned h = hslot(k, lg);
  while (true) {
    const int32_t old = cas_s32(kb + 4 * h, EMPTY, k);
    if (old == EMPTY) {
      if (claimed) *claimed = true;
      break;
    }
    if (old == k) break;
    h = (h + 1) & mask;
  }
  if (sizeof(VT) == 4) red_add_s32(vb + 4 * h, (uint32_t)v);
  else add_u64_split(vb + 8 * h, v);
  return h;
}

// ---- exact move scores S = 2W·v − δ·deg (Eq. 4 scaled by 2W², reading D4).  For
// every candidate of row i, 0 <= v = e_{i->C} <= δ_i and 0 <= deg_C <= 2W (likewise
// deg_own − δ_i for S_own), so |S| <= 2W·δ_i: rows with 2W·δ_i < 2^63 score in int64
// (row_s64), the rest in int128 (two 64x64->128 unsigned products).  Both are exact.
__device__ __forceinline__ bool row_s64(i64 twoW, i64 di) {
  return __umul64hi((u64)twoW, (u64)di) == 0 && (i64)((u64)twoW * (u64)di) >= 0;
}
__device__ __forceinline__ i128 move_score(i64 twoW, u64 v, i64 di, i64 dk) {
  const u128 a = ((u128)__umul64hi((u64)twoW, v) << 64) | (u128)((u64)twoW * v);
  const u128 b = ((u128)__umul64hi((u64)di, (u64)dk) << 64) | (u128)((u64)di * (u64)dk);
  return (i128)(a - b);
}

// smallest lg with 2^lg >= 2*d (d >= 1), clamped to [3, LGMAX]
__device__ __forceinline__ int row_lg(i64 d, int lgmax) {
  int lg = 64 - __clzll((unsigned long long)(2 * d - 1));
  lg = lg < 3 ? 3 : lg;
  return lg > lgmax ? lgmax : lg;
}

// Insert the row's edges [beg, end) into a table, U edges per lane per batch so the
// col/w loads and then the entry gathers of a batch are independent and in flight
// together (memory-level parallelism; the atomics would otherwise serialise them).
// SWEEP/MERGE: the key is the neighbour's packed entry; the thread that claims a slot
// records the candidate's deg_C next to the slot's list position (odeg[q]).
template <int G, int U, int MODE, class WT, bool LIST, class VT>
__device__ __forceinline__ void insert_range(const AggArgs &a, int lane, i64 beg, i64 end, int32_t *keys, VT *vals,
                                             unsigned mask, int lg, uint16_t *olist, uint32_t *odeg, int *ocnt) {
  const u64 pf = l2_policy_first(), pl = l2_policy_last();
  const uint32_t kb = saddr(keys), vb = saddr(vals), cb = saddr(ocnt);
  // lane-uniform trip count (every lane of the group runs every batch)
  for (i64 b0 = beg; b0 < end; b0 += (i64)G * U) {
    const i64 e0 = b0 + lane;
    int32_t k[U];
    uint32_t dg[U];
    u64 wv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const i64 e = e0 + (i64)u * G;
      k[u] = EMPTY;
      wv[u] = 0;
      dg[u] = 0;
      if (e < end) {
        if (a.hint & 1) {
          k[u] = ld_stream(&a.keys[e], pf);
          wv[u] = WT::get(a.w, e, pf);
        } else {
          k[u] = __ldg(&a.keys[e]);
          wv[u] = WT::get(a.w, e);
        }
      }
    }
    if (MODE != 2 /* M_EMIT */) {
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (k[u] != EMPTY) {
          const u64 p = ld_entry(a, k[u], pl);
          k[u] = (int32_t)(uint32_t)p;
          dg[u] = (uint32_t)(p >> 32);
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const u64 wsum = wv[u];
      if (k[u] == EMPTY) continue;
      bool claimed = false;
      const unsigned sl = tab_insert<VT>(kb, vb, mask, lg, k[u], wsum, LIST ? &claimed : nullptr);
      if (LIST && claimed) {
        const int q = (int)atom_add_s32(cb, 1);
        olist[q] = (uint16_t)sl;
        if (MODE != 2 && odeg) odeg[q] = dg[u];
      }
    }
  }
}

// ----------------------------------------------------------------- group primitives
// A "group" is the set of G threads that cooperate on one row: a segment of a warp
// (G <= 32) or the whole CTA (G == BLOCK > 32).
template <int G, int BLOCK>
struct Grp {
  unsigned mask;
  int lane;
  __device__ __forceinline__ Grp() {
    lane = threadIdx.x % G;
    if (G >= 32) mask = 0xffffffffu;
    else mask = ((1u << (G & 31)) - 1u) << (((threadIdx.x & 31) / G) * G);
  }
  __device__ __forceinline__ void sync() const {
    if (G <= 32) __syncwarp(mask);
    else __syncthreads();
  }
};

// Sum of v over the lanes of `peers` (this lane's __match_any_sync class within `mask`,
// the lanes executing the call), valid in every lane of the class.  __reduce_add_sync
// with a per-lane (non-uniform) mask compiles to a loop over the classes (one
// WARPSYNC.EXCLUSIVE + REDUX round per distinct key: ~24 rounds for a 32-entry row
// whose keys are mostly distinct — r2 ncu, k_agg_reg<32>: 26 warp instructions per
// edge); here every lane adds into its class leader's word of a per-warp shared buffer
// `wb` (32 words, zero between calls), so the cost is one shared reduction per lane.
// Lanes whose class is a singleton (the common case) skip the buffer when the whole
// warp has no duplicate (lanes with valid = false — padding — do not count).  Exact
// (integer adds).
__device__ __forceinline__ uint32_t class_sum32(unsigned mask, unsigned peers, uint32_t v, uint32_t *wb,
                                                bool valid = true) {
  if (!__any_sync(mask, valid && (peers & (peers - 1u)) != 0u)) return v;  // no class with two lanes
  const int leader = __ffs(peers) - 1;
  const uint32_t a = saddr(wb + leader);
  red_add_s32(a, v);
  __syncwarp(mask);
  const uint32_t t = (uint32_t)lds_i32(a);
  __syncwarp(mask);
  if ((int)(threadIdx.x & 31) == leader) wb[leader] = 0u;
  __syncwarp(mask);
  return t;
}

// Two class sums at once (one vote, one set of warp barriers): wb holds 64 words (the
// second sum uses wb + 32).
__device__ __forceinline__ void class_sum32x2(unsigned mask, unsigned peers, uint32_t &x, uint32_t &y, uint32_t *wb) {
  if (!__any_sync(mask, (peers & (peers - 1u)) != 0u)) return;  // no class with two lanes
  const int leader = __ffs(peers) - 1;
  const uint32_t a0 = saddr(wb + leader), a1 = saddr(wb + 32 + leader);
  red_add_s32(a0, x);
  red_add_s32(a1, y);
  __syncwarp(mask);
  x = (uint32_t)lds_i32(a0);
  y = (uint32_t)lds_i32(a1);
  __syncwarp(mask);
  if ((int)(threadIdx.x & 31) == leader) { wb[leader] = 0u; wb[32 + leader] = 0u; }
  __syncwarp(mask);
}

// Candidate: lexicographic key (S desc, label asc).  c is the packed key (label | singlet
// bit, see "packed entries") so the singlet flag travels with it.  "None" has S = -2^127
// (below every real score, |S| < 2^127) and c = INT32_MAX (no packed key equals it: that
// would be label 2^31 - 1 >= n).  Rows scored in int64 (row_s64) keep S in lo only.
struct Cand {
  i64 hi;
  u64 lo;
  int32_t c;
};

__device__ __forceinline__ Cand cand_none() {
  Cand x;
  x.hi = INT64_MIN; x.lo = 0; x.c = INT32_MAX;
  return x;
}
__device__ __forceinline__ Cand cand_none64() {
  Cand x;
  x.hi = -1; x.lo = (u64)INT64_MIN; x.c = INT32_MAX;
  return x;
}
__device__ __forceinline__ i128 cand_S(const Cand &x) { return (i128)(((u128)(u64)x.hi << 64) | (u128)x.lo); }
__device__ __forceinline__ bool cand_better(const Cand &a, const Cand &b) {
  const i128 sa = cand_S(a), sb = cand_S(b);
  return sa > sb || (sa == sb && key_label(a.c) < key_label(b.c));
}
__device__ __forceinline__ bool cand_better64(const Cand &a, const Cand &b) {
  const i64 sa = (i64)a.lo, sb = (i64)b.lo;
  return sa > sb || (sa == sb && key_label(a.c) < key_label(b.c));
}

// Argmax of the group's candidates; result valid in the group's lane 0 (thread 0 of the
// CTA for block groups).  S64: scores are int64 in lo (hi is made its sign extension).
template <int G, int BLOCK, bool S64>
__device__ __forceinline__ void grp_argmax(const Grp<G, BLOCK> &g, Cand &best) {
  constexpr int W = G < 32 ? G : 32;
#pragma unroll
  for (int o = W / 2; o > 0; o >>= 1) {
    Cand y;
    y.lo = __shfl_xor_sync(g.mask, best.lo, o, W);
    y.c = __shfl_xor_sync(g.mask, best.c, o, W);
    if (S64) {
      y.hi = 0;
      if (cand_better64(y, best)) { best.lo = y.lo; best.c = y.c; }
    } else {
      y.hi = __shfl_xor_sync(g.mask, best.hi, o, W);
      if (cand_better(y, best)) best = y;
    }
  }
  if (G > 32) {
    constexpr int NW = BLOCK / 32;
    __shared__ Cand sc[NW];
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) sc[w] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int i = 1; i < NW; ++i) {
        const Cand y = sc[i];
        if (S64 ? cand_better64(y, best) : cand_better(y, best)) best = y;
      }
    }
    __syncthreads();
  }
  if (S64) best.hi = (i64)best.lo >> 63;
}

// Reduce (sum a, sum b, max m) across the group; result valid in the group's lane 0.
template <int G, int BLOCK>
__device__ __forceinline__ void grp_reduce(const Grp<G, BLOCK> &g, u64 &a, u64 &b, int32_t &m) {
  constexpr int W = G < 32 ? G : 32;
#pragma unroll
  for (int o = W / 2; o > 0; o >>= 1) {
    a += __shfl_xor_sync(g.mask, a, o, W);
    b += __shfl_xor_sync(g.mask, b, o, W);
    m = max(m, __shfl_xor_sync(g.mask, m, o, W));
  }
  if (G > 32) {
    constexpr int NW = BLOCK / 32;
    __shared__ u64 sa[NW], sb[NW];
    __shared__ int32_t sm_[NW];
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) { sa[w] = a; sb[w] = b; sm_[w] = m; }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int i = 1; i < NW; ++i) {
        a += sa[i];
        b += sb[i];
        m = max(m, sm_[i]);
      }
    }
    __syncthreads();
  }
}

// Exclusive scan of v across the group; total returned in `tot` (valid in all lanes).
template <int G, int BLOCK>
__device__ __forceinline__ u64 grp_excl_scan(const Grp<G, BLOCK> &g, u64 v, u64 &tot) {
  constexpr int W = G < 32 ? G : 32;
  const int wl = threadIdx.x % W;
  u64 inc = v;
#pragma unroll
  for (int o = 1; o < W; o <<= 1) {
    u64 t = __shfl_up_sync(g.mask, inc, o, W);
    if (wl >= o) inc += t;
  }
  if (G <= 32) {
    tot = __shfl_sync(g.mask, inc, W - 1, W);
    return inc - v;
  } else {
    constexpr int NW = BLOCK / 32;
    __shared__ u64 ws[NW + 1];
    const int w = threadIdx.x >> 5;
    if (wl == 31) ws[w] = inc;
    __syncthreads();
    if (threadIdx.x == 0) {
      u64 r = 0;
      for (int i = 0; i < NW; ++i) { u64 t = ws[i]; ws[i] = r; r += t; }
      ws[NW] = r;
    }
    __syncthreads();
    u64 pre = ws[w] + inc - v;
    tot = ws[NW];
    __syncthreads();
    return pre;
  }
}

// Per-thread accumulators of the sweep counters, flushed once per CTA-thread at exit.
struct Acc {
  u64 i2 = 0, moved = 0, cand = 0, s2hi = 0, s2lo = 0;
  __device__ __forceinline__ void add_sq(i64 d) {
    u128 sq = (u128)(u64)d * (u64)d;
    add128(s2hi, s2lo, (u64)(sq >> 64), (u64)sq);
  }
  __device__ __forceinline__ void flush(u64 *ctr) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      i2 += __shfl_xor_sync(0xffffffffu, i2, o);
      moved += __shfl_xor_sync(0xffffffffu, moved, o);
      cand += __shfl_xor_sync(0xffffffffu, cand, o);
      u64 h = __shfl_xor_sync(0xffffffffu, s2hi, o), l = __shfl_xor_sync(0xffffffffu, s2lo, o);
      add128(s2hi, s2lo, h, l);
    }
    if ((threadIdx.x & 31) == 0) {
      if (i2) atomicAdd(&ctr[0], i2);
      if (moved) atomicAdd(&ctr[1], moved);
      if (s2hi | s2lo) atomic_add128(&ctr[2], &ctr[3], s2hi, s2lo);
      if (cand) atomicAdd(&ctr[4], cand);
    }
  }
};

// Record a move own -> tgt of vertex r (weighted degree di) in the next-state deg/size
// ("remove ... from the old community ... insert ... into the new").
// The passes normally leave deg_next NULL and apply every move afterwards with
// warp-aggregated atomics (k_apply_moves): a sweep moves millions of vertices into the
// same few large communities, and per-move atomics on those few addresses serialise in L2
// (measured r2: the <= 4-entry bin spent ~0.6 of its 0.8 ms on them).  The direct path
// (deg_next set) remains for callers that want it.
__device__ __forceinline__ void record_move(const AggArgs &a, int32_t own, int32_t tgt, i64 di) {
  if (!a.deg_next) return;
  atomicAdd((u64 *)&a.deg_next[own], (u64)(-di));
  atomicAdd((u64 *)&a.deg_next[tgt], (u64)di);
  atomicSub(&a.size_next[own], 1);
  atomicAdd(&a.size_next[tgt], 1);
}

// ----------------------------------------------------------------- row epilogue
// Per-row scalars the group's lane 0 prefetches before the insertion loop (SWEEP).
struct RowPre {
  i64 dq = 0, dr = 0;  // deg_own, deg_r
};

// Decision of Algorithm 1 for vertex r from its best candidate: move iff
// S(best) > S_own (D6), unless both communities are singlets and best's label is larger
// (singlet rule, D8).  ownk = packed key of r's own community.
template <bool S64>
__device__ __forceinline__ void sweep_decide(const AggArgs &a, Acc &acc, int32_t r, int32_t ownk, i64 di, i64 dq,
                                             i64 dr, const Cand &best, u64 eown) {
  const int32_t own = key_label(ownk);
  bool gain;
  if (S64) {
    const i64 so = (i64)((u64)a.twoW * eown) - (i64)((u64)di * (u64)(dq - di));
    gain = (i64)best.lo > so;
  } else {
    const i128 S_own = (i128)a.twoW * (i128)(i64)eown - (i128)di * ((i128)dq - (i128)di);
    gain = cand_S(best) > S_own;
  }
  int32_t tgt = own;
  if (best.c != INT32_MAX && gain) {
    tgt = key_label(best.c);
    if (key_sg(ownk) && key_sg(best.c) && tgt > own) tgt = own;  // singlet rule (D8)
  }
  a.label_next[r] = tgt;
  if (tgt != own) record_move(a, own, tgt, di);
  acc.moved += (tgt != own);
  if (!a.coloring) {
    acc.i2 += eown;
    acc.add_sq(dr);  // deg of label index r: Σ over all labels gives S2
  } else if (tgt != own) {
    // ΔI2 of a class (D29): a move own -> tgt changes I2 by 2(e_{i->tgt} - e_{i->own})
    // (its non-adjacent classmates add independently).  2W·e_{i->tgt} = S(best) + δ_i·deg_tgt
    // exactly; summed in 128 bits, divided by 2W once on the host.
    acc.i2 += eown;
    const i128 t = (S64 ? (i128)(i64)best.lo : cand_S(best)) + (i128)di * (i128)load_deg(a, tgt);
    add128(acc.s2hi, acc.s2lo, (u64)((u128)t >> 64), (u64)t);
  }
}

// Score candidate (packed key k, e_{i->C} = v, deg_C = dk) into best.
template <bool S64>
__device__ __forceinline__ void cand_push(Cand &best, i64 twoW, i64 di, int32_t k, u64 v, i64 dk) {
  if (S64) {  // branch-free select (bitwise, no short-circuit): no reconvergence per candidate
    const i64 sc = (i64)((u64)twoW * v) - (i64)((u64)di * (u64)dk);
    const i64 sb = (i64)best.lo;
    const bool bt = (sc > sb) | ((sc == sb) & (key_label(k) < key_label(best.c)));
    best.lo = bt ? (u64)sc : best.lo;
    best.c = bt ? k : best.c;
  } else {
    const i128 S = move_score(twoW, v, di, dk);
    Cand x;
    x.hi = (i64)(S >> 64); x.lo = (u64)S; x.c = k;
    if (cand_better(x, best)) best = x;
  }
}

// Isolated-node merge (D14) for a singlet r: cnt distinct neighbouring
// communities, T the largest label among them, nsg how many of them are singlets.
__device__ __forceinline__ void merge_decide(const AggArgs &a, Acc &acc, int32_t r, int32_t ownk, u64 cnt, int32_t T,
                                             u64 nsg) {
  const int32_t own = key_label(ownk);
  int32_t tgt = own;
  if (key_sg(ownk) && cnt == 1) tgt = (nsg && T > own) ? own : T;
  a.label_next[r] = tgt;
  if (tgt != own) record_move(a, own, tgt, a.delta[r]);
  acc.moved += (tgt != own);
}

// Visits the row's occupied entries — by scanning slots [0,n) (LIST = false) or through
// the occupied-slot list olist[0..n) (LIST = true) — resets every slot it reads, and
// applies the mode's epilogue.  Both EMIT passes visit entries in the same order.
// SWEEP/MERGE: own = packed key of r's community; with LIST, odeg[t] is the deg_C of the
// entry at list position t (else it is read from cpk).
// SWEEP epilogue of one row: score every entry, argmax over the group, decide.  The lane
// that meets r's own community stores e_{i->own} in the group's slot *eown_s (read and
// cleared by lane 0 after the argmax).
template <bool S64, int G, int BLOCK, bool LIST, class SlotT, class VT>
__device__ __forceinline__ void sweep_epilogue(const Grp<G, BLOCK> &g, int32_t *keys, VT *vals, const SlotT *olist,
                                               const uint32_t *odeg, i64 n, int32_t r, int32_t own, i64 di,
                                               const RowPre &pre, const AggArgs &a, Acc &acc, u64 *eown_s) {
  constexpr int U = G < 32 ? 2 : 4;  // entries per lane per batch
  Cand best = S64 ? cand_none64() : cand_none();
  u64 ncand = 0;
  for (i64 t0 = g.lane; t0 < n; t0 += (i64)G * U) {
    int32_t sl[U], k[U];
    uint32_t d31[U];
    u64 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const i64 t = t0 + (i64)u * G;
      sl[u] = t < n ? (LIST ? (int32_t)olist[t] : (int32_t)t) : -1;
      d31[u] = (odeg && t < n) ? odeg[t] : 0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      k[u] = sl[u] >= 0 ? keys[sl[u]] : EMPTY;
      v[u] = 0;
      if (k[u] != EMPTY) {
        v[u] = (u64)vals[sl[u]];
        keys[sl[u]] = EMPTY;
        vals[sl[u]] = 0;
        if (!odeg) d31[u] = __ldg(&a.cpk[key_label(k[u])]) & DEG_SAT;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (k[u] == EMPTY) continue;
      if (k[u] == own) {
        *eown_s = v[u];
      } else {
        ++ncand;
        cand_push<S64>(best, a.twoW, di, k[u], v[u], deg_of(a, d31[u], key_label(k[u])));
      }
    }
  }
  acc.cand += ncand;
  if (G <= 32) {
    grp_argmax<G, BLOCK, S64>(g, best);
    g.sync();  // *eown_s visible to lane 0
    if (g.lane == 0) {
      const u64 eown = *eown_s;
      *eown_s = 0;
      sweep_decide<S64>(a, acc, r, own, di, pre.dq, pre.dr, best, eown);
    }
  } else {
    // CTA group (the two-barrier row protocol of k_agg_smem): warp argmax, ONE barrier,
    // thread 0 combines the warps' candidates and decides while the CTA moves on
    Grp<32, BLOCK> wg;
    grp_argmax<32, BLOCK, S64>(wg, best);
    constexpr int NW = BLOCK / 32;
    __shared__ Cand sc[NW];
    if ((threadIdx.x & 31) == 0) sc[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int i = 1; i < NW; ++i) {
        const Cand y = sc[i];
        if (S64 ? cand_better64(y, best) : cand_better(y, best)) best = y;
      }
      if (S64) best.hi = (i64)best.lo >> 63;
      const u64 eown = *eown_s;
      *eown_s = 0;
      sweep_decide<S64>(a, acc, r, own, di, pre.dq, pre.dr, best, eown);
    }
  }
}

// Visits the row's occupied entries — by scanning slots [0,n) (LIST = false) or through
// the occupied-slot list olist[0..n) (LIST = true) — resets every slot it reads, and
// applies the mode's epilogue.  Both EMIT passes visit entries in the same order.
// SWEEP/MERGE: own = packed key of r's community; odeg[t] (if not NULL) is the deg_C of
// the entry at list position t (else it is read from cpk).
template <int G, int BLOCK, int MODE, bool LIST, class SlotT, class VT>
__device__ __forceinline__ void row_epilogue(const Grp<G, BLOCK> &g, int32_t *keys, VT *vals, const SlotT *olist,
                                             const uint32_t *odeg, i64 n, int32_t r, int32_t own, i64 di,
                                             const RowPre &pre, const AggArgs &a, Acc &acc, u64 *eown_s) {
  if (MODE == M_SWEEP) {
    if (row_s64(a.twoW, di)) sweep_epilogue<true, G, BLOCK, LIST>(g, keys, vals, olist, odeg, n, r, own, di, pre, a, acc, eown_s);
    else sweep_epilogue<false, G, BLOCK, LIST>(g, keys, vals, olist, odeg, n, r, own, di, pre, a, acc, eown_s);
  } else if (MODE == M_MERGE) {
    u64 cnt = 0, nsg = 0;
    int32_t T = -1;
    for (i64 t = g.lane; t < n; t += G) {
      const int32_t sl = LIST ? (int32_t)olist[t] : (int32_t)t;
      const int32_t k = keys[sl];
      if (k != EMPTY) {
        keys[sl] = EMPTY;
        vals[sl] = 0;
        if (k != own) { ++cnt; T = max(T, key_label(k)); nsg += key_sg(k); }
      }
    }
    grp_reduce<G, BLOCK>(g, cnt, nsg, T);
    if (g.lane == 0) merge_decide(a, acc, r, own, cnt, T, nsg);
  } else {  // M_EMIT
    u64 c = 0, selfw = 0, sumw = 0;
    for (i64 t = g.lane; t < n; t += G) {
      const int32_t sl = LIST ? (int32_t)olist[t] : (int32_t)t;
      const int32_t k = keys[sl];
      if (k != EMPTY) {
        const u64 v = (u64)vals[sl];
        sumw += v;
        if (k == r) selfw += v;
        else ++c;
      }
    }
    u64 tot;
    const u64 pre_ = grp_excl_scan<G, BLOCK>(g, c, tot);
    i64 o = (a.out_base ? a.out_base[r] : a.ptr[r]) + (i64)pre_;
    for (i64 t = g.lane; t < n; t += G) {
      const int32_t sl = LIST ? (int32_t)olist[t] : (int32_t)t;
      const int32_t k = keys[sl];
      if (k != EMPTY) {
        const u64 v = (u64)vals[sl];
        keys[sl] = EMPTY;
        vals[sl] = 0;
        if (k != r && a.out_key) {
          a.out_key[o] = k;
          store_w(a, o, v);
          ++o;
        }
      }
    }
    int32_t dummy = 0;
    grp_reduce<G, BLOCK>(g, selfw, sumw, dummy);
    if (g.lane == 0) {
      a.out_cnt[r] = (i64)tot;
      if (a.out_self) a.out_self[r] = selfw;
      if (a.out_sum) a.out_sum[r] = sumw;
    }
  }
}

// ----------------------------------------------------------------- shared-memory bins
// Tables of CAP >= 256 slots keep an occupied-slot list (uint16 indices) so the
// epilogue costs O(distinct keys), not O(capacity).
template <int CAP>
constexpr bool has_list() { return CAP >= 256; }
// Per group: CAP values, CAP keys, and with a list CAP/2 slot indices (a row of <= CAP/2
// entries) plus, in SWEEP/MERGE, CAP/2 candidate degrees.
// (the degree list is dropped — deg_C read from cpk — when it would not fit: u64 tables
// of the largest bin)
template <int G, int CAP, int BLOCK, class VT, int MODE>
constexpr bool has_deg_list() {
  return has_list<CAP>() && MODE != M_EMIT &&
         (size_t)(BLOCK / G) * ((size_t)CAP * (sizeof(VT) + sizeof(int32_t) + 3) + 16) <= (size_t)220 * 1024;
}
template <int G, int CAP, int BLOCK, class VT, int MODE>
constexpr size_t smem_bytes() {
  return (size_t)(BLOCK / G) * ((size_t)CAP * (sizeof(VT) + sizeof(int32_t)) + (has_list<CAP>() ? CAP : 0) +
                                (has_deg_list<G, CAP, BLOCK, VT, MODE>() ? (size_t)CAP * 2 : 0) + 16);
}

template <int G, int CAP, int BLOCK, int MODE, class WT, class VT>
__global__ void __launch_bounds__(BLOCK) k_agg_smem(AggArgs a) {
  constexpr int GPB = BLOCK / G;
  constexpr bool LIST = has_list<CAP>();
  constexpr bool DEGL = has_deg_list<G, CAP, BLOCK, VT, MODE>();
  constexpr int LG = (CAP >= 65536) ? 16 : (CAP >= 32768) ? 15 : (CAP >= 16384) ? 14 : (CAP >= 8192) ? 13
                   : (CAP >= 4096) ? 12 : (CAP >= 2048) ? 11 : (CAP >= 1024) ? 10 : (CAP >= 512) ? 9
                   : (CAP >= 256) ? 8 : (CAP >= 128) ? 7 : (CAP >= 64) ? 6 : (CAP >= 32) ? 5
                   : (CAP >= 16) ? 4 : 3;
  static_assert((1 << LG) == CAP, "CAP must be a power of two >= 8");
  extern __shared__ __align__(16) unsigned char sm[];
  constexpr size_t SB = sizeof(VT) + sizeof(int32_t);
  VT *svals = (VT *)sm;
  int32_t *skeys = (int32_t *)(sm + (size_t)GPB * CAP * sizeof(VT));
  uint32_t *sdeg = (uint32_t *)(sm + (size_t)GPB * CAP * SB);
  uint16_t *slist = (uint16_t *)(sm + (size_t)GPB * CAP * SB + (DEGL ? (size_t)GPB * CAP * 2 : 0));
  // per group 16 B: [0] occupied count (int), [8] e_{i->own} slot (u64)
  unsigned char *srec = (unsigned char *)slist + (LIST ? (size_t)GPB * CAP : 0);
  Grp<G, BLOCK> g;
  const int grp = threadIdx.x / G;
  int32_t *keys = skeys + grp * CAP;
  VT *vals = svals + grp * CAP;
  uint16_t *olist = slist + grp * (CAP / 2);
  uint32_t *odeg = DEGL ? sdeg + grp * (CAP / 2) : nullptr;
  int *ocnt2 = (int *)(srec + 16 * grp);  // two occupied counters, alternating per row
  u64 *eown_s = (u64 *)(srec + 16 * grp + 8);
  Acc acc;
  for (int s = g.lane; s < CAP; s += G) { keys[s] = EMPTY; vals[s] = 0; }
  if (g.lane == 0) { ocnt2[0] = 0; ocnt2[1] = 0; *eown_s = 0; }
  g.sync();
  // CTA groups sweep a row with two barriers: S1 after the inserts, S2 inside the
  // epilogue (before thread 0 decides).  Slots are reset by their readers before S2, and
  // the occupied counter alternates so the next row's is cleared (after S1) without one.
  constexpr bool TWO_BAR = G > 32 && MODE == M_SWEEP;
  int par = 0;
  const i64 stride = (i64)gridDim.x * GPB;
  i64 idx = (i64)blockIdx.x * GPB + grp;
  RowHdr nh;  // next row's header, prefetched one iteration ahead
  nh.beg = 0; nh.r = 0; nh.len = 0;
  if (idx < a.nrows) nh = a.hdr[idx];
  for (; idx < a.nrows; idx += stride) {
    const RowHdr hd = nh;
    if (idx + stride < a.nrows) nh = a.hdr[idx + stride];
    const int32_t r = hd.r;
    const i64 beg = hd.beg, end = hd.beg + hd.len;
    u64 pr = 0;  // r's own packed entry
    if (MODE != M_EMIT) pr = __ldg(&a.ldeg[r]);
    const int32_t own = (MODE == M_EMIT) ? r : (int32_t)(uint32_t)pr;
    const i64 di = (MODE == M_SWEEP) ? a.delta[r] : 0;
    RowPre pre;
    if (MODE == M_SWEEP && g.lane == 0) {  // issued before the edge loop: overlaps it
      pre.dq = deg_of(a, (uint32_t)(pr >> 32), key_label(own));
      pre.dr = load_deg(a, r);
    }
    if (MODE == M_MERGE) {
      if (!key_sg(own)) {
        if (g.lane == 0) a.label_next[r] = key_label(own);
        continue;
      }
    }
    const int lg = row_lg(end - beg, LG);  // table prefix sized for this row
    const unsigned mask = (1u << lg) - 1u;
    int *ocnt = ocnt2 + par;
    insert_range<G, (G >= 64 ? 8 : (G == 32 ? 4 : 1)), MODE, WT, LIST, VT>(a, g.lane, beg, end, keys, vals, mask, lg,
                                                                          olist, odeg, ocnt);
    g.sync();
    const i64 n = LIST ? (i64)(*(volatile int *)ocnt) : ((i64)1 << lg);
    if (TWO_BAR) {
      if (g.lane == 0) ocnt2[par ^ 1] = 0;
      row_epilogue<G, BLOCK, MODE, LIST>(g, keys, vals, olist, odeg, n, r, own, di, pre, a, acc, eown_s);
      par ^= 1;
    } else {
      row_epilogue<G, BLOCK, MODE, LIST>(g, keys, vals, olist, odeg, n, r, own, di, pre, a, acc, eown_s);
      g.sync();
      if (LIST && g.lane == 0) *ocnt = 0;
      g.sync();
    }
  }
  if (MODE != M_EMIT) acc.flush(a.counters);
}

// ----------------------------------------------------------------- register bins
// Rows of length <= G <= 32: one edge per lane, no shared memory.  Lanes holding the same
// key are found with __match_any_sync and their weights summed (__reduce_add_sync when the
// row sum fits 32 bits, else an exact shuffle loop); the first lane of each key group
// stands for that candidate community.
#ifndef LV_REG_MINB
#define LV_REG_MINB 6  // CTAs of 256 per SM the register bins are compiled for (<= 42 regs)
#endif
template <int G, int BLOCK, int MODE, class WT, bool NARROW>
__global__ void __launch_bounds__(BLOCK, LV_REG_MINB) k_agg_reg(AggArgs a) {
  constexpr int GPB = BLOCK / G;
  Grp<G, BLOCK> g;
  const int grp = threadIdx.x / G;
  const int wl = threadIdx.x & 31;
  Acc acc;
  __shared__ uint32_t segbuf[BLOCK / 32][32];  // class_sum32 buffers (one per warp)
  segbuf[threadIdx.x >> 5][wl] = 0u;
  __syncwarp();
  const u64 pf = l2_policy_first();
  const i64 stride = (i64)gridDim.x * GPB;
  i64 idx = (i64)blockIdx.x * GPB + grp;
  RowHdr nh;
  nh.beg = 0; nh.r = 0; nh.len = 0;
  if (idx < a.nrows) nh = a.hdr[idx];
  for (; idx < a.nrows; idx += stride) {
    const RowHdr hd = nh;
    if (idx + stride < a.nrows) nh = a.hdr[idx + stride];
    const int32_t r = hd.r;
    u64 pr = 0;  // r's own packed entry
    if (MODE != M_EMIT) pr = __ldg(&a.ldeg[r]);
    const int32_t own = (MODE == M_EMIT) ? r : (int32_t)(uint32_t)pr;
    i64 di = 0, dq = 0, dr = 0;
    if (MODE == M_SWEEP) {
      di = a.delta[r];
      if (g.lane == 0) {
        dq = deg_of(a, (uint32_t)(pr >> 32), key_label(own));
        dr = load_deg(a, r);
      }
    }
    if (MODE == M_MERGE) {
      if (!key_sg(own)) {
        if (g.lane == 0) a.label_next[r] = key_label(own);
        continue;
      }
    }
    int32_t k = EMPTY;
    uint32_t d31 = 0;
    u64 w = 0;
    if (g.lane < hd.len) {
      const i64 e = hd.beg + g.lane;
      if (a.hint & 1) {
        k = ld_stream(&a.keys[e], pf);
        w = WT::get(a.w, e, pf);
      } else {
        k = __ldg(&a.keys[e]);
        w = WT::get(a.w, e);
      }
      if (MODE != M_EMIT) {
        const u64 p = __ldg(&a.ldeg[k]);
        k = (int32_t)(uint32_t)p;
        d31 = (uint32_t)(p >> 32);
      }
    }
    bool lead;
    u64 sum;
    if (G <= 8 || !NARROW) {  // small groups: an O(G) shuffle scan beats MATCH.ANY
      constexpr int W = G < 32 ? G : 32;
      sum = 0;
      bool first = true;
      const int gl = g.lane;
#pragma unroll
      for (int j = 0; j < W; ++j) {
        const int32_t kj = __shfl_sync(g.mask, k, j, W);
        const u64 wj = NARROW ? (u64)__shfl_sync(g.mask, (uint32_t)w, j, W) : __shfl_sync(g.mask, w, j, W);
        if (kj == k) {
          sum += wj;
          if (j < gl) first = false;
        }
      }
      lead = first && k != EMPTY;
    } else {
      const unsigned peers = __match_any_sync(g.mask, k);
      lead = (__ffs(peers) - 1) == wl && k != EMPTY;
      sum = class_sum32(g.mask, peers, (uint32_t)w, segbuf[threadIdx.x >> 5], k != EMPTY);
    }
    if (MODE == M_SWEEP) {
      constexpr int W = G < 32 ? G : 32;
      const bool cand = lead && k != own;
      acc.cand += cand;
      // e_{i->own} from the lane leading r's own community (if any)
      const unsigned ob = __ballot_sync(g.mask, lead && k == own) & g.mask;
      const u64 eown = __shfl_sync(g.mask, sum, (__ffs(ob) - 1) & (W - 1), W);
      if (row_s64(a.twoW, di)) {  // group-uniform
        Cand best = cand_none64();
        if (cand) cand_push<true>(best, a.twoW, di, k, sum, deg_of(a, d31, key_label(k)));
        grp_argmax<G, BLOCK, true>(g, best);
        if (g.lane == 0) sweep_decide<true>(a, acc, r, own, di, dq, dr, best, ob ? eown : 0);
      } else {
        Cand best = cand_none();
        if (cand) cand_push<false>(best, a.twoW, di, k, sum, deg_of(a, d31, key_label(k)));
        grp_argmax<G, BLOCK, false>(g, best);
        if (g.lane == 0) sweep_decide<false>(a, acc, r, own, di, dq, dr, best, ob ? eown : 0);
      }
    } else if (MODE == M_MERGE) {
      const bool other = lead && k != own;
      u64 cnt = other ? 1 : 0, nsg = other ? (u64)key_sg(k) : 0;
      int32_t T = other ? key_label(k) : -1;
      grp_reduce<G, BLOCK>(g, cnt, nsg, T);
      if (g.lane == 0) merge_decide(a, acc, r, own, cnt, T, nsg);
    } else {  // M_EMIT: distinct keys != r written compactly at out_base[r]
      const bool emit = lead && k != r;
      const unsigned bal = __ballot_sync(g.mask, emit) & g.mask;
      if (emit && a.out_key) {
        const i64 o = (a.out_base ? a.out_base[r] : a.ptr[r]) + __popc(bal & ((1u << wl) - 1u));
        a.out_key[o] = k;
        store_w(a, o, sum);
      }
      u64 selfw = (lead && k == r) ? sum : 0, sumw = lead ? sum : 0;
      int32_t dummy = 0;
      grp_reduce<G, BLOCK>(g, selfw, sumw, dummy);
      if (g.lane == 0) {
        a.out_cnt[r] = (i64)__popc(bal);
        if (a.out_self) a.out_self[r] = selfw;
        if (a.out_sum) a.out_sum[r] = sumw;
      }
    }
  }
  if (MODE != M_EMIT) acc.flush(a.counters);
}

// SWEEP over rows of length <= G <= 32, software-pipelined: each group keeps four rows
// in flight — the header of row i+3, the edge / own-entry / δ loads of row i+2, the
// entry gather of row i+1 — while it decides row i, so the three dependent global
// round trips of a short row (header -> col -> ldeg[col]) overlap across rows instead
// of adding up.  Same arithmetic as k_agg_reg<M_SWEEP>.
#ifndef LV_REGP_MINB
#define LV_REGP_MINB 4
#endif
struct RegStage {  // per-lane loads of one row (stage B)
  int32_t col;
  uint32_t dr31;   // lane 0: cpk[r] (deg_r for S2)
  u64 w;
  u64 pr;          // r's own packed entry
  i64 di;          // δ_r
};

template <int G, int BLOCK, class WT, bool NARROW>
__global__ void __launch_bounds__(BLOCK, LV_REGP_MINB) k_sweep_reg(AggArgs a) {
  constexpr int GPB = BLOCK / G;
  constexpr int W = G < 32 ? G : 32;
  Grp<G, BLOCK> g;
  const int wl = threadIdx.x & 31;
  Acc acc;
  __shared__ uint32_t segbuf[BLOCK / 32][32];  // class_sum32 buffers (one per warp)
  segbuf[threadIdx.x >> 5][wl] = 0u;
  __syncwarp();
  const u64 pf = l2_policy_first(), pl = l2_policy_last();
  const i64 stride = (i64)gridDim.x * GPB;
  const i64 i0 = (i64)blockIdx.x * GPB + threadIdx.x / G;
  auto hdr_at = [&](i64 i) {
    RowHdr h;
    h.beg = 0; h.r = 0; h.len = 0;
    if (i < a.nrows) h = a.hdr[i];
    return h;
  };
  auto load_stage = [&](const RowHdr &h, RegStage &E) {
    E.col = EMPTY; E.w = 0; E.pr = 0; E.di = 0; E.dr31 = 0;
    if (h.len == 0) return;  // past the end
    if (g.lane < h.len) {
      const i64 e = h.beg + g.lane;
      if (a.hint & 1) {
        E.col = ld_stream(&a.keys[e], pf);
        E.w = WT::get(a.w, e, pf);
      } else {
        E.col = __ldg(&a.keys[e]);
        E.w = WT::get(a.w, e);
      }
    }
    E.pr = __ldg(&a.ldeg[h.r]);
    E.di = __ldg(&a.delta[h.r]);
    if (g.lane == 0) E.dr31 = __ldg(&a.cpk[h.r]) & DEG_SAT;
  };
  RowHdr h0 = hdr_at(i0), h1 = hdr_at(i0 + stride), h2 = hdr_at(i0 + 2 * stride);
  RegStage E0, E1;
  load_stage(h0, E0);
  load_stage(h1, E1);
  u64 p0 = E0.col != EMPTY ? ld_entry(a, E0.col, pl) : 0;
  for (i64 i = i0; i < a.nrows; i += stride) {
    // issue the loads of the rows behind this one
    const RowHdr h3 = hdr_at(i + 3 * stride);
    const u64 p1 = E1.col != EMPTY ? ld_entry(a, E1.col, pl) : 0;
    RegStage E2;
    load_stage(h2, E2);
    // decide row i
    const int32_t r = h0.r;
    const int32_t own = (int32_t)(uint32_t)E0.pr;
    const i64 di = E0.di;
    const int32_t k = E0.col != EMPTY ? (int32_t)(uint32_t)p0 : EMPTY;
    const uint32_t d31 = (uint32_t)(p0 >> 32);
    const u64 w = E0.w;
    bool lead;
    u64 sum;
    if (G <= 8 || !NARROW) {  // small groups: an O(G) shuffle scan beats MATCH.ANY
      sum = 0;
      bool first = true;
#pragma unroll
      for (int j = 0; j < W; ++j) {
        const int32_t kj = __shfl_sync(g.mask, k, j, W);
        const u64 wj = NARROW ? (u64)__shfl_sync(g.mask, (uint32_t)w, j, W) : __shfl_sync(g.mask, w, j, W);
        if (kj == k) {
          sum += wj;
          if (j < g.lane) first = false;
        }
      }
      lead = first && k != EMPTY;
    } else {
      const unsigned peers = __match_any_sync(g.mask, k);
      lead = (__ffs(peers) - 1) == wl && k != EMPTY;
      sum = class_sum32(g.mask, peers, (uint32_t)w, segbuf[threadIdx.x >> 5], k != EMPTY);
    }
    const bool cand = lead && k != own;
    acc.cand += cand;
    const unsigned ob = __ballot_sync(g.mask, lead && k == own) & g.mask;
    const u64 eown = __shfl_sync(g.mask, sum, (__ffs(ob) - 1) & (W - 1), W);
    i64 dq = 0, dr = 0;
    if (g.lane == 0) {
      dq = deg_of(a, (uint32_t)(E0.pr >> 32), key_label(own));
      dr = deg_of(a, E0.dr31, r);
    }
    if (row_s64(a.twoW, di)) {  // group-uniform
      Cand best = cand_none64();
      if (cand) cand_push<true>(best, a.twoW, di, k, sum, deg_of(a, d31, key_label(k)));
      grp_argmax<G, BLOCK, true>(g, best);
      if (g.lane == 0) sweep_decide<true>(a, acc, r, own, di, dq, dr, best, ob ? eown : 0);
    } else {
      Cand best = cand_none();
      if (cand) cand_push<false>(best, a.twoW, di, k, sum, deg_of(a, d31, key_label(k)));
      grp_argmax<G, BLOCK, false>(g, best);
      if (g.lane == 0) sweep_decide<false>(a, acc, r, own, di, dq, dr, best, ob ? eown : 0);
    }
    // advance the pipeline
    h0 = h1; h1 = h2; h2 = h3;
    E0 = E1; E1 = E2;
    p0 = p1;
  }
  acc.flush(a.counters);
}

// ----------------------------------------------------------------- thread per row
// SWEEP for rows of at most L entries (L <= 8): one thread per row.  A 4-lane group per
// 1..4-entry row (k_sweep_reg<4>) keeps only 8 rows of a warp in flight and spends
// shuffles on a handful of items; here a warp has 32 rows' header / stream / entry loads
// in flight and the row's keys are merged in registers.  Same decision as the group
// kernels: candidates are the distinct packed keys != own, scored with the same exact
// integers; argmax by (S desc, label asc) is order-independent.
template <int L, class WT, bool S64>
__device__ __forceinline__ void thr_decide(const AggArgs &a, Acc &acc, const RowHdr &h, u64 pr, i64 di, uint32_t dr31,
                                           const int32_t (&key)[L], const u64 (&wv)[L], const uint32_t (&d31)[L]) {
  const int32_t own = (int32_t)(uint32_t)pr;
  Cand best = S64 ? cand_none64() : cand_none();
  u64 eown = 0;
#pragma unroll
  for (int t = 0; t < L; ++t) {
    if (key[t] == EMPTY) continue;
    if (key[t] == own) {
      eown += wv[t];
      continue;
    }
    ++acc.cand;
    cand_push<S64>(best, a.twoW, di, key[t], wv[t], deg_of(a, d31[t], key_label(key[t])));
  }
  const i64 dq = deg_of(a, (uint32_t)(pr >> 32), key_label(own));
  const i64 dr = deg_of(a, dr31, h.r);
  sweep_decide<S64>(a, acc, h.r, own, di, dq, dr, best, eown);
}

template <int L, class WT>
__global__ void __launch_bounds__(256) k_sweep_thr(AggArgs a) {
  Acc acc;
  const u64 pf = l2_policy_first(), pl = l2_policy_last();
  for (i64 i = (i64)blockIdx.x * 256 + threadIdx.x; i < a.nrows; i += (i64)gridDim.x * 256) {
    const RowHdr h = a.hdr[i];
    int32_t col[L];
    u64 wv[L];
#pragma unroll
    for (int t = 0; t < L; ++t) {
      col[t] = EMPTY;
      wv[t] = 0;
      if (t < h.len) {
        if (a.hint & 1) {
          col[t] = ld_stream(&a.keys[h.beg + t], pf);
          wv[t] = WT::get(a.w, h.beg + t, pf);
        } else {
          col[t] = __ldg(&a.keys[h.beg + t]);
          wv[t] = WT::get(a.w, h.beg + t);
        }
      }
    }
    const u64 pr = __ldg(&a.ldeg[h.r]);
    const i64 di = __ldg(&a.delta[h.r]);
    const uint32_t dr31 = __ldg(&a.cpk[h.r]) & DEG_SAT;
    int32_t key[L];
    uint32_t d31[L];
#pragma unroll
    for (int t = 0; t < L; ++t) {
      const u64 p = col[t] != EMPTY ? ld_entry(a, col[t], pl) : 0;
      key[t] = col[t] != EMPTY ? (int32_t)(uint32_t)p : EMPTY;
      d31[t] = (uint32_t)(p >> 32);
    }
    // merge equal keys into their first occurrence (e_{i->C} per community, Eq. 1)
#pragma unroll
    for (int t = 1; t < L; ++t)
#pragma unroll
      for (int u = 0; u < t; ++u)
        if (key[t] != EMPTY && key[u] == key[t]) {
          wv[u] += wv[t];
          key[t] = EMPTY;
        }
    if (row_s64(a.twoW, di)) thr_decide<L, WT, true>(a, acc, h, pr, di, dr31, key, wv, d31);
    else thr_decide<L, WT, false>(a, acc, h, pr, di, dr31, key, wv, d31);
  }
  acc.flush(a.counters);
}

// ----------------------------------------------------------------- hub path
// Rows longer than the largest shared-memory bin (> 4096 entries).  Instead of one
// global hash table per row (random read-modify-writes over a table far larger than
// L2), a hub row is radix-partitioned by a second hash of the key:
//   k_hub_acc    one CTA per HUB_CHUNK-edge chunk: aggregate the chunk in a shared table
//                (<= 4096 distinct keys), then write its distinct (key, Σw) to the
//                chunk's pool region grouped by bucket, with the bucket boundaries in
//                the chunk's segment table.  Sequential writes only.
//   k_hub_fin    one CTA per (row, bucket): merge that bucket's segments of every chunk
//                of the row in a shared table (expected <= 1024 distinct keys), then score
//                / count / emit them and write one partial.
//   k_hub_decide one thread per row: combine the row's partials and decide.
constexpr i64 HUB_CHUNK = 4096;
constexpr int HUB_ACC_T = 512;
constexpr int HUB_SM_LG = 13;      // chunk table: 8192 slots >= 2 x 4096 distinct (exact bound)
constexpr int HUB_FIN_T = 256;
// bucket table: 2^fin_lg slots, <= 2^(fin_lg-1) distinct keys (load <= 0.5), buckets sized
// for an expected 2^(fin_lg-2); fin_lg = 12 normally, up to 14 (per launch) for giant rows
constexpr int HUB_FIN_LG = 12;
constexpr int HUB_FIN_LG_MAX = 14;
constexpr i64 HUB_BUCKET_TARGET = 1024;
constexpr int HUB_MAX_BLG = 15;    // <= 32768 buckets per row (histogram sized per launch)

__device__ __forceinline__ unsigned hbucket(int32_t k, int blg) {
  return blg == 0 ? 0u : (((uint32_t)k * 0x85EBCA77u) >> (32 - blg));
}

struct HubPartial {
  i64 hi;
  u64 lo;
  int32_t c, T, sg, pad;
  u64 eown, cnt, selfw, sumw;
};

struct HubArgs {
  const i64 *cfirst;      // per hub: first chunk (chunks of a hub are contiguous)
  const int32_t *ccount;  // per hub: number of chunks
  const int32_t *blg;     // per hub: log2 number of buckets
  const i64 *bfirst;      // per hub: first fin item (one per bucket)
  const i64 *segoff;      // per chunk: offset of its segment table (nb + 1 entries)
  int32_t *seg;           // segment boundaries, relative to the chunk's pool region
  uint4 *pent;            // pool: chunk c of this batch owns [(c - c0) * HUB_CHUNK, +HUB_CHUNK);
                          //   entries packed {key, deg_C (SWEEP/MERGE), Σw lo, Σw hi} — ONE
                          //   16-byte store / load per entry (not three scattered 4-8 byte
                          //   accesses to separate key / value / degree arrays)
  i64 c0, c1;            // chunk range of this batch (hub rows are processed in batches
  i64 f0, f1;             //   bounding the pool); fin-item range of the same rows
  i64 h0, h1;             // hub range of the batch
  const int2 *fitem;      // per fin item: (hub, bucket)
  HubPartial *part;       // per fin item
  u64 *emit_cur;          // per hub (EMIT output cursor)
  int *overflow;          // set if a bucket exceeds its distinct-key capacity
  i64 nhub, nchunks, nfin;
  int fin_lg;             // bucket table log2 capacity of this launch
};

// layouts: [vals | keys | list degrees (SWEEP/MERGE) | list | ...]
template <class VT, int MODE>
constexpr size_t hub_acc_smem(int max_blg) {
  return (size_t)(1 << HUB_SM_LG) * (sizeof(VT) + sizeof(int32_t)) +
         (MODE != M_EMIT ? (size_t)HUB_CHUNK * sizeof(uint32_t) : 0) + (size_t)HUB_CHUNK * sizeof(uint16_t) +
         (size_t)((1 << max_blg) + 1) * sizeof(int) + 64;
}
template <class VT, int MODE>
constexpr size_t hub_fin_smem(int fin_lg) {
  return ((size_t)1 << fin_lg) * (sizeof(VT) + sizeof(int32_t)) +
         (MODE != M_EMIT ? ((size_t)1 << (fin_lg - 1)) * sizeof(uint32_t) : 0) +
         ((size_t)1 << (fin_lg - 1)) * sizeof(uint16_t) + 64;
}

// exclusive scan of cnt[0..n) in shared memory by a CTA of T threads; returns the total
template <int T>
__device__ __forceinline__ int smem_excl_scan(int *cnt, int n) {
  __shared__ int part[T / 32 + 1];
  const int per = (n + T - 1) / T;
  const int base = threadIdx.x * per;
  const int lim = min(base + per, n);
  int sum = 0;
  for (int q = base; q < lim; ++q) sum += cnt[q];
  int inc = sum;
  const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, inc, o);
    if (l >= o) inc += t;
  }
  if (l == 31) part[w] = inc;
  __syncthreads();
  if (threadIdx.x == 0) {
    int r = 0;
    for (int i = 0; i < T / 32; ++i) { const int t = part[i]; part[i] = r; r += t; }
    part[T / 32] = r;
  }
  __syncthreads();
  int run = part[w] + inc - sum;
  for (int q = base; q < lim; ++q) {
    const int v = cnt[q];
    cnt[q] = run;
    run += v;
  }
  const int total = part[T / 32];
  __syncthreads();
  return total;
}

// Persistent: each CTA loops over chunks; the shared table is cleared once and every
// used slot is reset through the occupied list.
template <int MODE, class WT, class VT>
__global__ void __launch_bounds__(HUB_ACC_T) k_hub_acc(AggArgs a, HubArgs hb) {
  extern __shared__ __align__(16) unsigned char sm[];
  constexpr int CAPS = 1 << HUB_SM_LG;
  constexpr bool DEGL = MODE != M_EMIT;
  VT *svals = (VT *)sm;
  int32_t *skeys = (int32_t *)(sm + (size_t)CAPS * sizeof(VT));
  uint32_t *sdeg = (uint32_t *)(sm + (size_t)CAPS * (sizeof(VT) + sizeof(int32_t)));
  uint16_t *slist = (uint16_t *)((unsigned char *)sdeg + (DEGL ? (size_t)HUB_CHUNK * sizeof(uint32_t) : 0));
  int *hist = (int *)((unsigned char *)slist + (size_t)HUB_CHUNK * sizeof(uint16_t));
  __shared__ int scnt;
  for (int s = threadIdx.x; s < CAPS; s += HUB_ACC_T) { skeys[s] = EMPTY; svals[s] = 0; }
  if (threadIdx.x == 0) scnt = 0;
  __syncthreads();
  for (i64 ci = hb.c0 + blockIdx.x; ci < hb.c1; ci += gridDim.x) {
    const Chunk ch = a.chunks[ci];
    const int32_t r = a.rows[ch.h];
    if (MODE == M_MERGE) {
      if (!key_sg((int32_t)(uint32_t)__ldg(&a.ldeg[r]))) continue;  // CTA-uniform
    }
    const int blg = hb.blg[ch.h];
    const int nb = 1 << blg;
    for (int b = threadIdx.x; b <= nb; b += HUB_ACC_T) hist[b] = 0;
    insert_range<HUB_ACC_T, 8, MODE, WT, true, VT>(a, threadIdx.x, ch.beg, ch.end, skeys, svals, CAPS - 1,
                                                         HUB_SM_LG, slist, sdeg, &scnt);
    __syncthreads();
    const int n = scnt;
    for (int t = threadIdx.x; t < n; t += HUB_ACC_T) atomicAdd(&hist[hbucket(skeys[slist[t]], blg)], 1);
    __syncthreads();
    smem_excl_scan<HUB_ACC_T>(hist, nb);  // hist[b] = start of bucket b
    int32_t *seg = hb.seg + hb.segoff[ci];
    for (int b = threadIdx.x; b < nb; b += HUB_ACC_T) seg[b] = hist[b];
    if (threadIdx.x == 0) seg[nb] = n;
    __syncthreads();
    const i64 base = (ci - hb.c0) * HUB_CHUNK;
    for (int t = threadIdx.x; t < n; t += HUB_ACC_T) {
      const int sl = slist[t];
      const int32_t k = skeys[sl];
      const int pos = atomicAdd(&hist[hbucket(k, blg)], 1);
      const u64 val = (u64)svals[sl];
      hb.pent[base + pos] = make_uint4((uint32_t)k, DEGL ? sdeg[t] : 0u, (uint32_t)val, (uint32_t)(val >> 32));
      skeys[sl] = EMPTY;
      svals[sl] = 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) scnt = 0;
    __syncthreads();
  }
}

// SWEEP part of one (row, bucket) item: score the bucket's entries (list positions
// [0, n)), reset their slots, argmax over the CTA (result in thread 0).  The thread that
// meets r's own community stores e_{i->own} in *eown_s.
template <bool S64, class VT>
__device__ __forceinline__ Cand hub_fin_sweep(const Grp<HUB_FIN_T, HUB_FIN_T> &g, int32_t *skeys, VT *svals,
                                              const uint16_t *slist, const uint32_t *sdeg, int n, int32_t own, i64 di,
                                              const AggArgs &a, Acc &acc, u64 *eown_s) {
  constexpr int U = 4;
  Cand best = S64 ? cand_none64() : cand_none();
  u64 n1 = 0;
  for (int t0 = threadIdx.x; t0 < n; t0 += HUB_FIN_T * U) {
    int32_t sl[U], k[U];
    uint32_t d31[U];
    u64 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int t = t0 + u * HUB_FIN_T;
      sl[u] = t < n ? (int32_t)slist[t] : -1;
      d31[u] = t < n ? sdeg[t] : 0;
      k[u] = sl[u] >= 0 ? skeys[sl[u]] : EMPTY;
      v[u] = sl[u] >= 0 ? (u64)svals[sl[u]] : 0;
      if (sl[u] >= 0) { skeys[sl[u]] = EMPTY; svals[sl[u]] = 0; }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (k[u] == EMPTY) continue;
      if (k[u] == own) {
        *eown_s = v[u];
      } else {
        ++n1;
        cand_push<S64>(best, a.twoW, di, k[u], v[u], deg_of(a, d31[u], key_label(k[u])));
      }
    }
  }
  acc.cand += n1;
  grp_argmax<HUB_FIN_T, HUB_FIN_T, S64>(g, best);  // ends with __syncthreads: *eown_s visible
  return best;
}

// Persistent over (row, bucket) items; table reset through the occupied list.
template <int MODE, class VT>
__global__ void __launch_bounds__(HUB_FIN_T) k_hub_fin(AggArgs a, HubArgs hb) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int FLG = hb.fin_lg;
  const int CAPF = 1 << FLG;
  const int MAXD = CAPF / 2;
  constexpr bool DEGL = MODE != M_EMIT;
  VT *svals = (VT *)sm;
  int32_t *skeys = (int32_t *)(sm + (size_t)CAPF * sizeof(VT));
  uint32_t *sdeg = (uint32_t *)(sm + (size_t)CAPF * (sizeof(VT) + sizeof(int32_t)));
  uint16_t *slist = (uint16_t *)((unsigned char *)sdeg + (DEGL ? (size_t)MAXD * sizeof(uint32_t) : 0));
  __shared__ int scnt, sovf;
  __shared__ u64 sbase, seown;
  const uint32_t kb = saddr(skeys), vb = saddr(svals), cb = saddr(&scnt);
  Acc acc;
  for (int s = threadIdx.x; s < CAPF; s += HUB_FIN_T) { skeys[s] = EMPTY; svals[s] = 0; }
  if (threadIdx.x == 0) { scnt = 0; sovf = 0; seown = 0; }
  __syncthreads();
  Grp<HUB_FIN_T, HUB_FIN_T> g;
  for (i64 fi = hb.f0 + blockIdx.x; fi < hb.f1; fi += gridDim.x) {
    const int2 it = hb.fitem[fi];
    const int h = it.x, b = it.y;
    const int32_t r = a.rows[h];
    const int32_t own = (MODE == M_EMIT) ? r : (int32_t)(uint32_t)__ldg(&a.ldeg[r]);
    HubPartial P;
    P.hi = INT64_MIN; P.lo = 0; P.c = INT32_MAX; P.T = -1; P.sg = 0; P.pad = 0;
    P.eown = 0; P.cnt = 0; P.selfw = 0; P.sumw = 0;
    if (MODE == M_MERGE && !key_sg(own)) {  // CTA-uniform
      if (threadIdx.x == 0) hb.part[fi] = P;
      continue;
    }
    const i64 cf = hb.cfirst[h];
    const int nch = hb.ccount[h];
    {
      // every chunk's segment b gets Gc = 256 / nch lanes (a power of two, >= 1): the
      // segments of an item hold ~2^(fin_lg-2) entries in total, so ~equal work per lane
      const int per = nch < HUB_FIN_T ? HUB_FIN_T / nch : 1;
      const int Gc = 1 << (31 - __clz(per));
      const int ng = HUB_FIN_T / Gc, gid = threadIdx.x / Gc, gl = threadIdx.x % Gc;
      for (int j = gid; j < nch; j += ng) {
        const i64 c = cf + j;
        const int32_t *seg = hb.seg + hb.segoff[c];
        const int s0 = seg[b], s1 = seg[b + 1];
        const i64 base = (c - hb.c0) * HUB_CHUNK;
        for (int i = s0 + gl; i < s1; i += Gc) {
          const i64 e = base + i;
          const uint4 pe = hb.pent[e];
          const int32_t k = (int32_t)pe.x;
          const u64 v = (u64)pe.z | ((u64)pe.w << 32);
          if (*(volatile int *)&scnt >= MAXD - 1) { sovf = 1; continue; }
          bool claimed = false;
          const unsigned sl = tab_insert<VT>(kb, vb, CAPF - 1, FLG, k, v, &claimed);
          if (claimed) {
            const int q = (int)atom_add_s32(cb, 1);
            if (q < MAXD) {
              slist[q] = (uint16_t)sl;
              if (DEGL) sdeg[q] = pe.y;
            } else {
              sovf = 1;
            }
          }
        }
      }
      __syncthreads();
    }
    if (sovf) {
      if (threadIdx.x == 0) atomicOr(hb.overflow, 1);
    }
    const int n = min(scnt, MAXD);
    if (MODE == M_SWEEP) {
      const i64 di = a.delta[r];
      Cand best;
      if (row_s64(a.twoW, di)) best = hub_fin_sweep<true, VT>(g, skeys, svals, slist, sdeg, n, own, di, a, acc, &seown);
      else best = hub_fin_sweep<false, VT>(g, skeys, svals, slist, sdeg, n, own, di, a, acc, &seown);
      if (threadIdx.x == 0) {
        P.hi = best.hi; P.lo = best.lo; P.c = best.c; P.eown = seown;
        seown = 0;
      }
    } else if (MODE == M_MERGE) {
      u64 n1 = 0, nsg = 0;
      int32_t T = -1;
      for (int i = threadIdx.x; i < n; i += HUB_FIN_T) {
        const int sl = slist[i];
        const int32_t k = skeys[sl];
        skeys[sl] = EMPTY;
        svals[sl] = 0;
        if (k != own) { ++n1; T = max(T, key_label(k)); nsg += key_sg(k); }
      }
      grp_reduce<HUB_FIN_T, HUB_FIN_T>(g, n1, nsg, T);
      if (threadIdx.x == 0) { P.cnt = n1; P.T = T; P.selfw = nsg; }
    } else {
      u64 n1 = 0, selfw = 0, sumw = 0;
      for (int i = threadIdx.x; i < n; i += HUB_FIN_T) {
        const int sl = slist[i];
        const int32_t k = skeys[sl];
        const u64 v = (u64)svals[sl];
        sumw += v;
        if (k == r) selfw += v;
        else ++n1;
      }
      u64 tot;
      const u64 pre = grp_excl_scan<HUB_FIN_T, HUB_FIN_T>(g, n1, tot);
      if (threadIdx.x == 0) sbase = atomicAdd(&hb.emit_cur[h], tot);
      __syncthreads();
      i64 o = (a.out_base ? a.out_base[r] : a.ptr[r]) + (i64)(sbase + pre);
      for (int i = threadIdx.x; i < n; i += HUB_FIN_T) {
        const int sl = slist[i];
        const int32_t k = skeys[sl];
        if (k != r && a.out_key) {
          a.out_key[o] = k;
          store_w(a, o, (u64)svals[sl]);
          ++o;
        }
        skeys[sl] = -1;
        svals[sl] = 0;
      }
      int32_t dm = 0;
      grp_reduce<HUB_FIN_T, HUB_FIN_T>(g, selfw, sumw, dm);
      if (threadIdx.x == 0) { P.cnt = tot; P.selfw = selfw; P.sumw = sumw; }
    }
    if (threadIdx.x == 0) hb.part[fi] = P;
    __syncthreads();
    if (threadIdx.x == 0) { scnt = 0; sovf = 0; }
    __syncthreads();
  }
  if (MODE == M_SWEEP) acc.flush(a.counters);  // candidate count only
}

// SWEEP-mode specialisation of k_hub_fin with two CTA barriers per (row, bucket) item
// instead of five: the distinct-key counter and overflow flag alternate by item parity
// (the next item's pair is cleared between the two barriers), and the argmax combine is
// done by thread 0 after ONE barrier (the per-warp candidate slots are not rewritten
// before the next item's first barrier, which thread 0 reaches only after combining).
// Same arithmetic as k_hub_fin<M_SWEEP> (hub_fin_sweep): the bucket's (key, Σw, deg)
// entries of every chunk merged in a shared table, scored, argmax by (S desc, label asc).
template <class VT>
__global__ void __launch_bounds__(HUB_FIN_T) k_hub_fin_sw(AggArgs a, HubArgs hb) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int FLG = hb.fin_lg;
  const int CAPF = 1 << FLG;
  const int MAXD = CAPF / 2;
  VT *svals = (VT *)sm;
  int32_t *skeys = (int32_t *)(sm + (size_t)CAPF * sizeof(VT));
  uint32_t *sdeg = (uint32_t *)(sm + (size_t)CAPF * (sizeof(VT) + sizeof(int32_t)));
  uint16_t *slist = (uint16_t *)((unsigned char *)sdeg + (size_t)MAXD * sizeof(uint32_t));
  __shared__ int scnt[2], sovf[2];
  __shared__ u64 seown[2];
  __shared__ Cand wc[HUB_FIN_T / 32];
  const uint32_t kb = saddr(skeys), vb = saddr(svals);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  Acc acc;
  for (int s = threadIdx.x; s < CAPF; s += HUB_FIN_T) { skeys[s] = EMPTY; svals[s] = 0; }
  if (threadIdx.x == 0) { scnt[0] = scnt[1] = 0; sovf[0] = sovf[1] = 0; seown[0] = seown[1] = 0; }
  __syncthreads();
  int par = 0;
  for (i64 fi = hb.f0 + blockIdx.x; fi < hb.f1; fi += gridDim.x) {
    const int2 it = hb.fitem[fi];
    const int h = it.x, b = it.y;
    const int32_t r = a.rows[h];
    const int32_t own = (int32_t)(uint32_t)__ldg(&a.ldeg[r]);
    const i64 di = a.delta[r];
    const i64 cf = hb.cfirst[h];
    const int nch = hb.ccount[h];
    const uint32_t cb = saddr(&scnt[par]);
    {
      const int per = nch < HUB_FIN_T ? HUB_FIN_T / nch : 1;
      const int Gc = 1 << (31 - __clz(per));
      const int ng = HUB_FIN_T / Gc, gid = threadIdx.x / Gc, gl = threadIdx.x % Gc;
      for (int j = gid; j < nch; j += ng) {
        const i64 c = cf + j;
        const int32_t *seg = hb.seg + hb.segoff[c];
        const int s0 = seg[b], s1 = seg[b + 1];
        const i64 base = (c - hb.c0) * HUB_CHUNK;
        for (int i = s0 + gl; i < s1; i += Gc) {
          const i64 e = base + i;
          const uint4 pe = hb.pent[e];
          const int32_t k = (int32_t)pe.x;
          const u64 v = (u64)pe.z | ((u64)pe.w << 32);
          if (*(volatile int *)&scnt[par] >= MAXD - 1) { sovf[par] = 1; continue; }
          bool claimed = false;
          const unsigned sl = tab_insert<VT>(kb, vb, CAPF - 1, FLG, k, v, &claimed);
          if (claimed) {
            const int q = (int)atom_add_s32(cb, 1);
            if (q < MAXD) {
              slist[q] = (uint16_t)sl;
              sdeg[q] = pe.y;
            } else {
              sovf[par] = 1;
            }
          }
        }
      }
    }
    __syncthreads();  // B1: the item's inserts are complete
    const int n = min(scnt[par], MAXD);
    if (threadIdx.x == 0) {
      if (sovf[par]) atomicOr(hb.overflow, 1);
      scnt[par ^ 1] = 0;  // the next item's counter and flag (nobody touches them before B2)
      sovf[par ^ 1] = 0;
    }
    const bool s64 = row_s64(a.twoW, di);  // CTA-uniform
    Cand best = s64 ? cand_none64() : cand_none();
    u64 n1 = 0;
    for (int t = threadIdx.x; t < n; t += HUB_FIN_T) {
      const int sl = slist[t];
      const uint32_t d31 = sdeg[t];
      const int32_t k = skeys[sl];
      const u64 v = (u64)svals[sl];
      skeys[sl] = EMPTY;
      svals[sl] = 0;
      if (k == own) {
        seown[par] = v;
      } else {
        ++n1;
        if (s64) cand_push<true>(best, a.twoW, di, k, v, deg_of(a, d31, key_label(k)));
        else cand_push<false>(best, a.twoW, di, k, v, deg_of(a, d31, key_label(k)));
      }
    }
    acc.cand += n1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      Cand y;
      y.lo = __shfl_xor_sync(0xffffffffu, best.lo, o);
      y.hi = __shfl_xor_sync(0xffffffffu, best.hi, o);
      y.c = __shfl_xor_sync(0xffffffffu, best.c, o);
      if (s64 ? cand_better64(y, best) : cand_better(y, best)) best = y;
    }
    if (lane == 0) wc[wid] = best;
    __syncthreads();  // B2: partial candidates, e_own visible; every slot reset
    if (threadIdx.x == 0) {
      for (int w = 1; w < HUB_FIN_T / 32; ++w)
        if (s64 ? cand_better64(wc[w], best) : cand_better(wc[w], best)) best = wc[w];
      if (s64) best.hi = (i64)best.lo >> 63;
      HubPartial P;
      P.hi = best.hi; P.lo = best.lo; P.c = best.c; P.T = -1; P.sg = 0; P.pad = 0;
      P.eown = seown[par]; P.cnt = 0; P.selfw = 0; P.sumw = 0;
      seown[par] = 0;  // rewritten only after the next item's B1 (other parity) or the one after
      hb.part[fi] = P;
    }
    par ^= 1;
  }
  acc.flush(a.counters);  // candidate count only
}

// One warp per hub row: combine the row's per-bucket partials, then decide / emit.
template <int MODE>
__global__ void __launch_bounds__(128) k_hub_decide(AggArgs a, HubArgs hb) {
  Acc acc;
  const int lane = threadIdx.x & 31;
  const i64 h = hb.h0 + (i64)blockIdx.x * 4 + (threadIdx.x >> 5);
  if (h < hb.h1) {  // warp-uniform
    const int32_t r = a.rows[h];
    const u64 pr = (MODE == M_EMIT) ? 0 : __ldg(&a.ldeg[r]);
    const int32_t own = (MODE == M_EMIT) ? r : (int32_t)(uint32_t)pr;
    Cand best = cand_none();
    u64 eown = 0, cnt = 0, selfw = 0, sumw = 0;
    int32_t T = -1;
    const HubPartial *p = hb.part + hb.bfirst[h];
    const int np = 1 << hb.blg[h];
    for (int j = lane; j < np; j += 32) {
      Cand x;
      x.hi = p[j].hi; x.lo = p[j].lo; x.c = p[j].c;
      if (cand_better(x, best)) best = x;
      eown += p[j].eown; cnt += p[j].cnt; selfw += p[j].selfw; sumw += p[j].sumw;
      T = max(T, p[j].T);
    }
    Grp<32, 128> g;
    grp_argmax<32, 128, false>(g, best);
    eown = warp_sum_u64(eown);
    cnt = warp_sum_u64(cnt);
    selfw = warp_sum_u64(selfw);
    sumw = warp_sum_u64(sumw);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) T = max(T, __shfl_xor_sync(0xffffffffu, T, o));
    if (lane == 0) {
      if (MODE == M_SWEEP) {
        const i64 dq = deg_of(a, (uint32_t)(pr >> 32), key_label(own));
        sweep_decide<false>(a, acc, r, own, a.delta[r], dq, load_deg(a, r), best, eown);
      } else if (MODE == M_MERGE) {
        merge_decide(a, acc, r, own, cnt, T, selfw);  // selfw carries the singlet count
      } else {
        a.out_cnt[r] = (i64)cnt;
        if (a.out_self) a.out_self[r] = selfw;
        if (a.out_sum) a.out_sum[r] = sumw;
      }
      hb.emit_cur[h] = 0;
    }
  }
  if (MODE != M_EMIT) acc.flush(a.counters);
}

// Apply every move cur -> nxt of a pass to the next-state deg/size (remove from
// the old community, insert into the new), after the pass (and, sweep-sharded, after the
// label exchange: identical on every rank).  Exact and order-free (integer sums).
// A sweep moves millions of vertices into and out of the same few big communities, and
// per-move global atomics on those addresses serialise in L2, so the moves are combined
// in two stages before they reach global memory:
//  1. the lanes of a warp that share a community (__match_any_sync) sum their δ (the
//     16-bit halves with two 32-bit reductions: exact for δ < 2^32, "narrow");
//  2. a CTA sweeps a chunk of AM_CHUNK vertices (AM_U per thread and step, loads issued
//     together); the warp sums for HOT communities (snapshot deg_C >= AM_HOT, from cpk) go
//     to a shared-memory table (fire-and-forget 32-bit reductions of the 16-bit halves:
//     < AM_CHUNK·2^16 < 2^31 per chunk), flushed with one global atomic per hot community
//     and chunk; cold communities (and hot ones whose probe fails, and everything when
//     not narrow) take global atomics directly.
constexpr int AM_T = 512, AM_TLG = 11, AM_TS = 1 << AM_TLG, AM_PROBE = 8, AM_U = 4;
constexpr i64 AM_CHUNK = (i64)AM_T * AM_U * 4;  // 8192 vertices: 4 iterations of AM_U per thread
constexpr size_t AM_SMEM = (size_t)AM_TS * 24;
constexpr uint32_t AM_HOT = 1u << 12;

__device__ __forceinline__ void am_global(i64 *deg_next, int32_t *size_next, int32_t c, u64 d, int cnt) {
  atomicAdd((u64 *)&deg_next[c], d);
  atomicAdd(&size_next[c], cnt);
}

__global__ void __launch_bounds__(AM_T) k_apply_moves(i64 n, const int32_t *__restrict__ cur,
                                                      const int32_t *__restrict__ nxt, const i64 *__restrict__ delta,
                                                      const uint32_t *__restrict__ cpk, i64 *deg_next,
                                                      int32_t *size_next, int narrow) {
  extern __shared__ __align__(16) unsigned char sm[];  // AM_SMEM bytes
  uint32_t(*tv)[4] = (uint32_t(*)[4])sm;              // Σ lo16(+δ), Σ hi(+δ), Σ lo16(−δ), Σ hi(−δ)
  int32_t *tk = (int32_t *)(sm + (size_t)AM_TS * 16);
  int32_t *tc = (int32_t *)(sm + (size_t)AM_TS * 20);  // Σ ±1
  const int lane = threadIdx.x & 31;
  __shared__ uint32_t segbuf[AM_T / 32][64];  // class_sum32x2 buffers (one pair per warp)
  segbuf[threadIdx.x >> 5][lane] = 0u;
  segbuf[threadIdx.x >> 5][32 + lane] = 0u;
  __syncwarp();
  const uint32_t kb = saddr(tk);
  for (int s = threadIdx.x; s < AM_TS; s += AM_T) {
    tk[s] = EMPTY;
    tv[s][0] = tv[s][1] = tv[s][2] = tv[s][3] = 0;
    tc[s] = 0;
  }
  __syncthreads();
  // one warp group's (community c, hot?, sign, Σδ halves, count) -> table or global
  auto put = [&](int32_t c, bool hot, int neg, uint32_t lo, uint32_t hi, int cnt) {
    if (hot) {
      unsigned h = hslot(c, AM_TLG);
#pragma unroll 1
      for (int p = 0; p < AM_PROBE; ++p) {
        int32_t k = lds_i32(kb + 4 * h);
        if (k == EMPTY) k = cas_s32(kb + 4 * h, EMPTY, c);
        if (k == EMPTY || k == c) {
          red_add_s32(saddr(&tv[h][2 * neg]), lo);
          red_add_s32(saddr(&tv[h][2 * neg + 1]), hi);
          red_add_s32(saddr(&tc[h]), (uint32_t)(neg ? -cnt : cnt));
          return;
        }
        h = (h + 1) & (AM_TS - 1);
      }
    }
    const u64 v = (u64)lo + ((u64)hi << 16);
    am_global(deg_next, size_next, c, neg ? (u64)0 - v : v, neg ? -cnt : cnt);
  };
  for (i64 c0 = (i64)blockIdx.x * AM_CHUNK; c0 < n; c0 += (i64)gridDim.x * AM_CHUNK) {
    const i64 c1 = c0 + AM_CHUNK < n ? c0 + AM_CHUNK : n;
    for (i64 base = c0 + (threadIdx.x & ~31) * AM_U; base < c1; base += (i64)AM_T * AM_U) {  // warp-uniform
      int32_t av[AM_U], bv[AM_U];
      i64 dv[AM_U];
      uint32_t ha[AM_U], hb[AM_U];
#pragma unroll
      for (int u = 0; u < AM_U; ++u) {  // every load of the AM_U vertices issued together
        const i64 i = base + u * 32 + lane;
        av[u] = bv[u] = 0;
        dv[u] = 0;
        if (i < c1) { av[u] = cur[i]; bv[u] = nxt[i]; dv[u] = delta[i]; }
      }
#pragma unroll
      for (int u = 0; u < AM_U; ++u) {
        ha[u] = hb[u] = 0;
        if (narrow && av[u] != bv[u]) { ha[u] = __ldg(&cpk[av[u]]); hb[u] = __ldg(&cpk[bv[u]]); }
      }
#pragma unroll
      for (int u = 0; u < AM_U; ++u) {
        const bool moved = av[u] != bv[u];
        const unsigned mv = __ballot_sync(0xffffffffu, moved);
        if (!moved) continue;
        const i64 d = dv[u];
        const int32_t a = av[u], b = bv[u];
        if (narrow) {
          const uint32_t dlo = (uint32_t)(d & 0xFFFF), dhi = (uint32_t)((u64)d >> 16);
          uint32_t *wb = segbuf[threadIdx.x >> 5];
          const unsigned pt = __match_any_sync(mv, b);
          uint32_t tlo = dlo, thi = dhi;
          class_sum32x2(mv, pt, tlo, thi, wb);
          if (lane == __ffs(pt) - 1) put(b, (hb[u] & DEG_SAT) >= AM_HOT, 0, tlo, thi, __popc(pt));
          const unsigned po = __match_any_sync(mv, a);
          uint32_t olo = dlo, ohi = dhi;
          class_sum32x2(mv, po, olo, ohi, wb);
          if (lane == __ffs(po) - 1) put(a, (ha[u] & DEG_SAT) >= AM_HOT, 1, olo, ohi, __popc(po));
        } else {  // wide graphs (rare): per-vertex atomics
          am_global(deg_next, size_next, b, (u64)d, 1);
          am_global(deg_next, size_next, a, (u64)0 - (u64)d, -1);
        }
      }
    }
    __syncthreads();  // flush the chunk's hot communities, reset the table
    for (int s = threadIdx.x; s < AM_TS; s += AM_T) {
      const int32_t c = tk[s];
      if (c == EMPTY) continue;
      const u64 pv = (u64)tv[s][0] + ((u64)tv[s][1] << 16), mvv = (u64)tv[s][2] + ((u64)tv[s][3] << 16);
      const u64 v = pv - mvv;
      if (v) atomicAdd((u64 *)&deg_next[c], v);
      if (tc[s]) atomicAdd(&size_next[c], tc[s]);
      tk[s] = EMPTY;
      tv[s][0] = tv[s][1] = tv[s][2] = tv[s][3] = 0;
      tc[s] = 0;
    }
    __syncthreads();
  }
}

// cpk[c] = (|c| == 1) << 31 | min(deg_c, 2^31 - 1): the per-community half of the packed
// entries, built once per committed state
__global__ void __launch_bounds__(256) k_cpk(i64 n, const i64 *__restrict__ deg, const int32_t *__restrict__ size,
                                             uint32_t *cpk) {
  for (i64 c = (i64)blockIdx.x * 256 + threadIdx.x; c < n; c += (i64)gridDim.x * 256) {
    const i64 d = deg[c];
    cpk[c] = (size[c] == 1 ? SG_BIT : 0u) | (d >= (i64)DEG_SAT ? DEG_SAT : (uint32_t)d);
  }
}

// ldeg[v] = { C(v) | singlet bit, deg_C(v) }: the packed entry every edge gathers
__global__ void __launch_bounds__(256) k_ldeg(i64 n, const int32_t *__restrict__ label,
                                              const uint32_t *__restrict__ cpk, u64 *ldeg) {
  for (i64 v = (i64)blockIdx.x * 256 + threadIdx.x; v < n; v += (i64)gridDim.x * 256) {
    const int32_t l = label[v];
    const uint32_t p = cpk[l];
    ldeg[v] = ((u64)(p & DEG_SAT) << 32) | (u64)((uint32_t)l | (p & SG_BIT));
  }
}

}  // namespace lv
