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
//             S(best) > S_own (D6), singlet rule (D8).  It also emits
//             e_{i->own} and deg[i]² for the exact Eq. 3 numerators of the snapshot.
//   M_MERGE : isolated-node merge (D14): a singlet whose neighbours lie in
//             exactly one community T moves to T (singlet rule applies).
//   M_EMIT  : distinct (key, Σw) per row, for duplicate merging in "Neighbor
//             computation" (P:L271 reduce_by_key) and for graph contraction (P:L306-313:
//             sort_by_key + reduce_by_key).  Entries whose key equals the row id are
//             summed separately (intra-community weight -> the meta-vertex loop).
//
// Rows are binned by length (P:L438 motivates grouping by degree): bins of
// G ∈ {4,8,16,32} lanes per row with per-group shared-memory open-addressing tables,
// block-per-row bins with block-wide shared tables up to 16384 slots (192 KB), and a
// hub path for longer rows: a global-memory table per row filled by many CTAs
// (k_hub_acc), then one CTA per row runs the epilogue (k_hub_fin).  All sums are exact
// integers, so the result is independent of insertion order and schedule.
#pragma once
#include "lv_common.cuh"

namespace lv {

enum { M_SWEEP = 0, M_MERGE = 1, M_EMIT = 2 };
enum { WT_NONE = 0, WT_U32 = 1, WT_U64 = 2 };

struct WNone {
  static constexpr int id = WT_NONE;
  static constexpr int bytes = 0;
  __device__ __forceinline__ static u64 get(const void *, i64) { return 1ull; }
};
struct WU32 {
  static constexpr int id = WT_U32;
  static constexpr int bytes = 4;
  __device__ __forceinline__ static u64 get(const void *w, i64 e) { return __ldg((const uint32_t *)w + e); }
};
struct WU64 {
  static constexpr int id = WT_U64;
  static constexpr int bytes = 8;
  __device__ __forceinline__ static u64 get(const void *w, i64 e) { return __ldg((const u64 *)w + e); }
};

struct Chunk {
  i64 beg, end;
  int32_t h, pad;
};

struct AggArgs {
  const i64 *ptr;          // row offsets: row r = [ptr[r], ptr[r+1])
  const int32_t *rows;     // rows of this bin
  i64 nrows;
  const int32_t *keys;     // SWEEP/MERGE: col[] (key = label[col]); EMIT: key directly
  const void *w;           // weights (WT)
  const int32_t *label;    // snapshot labels C
  int32_t *label_next;     // decisions
  const i64 *deg;          // deg_C, indexed by label
  const int32_t *size;     // |C|, indexed by label
  const i64 *delta;        // δ_i
  i64 twoW;                // 2W
  const i64 *out_base;     // EMIT: output offset of row r (NULL -> ptr)
  int32_t *out_key;        // EMIT outputs (NULL -> count only)
  u64 *out_w;
  i64 *out_cnt;            // distinct keys ≠ row id
  u64 *out_self;           // Σ w with key == row id (may be NULL)
  u64 *out_sum;            // Σ w over the row (may be NULL)
  u64 *counters;           // SWEEP/MERGE: [0] I2 [1] moved [2] S2 lo [3] S2 hi [4] cand
  // hub tables
  int32_t *tkeys;
  u64 *tvals;
  const i64 *toff;         // table offset per hub index
  const int32_t *tlog;     // log2 capacity per hub index
  const Chunk *chunks;
};

__device__ __forceinline__ unsigned hslot(int32_t k, int lg) {
  return ((uint32_t)k * 0x9E3779B1u) >> (32 - lg);
}

// Exact 64-bit add (mod 2^64) with native 32-bit atomics: sm_100 has no native 64-bit
// shared-memory add (it compiles to a CAS loop, which collapses under the same-key
// contention of later sweeps); the low word's returned old value gives the carry.
__device__ __forceinline__ void add_u64_split(u64 *p, u64 v) {
  uint32_t *q = (uint32_t *)p;
  const uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
  const uint32_t old = atomicAdd(q, lo);
  const uint32_t carry = ((uint32_t)(old + lo) < old) ? 1u : 0u;
  if (hi + carry) atomicAdd(q + 1, hi + carry);
}

// Open-addressing insert with linear probing; keys -1 = empty.  Returns the slot.
template <bool SHARED>
__device__ __forceinline__ unsigned tab_insert(int32_t *keys, u64 *vals, unsigned mask, int lg, int32_t k, u64 v,
                                               bool *claimed = nullptr) {
  unsigned h = hslot(k, lg);
  while (true) {
    int32_t cur = ((volatile int32_t *)keys)[h];
    if (cur == k) break;
    if (cur == -1) {
      int32_t old = atomicCAS(&keys[h], -1, k);
      if (old == -1) {
        if (claimed) *claimed = true;
        break;
      }
      if (old == k) break;
    }
    h = (h + 1) & mask;
  }
  if (SHARED) add_u64_split(&vals[h], v);
  else atomicAdd(&vals[h], v);
  return h;
}

// smallest lg with 2^lg >= 2*d (d >= 1), clamped to [3, LGMAX]
__device__ __forceinline__ int row_lg(i64 d, int lgmax) {
  int lg = 64 - __clzll((unsigned long long)(2 * d - 1));
  lg = lg < 3 ? 3 : lg;
  return lg > lgmax ? lgmax : lg;
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

struct Cand {  // lexicographic key (S desc, c asc); c == INT32_MAX means "none"
  i64 hi;
  u64 lo;
  int32_t c;
};

__device__ __forceinline__ i128 cand_S(const Cand &x) { return (i128)(((u128)(u64)x.hi << 64) | (u128)x.lo); }
__device__ __forceinline__ bool cand_better(const Cand &a, const Cand &b) {
  if (a.c == INT32_MAX) return false;
  if (b.c == INT32_MAX) return true;
  i128 sa = cand_S(a), sb = cand_S(b);
  return sa > sb || (sa == sb && a.c < b.c);
}
__device__ __forceinline__ Cand cand_shfl_xor(const Cand &x, unsigned mask, int o, int width) {
  Cand y;
  y.hi = __shfl_xor_sync(mask, x.hi, o, width);
  y.lo = __shfl_xor_sync(mask, x.lo, o, width);
  y.c = __shfl_xor_sync(mask, x.c, o, width);
  return y;
}

// Reduce (best candidate, sum a, sum b, max m) across the group; result valid in the
// group's lane 0 (thread 0 of the CTA for block groups).
template <int G, int BLOCK>
__device__ __forceinline__ void grp_reduce(const Grp<G, BLOCK> &g, Cand &best, u64 &a, u64 &b, int32_t &m) {
  constexpr int W = G < 32 ? G : 32;
#pragma unroll
  for (int o = W / 2; o > 0; o >>= 1) {
    Cand y = cand_shfl_xor(best, g.mask, o, W);
    if (cand_better(y, best)) best = y;
    a += __shfl_xor_sync(g.mask, a, o, W);
    b += __shfl_xor_sync(g.mask, b, o, W);
    m = max(m, __shfl_xor_sync(g.mask, m, o, W));
  }
  if (G > 32) {
    constexpr int NW = BLOCK / 32;
    __shared__ Cand sc[NW];
    __shared__ u64 sa[NW], sb[NW];
    __shared__ int32_t sm_[NW];
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) { sc[w] = best; sa[w] = a; sb[w] = b; sm_[w] = m; }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int i = 1; i < NW; ++i) {
        if (cand_better(sc[i], best)) best = sc[i];
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

// ----------------------------------------------------------------- row epilogue
// Scans the row's table (capacity cap), resets every slot it reads, and applies the
// mode's epilogue.  Slots are visited by lane-strided order, identically in both passes.
template <int G, int BLOCK, int MODE>
__device__ __forceinline__ void row_epilogue(const Grp<G, BLOCK> &g, int32_t *keys, u64 *vals, i64 cap,
                                             int32_t r, int32_t own, const AggArgs &a, Acc &acc) {
  if (MODE == M_SWEEP) {
    const i64 di = a.delta[r];
    Cand best;
    best.hi = 0; best.lo = 0; best.c = INT32_MAX;
    u64 eown = 0, ncand = 0;
    int32_t dummy = 0;
    for (i64 s = g.lane; s < cap; s += G) {
      int32_t k = keys[s];
      if (k >= 0) {
        u64 v = vals[s];
        keys[s] = -1;
        vals[s] = 0;
        if (k == own) {
          eown = v;
        } else {
          ++ncand;
          i128 S = (i128)a.twoW * (i128)(i64)v - (i128)di * (i128)__ldg(&a.deg[k]);
          Cand x;
          x.hi = (i64)(S >> 64); x.lo = (u64)S; x.c = k;
          if (cand_better(x, best)) best = x;
        }
      }
    }
    grp_reduce<G, BLOCK>(g, best, eown, ncand, dummy);
    if (g.lane == 0) {
      const i64 dq = a.deg[own];
      i128 S_own = (i128)a.twoW * (i128)(i64)eown - (i128)di * ((i128)dq - (i128)di);
      int32_t tgt = own;
      if (best.c != INT32_MAX && cand_S(best) > S_own) {
        tgt = best.c;
        if (a.size[own] == 1 && a.size[best.c] == 1 && best.c > own) tgt = own;  // singlet rule
      }
      a.label_next[r] = tgt;
      acc.moved += (tgt != own);
      acc.i2 += eown;
      acc.cand += ncand;
      acc.add_sq(a.deg[r]);  // deg of label index r: Σ over all labels gives S2
    }
  } else if (MODE == M_MERGE) {
    Cand none;
    none.hi = 0; none.lo = 0; none.c = INT32_MAX;
    u64 cnt = 0, unused = 0;
    int32_t T = -1;
    for (i64 s = g.lane; s < cap; s += G) {
      int32_t k = keys[s];
      if (k >= 0) {
        keys[s] = -1;
        vals[s] = 0;
        if (k != own) { ++cnt; T = max(T, k); }
      }
    }
    grp_reduce<G, BLOCK>(g, none, cnt, unused, T);
    if (g.lane == 0) {
      int32_t tgt = own;
      if (cnt == 1) tgt = (a.size[T] == 1 && T > own) ? own : T;
      a.label_next[r] = tgt;
      acc.moved += (tgt != own);
    }
  } else {  // M_EMIT
    u64 c = 0, selfw = 0, sumw = 0;
    for (i64 s = g.lane; s < cap; s += G) {
      int32_t k = keys[s];
      if (k >= 0) {
        u64 v = vals[s];
        sumw += v;
        if (k == r) selfw += v;
        else ++c;
      }
    }
    u64 tot;
    u64 pre = grp_excl_scan<G, BLOCK>(g, c, tot);
    i64 o = (a.out_base ? a.out_base[r] : a.ptr[r]) + (i64)pre;
    for (i64 s = g.lane; s < cap; s += G) {
      int32_t k = keys[s];
      if (k >= 0) {
        u64 v = vals[s];
        keys[s] = -1;
        vals[s] = 0;
        if (k != r && a.out_key) {
          a.out_key[o] = k;
          a.out_w[o] = v;
          ++o;
        }
      }
    }
    Cand none;
    none.hi = 0; none.lo = 0; none.c = INT32_MAX;
    int32_t dummy = 0;
    grp_reduce<G, BLOCK>(g, none, selfw, sumw, dummy);
    if (g.lane == 0) {
      a.out_cnt[r] = (i64)tot;
      if (a.out_self) a.out_self[r] = selfw;
      if (a.out_sum) a.out_sum[r] = sumw;
    }
  }
}

// ----------------------------------------------------------------- shared-memory bins
template <int G, int CAP, int BLOCK, int MODE, class WT>
__global__ void __launch_bounds__(BLOCK) k_agg_smem(AggArgs a) {
  constexpr int GPB = BLOCK / G;
  constexpr int LG = (CAP >= 65536) ? 16 : (CAP >= 32768) ? 15 : (CAP >= 16384) ? 14 : (CAP >= 8192) ? 13
                   : (CAP >= 4096) ? 12 : (CAP >= 2048) ? 11 : (CAP >= 1024) ? 10 : (CAP >= 512) ? 9
                   : (CAP >= 256) ? 8 : (CAP >= 128) ? 7 : (CAP >= 64) ? 6 : (CAP >= 32) ? 5
                   : (CAP >= 16) ? 4 : 3;
  static_assert((1 << LG) == CAP, "CAP must be a power of two >= 8");
  extern __shared__ __align__(16) unsigned char sm[];
  u64 *svals = (u64 *)sm;
  int32_t *skeys = (int32_t *)(sm + (size_t)GPB * CAP * sizeof(u64));
  Grp<G, BLOCK> g;
  const int grp = threadIdx.x / G;
  int32_t *keys = skeys + grp * CAP;
  u64 *vals = svals + grp * CAP;
  Acc acc;
  for (int s = g.lane; s < CAP; s += G) { keys[s] = -1; vals[s] = 0; }
  g.sync();
  for (i64 idx = (i64)blockIdx.x * GPB + grp; idx < a.nrows; idx += (i64)gridDim.x * GPB) {
    const int32_t r = a.rows[idx];
    const i64 beg = a.ptr[r], end = a.ptr[r + 1];
    const int32_t own = (MODE == M_EMIT) ? r : a.label[r];
    if (MODE == M_MERGE) {
      if (a.size[own] != 1) {
        if (g.lane == 0) a.label_next[r] = own;
        continue;
      }
    }
    const int lg = row_lg(end - beg, LG);  // table prefix sized for this row
    const unsigned mask = (1u << lg) - 1u;
    for (i64 e = beg + g.lane; e < end; e += G) {
      int32_t k = __ldg(&a.keys[e]);
      if (MODE != M_EMIT) k = __ldg(&a.label[k]);
      tab_insert<true>(keys, vals, mask, lg, k, WT::get(a.w, e));
    }
    g.sync();
    row_epilogue<G, BLOCK, MODE>(g, keys, vals, (i64)1 << lg, r, own, a, acc);
    g.sync();
  }
  if (MODE != M_EMIT) acc.flush(a.counters);
}

// ----------------------------------------------------------------- hub path
// Rows longer than the largest shared-memory bin.  Per hub row h:
//   k_hub_acc    one CTA per HUB_CHUNK edges: aggregate the chunk in a shared-memory table,
//                then flush its distinct (key, Σw) into the row's global table; a slot
//                claimed for the first time is appended to the row's occupied list.
//   k_hub_fin    nparts CTAs per row, each over a strided share of the occupied list:
//                score / count / emit, reset the slots, write one partial per CTA.
//   k_hub_decide one thread per row: combine the partials, decide, reset the row's counters.
constexpr int HUB_ACC_T = 512;
constexpr int HUB_SM_LG = 13;  // 8192-slot pre-aggregation table (chunk of 4096 edges)
constexpr int HUB_FIN_T = 256;
constexpr i64 HUB_FIN_PER = 8192;  // occupied entries per fin CTA

struct FinChunk {
  int32_t h, j, nparts, pad;
};

struct HubPartial {
  i64 hi;
  u64 lo;
  int32_t c, T;
  u64 eown, cnt, selfw, sumw;
};

struct HubArgs {
  const FinChunk *fchunks;
  const i64 *pstart;    // first partial of hub h
  const int32_t *nparts;
  int32_t *occ;         // occupied-slot lists (offset toff[h]/2)
  uint32_t *occ_cnt;    // per hub
  u64 *emit_cur;        // per hub (EMIT output cursor)
  HubPartial *part;
  i64 nhub;
};

template <int MODE, class WT>
__global__ void __launch_bounds__(HUB_ACC_T) k_hub_acc(AggArgs a, HubArgs hb) {
  extern __shared__ __align__(16) unsigned char sm[];
  constexpr int CAPS = 1 << HUB_SM_LG;
  u64 *svals = (u64 *)sm;
  int32_t *skeys = (int32_t *)(sm + (size_t)CAPS * sizeof(u64));
  const Chunk ch = a.chunks[blockIdx.x];
  const int32_t r = a.rows[ch.h];
  if (MODE == M_MERGE) {
    if (a.size[a.label[r]] != 1) return;
  }
  for (int s = threadIdx.x; s < CAPS; s += HUB_ACC_T) { skeys[s] = -1; svals[s] = 0; }
  __syncthreads();
  for (i64 e = ch.beg + threadIdx.x; e < ch.end; e += HUB_ACC_T) {
    int32_t k = __ldg(&a.keys[e]);
    if (MODE != M_EMIT) k = __ldg(&a.label[k]);
    tab_insert<true>(skeys, svals, CAPS - 1, HUB_SM_LG, k, WT::get(a.w, e));
  }
  __syncthreads();
  const int lg = a.tlog[ch.h];
  const i64 off = a.toff[ch.h];
  int32_t *gk = a.tkeys + off;
  u64 *gv = a.tvals + off;
  int32_t *occ = hb.occ + off / 2;
  const unsigned mask = (1u << lg) - 1u;
  for (int s = threadIdx.x; s < CAPS; s += HUB_ACC_T) {
    const int32_t k = skeys[s];
    if (k >= 0) {
      bool claimed = false;
      const unsigned slot = tab_insert<false>(gk, gv, mask, lg, k, svals[s], &claimed);
      if (claimed) occ[atomicAdd(&hb.occ_cnt[ch.h], 1u)] = (int32_t)slot;
    }
  }
}

template <int MODE>
__global__ void __launch_bounds__(HUB_FIN_T) k_hub_fin(AggArgs a, HubArgs hb) {
  const FinChunk fc = hb.fchunks[blockIdx.x];
  const int h = fc.h;
  const int32_t r = a.rows[h];
  const int32_t own = (MODE == M_EMIT) ? r : a.label[r];
  HubPartial P;
  P.hi = 0; P.lo = 0; P.c = INT32_MAX; P.T = -1;
  P.eown = 0; P.cnt = 0; P.selfw = 0; P.sumw = 0;
  const bool skip = (MODE == M_MERGE) && a.size[own] != 1;
  if (!skip) {
    const i64 off = a.toff[h];
    int32_t *gk = a.tkeys + off;
    u64 *gv = a.tvals + off;
    const int32_t *occ = hb.occ + off / 2;
    const int32_t cnt = (int32_t)hb.occ_cnt[h];
    const int stride = fc.nparts * HUB_FIN_T;
    Cand best;
    best.hi = 0; best.lo = 0; best.c = INT32_MAX;
    u64 eown = 0, n1 = 0, selfw = 0, sumw = 0;
    int32_t T = -1;
    const i64 di = (MODE == M_SWEEP) ? a.delta[r] : 0;
    for (int t = fc.j * HUB_FIN_T + threadIdx.x; t < cnt; t += stride) {
      const int32_t slot = occ[t];
      const int32_t k = gk[slot];
      const u64 v = gv[slot];
      if (MODE != M_EMIT) { gk[slot] = -1; gv[slot] = 0; }
      if (MODE == M_SWEEP) {
        if (k == own) eown = v;
        else {
          ++n1;
          i128 S = (i128)a.twoW * (i128)(i64)v - (i128)di * (i128)__ldg(&a.deg[k]);
          Cand x;
          x.hi = (i64)(S >> 64); x.lo = (u64)S; x.c = k;
          if (cand_better(x, best)) best = x;
        }
      } else if (MODE == M_MERGE) {
        if (k != own) { ++n1; T = max(T, k); }
      } else {
        sumw += v;
        if (k == r) selfw += v;
        else ++n1;
      }
    }
    if (MODE == M_EMIT) {
      // second pass: write this CTA's entries at a cursor reserved for the CTA
      u64 tot;
      Grp<HUB_FIN_T, HUB_FIN_T> g;
      const u64 pre = grp_excl_scan<HUB_FIN_T, HUB_FIN_T>(g, n1, tot);
      __shared__ u64 sbase;
      if (threadIdx.x == 0) sbase = atomicAdd(&hb.emit_cur[h], tot);
      __syncthreads();
      i64 o = (a.out_base ? a.out_base[r] : a.ptr[r]) + (i64)(sbase + pre);
      for (int t = fc.j * HUB_FIN_T + threadIdx.x; t < cnt; t += stride) {
        const int32_t slot = occ[t];
        const int32_t k = gk[slot];
        const u64 v = gv[slot];
        gk[slot] = -1;
        gv[slot] = 0;
        if (k != r && a.out_key) {
          a.out_key[o] = k;
          a.out_w[o] = v;
          ++o;
        }
      }
    }
    Grp<HUB_FIN_T, HUB_FIN_T> g;
    grp_reduce<HUB_FIN_T, HUB_FIN_T>(g, best, eown, n1, T);
    Cand none;
    none.hi = 0; none.lo = 0; none.c = INT32_MAX;
    int32_t dummy = 0;
    grp_reduce<HUB_FIN_T, HUB_FIN_T>(g, none, selfw, sumw, dummy);
    if (threadIdx.x == 0) {
      P.hi = best.hi; P.lo = best.lo; P.c = best.c; P.T = T;
      P.eown = eown; P.cnt = n1; P.selfw = selfw; P.sumw = sumw;
    }
  }
  if (threadIdx.x == 0) hb.part[hb.pstart[h] + fc.j] = P;
}

template <int MODE>
__global__ void __launch_bounds__(128) k_hub_decide(AggArgs a, HubArgs hb) {
  Acc acc;
  const i64 h = (i64)blockIdx.x * 128 + threadIdx.x;
  if (h < hb.nhub) {
    const int32_t r = a.rows[h];
    const int32_t own = (MODE == M_EMIT) ? r : a.label[r];
    Cand best;
    best.hi = 0; best.lo = 0; best.c = INT32_MAX;
    u64 eown = 0, cnt = 0, selfw = 0, sumw = 0;
    int32_t T = -1;
    const HubPartial *p = hb.part + hb.pstart[h];
    for (int j = 0; j < hb.nparts[h]; ++j) {
      Cand x;
      x.hi = p[j].hi; x.lo = p[j].lo; x.c = p[j].c;
      if (cand_better(x, best)) best = x;
      eown += p[j].eown; cnt += p[j].cnt; selfw += p[j].selfw; sumw += p[j].sumw;
      T = max(T, p[j].T);
    }
    if (MODE == M_SWEEP) {
      const i64 di = a.delta[r];
      const i64 dq = a.deg[own];
      i128 S_own = (i128)a.twoW * (i128)(i64)eown - (i128)di * ((i128)dq - (i128)di);
      int32_t tgt = own;
      if (best.c != INT32_MAX && cand_S(best) > S_own) {
        tgt = best.c;
        if (a.size[own] == 1 && a.size[best.c] == 1 && best.c > own) tgt = own;
      }
      a.label_next[r] = tgt;
      acc.moved += (tgt != own);
      acc.i2 += eown;
      acc.cand += cnt;
      acc.add_sq(a.deg[r]);
    } else if (MODE == M_MERGE) {
      int32_t tgt = own;
      if (a.size[own] == 1 && cnt == 1) tgt = (a.size[T] == 1 && T > own) ? own : T;
      a.label_next[r] = tgt;
      acc.moved += (tgt != own);
    } else {
      a.out_cnt[r] = (i64)cnt;
      if (a.out_self) a.out_self[r] = selfw;
      if (a.out_sum) a.out_sum[r] = sumw;
    }
    hb.occ_cnt[h] = 0;
    hb.emit_cur[h] = 0;
  }
  if (MODE != M_EMIT) acc.flush(a.counters);
}

// ----------------------------------------------------------------- commit
// deg_C / |C| update for every vertex whose decision differs from the snapshot
// ("remove ... insert ... atomicSub/atomicAdd").  Exact int64 atomics: the
// result is independent of their order.
__global__ void __launch_bounds__(256) k_commit(i64 n, const int32_t *__restrict__ cur,
                                                const int32_t *__restrict__ nxt, const i64 *__restrict__ delta,
                                                i64 *deg, int32_t *size) {
  for (i64 i = (i64)blockIdx.x * 256 + threadIdx.x; i < n; i += (i64)gridDim.x * 256) {
    const int32_t a = cur[i], b = nxt[i];
    if (a != b) {
      const i64 d = delta[i];
      atomicAdd((u64 *)&deg[a], (u64)(-d));
      atomicAdd((u64 *)&deg[b], (u64)d);
      atomicSub(&size[a], 1);
      atomicAdd(&size[b], 1);
    }
  }
}

}  // namespace lv
