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
  const int32_t *keys;     // SWEEP/MERGE: col[] (key = label[col]); EMIT: key directly
  const void *w;           // weights (WT)
  const int32_t *label;    // snapshot labels C
  int32_t *label_next;     // decisions
  const i64 *deg;          // deg_C, indexed by label (snapshot)
  const uint32_t *deg32;   // min(deg_C, 2^32-1): the gathered copy (half the bytes);
                           // 0xFFFFFFFF means "read deg" (at most one community: Σ deg = 2W)
  const int32_t *size;     // |C|, indexed by label (snapshot)
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
};

__device__ __forceinline__ void store_w(const AggArgs &a, i64 o, u64 v) {
  if (a.out_wnone) return;
  if (a.out_w32) ((uint32_t *)a.out_w)[o] = (uint32_t)v;
  else ((u64 *)a.out_w)[o] = v;
}

// deg_C through the 32-bit mirror (exact: saturated entries fall back to the 64-bit array)
__device__ __forceinline__ i64 load_deg(const AggArgs &a, int32_t c) {
  const uint32_t d = __ldg(&a.deg32[c]);
  return d != 0xFFFFFFFFu ? (i64)d : __ldg(&a.deg[c]);
}

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
// VT = table value type: uint32_t when the caller has proved every row sum < 2^32
// (native 32-bit atomics, 9 B per shared slot), else u64.
template <bool SHARED, class VT>
__device__ __forceinline__ unsigned tab_insert(int32_t *keys, VT *vals, unsigned mask, int lg, int32_t k, u64 v,
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
  if (sizeof(VT) == 4) atomicAdd((uint32_t *)&vals[h], (uint32_t)v);
  else if (SHARED) add_u64_split((u64 *)&vals[h], v);
  else atomicAdd((u64 *)&vals[h], v);
  return h;
}

// Exact move score S = 2W·v − δ·deg (Eq. 4 scaled by 2W², reading D4); all four
// operands are non-negative, so two 64x64->128 unsigned products suffice.
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
// col/w loads and then the label gathers of a batch are independent and in flight
// together (memory-level parallelism; the atomics would otherwise serialise them).
template <int G, int U, int MODE, class WT, bool SHARED, bool LIST, class VT>
__device__ __forceinline__ void insert_range(const AggArgs &a, int lane, i64 beg, i64 end, int32_t *keys, VT *vals,
                                             unsigned mask, int lg, uint16_t *olist, int *ocnt) {
  const u64 pf = l2_policy_first(), pl = l2_policy_last();
  // lane-uniform trip count (every lane of the group runs every batch): required by the
  // warp-synchronous pre-aggregation below
  for (i64 b0 = beg; b0 < end; b0 += (i64)G * U) {
    const i64 e0 = b0 + lane;
    int32_t k[U];
    u64 wv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const i64 e = e0 + (i64)u * G;
      k[u] = -1;
      wv[u] = 0;
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
        if (k[u] >= 0) k[u] = (a.hint & 2) ? ld_keep(&a.label[k[u]], pl) : __ldg(&a.label[k[u]]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const u64 wsum = wv[u];
      if (k[u] < 0) continue;
      bool claimed = false;
      const unsigned sl = tab_insert<SHARED, VT>(keys, vals, mask, lg, k[u], wsum, LIST ? &claimed : nullptr);
      if (LIST && claimed) olist[atomicAdd(ocnt, 1)] = (uint16_t)sl;
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

struct Cand {  // lexicographic key (S desc, c asc); c == INT32_MAX means "none"
  i64 hi;
  u64 lo;
  int32_t c;
  int32_t sg;  // |C| == 1 (singlet rule), carried with the candidate
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

// Record a move own -> tgt of vertex r (weighted degree di) in the next-state deg/size
// ("remove ... from the old community ... insert ... into the new").
// (In the sweep-sharded mode deg_next is NULL: every rank applies all moves after the
// label exchange instead, see k_apply_moves.)
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
  int32_t szo = 0;     // |own|
};

// Visits the row's occupied entries — by scanning slots [0,n) (LIST = false) or through
// the occupied-slot list olist[0..n) (LIST = true) — resets every slot it reads, and
// applies the mode's epilogue.  Both EMIT passes visit entries in the same order.
template <int G, int BLOCK, int MODE, bool LIST, class SlotT, class VT>
__device__ __forceinline__ void row_epilogue(const Grp<G, BLOCK> &g, int32_t *keys, VT *vals, const SlotT *olist,
                                             i64 n, int32_t r, int32_t own, i64 di, const RowPre &pre,
                                             const AggArgs &a, Acc &acc) {
  constexpr int U = G < 32 ? 2 : 4;  // entries per lane per batch: their deg_C gathers overlap
  if (MODE == M_SWEEP) {
    Cand best;
    best.hi = 0; best.lo = 0; best.c = INT32_MAX; best.sg = 0;
    u64 eown = 0, ncand = 0;
    int32_t dummy = 0;
    for (i64 t0 = g.lane; t0 < n; t0 += (i64)G * U) {
      int32_t sl[U], k[U];
      u64 v[U];
      i64 dk[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const i64 t = t0 + (i64)u * G;
        sl[u] = t < n ? (LIST ? (int32_t)olist[t] : (int32_t)t) : -1;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        k[u] = sl[u] >= 0 ? keys[sl[u]] : -1;
        v[u] = 0;
        if (k[u] >= 0) {
          v[u] = (u64)vals[sl[u]];
          keys[sl[u]] = -1;
          vals[sl[u]] = 0;
        }
      }
#pragma unroll
#pragma unroll
      for (int u = 0; u < U; ++u)
        dk[u] = (k[u] >= 0 && k[u] != own) ? load_deg(a, k[u]) : 0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (k[u] < 0) continue;
        if (k[u] == own) {
          eown = v[u];
        } else {
          ++ncand;
          const i128 S = move_score(a.twoW, v[u], di, dk[u]);
          Cand x;
          x.hi = (i64)(S >> 64); x.lo = (u64)S; x.c = k[u];
          if (cand_better(x, best)) best = x;
        }
      }
    }
    grp_reduce<G, BLOCK>(g, best, eown, ncand, dummy);
    if (g.lane == 0) {
      i128 S_own = (i128)a.twoW * (i128)(i64)eown - (i128)di * ((i128)pre.dq - (i128)di);
      int32_t tgt = own;
      if (best.c != INT32_MAX && cand_S(best) > S_own) {
        tgt = best.c;
        if (pre.szo == 1 && best.c > own && a.size[best.c] == 1) tgt = own;  // singlet rule (D8)
      }
      a.label_next[r] = tgt;
      if (tgt != own) record_move(a, own, tgt, di);
      acc.moved += (tgt != own);
      acc.i2 += eown;
      acc.cand += ncand;
      acc.add_sq(pre.dr);  // deg of label index r: Σ over all labels gives S2
    }
  } else if (MODE == M_MERGE) {
    Cand none;
    none.hi = 0; none.lo = 0; none.c = INT32_MAX; none.sg = 0;
    u64 cnt = 0, unused = 0;
    int32_t T = -1;
    for (i64 t = g.lane; t < n; t += G) {
      const int32_t sl = LIST ? (int32_t)olist[t] : (int32_t)t;
      const int32_t k = keys[sl];
      if (k >= 0) {
        keys[sl] = -1;
        vals[sl] = 0;
        if (k != own) { ++cnt; T = max(T, k); }
      }
    }
    grp_reduce<G, BLOCK>(g, none, cnt, unused, T);
    if (g.lane == 0) {
      int32_t tgt = own;
      if (cnt == 1) tgt = (a.size[T] == 1 && T > own) ? own : T;
      a.label_next[r] = tgt;
      if (tgt != own) record_move(a, own, tgt, a.delta[r]);
      acc.moved += (tgt != own);
    }
  } else {  // M_EMIT
    u64 c = 0, selfw = 0, sumw = 0;
    for (i64 t = g.lane; t < n; t += G) {
      const int32_t sl = LIST ? (int32_t)olist[t] : (int32_t)t;
      const int32_t k = keys[sl];
      if (k >= 0) {
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
      if (k >= 0) {
        const u64 v = (u64)vals[sl];
        keys[sl] = -1;
        vals[sl] = 0;
        if (k != r && a.out_key) {
          a.out_key[o] = k;
          store_w(a, o, v);
          ++o;
        }
      }
    }
    Cand none;
    none.hi = 0; none.lo = 0; none.c = INT32_MAX; none.sg = 0;
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
// Tables of CAP >= 256 slots keep an occupied-slot list (uint16 indices) so the
// epilogue costs O(distinct keys), not O(capacity).
template <int CAP>
constexpr bool has_list() { return CAP >= 256; }
template <int G, int CAP, int BLOCK, class VT>
constexpr size_t smem_bytes() {
  return (size_t)(BLOCK / G) * ((size_t)CAP * (sizeof(VT) + sizeof(int32_t)) + (has_list<CAP>() ? CAP : 0) + 16);
}

template <int G, int CAP, int BLOCK, int MODE, class WT, class VT>
__global__ void __launch_bounds__(BLOCK) k_agg_smem(AggArgs a) {
  constexpr int GPB = BLOCK / G;
  constexpr bool LIST = has_list<CAP>();
  constexpr int LG = (CAP >= 65536) ? 16 : (CAP >= 32768) ? 15 : (CAP >= 16384) ? 14 : (CAP >= 8192) ? 13
                   : (CAP >= 4096) ? 12 : (CAP >= 2048) ? 11 : (CAP >= 1024) ? 10 : (CAP >= 512) ? 9
                   : (CAP >= 256) ? 8 : (CAP >= 128) ? 7 : (CAP >= 64) ? 6 : (CAP >= 32) ? 5
                   : (CAP >= 16) ? 4 : 3;
  static_assert((1 << LG) == CAP, "CAP must be a power of two >= 8");
  extern __shared__ __align__(16) unsigned char sm[];
  constexpr size_t SB = sizeof(VT) + sizeof(int32_t);
  VT *svals = (VT *)sm;
  int32_t *skeys = (int32_t *)(sm + (size_t)GPB * CAP * sizeof(VT));
  uint16_t *slist = (uint16_t *)(sm + (size_t)GPB * CAP * SB);
  int *scnt = (int *)(sm + (size_t)GPB * CAP * SB + (LIST ? (size_t)GPB * CAP : 0));
  Grp<G, BLOCK> g;
  const int grp = threadIdx.x / G;
  int32_t *keys = skeys + grp * CAP;
  VT *vals = svals + grp * CAP;
  uint16_t *olist = slist + grp * (CAP / 2);
  int *ocnt = scnt + grp;
  Acc acc;
  for (int s = g.lane; s < CAP; s += G) { keys[s] = -1; vals[s] = 0; }
  if (LIST && g.lane == 0) *ocnt = 0;
  g.sync();
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
    const int32_t own = (MODE == M_EMIT) ? r : a.label[r];
    const i64 di = (MODE == M_SWEEP) ? a.delta[r] : 0;
    RowPre pre;
    if (MODE == M_SWEEP && g.lane == 0) {  // issued before the edge loop: overlaps it
      pre.dq = load_deg(a, own);
      pre.dr = load_deg(a, r);
      pre.szo = __ldg(&a.size[own]);
    }
    if (MODE == M_MERGE) {
      if (a.size[own] != 1) {
        if (g.lane == 0) a.label_next[r] = own;
        continue;
      }
    }
    const int lg = row_lg(end - beg, LG);  // table prefix sized for this row
    const unsigned mask = (1u << lg) - 1u;
    insert_range<G, (G >= 64 ? 8 : (G == 32 ? 4 : 1)), MODE, WT, true, LIST, VT>(a, g.lane, beg, end, keys, vals, mask,
                                                                                lg, olist, ocnt);
    g.sync();
    const i64 n = LIST ? (i64)(*(volatile int *)ocnt) : ((i64)1 << lg);
    row_epilogue<G, BLOCK, MODE, LIST>(g, keys, vals, olist, n, r, own, di, pre, a, acc);
    g.sync();
    if (LIST && g.lane == 0) *ocnt = 0;
    g.sync();
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
    const int32_t own = (MODE == M_EMIT) ? r : a.label[r];
    i64 di = 0, dq = 0, dr = 0;
    int32_t szo = 0;
    if (MODE == M_SWEEP) {
      di = a.delta[r];
      if (g.lane == 0) {
        dq = load_deg(a, own);
        dr = load_deg(a, r);
        szo = __ldg(&a.size[own]);
      }
    }
    if (MODE == M_MERGE) {
      if (a.size[own] != 1) {
        if (g.lane == 0) a.label_next[r] = own;
        continue;
      }
    }
    int32_t k = -1;
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
      if (MODE != M_EMIT) k = __ldg(&a.label[k]);
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
      lead = first && k >= 0;
    } else {
      const unsigned peers = __match_any_sync(g.mask, k);
      lead = (__ffs(peers) - 1) == wl && k >= 0;
      sum = __reduce_add_sync(peers, (uint32_t)w);
    }
    if (MODE == M_SWEEP) {
      Cand best;
      best.hi = 0; best.lo = 0; best.c = INT32_MAX; best.sg = 0;
      u64 eown = 0, ncand = 0;
      int32_t dummy = 0;
      if (lead) {
        if (k == own) {
          eown = sum;
        } else {
          ncand = 1;
          const i64 dk = load_deg(a, k);
          const i128 S = move_score(a.twoW, sum, di, dk);
          best.hi = (i64)(S >> 64); best.lo = (u64)S; best.c = k;
        }
      }
      grp_reduce<G, BLOCK>(g, best, eown, ncand, dummy);
      if (g.lane == 0) {
        const i128 S_own = (i128)a.twoW * (i128)(i64)eown - (i128)di * ((i128)dq - (i128)di);
        int32_t tgt = own;
        if (best.c != INT32_MAX && cand_S(best) > S_own) {
          tgt = best.c;
          if (szo == 1 && best.c > own && a.size[best.c] == 1) tgt = own;  // singlet rule (D8)
        }
        a.label_next[r] = tgt;
        if (tgt != own) record_move(a, own, tgt, di);
        acc.moved += (tgt != own);
        acc.i2 += eown;
        acc.cand += ncand;
        acc.add_sq(dr);
      }
    } else if (MODE == M_MERGE) {
      Cand none;
      none.hi = 0; none.lo = 0; none.c = INT32_MAX; none.sg = 0;
      u64 cnt = (lead && k != own) ? 1 : 0, unused = 0;
      int32_t T = (lead && k != own) ? k : -1;
      grp_reduce<G, BLOCK>(g, none, cnt, unused, T);
      if (g.lane == 0) {
        int32_t tgt = own;
        if (cnt == 1) tgt = (a.size[T] == 1 && T > own) ? own : T;
        a.label_next[r] = tgt;
        if (tgt != own) record_move(a, own, tgt, a.delta[r]);
        acc.moved += (tgt != own);
      }
    } else {  // M_EMIT: distinct keys != r written compactly at out_base[r]
      const bool emit = lead && k != r;
      const unsigned bal = __ballot_sync(g.mask, emit) & g.mask;
      if (emit && a.out_key) {
        const i64 o = (a.out_base ? a.out_base[r] : a.ptr[r]) + __popc(bal & ((1u << wl) - 1u));
        a.out_key[o] = k;
        store_w(a, o, sum);
      }
      Cand none;
      none.hi = 0; none.lo = 0; none.c = INT32_MAX; none.sg = 0;
      u64 selfw = (lead && k == r) ? sum : 0, sumw = lead ? sum : 0;
      int32_t dummy = 0;
      grp_reduce<G, BLOCK>(g, none, selfw, sumw, dummy);
      if (g.lane == 0) {
        a.out_cnt[r] = (i64)__popc(bal);
        if (a.out_self) a.out_self[r] = selfw;
        if (a.out_sum) a.out_sum[r] = sumw;
      }
    }
  }
  if (MODE != M_EMIT) acc.flush(a.counters);
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
constexpr int HUB_FIN_TILE = 1024; // chunks staged per pass in k_hub_fin

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
  int32_t *pkey;          // pool: chunk c of this batch owns [(c - c0) * HUB_CHUNK, +HUB_CHUNK)
  void *pval;             // pool values: uint32 when VT is 32-bit, else u64
  i64 c0, c1;             // chunk range of this batch (hub rows are processed in batches
  i64 f0, f1;             //   bounding the pool); fin-item range of the same rows
  i64 h0, h1;             // hub range of the batch
  const int2 *fitem;      // per fin item: (hub, bucket)
  HubPartial *part;       // per fin item
  u64 *emit_cur;          // per hub (EMIT output cursor)
  int *overflow;          // set if a bucket exceeds its distinct-key capacity
  i64 nhub, nchunks, nfin;
  int fin_lg;             // bucket table log2 capacity of this launch
};

template <class VT>
constexpr size_t hub_acc_smem(int max_blg) {
  return (size_t)(1 << HUB_SM_LG) * (sizeof(VT) + sizeof(int32_t)) + (size_t)HUB_CHUNK * sizeof(uint16_t) +
         (size_t)((1 << max_blg) + 1) * sizeof(int) + 64;
}
template <class VT>
constexpr size_t hub_fin_smem(int fin_lg) {
  return ((size_t)1 << fin_lg) * (sizeof(VT) + sizeof(int32_t)) + ((size_t)1 << (fin_lg - 1)) * sizeof(uint16_t) +
         (size_t)HUB_FIN_TILE * (sizeof(i64) + sizeof(int)) + 64;
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
  VT *svals = (VT *)sm;
  int32_t *skeys = (int32_t *)(sm + (size_t)CAPS * sizeof(VT));
  uint16_t *slist = (uint16_t *)(sm + (size_t)CAPS * (sizeof(VT) + sizeof(int32_t)));
  int *hist = (int *)(sm + (size_t)CAPS * (sizeof(VT) + sizeof(int32_t)) + (size_t)HUB_CHUNK * sizeof(uint16_t));
  __shared__ int scnt;
  for (int s = threadIdx.x; s < CAPS; s += HUB_ACC_T) { skeys[s] = -1; svals[s] = 0; }
  if (threadIdx.x == 0) scnt = 0;
  __syncthreads();
  VT *pv = (VT *)hb.pval;
  for (i64 ci = hb.c0 + blockIdx.x; ci < hb.c1; ci += gridDim.x) {
    const Chunk ch = a.chunks[ci];
    const int32_t r = a.rows[ch.h];
    if (MODE == M_MERGE) {
      if (a.size[a.label[r]] != 1) continue;  // CTA-uniform
    }
    const int blg = hb.blg[ch.h];
    const int nb = 1 << blg;
    for (int b = threadIdx.x; b <= nb; b += HUB_ACC_T) hist[b] = 0;
    insert_range<HUB_ACC_T, 8, MODE, WT, true, true, VT>(a, threadIdx.x, ch.beg, ch.end, skeys, svals, CAPS - 1,
                                                         HUB_SM_LG, slist, &scnt);
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
      hb.pkey[base + pos] = k;
      pv[base + pos] = svals[sl];
      skeys[sl] = -1;
      svals[sl] = 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) scnt = 0;
    __syncthreads();
  }
}

// Persistent over (row, bucket) items; table reset through the occupied list.
template <int MODE, class VT>
__global__ void __launch_bounds__(HUB_FIN_T) k_hub_fin(AggArgs a, HubArgs hb) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int FLG = hb.fin_lg;
  const int CAPF = 1 << FLG;
  const int MAXD = CAPF / 2;
  VT *svals = (VT *)sm;
  int32_t *skeys = (int32_t *)(sm + (size_t)CAPF * sizeof(VT));
  uint16_t *slist = (uint16_t *)(sm + (size_t)CAPF * (sizeof(VT) + sizeof(int32_t)));
  i64 *tst = (i64 *)(sm + (size_t)CAPF * (sizeof(VT) + sizeof(int32_t)) + (size_t)MAXD * sizeof(uint16_t));
  int *tlen = (int *)(tst + HUB_FIN_TILE);
  __shared__ int scnt, sovf;
  __shared__ u64 sbase;
  for (int s = threadIdx.x; s < CAPF; s += HUB_FIN_T) { skeys[s] = -1; svals[s] = 0; }
  if (threadIdx.x == 0) { scnt = 0; sovf = 0; }
  __syncthreads();
  Grp<HUB_FIN_T, HUB_FIN_T> g;
  for (i64 fi = hb.f0 + blockIdx.x; fi < hb.f1; fi += gridDim.x) {
    const int2 it = hb.fitem[fi];
    const int h = it.x, b = it.y;
    const int32_t r = a.rows[h];
    const int32_t own = (MODE == M_EMIT) ? r : a.label[r];
    HubPartial P;
    P.hi = 0; P.lo = 0; P.c = INT32_MAX; P.T = -1; P.sg = 0; P.pad = 0;
    P.eown = 0; P.cnt = 0; P.selfw = 0; P.sumw = 0;
    if (MODE == M_MERGE && a.size[own] != 1) {  // CTA-uniform
      if (threadIdx.x == 0) hb.part[fi] = P;
      continue;
    }
    const i64 cf = hb.cfirst[h];
    const int nch = hb.ccount[h];
    for (int t0 = 0; t0 < nch; t0 += HUB_FIN_TILE) {
      const int m = min(HUB_FIN_TILE, nch - t0);
      for (int j = threadIdx.x; j < m; j += HUB_FIN_T) {
        const i64 c = cf + t0 + j;
        const int32_t *seg = hb.seg + hb.segoff[c];
        const int s0 = seg[b], s1 = seg[b + 1];
        tlen[j] = s1 - s0;
        tst[j] = (c - hb.c0) * HUB_CHUNK + s0;
      }
      __syncthreads();
      const int total = smem_excl_scan<HUB_FIN_T>(tlen, m);  // tlen[j] = prefix
      for (int i = threadIdx.x; i < total; i += HUB_FIN_T) {
        int lo = 0, hi = m - 1;  // last j with tlen[j] <= i
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (tlen[mid] <= i) lo = mid;
          else hi = mid - 1;
        }
        const i64 e = tst[lo] + (i - tlen[lo]);
        const int32_t k = hb.pkey[e];
        const u64 v = (u64)((const VT *)hb.pval)[e];
        if (*(volatile int *)&scnt >= MAXD - 1) { sovf = 1; continue; }
        bool claimed = false;
        const unsigned sl = tab_insert<true, VT>(skeys, svals, CAPF - 1, FLG, k, v, &claimed);
        if (claimed) {
          const int q = atomicAdd(&scnt, 1);
          if (q < MAXD) slist[q] = (uint16_t)sl;
          else sovf = 1;
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
      constexpr int U = 4;
      Cand best;
      best.hi = 0; best.lo = 0; best.c = INT32_MAX; best.sg = 0;
      u64 eown = 0, n1 = 0;
      int32_t dm = 0;
      for (int t0 = threadIdx.x; t0 < n; t0 += HUB_FIN_T * U) {
        int32_t sl[U], k[U];
        u64 v[U];
        i64 dk[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int t = t0 + u * HUB_FIN_T;
          sl[u] = t < n ? (int32_t)slist[t] : -1;
          k[u] = sl[u] >= 0 ? skeys[sl[u]] : -1;
          v[u] = sl[u] >= 0 ? (u64)svals[sl[u]] : 0;
          if (sl[u] >= 0) { skeys[sl[u]] = -1; svals[sl[u]] = 0; }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          dk[u] = (k[u] >= 0 && k[u] != own) ? load_deg(a, k[u]) : 0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (k[u] < 0) continue;
          if (k[u] == own) {
            eown = v[u];
          } else {
            ++n1;
            const i128 S = move_score(a.twoW, v[u], di, dk[u]);
            Cand x;
            x.hi = (i64)(S >> 64); x.lo = (u64)S; x.c = k[u];
            if (cand_better(x, best)) best = x;
          }
        }
      }
      grp_reduce<HUB_FIN_T, HUB_FIN_T>(g, best, eown, n1, dm);
      if (threadIdx.x == 0) { P.hi = best.hi; P.lo = best.lo; P.c = best.c; P.eown = eown; P.cnt = n1; }
    } else if (MODE == M_MERGE) {
      Cand none;
      none.hi = 0; none.lo = 0; none.c = INT32_MAX; none.sg = 0;
      u64 n1 = 0, unused = 0;
      int32_t T = -1;
      for (int i = threadIdx.x; i < n; i += HUB_FIN_T) {
        const int sl = slist[i];
        const int32_t k = skeys[sl];
        skeys[sl] = -1;
        svals[sl] = 0;
        if (k != own) { ++n1; T = max(T, k); }
      }
      grp_reduce<HUB_FIN_T, HUB_FIN_T>(g, none, n1, unused, T);
      if (threadIdx.x == 0) { P.cnt = n1; P.T = T; }
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
      Cand none;
      none.hi = 0; none.lo = 0; none.c = INT32_MAX; none.sg = 0;
      int32_t dm = 0;
      grp_reduce<HUB_FIN_T, HUB_FIN_T>(g, none, selfw, sumw, dm);
      if (threadIdx.x == 0) { P.cnt = tot; P.selfw = selfw; P.sumw = sumw; }
    }
    if (threadIdx.x == 0) hb.part[fi] = P;
    __syncthreads();
    if (threadIdx.x == 0) { scnt = 0; sovf = 0; }
    __syncthreads();
  }
}

template <int MODE>
__global__ void __launch_bounds__(128) k_hub_decide(AggArgs a, HubArgs hb) {
  Acc acc;
  const i64 h = hb.h0 + (i64)blockIdx.x * 128 + threadIdx.x;
  if (h < hb.h1) {
    const int32_t r = a.rows[h];
    const int32_t own = (MODE == M_EMIT) ? r : a.label[r];
    Cand best;
    best.hi = 0; best.lo = 0; best.c = INT32_MAX; best.sg = 0;
    u64 eown = 0, cnt = 0, selfw = 0, sumw = 0;
    int32_t T = -1;
    const HubPartial *p = hb.part + hb.bfirst[h];
    const int np = 1 << hb.blg[h];
    for (int j = 0; j < np; ++j) {
      Cand x;
      x.hi = p[j].hi; x.lo = p[j].lo; x.c = p[j].c; x.sg = p[j].sg;
      if (cand_better(x, best)) best = x;
      eown += p[j].eown; cnt += p[j].cnt; selfw += p[j].selfw; sumw += p[j].sumw;
      T = max(T, p[j].T);
    }
    if (MODE == M_SWEEP) {
      const i64 di = a.delta[r];
      const i64 dq = load_deg(a, own);
      i128 S_own = (i128)a.twoW * (i128)(i64)eown - (i128)di * ((i128)dq - (i128)di);
      int32_t tgt = own;
      if (best.c != INT32_MAX && cand_S(best) > S_own) {
        tgt = best.c;
        if (a.size[own] == 1 && a.size[best.c] == 1 && best.c > own) tgt = own;
      }
      a.label_next[r] = tgt;
      if (tgt != own) record_move(a, own, tgt, di);
      acc.moved += (tgt != own);
      acc.i2 += eown;
      acc.cand += cnt;
      acc.add_sq(load_deg(a, r));
    } else if (MODE == M_MERGE) {
      int32_t tgt = own;
      if (a.size[own] == 1 && cnt == 1) tgt = (a.size[T] == 1 && T > own) ? own : T;
      a.label_next[r] = tgt;
      if (tgt != own) record_move(a, own, tgt, a.delta[r]);
      acc.moved += (tgt != own);
    } else {
      a.out_cnt[r] = (i64)cnt;
      if (a.out_self) a.out_self[r] = selfw;
      if (a.out_sum) a.out_sum[r] = sumw;
    }
    hb.emit_cur[h] = 0;
  }
  if (MODE != M_EMIT) acc.flush(a.counters);
}

// Apply every move cur -> nxt to the next-state deg/size (sweep-sharded mode: run
// identically on every rank after the label exchange; exact atomics, order-free).
__global__ void __launch_bounds__(256) k_apply_moves(i64 n, const int32_t *__restrict__ cur,
                                                     const int32_t *__restrict__ nxt, const i64 *__restrict__ delta,
                                                     i64 *deg_next, int32_t *size_next) {
  for (i64 i = (i64)blockIdx.x * 256 + threadIdx.x; i < n; i += (i64)gridDim.x * 256) {
    const int32_t a = cur[i], b = nxt[i];
    if (a != b) {
      const i64 d = delta[i];
      atomicAdd((u64 *)&deg_next[a], (u64)(-d));
      atomicAdd((u64 *)&deg_next[b], (u64)d);
      atomicSub(&size_next[a], 1);
      atomicAdd(&size_next[b], 1);
    }
  }
}

// deg32[c] = min(deg[c], 2^32 - 1) (the gathered mirror of deg_C)
__global__ void __launch_bounds__(256) k_deg32(i64 n, const i64 *__restrict__ deg, uint32_t *deg32) {
  for (i64 c = (i64)blockIdx.x * 256 + threadIdx.x; c < n; c += (i64)gridDim.x * 256) {
    const i64 d = deg[c];
    deg32[c] = d >= (i64)0xFFFFFFFF ? 0xFFFFFFFFu : (uint32_t)d;
  }
}

}  // namespace lv
