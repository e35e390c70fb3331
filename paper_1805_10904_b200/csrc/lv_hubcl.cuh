// lv_hubcl.cuh — the local-move sweep for hub rows (> 8192 entries) on thread-block
// clusters: one row at a time per cluster, its e_{i->C} table distributed over the
// cluster's CTAs' shared memory (DSMEM) and filled with remote shared-memory atomics.
//
// Same method as every sweep kernel (Algorithm 1 body; Eq. 1, 2, 4, 5 and the
// heuristics of P:L92 / P:L95; readings D4-D8): e_{i->C} = Σ_{j∈Γ(i)} ω(i,j) per
// community C = C(j), S(C) = 2W·e_{i->C} − δ_i·deg_C, S_own = 2W·e_{i->own} −
// δ_i(deg_own − δ_i), argmax by (S desc, label asc), move iff S(best) > S_own, singlet
// rule.  What differs is where the per-row table lives.  A hub row has more distinct
// neighbouring communities than one CTA's shared memory holds (C4: 2,325 rows of 8k-406k
// entries), so the paper's block-per-vertex shared table does not fit; the
// previous design (k_hub_acc / k_hub_fin) aggregated 4096-edge chunks and merged them
// through a global-memory pool — 1.7x the algorithmic DRAM traffic (write + re-read of
// the pool).  Here the table is sharded by key hash over the CS CTAs of a cluster:
//
//  * slot owner = top lg(CS) bits of the key's multiplicative hash, slot within the
//    owner's partition = the next lg(TP) bits; TP = pow2 >= 2·len / CS (load <= 0.5);
//  * CTA q streams the row's edges beg + q·T + t + j·CS·T (coalesced), gathers the
//    packed entry of each neighbour (community key + deg_C, see lv_agg.cuh) and inserts
//    (key, ω) into the owner's partition: atom.shared::cluster.cas.b32 on the key slot,
//    red.shared::cluster.add.u32 on the value, and the claiming thread stores deg_C next
//    to the slot.  The U first-probe CASes of a batch are issued back to back so their
//    DSMEM round trips overlap;
//  * barrier.cluster (release / acquire) — every remote insert is visible;
//  * every CTA scans its own partition (TP slots), resets it, scores the candidates and
//    reduces them to one (S, label) per CTA plus e_{i->own} and the candidate count;
//  * barrier.cluster — rank 0 reads the CS partials over DSMEM and decides (sweep_decide,
//    identical to the other kernels).  The partial records are double-buffered by row
//    parity, so the next row's inserts start right after this barrier.
// Rows are pre-sorted by decreasing length and dealt round-robin to the persistent
// clusters.  No global-memory intermediate: DRAM traffic = the row streams + gathers.
// Narrow tables only (uint32 values: the caller guarantees every row sum < 2^32).
#pragma once
#include "lv_agg.cuh"

namespace lv {

constexpr int HCL_T = 1024;               // threads per CTA
constexpr int HCL_LGTP = 14;              // max slots per CTA partition (16384)
constexpr int HCL_TP = 1 << HCL_LGTP;
constexpr int HCL_U = 4;                  // edges per thread per batch
// per CTA: keys, vals, degs (4 B each per slot) + two partial records
struct HclRec {
  i64 hi;
  u64 lo;
  u64 eown;
  u64 cand;
  int32_t c, pad;
};
constexpr size_t HCL_SMEM = (size_t)HCL_TP * 12 + 2 * sizeof(HclRec) + 64;

// rows of at most this many entries fit a cluster of cs CTAs (load <= 0.5)
inline i64 hcl_max_len(int cs) { return (i64)cs * HCL_TP / 2; }

__device__ __forceinline__ uint32_t cl_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cl_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cl_count() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
// shared::cluster address of the same variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t cl_map(uint32_t sa, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(sa), "r"(rank));
  return r;
}
__device__ __forceinline__ int32_t cl_cas(uint32_t a, int32_t cmp, int32_t val) {
  int32_t old;
  asm volatile("atom.shared::cluster.cas.b32 %0, [%1], %2, %3;" : "=r"(old) : "r"(a), "r"(cmp), "r"(val) : "memory");
  return old;
}
__device__ __forceinline__ void cl_red_add(uint32_t a, uint32_t v) {
  asm volatile("red.shared::cluster.add.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void cl_red_max(uint32_t a, uint32_t v) {
  asm volatile("red.shared::cluster.max.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void cl_st(uint32_t a, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ u64 cl_ld64(uint32_t a) {
  u64 v;
  asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ int32_t cl_ld32(uint32_t a) {
  int32_t v;
  asm volatile("ld.shared::cluster.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Remote insert of (key k, weight w, deg d) into a CTA's partition (shared::cluster
// address kb of its keys; values / degs at +TP·4 / +TP·8), starting at slot s whose
// first CAS already returned `old`.  Hashing uses the row's TPR = 2^lgp slots; linear
// probing continues over the whole partition (HCL_TP slots), and a claim beyond TPR
// raises the partition's high-water mark hw so the epilogue scans it.  A partition
// that is completely full (impossible unless > HCL_TP distinct keys of one row hash to
// one CTA) sets *ovf — the pass is then reported as failed, like the pool path's
// bucket overflow — instead of probing forever.
__device__ __forceinline__ void hcl_finish(uint32_t kb, unsigned s, int32_t old, int32_t k, uint32_t w, uint32_t d,
                                           unsigned tpr, uint32_t hw, int *ovf) {
  int p = 0;
  while (old != EMPTY && old != k) {
    if (++p >= HCL_TP) {
      atomicOr(ovf, 1);
      return;
    }
    s = (s + 1) & (HCL_TP - 1);
    old = cl_cas(kb + 4 * s, EMPTY, k);
  }
  cl_red_add(kb + HCL_TP * 4 + 4 * s, w);
  if (old == EMPTY) {  // the claiming thread records deg_C
    cl_st(kb + HCL_TP * 8 + 4 * s, d);
    if (s >= tpr) cl_red_max(hw, s + 1);
  }
}

template <int CS, class WT, bool S64ALL>
__global__ void __launch_bounds__(HCL_T, 1) k_hub_cl(AggArgs a, const RowHdr *__restrict__ rows, i64 nrows, int *ovf) {
  constexpr int LGCS = CS == 16 ? 4 : CS == 8 ? 3 : CS == 4 ? 2 : CS == 2 ? 1 : 0;
  static_assert((1 << LGCS) == CS, "cluster size: power of two <= 16");
  extern __shared__ __align__(16) unsigned char sm[];
  int32_t *keys = (int32_t *)sm;
  uint32_t *vals = (uint32_t *)(sm + (size_t)HCL_TP * 4);
  uint32_t *degs = (uint32_t *)(sm + (size_t)HCL_TP * 8);
  HclRec *rec = (HclRec *)(sm + (size_t)HCL_TP * 12);
  uint32_t *hwm = (uint32_t *)(rec + 2);  // high-water mark of this partition (row-local)
  __shared__ Cand wbest[HCL_T / 32];
  __shared__ u64 weown[HCL_T / 32], wcand[HCL_T / 32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t q = cl_rank();
  for (int s = tid; s < HCL_TP; s += HCL_T) { keys[s] = EMPTY; vals[s] = 0; }
  if (tid == 0) *hwm = 0;
  // shared::cluster bases of every CTA's partition (lane r < CS holds rank r's)
  // (the partition arrays are contiguous: vals / degs at +TP·4 / +TP·8 of keys, in every
  // CTA's window)
  const uint32_t kl = saddr(keys), rl = saddr(rec), hl = saddr(hwm);
  const uint32_t kb_r = lane < CS ? cl_map(kl, lane) : 0u;
  const uint32_t hw_r = lane < CS ? cl_map(hl, lane) : 0u;
  cl_sync();  // every partition initialised before any remote insert
  const u64 pf = l2_policy_first();
  const u64 *__restrict__ ldeg = a.ldeg;
  const i64 ncl = cl_count();
  Acc acc;
  int par = 0;
  for (i64 idx = cl_id(); idx < nrows; idx += ncl) {
    const RowHdr hd = rows[idx];
    const int32_t r = hd.r;
    const int len = hd.len;
    // partition size: TP = pow2 >= 2·len / CS (>= 32)
    int lgt = 64 - __clzll((unsigned long long)(2 * (i64)len - 1));  // 2^lgt >= 2·len
    int lgp = lgt - LGCS;
    lgp = lgp < 5 ? 5 : (lgp > HCL_LGTP ? HCL_LGTP : lgp);
    const unsigned mask = (1u << lgp) - 1u;
    const int sh = 32 - LGCS - lgp;
    const bool decider = q == 0 && tid == 0;
    i64 dq = 0, dr = 0, di = 0;
    int32_t own = 0;
    {
      const u64 pr = __ldg(&ldeg[r]);
      own = (int32_t)(uint32_t)pr;
      di = __ldg(&a.delta[r]);
      if (decider) {
        dq = deg_of(a, (uint32_t)(pr >> 32), key_label(own));
        dr = load_deg(a, r);
      }
    }
    // ---- insert phase
    const int32_t *col = a.keys + hd.beg;
    const void *wp = WT::bytes == 4 ? (const void *)((const uint32_t *)a.w + hd.beg)
                   : WT::bytes == 8 ? (const void *)((const u64 *)a.w + hd.beg) : nullptr;
    constexpr int STRIDE = CS * HCL_T;
    // warp-uniform trip count (the owner-base shuffles below need every lane)
    for (int b0 = (int)q * HCL_T + wid * 32; b0 < len; b0 += STRIDE * HCL_U) {
      const int t0 = b0 + lane;
      int32_t k[HCL_U];
      uint32_t w[HCL_U], d[HCL_U];
#pragma unroll
      for (int u = 0; u < HCL_U; ++u) {
        const int t = t0 + u * STRIDE;
        k[u] = t < len ? ld_stream(col + t, pf) : EMPTY;
        w[u] = 0u;
        if (t < len) {
          if (WT::bytes == 0) w[u] = 1u;
          else if (WT::bytes == 4) w[u] = ld_stream((const uint32_t *)wp + t, pf);
          else w[u] = (uint32_t)ld_stream((const u64 *)wp + t, pf);
        }
      }
#pragma unroll
      for (int u = 0; u < HCL_U; ++u) {
        const u64 p = k[u] != EMPTY ? __ldg(&ldeg[k[u]]) : 0ull;
        d[u] = (uint32_t)(p >> 32);
        k[u] = k[u] != EMPTY ? (int32_t)(uint32_t)p : EMPTY;
      }
      unsigned s[HCL_U];
      uint32_t kb[HCL_U], hw[HCL_U];
      int32_t old[HCL_U];
#pragma unroll
      for (int u = 0; u < HCL_U; ++u) {
        const uint32_t h = (uint32_t)k[u] * 0x9E3779B1u;
        const int o = LGCS ? (int)(h >> (32 - LGCS)) : 0;
        s[u] = (h >> sh) & mask;
        kb[u] = __shfl_sync(0xffffffffu, kb_r, o);
        hw[u] = __shfl_sync(0xffffffffu, hw_r, o);
        old[u] = k[u] != EMPTY ? cl_cas(kb[u] + 4 * s[u], EMPTY, k[u]) : 0;  // first probes in flight together
      }
#pragma unroll
      for (int u = 0; u < HCL_U; ++u)
        if (k[u] != EMPTY) hcl_finish(kb[u], s[u], old[u], k[u], w[u], d[u], mask + 1u, hw[u], ovf);
    }
    cl_sync();  // S1: the row's inserts are complete and visible in every partition
    // ---- epilogue over this CTA's partition
    const bool s64 = S64ALL || row_s64(a.twoW, di);  // cluster-uniform
    Cand best = s64 ? cand_none64() : cand_none();
    u64 eown = 0, ncand = 0;
    const int tp = max(1 << lgp, (int)*hwm);  // + slots claimed beyond the row's range
    for (int sl = tid; sl < tp; sl += HCL_T) {
      const int32_t kk = keys[sl];
      if (kk == EMPTY) continue;
      const u64 v = vals[sl];
      const uint32_t d31 = degs[sl];
      keys[sl] = EMPTY;
      vals[sl] = 0;
      if (kk == own) {
        eown = v;
      } else {
        ++ncand;
        if (s64) cand_push<true>(best, a.twoW, di, kk, v, deg_of(a, d31, key_label(kk)));
        else cand_push<false>(best, a.twoW, di, kk, v, deg_of(a, d31, key_label(kk)));
      }
    }
    // CTA reduction: warp argmax / sums, then warp 0 over the 32 warps
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      Cand y;
      y.lo = __shfl_xor_sync(0xffffffffu, best.lo, o);
      y.hi = __shfl_xor_sync(0xffffffffu, best.hi, o);
      y.c = __shfl_xor_sync(0xffffffffu, best.c, o);
      if (s64 ? cand_better64(y, best) : cand_better(y, best)) best = y;
      eown += __shfl_xor_sync(0xffffffffu, eown, o);
      ncand += __shfl_xor_sync(0xffffffffu, ncand, o);
    }
    if (lane == 0) { wbest[wid] = best; weown[wid] = eown; wcand[wid] = ncand; }
    __syncthreads();
    if (tid == 0) *hwm = 0;  // every thread read it before the barrier above
    HclRec *R = rec + par;
    if (wid == 0) {
      best = wbest[lane];
      eown = weown[lane];
      ncand = wcand[lane];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        Cand y;
        y.lo = __shfl_xor_sync(0xffffffffu, best.lo, o);
        y.hi = __shfl_xor_sync(0xffffffffu, best.hi, o);
        y.c = __shfl_xor_sync(0xffffffffu, best.c, o);
        if (s64 ? cand_better64(y, best) : cand_better(y, best)) best = y;
        eown += __shfl_xor_sync(0xffffffffu, eown, o);
        ncand += __shfl_xor_sync(0xffffffffu, ncand, o);
      }
      if (lane == 0) {
        R->hi = best.hi; R->lo = best.lo; R->c = best.c; R->eown = eown; R->cand = ncand;
      }
    }
    cl_sync();  // S2: partials visible; every partition reset (next row may insert)
    if (decider) {
      const uint32_t rb = rl + (uint32_t)(par * sizeof(HclRec));
      best.hi = R->hi; best.lo = R->lo; best.c = R->c;
      eown = R->eown;
      ncand = R->cand;
      for (int o = 1; o < CS; ++o) {
        const uint32_t ra = cl_map(rb, o);
        Cand y;
        y.hi = (i64)cl_ld64(ra + offsetof(HclRec, hi));
        y.lo = cl_ld64(ra + offsetof(HclRec, lo));
        y.c = cl_ld32(ra + offsetof(HclRec, c));
        eown += cl_ld64(ra + offsetof(HclRec, eown));
        ncand += cl_ld64(ra + offsetof(HclRec, cand));
        if (s64 ? cand_better64(y, best) : cand_better(y, best)) best = y;
      }
      if (s64) {
        best.hi = (i64)best.lo >> 63;
        sweep_decide<true>(a, acc, r, own, di, dq, dr, best, eown);
      } else {
        sweep_decide<false>(a, acc, r, own, di, dq, dr, best, eown);
      }
      acc.cand += ncand;
    }
    par ^= 1;
  }
  // rank 0's reads of the last row's partials must finish before any CTA of the cluster
  // exits (its shared memory would go away)
  cl_sync();
  acc.flush(a.counters);
}

}  // namespace lv
