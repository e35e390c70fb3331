// lv_sweep.cuh — the local-move sweep kernel for rows of 33..8192 entries (the bulk of
// every sweep's edges: 89 % at C4 level 0), specialised for the sweep epilogue.
//
// Same method as k_agg_smem<M_SWEEP> (lv_agg.cuh; Algorithm 1 body, Eq. 1,
// 2, 4, 5 + the heuristics of P:L92/P:L95, readings D4-D8): for row i, e_{i->C} per
// neighbouring community C in a shared-memory open-addressing table, then the exact
// scores S(C) = 2W·e_{i->C} − δ_i·deg_C and S_own = 2W·e_{i->own} − δ_i(deg_own − δ_i),
// argmax by (S desc, label asc), move iff S(best) > S_own, singlet rule.  What differs is
// the work decomposition, chosen to cut the per-row instruction overhead (r1 ncu:
// 10.3 warp instructions per edge in the CTA-per-row kernels, ~940 per warp and row):
//
//  * a GROUP of WARPS warps owns one table and sweeps one row at a time; rows of a bin
//    get the fewest warps whose table fits (1 warp per row up to 512 entries), so each
//    warp handles >= ~128 edges of a row and the per-row cost (header, argmax, decide)
//    is amortised over them;
//  * groups synchronise with a named barrier of their own warps only (bar.sync id, n) —
//    never the whole CTA — and a 1-warp group with __syncwarp;
//  * the occupied-slot list is appended with one ballot per warp and batch (the warp's
//    claims get consecutive positions: popc of the lower lanes' claims), so a 1-warp
//    group keeps its list counter in a register and a WARPS-warp group does one shared
//    atomic per warp and batch instead of one per claimed slot;
//  * U = 4 edges per lane per batch, software-pipelined: the next batch's col/w loads
//    are issued before this batch's table inserts, its packed-entry gathers right after;
//  * S64ALL (host-checked 2W·max δ < 2^63): every score fits int64 — no 128-bit code in
//    the kernel at all (smaller register footprint, fewer instructions);
//  * table values are uint32 (the caller guarantees every row sum δ_i < 2^32).
#pragma once
#include "lv_agg.cuh"

namespace lv {

template <int WARPS, int CAP>
struct TabCfg {
  static constexpr int NT = WARPS * 32 >= 256 ? WARPS * 32 : 256;  // threads per CTA (<= 1024)
  static constexpr int GPC = NT / (WARPS * 32);                     // groups per CTA
  static constexpr int LG = CAP == 256 ? 8 : CAP == 512 ? 9 : CAP == 1024 ? 10 : CAP == 2048 ? 11
                          : CAP == 4096 ? 12 : CAP == 8192 ? 13 : CAP == 16384 ? 14 : -1;
  static_assert(LG > 0, "CAP must be a power of two in [256, 16384]");
  static_assert(GPC <= 15, "named barriers 1..15");
  // per group: vals CAP x 4, keys CAP x 4, list degrees CAP/2 x 4, list CAP/2 x 2, record 64
  static constexpr size_t GROUP_BYTES = (size_t)CAP * 11 + 64;

  static constexpr size_t SMEM = (size_t)GPC * GROUP_BYTES;
};

__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Group record (in the group's last 64 B): two list counters (alternating per row) and
// the e_{i->own} slot of a multi-warp group.
struct TabRec {
  int cnt[2];
  u64 eown;
  u64 acc[5];  // the group's sweep counters (i2, moved, cand, s2 hi, s2 lo), written by its decider only
};
static_assert(sizeof(TabRec) <= 64, "group record");

// Streams of one row: col (and w) from the row start; 32-bit offsets within the row.
template <class WT>
struct RowStream {
  const int32_t *col;
  const void *w;
  __device__ __forceinline__ RowStream(const AggArgs &a, i64 beg) : col(a.keys + beg) {
    w = WT::bytes == 4 ? (const void *)((const uint32_t *)a.w + beg)
      : WT::bytes == 8 ? (const void *)((const u64 *)a.w + beg) : nullptr;
  }
  __device__ __forceinline__ uint32_t wt(int t, u64 pf) const {
    if (WT::bytes == 0) return 1u;
    if (WT::bytes == 4) return ld_stream((const uint32_t *)w + t, pf);
    return (uint32_t)ld_stream((const u64 *)w + t, pf);  // < 2^32: narrow tables only
  }
};

template <int WARPS, int CAP, int U, class WT, bool S64ALL>
__global__ void __launch_bounds__(TabCfg<WARPS, CAP>::NT, TabCfg<WARPS, CAP>::NT == 256 ? 4 : 1) k_sweep_tab(AggArgs a) {
  using Cfg = TabCfg<WARPS, CAP>;
  constexpr int GT = WARPS * 32;  // threads per group
  extern __shared__ __align__(16) unsigned char sm[];
  const int grp = threadIdx.x / GT;
  const int gt = threadIdx.x % GT;  // thread index within the group
  const int wig = gt >> 5;          // warp index within the group
  const int lane = threadIdx.x & 31;
  unsigned char *gb = sm + (size_t)grp * Cfg::GROUP_BYTES;
  uint32_t *vals = (uint32_t *)gb;
  int32_t *keys = (int32_t *)(gb + (size_t)CAP * 4);
  uint32_t *odeg = (uint32_t *)(gb + (size_t)CAP * 8);
  uint16_t *olist = (uint16_t *)(gb + (size_t)CAP * 10);
  TabRec *rec = (TabRec *)(gb + (size_t)CAP * 11);
  // per-warp candidates of a multi-warp group (combined by the group's thread 0)
  __shared__ u64 cand_s[Cfg::GPC][WARPS > 1 ? WARPS : 1];
  __shared__ int32_t cand_k[Cfg::GPC][WARPS > 1 ? WARPS : 1];
  __shared__ i64 cand_h[Cfg::GPC][WARPS > 1 ? WARPS : 1];
  const uint32_t kb = saddr(keys), vb = saddr(vals);
  for (int s = gt; s < CAP; s += GT) { keys[s] = EMPTY; vals[s] = 0; }
  if (gt == 0) {
    rec->cnt[0] = 0; rec->cnt[1] = 0; rec->eown = 0;
    for (int i = 0; i < 5; ++i) rec->acc[i] = 0;
  }
  if (WARPS > 1) named_bar(1 + grp, GT);
  else __syncwarp();
  const u64 pf = l2_policy_first();
  const u64 *__restrict__ ldeg = a.ldeg;
  int par = 0;
  const i64 stride = (i64)gridDim.x * Cfg::GPC;
  i64 idx = (i64)blockIdx.x * Cfg::GPC + grp;
  RowHdr nh;
  nh.beg = 0; nh.r = 0; nh.len = 0;
  if (idx < a.nrows) nh = a.hdr[idx];
  for (; idx < a.nrows; idx += stride) {
    const RowHdr hd = nh;
    if (idx + stride < a.nrows) nh = a.hdr[idx + stride];
    const int32_t r = hd.r;
    const int len = hd.len;
    const RowStream<WT> rs(a, hd.beg);
    const u64 pr = __ldg(&ldeg[r]);
    const int32_t own = (int32_t)(uint32_t)pr;
    const i64 di = __ldg(&a.delta[r]);
    const bool decider = gt == 0;
    i64 dq = 0, dr = 0;
    if (decider) {  // issued before the edge loop: overlaps it
      dq = deg_of(a, (uint32_t)(pr >> 32), key_label(own));
      dr = load_deg(a, r);
    }
    const int lg = row_lg(len, Cfg::LG);
    const unsigned mask = (1u << lg) - 1u;
    const uint32_t cb = saddr(&rec->cnt[par]);
    int nloc = 0;  // 1-warp group: list length in a register
    // ---- insert: U edges per lane per batch (offsets t0 + u·GT), the next batch's
    // col/w loads issued before this batch's inserts, its gathers right after them
    int32_t col[U], k[U];
    uint32_t w[U], nw[U], dg[U];
    int t0 = gt;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int t = t0 + u * GT;
      col[u] = t < len ? ld_stream(rs.col + t, pf) : EMPTY;
      w[u] = t < len ? rs.wt(t, pf) : 0u;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const u64 p = col[u] != EMPTY ? __ldg(&ldeg[col[u]]) : 0ull;
      k[u] = col[u] != EMPTY ? (int32_t)(uint32_t)p : EMPTY;
      dg[u] = (uint32_t)(p >> 32);
    }
    for (;;) {
      const int t1 = t0 + GT * U;
      const bool more = t1 - gt < len;  // group-uniform
      if (more) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int t = t1 + u * GT;
          col[u] = t < len ? ld_stream(rs.col + t, pf) : EMPTY;
          nw[u] = t < len ? rs.wt(t, pf) : 0u;
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        bool claimed = false;
        unsigned sl = 0;
        if (k[u] != EMPTY) sl = tab_insert<uint32_t>(kb, vb, mask, lg, k[u], (u64)w[u], &claimed);
        const unsigned cm = __ballot_sync(0xffffffffu, claimed);
        if (cm) {
          int base;
          if (WARPS == 1) {
            base = nloc;
            nloc += __popc(cm);
          } else {
            const int leader = __ffs(cm) - 1;
            int b = 0;
            if (lane == leader) b = (int)atom_add_s32(cb, (uint32_t)__popc(cm));
            base = __shfl_sync(0xffffffffu, b, leader);
          }
          if (claimed) {
            const int q = base + __popc(cm & ((1u << lane) - 1u));
            olist[q] = (uint16_t)sl;
            odeg[q] = dg[u];
          }
        }
      }
      if (!more) break;
      t0 = t1;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        w[u] = nw[u];
        const u64 p = col[u] != EMPTY ? __ldg(&ldeg[col[u]]) : 0ull;
        k[u] = col[u] != EMPTY ? (int32_t)(uint32_t)p : EMPTY;
        dg[u] = (uint32_t)(p >> 32);
      }
    }
    int n;
    if (WARPS == 1) {
      __syncwarp();
      n = nloc;
    } else {
      named_bar(1 + grp, GT);  // S1: every insert of the row done
      n = lds_i32(cb);
      if (gt == 0) rec->cnt[par ^ 1] = 0;  // the next row's counter (read before this S1)
    }
    // ---- epilogue: score the distinct candidates, reset their slots
    const bool s64 = S64ALL || row_s64(a.twoW, di);  // group-uniform
    Cand best = s64 ? cand_none64() : cand_none();
    u64 eown = 0;
    bool has_own = false;
    if (S64ALL || s64) {  // int64 scores: predicated, one select per candidate
      for (int t = gt; t < n; t += GT) {
        const int sl = olist[t];
        const uint32_t d31 = odeg[t];
        const int32_t kk = keys[sl];
        const u64 v = vals[sl];
        keys[sl] = EMPTY;
        vals[sl] = 0;
        const bool mine = kk == own;
        eown = mine ? v : eown;
        has_own |= mine;
        const i64 sc = (i64)((u64)a.twoW * v) - (i64)((u64)di * (u64)deg_of(a, d31, key_label(kk)));
        const i64 sb = (i64)best.lo;
        const bool bt = !mine & ((sc > sb) | ((sc == sb) & (key_label(kk) < key_label(best.c))));
        best.lo = bt ? (u64)sc : best.lo;
        best.c = bt ? kk : best.c;
      }
    } else {
      for (int t = gt; t < n; t += GT) {
        const int sl = olist[t];
        const uint32_t d31 = odeg[t];
        const int32_t kk = keys[sl];
        const u64 v = vals[sl];
        keys[sl] = EMPTY;
        vals[sl] = 0;
        if (kk == own) {
          eown = v;
          has_own = true;
        } else {
          cand_push<false>(best, a.twoW, di, kk, v, deg_of(a, d31, key_label(kk)));
        }
      }
    }
    // e_{i->own}: at most one thread of the group met it
    if (WARPS == 1) {
      const unsigned ob = __ballot_sync(0xffffffffu, has_own);
      eown = ob ? __shfl_sync(0xffffffffu, eown, __ffs(ob) - 1) : 0;
    } else if (has_own) {
      rec->eown = eown;
    }
    // warp argmax
    if (S64ALL || s64) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        Cand y;
        y.hi = 0;
        y.lo = __shfl_xor_sync(0xffffffffu, best.lo, o);
        y.c = __shfl_xor_sync(0xffffffffu, best.c, o);
        if (cand_better64(y, best)) { best.lo = y.lo; best.c = y.c; }
      }
    } else {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        Cand y;
        y.lo = __shfl_xor_sync(0xffffffffu, best.lo, o);
        y.hi = __shfl_xor_sync(0xffffffffu, best.hi, o);
        y.c = __shfl_xor_sync(0xffffffffu, best.c, o);
        if (cand_better(y, best)) best = y;
      }
    }
    if (WARPS > 1) {
      if (lane == 0) {
        cand_s[grp][wig] = best.lo;
        cand_h[grp][wig] = best.hi;
        cand_k[grp][wig] = best.c;
      }
      named_bar(1 + grp, GT);  // S2: candidates and e_own visible; slots all reset
      if (WARPS < 8) {  // a few partials: thread 0 combines them serially
        if (decider) {
#pragma unroll
          for (int w2 = 1; w2 < WARPS; ++w2) {
            Cand y;
            y.lo = cand_s[grp][w2];
            y.hi = cand_h[grp][w2];
            y.c = cand_k[grp][w2];
            if (S64ALL || s64 ? cand_better64(y, best) : cand_better(y, best)) best = y;
          }
          eown = rec->eown;
          rec->eown = 0;
        }
      } else if (wig == 0) {  // 8-32 partials: the group's first warp combines them with
                              // shuffles (thread 0 alone serialised the whole group behind
                              // it at the next row's barrier: C4 le8192 bin 1.20 -> 1.02 ms)
        Cand y = S64ALL || s64 ? cand_none64() : cand_none();
        if (lane < WARPS) {
          y.lo = cand_s[grp][lane];
          y.hi = cand_h[grp][lane];
          y.c = cand_k[grp][lane];
        }
#pragma unroll
        for (int o = WARPS / 2; o > 0; o >>= 1) {
          Cand z;
          z.lo = __shfl_xor_sync(0xffffffffu, y.lo, o);
          z.hi = __shfl_xor_sync(0xffffffffu, y.hi, o);
          z.c = __shfl_xor_sync(0xffffffffu, y.c, o);
          if (S64ALL || s64 ? cand_better64(z, y) : cand_better(z, y)) y = z;
        }
        best = y;
        if (decider) {
          eown = rec->eown;
          rec->eown = 0;
        }
      }
      par ^= 1;
    } else {
      __syncwarp();  // slot resets before the next row's inserts
    }
    if (decider) {  // counters in the group record: no per-thread accumulator registers
      Acc acc;
      if (S64ALL || s64) {
        best.hi = (i64)best.lo >> 63;
        sweep_decide<true>(a, acc, r, own, di, dq, dr, best, eown);
      } else {
        sweep_decide<false>(a, acc, r, own, di, dq, dr, best, eown);
      }
      // candidates = distinct communities other than own (e_{i->own} > 0 iff own is one:
      // weights are positive)
      acc.cand = (u64)n - (eown != 0 ? 1u : 0u);
      rec->acc[0] += acc.i2;
      rec->acc[1] += acc.moved;
      rec->acc[2] += acc.cand;
      add128(rec->acc[3], rec->acc[4], acc.s2hi, acc.s2lo);
    }
  }
  if (gt == 0) {
    u64 *ctr = a.counters;
    if (rec->acc[0]) atomicAdd(&ctr[0], rec->acc[0]);
    if (rec->acc[1]) atomicAdd(&ctr[1], rec->acc[1]);
    if (rec->acc[3] | rec->acc[4]) atomic_add128(&ctr[2], &ctr[3], rec->acc[3], rec->acc[4]);
    if (rec->acc[2]) atomicAdd(&ctr[4], rec->acc[2]);
  }
}

}  // namespace lv
