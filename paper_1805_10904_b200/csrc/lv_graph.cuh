// lv_graph.cuh — device graph (CSR) construction, renumbering and contraction.
//
//   build_csr  : §5.1.2 "Neighbor computation": loops to loop[] (reading
//                D2), mirror every non-loop record, group by source (counting pass +
//                prefix sum instead of the paper's sort_by_key), merge duplicates with the
//                hash aggregation (instead of reduce_by_key, reading D25), offsets by
//                exclusive scan, δ_i = Σ_j ω(i,j) + 2·loop_i, W = Σ ω.
//   renumber   : "Renumbering nodes": flag non-empty labels, exclusive scan,
//                order-preserving dense ids (reading D18).
//   contract   : "Inducing new graph" / graph rebuilding: rows of
//                each community's members are gathered into one contiguous range with
//                their neighbours' new ids, then hash-aggregated (instead of sort_by_key +
//                reduce_by_key): inter-community weights summed per pair, intra weight to
//                the meta-vertex loop (old loops once; reading D19); δ' = deg_C, W' = W.
#pragma once
#include <functional>
#include <cstring>

#include "lv_bins.cuh"

namespace lv {

struct DGraph {
  i64 n = 0, nnz = 0, W = 0;
  i64 max_delta = 0;      // max δ_i: bounds every row sum (u32 tables iff < 2^32)
  int wt = WT_NONE;
  Buf<i64> row_ptr;       // n+1
  Buf<int32_t> col;       // nnz
  Buf<unsigned char> w;   // nnz * wbytes(wt)
  Buf<i64> loop, delta;   // n
};

inline int wbytes(int wt) { return wt == WT_NONE ? 0 : wt == WT_U32 ? 4 : 8; }

// ------------------------------------------------------------------ COO -> CSR
struct RNone { __device__ __forceinline__ static i64 get(const void *, i64) { return 1; } };
struct RI32 { __device__ __forceinline__ static i64 get(const void *w, i64 k) { return ((const int32_t *)w)[k]; } };
struct RI64 { __device__ __forceinline__ static i64 get(const void *w, i64 k) { return ((const i64 *)w)[k]; } };

template <class R>
__global__ void __launch_bounds__(256) k_coo_count(i64 m, i64 n, const int32_t *__restrict__ src,
                                                   const int32_t *__restrict__ dst, const void *w, i64 *loop,
                                                   uint32_t *cnt, u64 *Wacc, int *err) {
  u64 s = 0, mx = 0;
  for (i64 k = (i64)blockIdx.x * 256 + threadIdx.x; k < m; k += (i64)gridDim.x * 256) {
    const int32_t u = src[k], v = dst[k];
    const i64 wk = R::get(w, k);
    if (u < 0 || v < 0 || u >= n || v >= n || wk <= 0) {
      atomicOr(err, 1);
      continue;
    }
    s += (u64)wk;
    mx = (u64)wk > mx ? (u64)wk : mx;
    if (u == v) {
      atomicAdd((u64 *)&loop[u], (u64)wk);
    } else {
      atomicAdd(&cnt[u], 1u);
      atomicAdd(&cnt[v], 1u);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const u64 y = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = y > mx ? y : mx;
  }
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(Wacc + 2, mx);
  s = block_sum_u64<256>(s);
  if (threadIdx.x == 0 && s) atomicAdd(Wacc, s);
}

template <class R, class WOUT>
__global__ void __launch_bounds__(256) k_coo_fill(i64 m, const int32_t *__restrict__ src,
                                                  const int32_t *__restrict__ dst, const void *w,
                                                  const i64 *__restrict__ rptr, uint32_t *cur, int32_t *rcol,
                                                  void *rw, int32_t lo, int32_t hi) {
  // rows outside [lo, hi) are left empty (the sharded build's other parts)
  for (i64 k = (i64)blockIdx.x * 256 + threadIdx.x; k < m; k += (i64)gridDim.x * 256) {
    const int32_t u = src[k], v = dst[k];
    if (u == v) continue;
    const i64 wk = R::get(w, k);
    if (u >= lo && u < hi) {
      const i64 pu = rptr[u] + atomicAdd(&cur[u], 1u);
      rcol[pu] = v;
      if (WOUT::bytes == 4) ((uint32_t *)rw)[pu] = (uint32_t)wk;
      if (WOUT::bytes == 8) ((u64 *)rw)[pu] = (u64)wk;
    }
    if (v >= lo && v < hi) {
      const i64 pv = rptr[v] + atomicAdd(&cur[v], 1u);
      rcol[pv] = u;
      if (WOUT::bytes == 4) ((uint32_t *)rw)[pv] = (uint32_t)wk;
      if (WOUT::bytes == 8) ((u64 *)rw)[pv] = (u64)wk;
    }
  }
}

__global__ void k_delta(i64 n, const u64 *__restrict__ rowsum, const i64 *__restrict__ loop, i64 *delta) {
  for (i64 i = (i64)blockIdx.x * 256 + threadIdx.x; i < n; i += (i64)gridDim.x * 256)
    delta[i] = (i64)rowsum[i] + 2 * loop[i];
}

struct U32AsI64 {
  const uint32_t *a;
  __device__ __forceinline__ i64 operator()(i64 i) const { return (i64)a[i]; }
};
struct I64Arr {
  const i64 *a;
  __device__ __forceinline__ i64 operator()(i64 i) const { return a[i]; }
};

inline i64 max_of(Ctx &c, const i64 *p, i64 n) {
  Buf<u64> t(c.A, 1);
  LV_CUDA(cudaMemsetAsync(t.p, 0, sizeof(u64), c.s));
  LV_LAUNCH(c, k_max_u64<I64Arr>, grid_for(c, n), 256, 0, I64Arr{p}, n, t.p);
  u64 v;
  LV_CUDA(cudaMemcpyAsync(&v, t.p, sizeof(u64), cudaMemcpyDeviceToHost, c.s));
  LV_CUDA(cudaStreamSynchronize(c.s));
  return (i64)v;
}

inline i64 d2h_i64(Ctx &c, const i64 *p) {
  i64 v;
  LV_CUDA(cudaMemcpyAsync(&v, p, sizeof(i64), cudaMemcpyDeviceToHost, c.s));
  LV_CUDA(cudaStreamSynchronize(c.s));
  return v;
}

// ------------------------------------------------- real weights
// The paper stores float weights.  Reading D28 maps them to fixed-point
// integers w~ = rint(w * 2^s) (round half to even; w * 2^s is an exact power-of-two
// scaling in binary64), s the largest integer with T(s) = sum_k w~_k <= 2^52, and runs
// the integer method on w~: exact, schedule-independent sums and scores as for integer
// graphs, and Q of the fixed-point graph within m * 2^-s (relative) of the real one.
template <class T>
__global__ void __launch_bounds__(256) k_fx_sum(i64 m, const T *__restrict__ w, int s, u64 *acc, int *bad) {
  constexpr u64 CAP = (u64)1 << 53;  // anything above 2^52 only needs to be "too big"
  u64 t = 0;
  for (i64 k = (i64)blockIdx.x * 256 + threadIdx.x; k < m; k += (i64)gridDim.x * 256) {
    const double x = (double)w[k];
    if (!(x > 0.0) || !isfinite(x)) {
      atomicOr(bad, 1);
      continue;
    }
    const double f = rint(ldexp(x, s));
    t += f < (double)CAP ? (u64)f : CAP;
    t = t < CAP ? t : CAP;
  }
  t = block_sum_u64<256>(t);  // <= 256 * 2^53
  if (threadIdx.x == 0 && t) atomicAdd(acc, t < CAP ? t : CAP);  // <= 1024 blocks * 2^53
}

template <class T>
__global__ void __launch_bounds__(256) k_fx_conv(i64 m, const T *__restrict__ w, int s, i64 *out, int *bad) {
  for (i64 k = (i64)blockIdx.x * 256 + threadIdx.x; k < m; k += (i64)gridDim.x * 256) {
    const i64 q = (i64)rint(ldexp((double)w[k], s));
    if (q <= 0) atomicOr(bad, 2);  // dynamic range beyond the 52-bit budget
    out[k] = q;
  }
}

// Quantise m real weights (in_wt LV_W_F32 / LV_W_F64, device pointer) into out (int64).
// Returns s.  Errors: LV_EGRAPH for a weight that is not finite and > 0, or that rounds
// to 0 at s.
inline int quantize_real(Ctx &c, i64 m, const void *w, int in_wt, Buf<i64> &out) {
  out.alloc(c.A, m > 0 ? m : 1);
  if (m == 0) return 0;
  Buf<u64> t(c.A, 2);
  int *bad = (int *)(t.p + 1);
  const unsigned gm = std::min(grid_for(c, m), 1024u);
  const u64 lim = (u64)1 << 52;
  auto T = [&](int s) {
    LV_CUDA(cudaMemsetAsync(t.p, 0, 2 * sizeof(u64), c.s));
    if (in_wt == LV_W_F32) LV_LAUNCH(c, k_fx_sum<float>, gm, 256, 0, m, (const float *)w, s, t.p, bad);
    else LV_LAUNCH(c, k_fx_sum<double>, gm, 256, 0, m, (const double *)w, s, t.p, bad);
    u64 h[2];
    LV_CUDA(cudaMemcpyAsync(h, t.p, sizeof(h), cudaMemcpyDeviceToHost, c.s));
    LV_CUDA(cudaStreamSynchronize(c.s));
    LV_REQUIRE((int)h[1] == 0, LV_EGRAPH, "real weight not finite and > 0 (P:L43: positive weights)");
    return h[0];
  };
  // T is non-decreasing in s: binary search the largest s with T(s) <= 2^52
  int lo = -1100, hi = 1100;  // T(lo) = 0 <= 2^52 < T(hi) for any m >= 1 positive weights
  while (hi - lo > 1) {
    const int mid = lo + (hi - lo) / 2;
    if (T(mid) <= lim) lo = mid;
    else hi = mid;
  }
  LV_CUDA(cudaMemsetAsync(t.p, 0, 2 * sizeof(u64), c.s));
  if (in_wt == LV_W_F32) LV_LAUNCH(c, k_fx_conv<float>, grid_for(c, m), 256, 0, m, (const float *)w, lo, out.p, bad);
  else LV_LAUNCH(c, k_fx_conv<double>, grid_for(c, m), 256, 0, m, (const double *)w, lo, out.p, bad);
  u64 h[2];
  LV_CUDA(cudaMemcpyAsync(h, t.p, sizeof(h), cudaMemcpyDeviceToHost, c.s));
  LV_CUDA(cudaStreamSynchronize(c.s));
  LV_REQUIRE((int)h[1] == 0, LV_EGRAPH, "real weights span more than the 52-bit fixed-point budget (reading D28)");
  return lo;
}

// Sharded CSR build and contraction: the rows of the graph being
// built (level-0 vertices / the next level's communities) are split into nparts contiguous
// ranges balanced by their raw entry counts; part p fills and aggregates only its rows.  A process computes the parts in `mine` (all of them
// for in-process simulated ranks, its own rank with NCCL) and `exchange` (NCCL) then
// broadcasts each part's slices from the rank that computed it — so every rank ends with
// the whole (replicated) next-level graph while the gather + hash aggregation work is
// split.  nparts = 1: the whole graph in one part.
struct ShardParts {
  int nparts = 1;
  std::vector<int> mine{0};
  // exchange(buf, elem_bytes, off): slice p = elements [off[p], off[p+1]) of buf, from rank p
  std::function<void(void *, size_t, const std::vector<i64> &)> exchange;
};

// Build the level-0 CSR from device COO records.  Returns LV_OK / LV_EGRAPH / LV_EZEROW
// through exceptions.  in_wt: 0 none, 1 int32, 2 int64 (louvain_wtype).
inline void build_csr(Ctx &c, i64 n, i64 m, const int32_t *src, const int32_t *dst, const void *w, int in_wt,
                      DGraph &g, const ShardParts &S = ShardParts()) {
  g.n = n;
  g.loop.alloc(c.A, n);
  g.delta.alloc(c.A, n);
  LV_CUDA(cudaMemsetAsync(g.loop.p, 0, n * sizeof(i64), c.s));
  Buf<uint32_t> cnt(c.A, n);
  LV_CUDA(cudaMemsetAsync(cnt.p, 0, n * sizeof(uint32_t), c.s));
  Buf<u64> scal(c.A, 3);  // [0] W, [1] err, [2] max weight
  LV_CUDA(cudaMemsetAsync(scal.p, 0, 3 * sizeof(u64), c.s));
  int *err = (int *)(scal.p + 1);
  const unsigned gm = grid_for(c, m);
  if (m > 0) {
    if (in_wt == LV_W_NONE) LV_LAUNCH(c, k_coo_count<RNone>, gm, 256, 0, m, n, src, dst, w, g.loop.p, cnt.p, scal.p, err);
    else if (in_wt == LV_W_I32) LV_LAUNCH(c, k_coo_count<RI32>, gm, 256, 0, m, n, src, dst, w, g.loop.p, cnt.p, scal.p, err);
    else LV_LAUNCH(c, k_coo_count<RI64>, gm, 256, 0, m, n, src, dst, w, g.loop.p, cnt.p, scal.p, err);
  }
  u64 hs[3];
  LV_CUDA(cudaMemcpyAsync(hs, scal.p, 3 * sizeof(u64), cudaMemcpyDeviceToHost, c.s));
  LV_CUDA(cudaStreamSynchronize(c.s));
  LV_REQUIRE(((int)hs[1]) == 0, LV_EGRAPH, "vertex id outside [0,n) or weight <= 0 (P:L43: positive weights)");
  g.W = (i64)hs[0];
  LV_REQUIRE(g.W > 0, LV_EZEROW, "W = 0: modularity (Eq. 3) is undefined");
  // raw (duplicated) adjacency
  Buf<i64> rptr(c.A, n + 1);
  exclusive_scan<i64>(c, U32AsI64{cnt.p}, n, rptr.p, true);
  const i64 rnnz = d2h_i64(c, rptr.p + n);
  // longest raw (duplicated) row: bounds every shared-table sum of the merge below
  u64 maxcnt = 0;
  {
    Buf<u64> t(c.A, 1);
    LV_CUDA(cudaMemsetAsync(t.p, 0, sizeof(u64), c.s));
    LV_LAUNCH(c, k_max_u64<ArrayIn<uint32_t>>, grid_for(c, n), 256, 0, ArrayIn<uint32_t>{cnt.p}, n, t.p);
    LV_CUDA(cudaMemcpyAsync(&maxcnt, t.p, sizeof(u64), cudaMemcpyDeviceToHost, c.s));
    LV_CUDA(cudaStreamSynchronize(c.s));
  }
  const int raw_wt = in_wt == LV_W_NONE ? WT_NONE : in_wt == LV_W_I32 ? WT_U32 : WT_U64;
  // row parts (sharded build): balanced by raw entries; this process fills the rows of its
  // parts ([rlo, rhi) = their union, contiguous: all parts in-process, or one rank's)
  const int P = S.nparts;
  std::vector<i64> rb(P + 1, 0);
  rb[P] = n;
  if (P > 1) {
    Buf<i64> db(c.A, P + 1);
    LV_LAUNCH(c, k_shard_bounds, 1, 1024, 0, n, rptr.p, P, db.p);
    LV_CUDA(cudaMemcpyAsync(rb.data(), db.p, (P + 1) * sizeof(i64), cudaMemcpyDeviceToHost, c.s));
    LV_CUDA(cudaStreamSynchronize(c.s));
  }
  i64 rlo = n, rhi = 0;
  for (int p : S.mine) { rlo = std::min(rlo, rb[p]); rhi = std::max(rhi, rb[p + 1]); }
  Buf<int32_t> rcol(c.A, rnnz > 0 ? rnnz : 1);
  Buf<unsigned char> rw(c.A, rnnz * (i64)wbytes(raw_wt) + 8);
  LV_CUDA(cudaMemsetAsync(cnt.p, 0, n * sizeof(uint32_t), c.s));
  if (m > 0) {
    const int32_t flo = (int32_t)rlo, fhi = (int32_t)rhi;
    if (in_wt == LV_W_NONE) LV_LAUNCH(c, (k_coo_fill<RNone, WNone>), gm, 256, 0, m, src, dst, w, rptr.p, cnt.p, rcol.p, (void *)rw.p, flo, fhi);
    else if (in_wt == LV_W_I32) LV_LAUNCH(c, (k_coo_fill<RI32, WU32>), gm, 256, 0, m, src, dst, w, rptr.p, cnt.p, rcol.p, (void *)rw.p, flo, fhi);
    else LV_LAUNCH(c, (k_coo_fill<RI64, WU64>), gm, 256, 0, m, src, dst, w, rptr.p, cnt.p, rcol.p, (void *)rw.p, flo, fhi);
  }
  cnt.release();
  // merge duplicates per row (hash aggregation, emit mode), two passes: count the distinct
  // entries of every row, then write them straight into the final CSR (no temporaries)
  std::vector<std::unique_ptr<Bins>> BP(P);
  for (int p : S.mine) {
    BP[p] = std::make_unique<Bins>();
    build_bins(c, rptr.p, n, n, *BP[p], rb[p], rb[p + 1]);
  }
  Buf<i64> ocnt(c.A, n);
  Buf<u64> osum(c.A, n);
  LV_CUDA(cudaMemsetAsync(ocnt.p, 0, n * sizeof(i64), c.s));
  LV_CUDA(cudaMemsetAsync(osum.p, 0, n * sizeof(u64), c.s));
  AggArgs a;
  memset(&a, 0, sizeof(a));
  a.ptr = rptr.p;
  a.keys = rcol.p;
  a.w = rw.p;
  a.out_cnt = ocnt.p;
  a.out_sum = osum.p;
  // 32-bit table sums only when no row sum can reach 2^32: every entry of a row's table
  // (and every hub bucket merge across chunks) sums at most (raw row length) x (max w)
  const bool narrow = (unsigned __int128)hs[2] * (unsigned __int128)(maxcnt > 0 ? maxcnt : 1) < ((unsigned __int128)1 << 32);
  for (int p : S.mine) launch_agg_wt<M_EMIT>(c, raw_wt, narrow, *BP[p], a);  // count pass (out_key == NULL)
  if (S.exchange) {  // every part's distinct counts and row sums (δ) from the rank that has them
    S.exchange(ocnt.p, sizeof(i64), rb);
    S.exchange(osum.p, sizeof(u64), rb);
  }
  g.row_ptr.alloc(c.A, n + 1);
  exclusive_scan<i64>(c, I64Arr{ocnt.p}, n, g.row_ptr.p, true);
  g.nnz = d2h_i64(c, g.row_ptr.p + n);
  // weight storage: every merged entry is at most its row sum (<= max δ), so uint32 suffices
  // whenever max row sum < 2^32, even when W itself is larger (C5)
  u64 maxrow = 0;
  {
    Buf<u64> t(c.A, 1);
    LV_CUDA(cudaMemsetAsync(t.p, 0, sizeof(u64), c.s));
    LV_LAUNCH(c, k_max_u64<ArrayIn<u64>>, grid_for(c, n), 256, 0, ArrayIn<u64>{osum.p}, n, t.p);
    LV_CUDA(cudaMemcpyAsync(&maxrow, t.p, sizeof(u64), cudaMemcpyDeviceToHost, c.s));
    LV_CUDA(cudaStreamSynchronize(c.s));
  }
  if (raw_wt == WT_NONE && g.nnz == rnnz) g.wt = WT_NONE;
  else g.wt = (maxrow < ((u64)1 << 32)) ? WT_U32 : WT_U64;
  g.col.alloc(c.A, g.nnz > 0 ? g.nnz : 1);
  g.w.alloc(c.A, g.nnz * (i64)wbytes(g.wt) + 8);
  a.out_base = g.row_ptr.p;
  a.out_key = g.col.p;
  a.out_w = g.w.p;
  a.out_w32 = g.wt == WT_U32;
  a.out_wnone = g.wt == WT_NONE;
  for (int p : S.mine) launch_agg_wt<M_EMIT>(c, raw_wt, narrow, *BP[p], a);  // write pass
  if (S.exchange) {  // every part's rows
    std::vector<i64> ro(P + 1);
    for (int p = 0; p <= P; ++p) ro[p] = d2h_i64(c, g.row_ptr.p + rb[p]);
    S.exchange(g.col.p, sizeof(int32_t), ro);
    if (wbytes(g.wt)) S.exchange(g.w.p, wbytes(g.wt), ro);
  }
  rcol.release();
  rw.release();
  LV_LAUNCH(c, k_delta, grid_for(c, n), 256, 0, n, osum.p, g.loop.p, g.delta.p);
  g.max_delta = max_of(c, g.delta.p, n);
}

// ------------------------------------------------------------------ renumber
struct NonEmpty {
  const int32_t *size;
  __device__ __forceinline__ i64 operator()(i64 c) const { return size[c] > 0 ? 1 : 0; }
};

__global__ void k_apply_newid(i64 n, const i64 *__restrict__ newid, const int32_t *__restrict__ lab_in, int32_t *lab_out) {
  for (i64 i = (i64)blockIdx.x * 256 + threadIdx.x; i < n; i += (i64)gridDim.x * 256)
    lab_out[i] = (int32_t)newid[lab_in[i]];
}

__global__ void k_newcomm(i64 n, const i64 *__restrict__ newid, const int32_t *__restrict__ size,
                          const i64 *__restrict__ deg, i64 *ndelta) {
  for (i64 c = (i64)blockIdx.x * 256 + threadIdx.x; c < n; c += (i64)gridDim.x * 256)
    if (size[c] > 0) ndelta[newid[c]] = deg[c];
}

// Order-preserving renumbering (D18): lab_out[i] = rank of lab_in[i] among non-empty
// labels.  Returns k; ndelta (allocated here, length k) receives deg of each community.
inline i64 renumber(Ctx &c, i64 n, const int32_t *lab_in, const int32_t *size, const i64 *deg, int32_t *lab_out,
                    Buf<i64> &ndelta) {
  Buf<i64> newid(c.A, n + 1);
  exclusive_scan<i64>(c, NonEmpty{size}, n, newid.p, true);
  const i64 k = d2h_i64(c, newid.p + n);
  LV_LAUNCH(c, k_apply_newid, grid_for(c, n), 256, 0, n, newid.p, lab_in, lab_out);
  ndelta.alloc(c.A, k > 0 ? k : 1);
  LV_LAUNCH(c, k_newcomm, grid_for(c, n), 256, 0, n, newid.p, size, deg, ndelta.p);
  return k;
}

// ------------------------------------------------------------------ contraction
__global__ void k_comm_edges(i64 n, const int32_t *__restrict__ lab, const i64 *__restrict__ rp,
                             const i64 *__restrict__ loop, i64 *ecnt, i64 *nloop) {
  for (i64 i = (i64)blockIdx.x * 256 + threadIdx.x; i < n; i += (i64)gridDim.x * 256) {
    const int32_t c = lab[i];
    const i64 d = rp[i + 1] - rp[i];
    if (d) atomicAdd((u64 *)&ecnt[c], (u64)d);
    if (loop[i]) atomicAdd((u64 *)&nloop[c], (u64)loop[i]);
  }
}

// Gather each vertex's row into its community's contiguous range, mapping neighbours
// to their new ids.  One group of G lanes per vertex (vertex bins of the level graph).
template <int G, int BLOCK, class WT>
__global__ void __launch_bounds__(BLOCK) k_permute(const int32_t *__restrict__ rows, i64 nrows,
                                                   const i64 *__restrict__ rp, const int32_t *__restrict__ col,
                                                   const void *w, const int32_t *__restrict__ lab,
                                                   const i64 *__restrict__ cptr, u64 *ecur, int32_t *pk, void *pw,
                                                   int32_t clo, int32_t chi) {
  constexpr int GPB = BLOCK / G;
  __shared__ i64 sbase[GPB];
  const int grp = threadIdx.x / G, lane = threadIdx.x % G;
  const unsigned mask = G >= 32 ? 0xffffffffu : (((1u << (G & 31)) - 1u) << (((threadIdx.x & 31) / G) * G));
  for (i64 idx = (i64)blockIdx.x * GPB + grp; idx < nrows; idx += (i64)gridDim.x * GPB) {
    const int32_t v = rows[idx];
    const int32_t c = lab[v];
    if (c < clo || c >= chi) continue;  // group-uniform: another part's community (sharded contraction)
    const i64 b = rp[v], d = rp[v + 1] - b;
    i64 base = 0;
    if (lane == 0) base = cptr[c] + (i64)atomicAdd(&ecur[c], (u64)d);
    if (G <= 32) {
      base = __shfl_sync(mask, base, 0, G < 32 ? G : 32);
    } else {
      if (lane == 0) sbase[grp] = base;
      __syncthreads();
      base = sbase[grp];
    }
    for (i64 t = lane; t < d; t += G) {
      pk[base + t] = lab[col[b + t]];
      if (WT::bytes == 4) ((uint32_t *)pw)[base + t] = ((const uint32_t *)w)[b + t];
      if (WT::bytes == 8) ((u64 *)pw)[base + t] = ((const u64 *)w)[b + t];
    }
    if (G > 32) __syncthreads();
  }
}

template <class WT>
__global__ void __launch_bounds__(256) k_permute_hub(const Chunk *__restrict__ chunks, const int32_t *__restrict__ rows,
                                                     const i64 *__restrict__ rp, const int32_t *__restrict__ col,
                                                     const void *w, const int32_t *__restrict__ lab,
                                                     const i64 *__restrict__ hub_base, int32_t *pk, void *pw,
                                                     int32_t clo, int32_t chi) {
  const Chunk ch = chunks[blockIdx.x];
  const int32_t v = rows[ch.h];
  if (lab[v] < clo || lab[v] >= chi) return;  // CTA-uniform
  const i64 b = rp[v], base = hub_base[ch.h];
  for (i64 e = ch.beg + threadIdx.x; e < ch.end; e += 256) {
    const i64 t = e - b;
    pk[base + t] = lab[col[e]];
    if (WT::bytes == 4) ((uint32_t *)pw)[base + t] = ((const uint32_t *)w)[e];
    if (WT::bytes == 8) ((u64 *)pw)[base + t] = ((const u64 *)w)[e];
  }
}

__global__ void k_hub_bases(i64 nhub, const int32_t *__restrict__ rows, const i64 *__restrict__ rp,
                            const int32_t *__restrict__ lab, const i64 *__restrict__ cptr, u64 *ecur, i64 *hub_base,
                            int32_t clo, int32_t chi) {
  for (i64 h = (i64)blockIdx.x * 256 + threadIdx.x; h < nhub; h += (i64)gridDim.x * 256) {
    const int32_t v = rows[h];
    const i64 d = rp[v + 1] - rp[v];
    const int32_t c = lab[v];
    if (c < clo || c >= chi) continue;
    hub_base[h] = cptr[c] + (i64)atomicAdd(&ecur[c], (u64)d);
  }
}

// Rows of vertices whose community lies in [clo, chi) only (a part of the sharded
// contraction; [0, k) = all).
template <class WT>
void permute_t(Ctx &c, const DGraph &g, const Bins &VB, const int32_t *lab, const i64 *cptr, u64 *ecur, int32_t *pk,
               void *pw, int32_t clo, int32_t chi) {
  auto one = [&](int b, auto kern, int GPB, int BLOCK) {
    if (!VB.count(b)) return;
    i64 grid = cdiv(VB.count(b), GPB);
    if (grid > (i64)c.sms * 16) grid = (i64)c.sms * 16;
    LV_LAUNCH(c, kern, (unsigned)grid, BLOCK, 0, VB.rows.p + VB.off[b], VB.count(b), g.row_ptr.p, g.col.p,
              (const void *)g.w.p, lab, cptr, ecur, pk, pw, clo, chi);
  };
  one(0, k_permute<4, 256, WT>, 64, 256);
  one(1, k_permute<8, 256, WT>, 32, 256);
  one(2, k_permute<16, 256, WT>, 16, 256);
  one(3, k_permute<32, 256, WT>, 8, 256);
  one(4, k_permute<32, 256, WT>, 8, 256);
  one(5, k_permute<128, 128, WT>, 1, 128);
  one(6, k_permute<128, 128, WT>, 1, 128);
  static_assert(NSMEM == 11, "one launch per degree bin below");
  for (int b = 7; b < NSMEM; ++b) one(b, k_permute<256, 256, WT>, 1, 256);
  if (VB.nhub) {
    Buf<i64> hb(c.A, VB.nhub);
    LV_LAUNCH(c, k_hub_bases, grid_for(c, VB.nhub), 256, 0, VB.nhub, VB.rows.p + VB.off[NSMEM], g.row_ptr.p, lab,
              cptr, ecur, hb.p, clo, chi);
    LV_LAUNCH(c, k_permute_hub<WT>, (unsigned)VB.nchunks, 256, 0, VB.chunks.p, VB.rows.p + VB.off[NSMEM], g.row_ptr.p,
              g.col.p, (const void *)g.w.p, lab, hb.p, pk, pw, clo, chi);
  }
}

__global__ void k_finish_loop(i64 k, const i64 *__restrict__ nloop, const u64 *__restrict__ selfw, i64 *loop_out) {
  for (i64 c = (i64)blockIdx.x * 256 + threadIdx.x; c < k; c += (i64)gridDim.x * 256)
    loop_out[c] = nloop[c] + (i64)(selfw[c] / 2);  // each undirected intra edge seen twice
}

// Contract g by dense labels lab (values in [0,k)); ndelta = deg of each community.
// VB = vertex bins of g (reused from the sweeps).
inline void contract(Ctx &c, const DGraph &g, const Bins &VB, const int32_t *lab, i64 k, Buf<i64> &&ndelta,
                     DGraph &h, const ShardParts &S = ShardParts()) {
  const i64 n = g.n;
  Buf<i64> ecnt(c.A, k + 1), nloop(c.A, k);
  LV_CUDA(cudaMemsetAsync(ecnt.p, 0, (k + 1) * sizeof(i64), c.s));
  LV_CUDA(cudaMemsetAsync(nloop.p, 0, k * sizeof(i64), c.s));
  LV_LAUNCH(c, k_comm_edges, grid_for(c, n), 256, 0, n, lab, g.row_ptr.p, g.loop.p, ecnt.p, nloop.p);
  Buf<i64> cptr(c.A, k + 1);
  exclusive_scan<i64>(c, I64Arr{ecnt.p}, k, cptr.p, true);
  // part boundaries over the communities
  const int P = S.nparts;
  std::vector<i64> cb(P + 1, 0);
  cb[P] = k;
  if (P > 1) {
    Buf<i64> db(c.A, P + 1);
    LV_LAUNCH(c, k_shard_bounds, 1, 1024, 0, k, cptr.p, P, db.p);
    LV_CUDA(cudaMemcpyAsync(cb.data(), db.p, (P + 1) * sizeof(i64), cudaMemcpyDeviceToHost, c.s));
    LV_CUDA(cudaStreamSynchronize(c.s));
  }
  const i64 tot = g.nnz;
  Buf<int32_t> pk(c.A, tot > 0 ? tot : 1);
  Buf<unsigned char> pw(c.A, tot * (i64)wbytes(g.wt) + 8);
  LV_CUDA(cudaMemsetAsync(ecnt.p, 0, (k + 1) * sizeof(i64), c.s));  // reuse as cursor
  for (int p : S.mine) {
    const int32_t clo = (int32_t)cb[p], chi = (int32_t)cb[p + 1];
    if (g.wt == WT_NONE) permute_t<WNone>(c, g, VB, lab, cptr.p, (u64 *)ecnt.p, pk.p, pw.p, clo, chi);
    else if (g.wt == WT_U32) permute_t<WU32>(c, g, VB, lab, cptr.p, (u64 *)ecnt.p, pk.p, pw.p, clo, chi);
    else permute_t<WU64>(c, g, VB, lab, cptr.p, (u64 *)ecnt.p, pk.p, pw.p, clo, chi);
  }
  ecnt.release();
  // aggregate each community's range: count pass, then write straight into the new CSR
  std::vector<std::unique_ptr<Bins>> CB(P);
  for (int p : S.mine) {
    CB[p] = std::make_unique<Bins>();
    build_bins(c, cptr.p, k, k, *CB[p], cb[p], cb[p + 1]);
  }
  Buf<i64> ocnt(c.A, k);
  Buf<u64> oself(c.A, k);
  LV_CUDA(cudaMemsetAsync(ocnt.p, 0, k * sizeof(i64), c.s));
  LV_CUDA(cudaMemsetAsync(oself.p, 0, k * sizeof(u64), c.s));
  AggArgs a;
  memset(&a, 0, sizeof(a));
  a.ptr = cptr.p;
  a.keys = pk.p;
  a.w = pw.p;
  a.out_cnt = ocnt.p;
  a.out_self = oself.p;
  // a community's row sum is at most its deg_C
  const i64 maxdeg = max_of(c, ndelta.p, k);
  const bool narrow = maxdeg < ((i64)1 << 32);
  for (int p : S.mine) launch_agg_wt<M_EMIT>(c, g.wt, narrow, *CB[p], a);  // count pass (out_key == NULL)
  if (S.exchange) {
    S.exchange(ocnt.p, sizeof(i64), cb);
    S.exchange(oself.p, sizeof(u64), cb);
  }
  h.n = k;
  h.W = g.W;
  h.row_ptr.alloc(c.A, k + 1);
  exclusive_scan<i64>(c, I64Arr{ocnt.p}, k, h.row_ptr.p, true);
  h.nnz = d2h_i64(c, h.row_ptr.p + k);
  h.wt = narrow ? WT_U32 : WT_U64;  // an entry (c,d) weighs at most deg_C <= maxdeg
  h.col.alloc(c.A, h.nnz > 0 ? h.nnz : 1);
  h.w.alloc(c.A, h.nnz * (i64)wbytes(h.wt) + 8);
  a.out_base = h.row_ptr.p;
  a.out_key = h.col.p;
  a.out_w = h.w.p;
  a.out_w32 = h.wt == WT_U32;
  a.out_wnone = 0;
  for (int p : S.mine) launch_agg_wt<M_EMIT>(c, g.wt, narrow, *CB[p], a);  // write pass
  if (S.exchange) {  // every part's rows from the rank that computed them
    std::vector<i64> ro(P + 1);
    for (int p = 0; p <= P; ++p) ro[p] = d2h_i64(c, h.row_ptr.p + cb[p]);
    S.exchange(h.col.p, sizeof(int32_t), ro);
    S.exchange(h.w.p, wbytes(h.wt), ro);
  }
  pk.release();
  pw.release();
  h.loop.alloc(c.A, k);
  LV_LAUNCH(c, k_finish_loop, grid_for(c, k), 256, 0, k, nloop.p, oself.p, h.loop.p);
  h.delta = std::move(ndelta);
  h.max_delta = maxdeg;
  LV_CUDA(cudaStreamSynchronize(c.s));
}

// ------------------------------------------------------------------ compaction + layout
// The graph a level sweeps is a relabelled copy of the level graph g:
//  * compaction: vertices without non-loop neighbours are removed (they never move and
//    are never gathered).  rank m[v] of v among the active vertices is monotone, and the
//    LABEL VALUES of the sweep are these ranks, so every label comparison the method
//    makes (min-label ties, the singlet rule, the order-preserving renumbering) is the
//    one it makes on g;
//  * layout: the vertex POSITIONS (row index, index of every per-vertex array, and of
//    the edges' neighbour ids) are the ranks ordered by degree bin (ascending rank within
//    a bin), so each bin's rows, headers and edges are contiguous in HBM (coalesced
//    streams for the short-row bins) and the high-degree vertices — gathered most often —
//    share sectors and L2 lines.
// rk[p] = rank of the vertex at position p (its initial label), pos[i] = position of rank i.
struct ActiveFlag {
  const i64 *rp;
  __device__ __forceinline__ i64 operator()(i64 v) const { return rp[v + 1] > rp[v] ? 1 : 0; }
};

__global__ void k_compact_build(i64 n, const i64 *__restrict__ rp, const i64 *__restrict__ m, int32_t *inv,
                                i64 *rp_r) {
  for (i64 v = (i64)blockIdx.x * 256 + threadIdx.x; v < n; v += (i64)gridDim.x * 256) {
    if (rp[v + 1] > rp[v]) {
      const i64 i = m[v];
      inv[i] = (int32_t)v;
      rp_r[i] = rp[v];  // rank-space row starts (original edge offsets)
    }
  }
}

// per position p: pos[rk[p]] = p, and the position-space row length / δ / loop
__global__ void k_layout_rows(i64 na, const int32_t *__restrict__ rk, const int32_t *__restrict__ inv,
                              const i64 *__restrict__ rp, const i64 *__restrict__ delta, const i64 *__restrict__ loop,
                              int32_t *pos, i64 *len_p, i64 *delta_p, i64 *loop_p) {
  for (i64 p = (i64)blockIdx.x * 256 + threadIdx.x; p < na; p += (i64)gridDim.x * 256) {
    const int32_t i = rk[p];
    const int32_t v = inv[i];
    pos[i] = (int32_t)p;
    len_p[p] = rp[v + 1] - rp[v];
    delta_p[p] = delta[v];
    loop_p[p] = loop[v];
  }
}

struct LenArr {
  const i64 *len;
  __device__ __forceinline__ i64 operator()(i64 p) const { return len[p]; }
};

// Copy every row of g to its position, neighbour ids mapped to positions (pos[m[col]]).
// One warp per row (rows of positions [p0, p1)); CTA-per-row for the hub rows.
template <int T>
__global__ void __launch_bounds__(T == 32 ? 256 : T) k_layout_edges(i64 p0, i64 p1, const int32_t *__restrict__ rk,
                                                    const int32_t *__restrict__ inv, const i64 *__restrict__ rp,
                                                    const int32_t *__restrict__ col, const void *w, int wb,
                                                    const i64 *__restrict__ m, const int32_t *__restrict__ pos,
                                                    const i64 *__restrict__ rp_p, int32_t *col_p, void *w_p) {
  constexpr int G = T == 32 ? 32 : T;  // lanes per row
  const int per = T == 32 ? (int)(blockDim.x / 32) : 1;
  const i64 first = (i64)blockIdx.x * per + (T == 32 ? threadIdx.x / 32 : 0);
  const int lane = threadIdx.x % G;
  for (i64 p = p0 + first; p < p1; p += (i64)gridDim.x * per) {
    const int32_t v = inv[rk[p]];
    const i64 b = rp[v], d = rp[v + 1] - b, o = rp_p[p];
    for (i64 t = lane; t < d; t += G) {
      col_p[o + t] = pos[m[col[b + t]]];
      if (wb == 4) ((uint32_t *)w_p)[o + t] = ((const uint32_t *)w)[b + t];
      else if (wb == 8) ((u64 *)w_p)[o + t] = ((const u64 *)w)[b + t];
    }
  }
}

// Back to g's index space: labels (rank-valued community ids -> original vertex ids) and
// per-community size / deg (indexed by the label value = rank).
__global__ void k_expand_state(i64 n, const i64 *__restrict__ rp, const i64 *__restrict__ m,
                               const int32_t *__restrict__ inv, const int32_t *__restrict__ pos,
                               const int32_t *__restrict__ lab_c, const int32_t *__restrict__ size_c,
                               const i64 *__restrict__ deg_c, const i64 *__restrict__ delta, int32_t *lab_o,
                               int32_t *size_o, i64 *deg_o) {
  for (i64 v = (i64)blockIdx.x * 256 + threadIdx.x; v < n; v += (i64)gridDim.x * 256) {
    if (rp[v + 1] > rp[v]) {
      const i64 i = m[v];
      lab_o[v] = inv[lab_c[pos[i]]];
      size_o[v] = size_c[i];
      deg_o[v] = deg_c[i];
    } else {
      lab_o[v] = (int32_t)v;
      size_o[v] = 1;
      deg_o[v] = delta[v];
    }
  }
}

constexpr i64 LONG_ROW = BIN_MAX[NSMEM - 1];  // longer rows take the hub path
struct LongRow {
  const i64 *rp;
  __device__ __forceinline__ i64 operator()(i64 p) const { return rp[p + 1] - rp[p] > LONG_ROW ? 1 : 0; }
};
inline i64 count_long_rows(Ctx &c, const DGraph &gc, i64 na) {
  Buf<u64> t(c.A, 1);
  LV_CUDA(cudaMemsetAsync(t.p, 0, sizeof(u64), c.s));
  LV_LAUNCH(c, k_sum_u64<LongRow>, grid_for(c, na), 256, 0, LongRow{gc.row_ptr.p}, na, t.p);
  u64 h = 0;
  LV_CUDA(cudaMemcpyAsync(&h, t.p, sizeof(u64), cudaMemcpyDeviceToHost, c.s));
  LV_CUDA(cudaStreamSynchronize(c.s));
  return (i64)h;
}

struct Compaction {
  i64 na = 0;
  Buf<i64> m;        // original id -> rank (n + 1; m[n] = na)
  Buf<int32_t> inv;  // rank -> original id
  Buf<int32_t> pos;  // rank -> position
  Buf<int32_t> rk;   // position -> rank
};

// Builds gc (the compacted, bin-ordered level graph); false when g has no active vertex.
inline bool compact_graph(Ctx &c, const DGraph &g, DGraph &gc, Compaction &cp) {
  cp.m.alloc(c.A, g.n + 1);
  exclusive_scan<i64>(c, ActiveFlag{g.row_ptr.p}, g.n, cp.m.p, true);
  cp.na = d2h_i64(c, cp.m.p + g.n);
  if (cp.na == 0) {
    cp.m.release();
    return false;
  }
  const i64 na = cp.na;
  cp.inv.alloc(c.A, na);
  cp.pos.alloc(c.A, na);
  cp.rk.alloc(c.A, na);
  {
    Buf<i64> rp_r(c.A, na + 1);
    LV_LAUNCH(c, k_compact_build, grid_for(c, g.n), 256, 0, g.n, g.row_ptr.p, cp.m.p, cp.inv.p, rp_r.p);
    LV_CUDA(cudaMemcpyAsync(rp_r.p + na, g.row_ptr.p + g.n, sizeof(i64), cudaMemcpyDeviceToDevice, c.s));
    Bins Br;  // rank-space rows per degree bin
    build_bins(c, rp_r.p, na, na, Br, 0, -1, true);
    LV_CUDA(cudaMemcpyAsync(cp.rk.p, Br.rows.p, na * sizeof(int32_t), cudaMemcpyDeviceToDevice, c.s));
  }
  gc.n = na;
  gc.nnz = g.nnz;
  gc.W = g.W;
  gc.wt = g.wt;
  gc.max_delta = g.max_delta;
  gc.row_ptr.alloc(c.A, na + 1);
  gc.delta.alloc(c.A, na);
  gc.loop.alloc(c.A, na);
  {
    Buf<i64> len_p(c.A, na);
    LV_LAUNCH(c, k_layout_rows, grid_for(c, na), 256, 0, na, cp.rk.p, cp.inv.p, g.row_ptr.p, g.delta.p, g.loop.p,
              cp.pos.p, len_p.p, gc.delta.p, gc.loop.p);
    exclusive_scan<i64>(c, LenArr{len_p.p}, na, gc.row_ptr.p, true);
  }
  gc.col.alloc(c.A, g.nnz > 0 ? g.nnz : 1);
  gc.w.alloc(c.A, g.nnz * (i64)wbytes(g.wt) + 8);
  // hub rows (> BIN_MAX[NSMEM-1] entries) sit at the end of the layout: a CTA each
  const i64 nh = count_long_rows(c, gc, na);
  const i64 ps = na - nh;
  if (ps > 0)
    LV_LAUNCH(c, k_layout_edges<32>, grid_for(c, ps, 8), 256, 0, (i64)0, ps, cp.rk.p, cp.inv.p, g.row_ptr.p, g.col.p,
              (const void *)g.w.p, wbytes(g.wt), cp.m.p, cp.pos.p, gc.row_ptr.p, gc.col.p, (void *)gc.w.p);
  if (nh > 0)
    LV_LAUNCH(c, k_layout_edges<512>, (unsigned)std::min<i64>(nh, (i64)c.sms * 4), 512, 0, ps, na, cp.rk.p, cp.inv.p,
              g.row_ptr.p, g.col.p, (const void *)g.w.p, wbytes(g.wt), cp.m.p, cp.pos.p, gc.row_ptr.p, gc.col.p,
              (void *)gc.w.p);
  return true;
}

}  // namespace lv
