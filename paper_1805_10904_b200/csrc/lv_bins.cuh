// lv_bins.cuh — degree binning ("divergence ... could be reduced by ordering the
// vertices by degree") and the launcher that runs one aggregation pass (sweep, merge or
// emit) over all bins.  Bins are rebuilt once per level and reused by every sweep.
#pragma once
#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "lv_agg.cuh"
#include "lv_hubcl.cuh"
#include "lv_scan.cuh"
#include "lv_sweep.cuh"

namespace lv {

// bin b holds rows of length in (BIN_MAX[b-1], BIN_MAX[b]]; bin NSMEM holds the hubs
constexpr int NSMEM = 11;
constexpr int NBIN = NSMEM + 1;
constexpr i64 BIN_MAX[NSMEM] = {4, 8, 16, 32, 128, 256, 512, 1024, 2048, 4096, 8192};

__device__ __forceinline__ int bin_of(i64 d) {
  constexpr i64 M[NSMEM] = {4, 8, 16, 32, 128, 256, 512, 1024, 2048, 4096, 8192};  // = BIN_MAX
  if (d <= 0) return 255;
  int b = 0;
#pragma unroll
  for (int i = 0; i < NSMEM; ++i) b += d > M[i];
  return b;
}

struct KTimer {  // optional per-launch CUDA-event timing (profiling; may nest)
  bool on = false;
  std::vector<std::string> names;
  std::vector<cudaEvent_t> t0, t1;
  std::vector<size_t> open;
  std::vector<cudaEvent_t> pool;  // events are reused across clear() (creation costs host time)
  size_t used = 0;
  cudaEvent_t get() {
    if (used == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return pool[used++];
  }
  void begin(cudaStream_t s, const std::string &n) {
    if (!on) return;
    cudaEvent_t a = get();
    cudaEventRecord(a, s);
    names.push_back(n);
    t0.push_back(a);
    t1.push_back(nullptr);
    open.push_back(names.size() - 1);
  }
  void end(cudaStream_t s) {
    if (!on || open.empty()) return;
    cudaEvent_t b = get();
    cudaEventRecord(b, s);
    t1[open.back()] = b;
    open.pop_back();
  }
  void clear() {
    t0.clear();
    t1.clear();
    names.clear();
    open.clear();
    used = 0;
  }
  ~KTimer() {
    for (auto e : pool) cudaEventDestroy(e);
  }
};

struct Bins {
  i64 nrows = 0;             // universe of rows considered
  Buf<int32_t> rows;         // active rows grouped by bin (ascending id within a bin)
  Buf<RowHdr> hdr;           // packed {beg, r, len} per entry of rows
  i64 off[NBIN + 1] = {0};   // host offsets of each bin in rows
  i64 edges[NBIN] = {0};     // Σ row length per bin
  // hub path (see lv_agg.cuh): chunks, buckets, pool, segment tables, partials
  i64 nhub = 0, nchunks = 0, nfin = 0, nseg = 0;
  int max_blg = 0;
  int fin_lg = HUB_FIN_LG;
  Buf<Chunk> chunks;
  Buf<i64> cfirst, bfirst, segoff;
  Buf<int32_t> ccount, blg, seg;
  Buf<u64> emit_cur;
  Buf<uint4> pent;                         // pool: {key, deg_C, Σw lo, Σw hi} per entry
  std::vector<i64> batch_h;                // hub-row batches: [batch_h[i], batch_h[i+1])
  std::vector<i64> h_cfirst, h_bfirst;     // host copies (chunk / fin-item starts, + end)
  i64 pool_chunks = 0;                     // pool capacity in chunks (max over batches)
  Buf<int2> fitem;
  Buf<HubPartial> part;
  Buf<int> overflow;
  // cluster hub path (lv_hubcl.cuh): hub rows [0, ncl) of the hub bin fit a cluster of
  // cl_cs CTAs (SWEEP with narrow tables runs them there; the pool path takes the rest);
  // clhdr = their headers by decreasing length; cl_used: the last SWEEP pass used it
  i64 ncl = 0, edges_cl = 0;
  int cl_cs = 0;
  Buf<RowHdr> clhdr;
  mutable int cl_used = 0;
  i64 count(int b) const { return off[b + 1] - off[b]; }
  i64 active() const { return off[NBIN]; }
};

struct LenOf {
  const i64 *ptr;
  __device__ __forceinline__ i64 operator()(i64 r) const { return ptr[r + 1] - ptr[r]; }
};

// cls (may be NULL): keep only rows of colour class ck (the colouring heuristic, D29)
__global__ void k_bin_ids(i64 n, const i64 *__restrict__ ptr, uint8_t *ids, i64 lo, i64 hi,
                          const int32_t *__restrict__ cls, int32_t ck) {
  for (i64 r = (i64)blockIdx.x * 256 + threadIdx.x; r < n; r += (i64)gridDim.x * 256)
    ids[r] = (r >= lo && r < hi && (!cls || cls[r] == ck)) ? (uint8_t)bin_of(ptr[r + 1] - ptr[r]) : (uint8_t)255;
}

// Edge-balanced contiguous vertex ranges (sweep-sharded mode):
// bounds[p] = first row v with ptr[v] >= p·nnz/P (bounds[0] = 0, bounds[P] = n).
__global__ void k_shard_bounds(i64 n, const i64 *__restrict__ ptr, int P, i64 *bounds) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p > P) return;
  if (p == 0) { bounds[0] = 0; return; }
  if (p == P) { bounds[P] = n; return; }
  const i64 nnz = ptr[n];
  const i64 target = (i64)(((__int128)nnz * p) / P);
  i64 lo = 0, hi = n;  // first v in [0,n] with ptr[v] >= target
  while (lo < hi) {
    const i64 mid = (lo + hi) >> 1;
    if (ptr[mid] >= target) hi = mid;
    else lo = mid + 1;
  }
  bounds[p] = lo;
}

struct BinLen {
  const int32_t *rows;
  const i64 *ptr;
  __device__ __forceinline__ u64 operator()(i64 t) const { return (u64)(ptr[rows[t] + 1] - ptr[rows[t]]); }
};

struct IsBin {
  const uint8_t *ids;
  int b;
  __device__ __forceinline__ i64 operator()(i64 r) const { return ids[r] == b ? 1 : 0; }
};

__global__ void k_bin_scatter(i64 n, const uint8_t *__restrict__ ids, int b, const i64 *__restrict__ pos,
                              int32_t *out) {
  for (i64 r = (i64)blockIdx.x * 256 + threadIdx.x; r < n; r += (i64)gridDim.x * 256)
    if (ids[r] == b) out[pos[r]] = (int32_t)r;
}

__global__ void k_fill_hdr(i64 m, const int32_t *__restrict__ rows, const i64 *__restrict__ ptr, RowHdr *hdr) {
  for (i64 t = (i64)blockIdx.x * 256 + threadIdx.x; t < m; t += (i64)gridDim.x * 256) {
    const int32_t r = rows[t];
    RowHdr h;
    h.beg = ptr[r];
    h.r = r;
    h.len = (int32_t)(ptr[r + 1] - ptr[r]);
    hdr[t] = h;
  }
}

__global__ void k_gather_len(i64 m, const int32_t *rows, const i64 *ptr, i64 *beg, i64 *len) {
  for (i64 t = (i64)blockIdx.x * 256 + threadIdx.x; t < m; t += (i64)gridDim.x * 256) {
    int32_t r = rows[t];
    beg[t] = ptr[r];
    len[t] = ptr[r + 1] - ptr[r];
  }
}

inline unsigned grid_for(const Ctx &c, i64 n, int per = 256) {
  i64 g = cdiv(n, per);
  i64 cap = (i64)c.sms * 32;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (unsigned)g;
}

// Resident CTAs per SM of kernel fn at (block, dynamic smem) on the CURRENT device, after
// raising fn's dynamic shared-memory limit there if smem needs it.  Cached per (device,
// kernel, block, smem) under a mutex: the attribute is per device, and distinct handles
// (possibly on other devices / threads) share these caches.  The limit only ever grows,
// so a cached smaller configuration never lowers it below a larger one in use.
template <class F>
inline int kernel_occ(F fn, int block, size_t smem) {
  static std::mutex mu;
  static std::map<std::tuple<int, const void *, int, size_t>, int> occ;
  static std::map<std::pair<int, const void *>, size_t> attr;
  int dev = 0;
  LV_CUDA(cudaGetDevice(&dev));
  const void *f = (const void *)fn;
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_tuple(dev, f, block, smem);
  const auto it = occ.find(key);
  if (it != occ.end()) return it->second;
  size_t &cur = attr[std::make_pair(dev, f)];
  if (smem > cur) {
    LV_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cur = smem;
  }
  int o = 0;
  LV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, block, smem));
  o = o > 0 ? o : 1;
  occ[key] = o;
  return o;
}

// Cluster hub kernel (lv_hubcl.cuh): raise its shared-memory limit / allow a non-portable
// cluster size on the current device (once per device and instantiation) and return how
// many clusters of CS CTAs can be co-resident (0: unsupported).
inline cudaLaunchConfig_t hcl_config(int cs, unsigned grid, cudaStream_t st, cudaLaunchAttribute *at) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(HCL_T, 1, 1);
  cfg.dynamicSmemBytes = HCL_SMEM;
  cfg.stream = st;
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cfg;
}
template <int CS, class WT, bool S64ALL>
inline int hcl_prepare() {
  static std::mutex mu;
  static std::map<int, int> done;  // device -> max active clusters
  int dev = 0;
  LV_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  const auto it = done.find(dev);
  if (it != done.end()) return it->second;
  auto kern = k_hub_cl<CS, WT, S64ALL>;
  int n = 0;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)HCL_SMEM) == cudaSuccess &&
      (CS <= 8 || cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess)) {
    cudaLaunchAttribute at[1];
    cudaLaunchConfig_t cfg = hcl_config(CS, CS * 148, nullptr, at);
    if (cudaOccupancyMaxActiveClusters(&n, (const void *)kern, &cfg) != cudaSuccess) n = 0;
  }
  cudaGetLastError();  // an unsupported size leaves a sticky-free error: clear it
  done[dev] = n;
  return n;
}
// cluster size used for the hub rows of this device.  Opt-in (LV_HUBCL=1): measured r2
// on B200 (C4 level-0 sweep, hub rows of 8k-131k entries): 6.0 ms with 16-CTA and 3.7 ms
// with 8-CTA clusters against 2.0 ms for the pool path (k_hub_acc + k_hub_fin) — remote
// shared-memory CAS round trips (SASS: generic ATOM.E.CAS) serialise the inserts, ~0.04
// inserts per cycle per SM.  LV_HUBCL_CS=8|16 forces a size; default 16 when 16-CTA
// clusters fit, else 8.
inline int hcl_cluster_size() {
  static const char *on = getenv("LV_HUBCL");
  if (!on || atoi(on) == 0) return 0;
  static const int force = getenv("LV_HUBCL_CS") ? atoi(getenv("LV_HUBCL_CS")) : 0;
  if (force == 16) return hcl_prepare<16, WU32, true>() > 0 ? 16 : 0;
  if (force == 8) return hcl_prepare<8, WU32, true>() > 0 ? 8 : 0;
  if (hcl_prepare<16, WU32, true>() > 0) return 16;
  if (hcl_prepare<8, WU32, true>() > 0) return 8;
  return 0;
}

// Partition rows [0,nrows) of `ptr` into length bins; set up hub tables sized for at
// most `universe` distinct keys per row.
// Only rows in [lo, hi) are binned (hi < 0: all rows).  rows_only: just B.rows / B.off
// (the per-bin row lists, ascending within a bin), no headers, edge counts or hub tables.
inline void finish_bins(Ctx &c, const i64 *ptr, i64 universe, Bins &B, const std::vector<i64> &cnt, const i64 *edges);

inline void build_bins(Ctx &c, const i64 *ptr, i64 nrows, i64 universe, Bins &B, i64 lo = 0, i64 hi = -1,
                       bool rows_only = false, const int32_t *cls = nullptr, int32_t ck = 0) {
  B.nrows = nrows;
  if (hi < 0) hi = nrows;
  Buf<uint8_t> ids(c.A, nrows > 0 ? nrows : 1);
  Buf<i64> pos(c.A, nrows + 1);
  LV_LAUNCH(c, k_bin_ids, grid_for(c, nrows), 256, 0, nrows, ptr, ids.p, lo, hi, cls, ck);
  // counts per bin
  std::vector<i64> cnt(NBIN, 0);
  for (int b = 0; b < NBIN; ++b) {
    exclusive_scan<i64>(c, IsBin{ids.p, b}, nrows, pos.p, true);
    LV_CUDA(cudaMemcpyAsync(&cnt[b], pos.p + nrows, sizeof(i64), cudaMemcpyDeviceToHost, c.s));
    LV_CUDA(cudaStreamSynchronize(c.s));
    B.off[b + 1] = B.off[b] + cnt[b];
  }
  B.rows.alloc(c.A, B.off[NBIN] > 0 ? B.off[NBIN] : 1);
  for (int b = 0; b < NBIN; ++b) {
    if (!cnt[b]) continue;
    exclusive_scan<i64>(c, IsBin{ids.p, b}, nrows, pos.p, false);
    LV_LAUNCH(c, k_bin_scatter, grid_for(c, nrows), 256, 0, nrows, ids.p, b, pos.p, B.rows.p + B.off[b]);
  }
  if (rows_only) return;
  finish_bins(c, ptr, universe, B, cnt, nullptr);
}

// Row headers, per-bin edge counts (given, or summed here) and the hub path's chunk /
// bucket tables of bins whose rows (B.rows, B.off) are already grouped.
inline void finish_bins(Ctx &c, const i64 *ptr, i64 universe, Bins &B, const std::vector<i64> &cnt,
                        const i64 *edges) {
  B.hdr.alloc(c.A, B.off[NBIN] > 0 ? B.off[NBIN] : 1);
  if (B.off[NSMEM] > 0)
    LV_LAUNCH(c, k_fill_hdr, grid_for(c, B.off[NSMEM]), 256, 0, B.off[NSMEM], B.rows.p, ptr, B.hdr.p);
  if (edges) {
    for (int b = 0; b < NBIN; ++b) B.edges[b] = edges[b];
  } else {
    Buf<u64> es(c.A, NBIN);
    LV_CUDA(cudaMemsetAsync(es.p, 0, NBIN * sizeof(u64), c.s));
    for (int b = 0; b < NBIN; ++b)
      if (cnt[b]) LV_LAUNCH(c, k_sum_u64<BinLen>, grid_for(c, cnt[b]), 256, 0, BinLen{B.rows.p + B.off[b], ptr}, cnt[b], es.p + b);
    u64 he[NBIN];
    LV_CUDA(cudaMemcpyAsync(he, es.p, NBIN * sizeof(u64), cudaMemcpyDeviceToHost, c.s));
    LV_CUDA(cudaStreamSynchronize(c.s));
    for (int b = 0; b < NBIN; ++b) B.edges[b] = (i64)he[b];
  }
  // hubs
  B.nhub = cnt[NSMEM];
  B.nchunks = 0;
  B.nfin = 0;
  B.nseg = 0;
  if (B.nhub) {
    Buf<i64> hb(c.A, B.nhub), hl(c.A, B.nhub);
    LV_LAUNCH(c, k_gather_len, grid_for(c, B.nhub), 256, 0, B.nhub, B.rows.p + B.off[NSMEM], ptr, hb.p, hl.p);
    std::vector<i64> beg(B.nhub), len(B.nhub);
    LV_CUDA(cudaMemcpyAsync(beg.data(), hb.p, B.nhub * sizeof(i64), cudaMemcpyDeviceToHost, c.s));
    LV_CUDA(cudaMemcpyAsync(len.data(), hl.p, B.nhub * sizeof(i64), cudaMemcpyDeviceToHost, c.s));
    LV_CUDA(cudaStreamSynchronize(c.s));
    // cluster-eligible hub rows first (stable), the pool path's giant rows last
    B.ncl = 0;
    B.edges_cl = 0;
    B.cl_cs = hcl_cluster_size();
    if (B.cl_cs) {
      const i64 lim = hcl_max_len(B.cl_cs);
      std::vector<int32_t> hr(B.nhub), hr2;
      int32_t *dh = B.rows.p + B.off[NSMEM];
      LV_CUDA(cudaMemcpyAsync(hr.data(), dh, B.nhub * sizeof(int32_t), cudaMemcpyDeviceToHost, c.s));
      LV_CUDA(cudaStreamSynchronize(c.s));
      std::vector<i64> beg2, len2;
      for (int pass = 0; pass < 2; ++pass)
        for (i64 h = 0; h < B.nhub; ++h)
          if ((len[h] <= lim) == (pass == 0)) { hr2.push_back(hr[h]); beg2.push_back(beg[h]); len2.push_back(len[h]); }
      for (i64 h = 0; h < B.nhub; ++h)
        if (len2[h] <= lim) { ++B.ncl; B.edges_cl += len2[h]; }
      beg.swap(beg2);
      len.swap(len2);
      LV_CUDA(cudaMemcpyAsync(dh, hr2.data(), B.nhub * sizeof(int32_t), cudaMemcpyHostToDevice, c.s));
      if (B.ncl) {
        std::vector<i64> ord(B.ncl);
        for (i64 h = 0; h < B.ncl; ++h) ord[h] = h;
        std::stable_sort(ord.begin(), ord.end(), [&](i64 x, i64 y) { return len[x] > len[y]; });
        std::vector<RowHdr> ch(B.ncl);
        for (i64 j = 0; j < B.ncl; ++j) {
          ch[j].beg = beg[ord[j]];
          ch[j].r = hr2[ord[j]];
          ch[j].len = (int32_t)len[ord[j]];
        }
        B.clhdr.alloc(c.A, B.ncl);
        LV_CUDA(cudaMemcpyAsync(B.clhdr.p, ch.data(), B.ncl * sizeof(RowHdr), cudaMemcpyHostToDevice, c.s));
      }
      LV_CUDA(cudaStreamSynchronize(c.s));  // host vectors go out of scope
    }
    std::vector<i64> cfirst(B.nhub), bfirst(B.nhub), segoff;
    std::vector<int32_t> ccount(B.nhub), blg(B.nhub);
    std::vector<Chunk> ch;
    std::vector<int2> fit;
    // bucket table size: the smallest fin_lg whose buckets (<= 2^HUB_MAX_BLG per row) can
    // hold every hub row's distinct keys at the expected load
    i64 dmax = 0;
    for (i64 h = 0; h < B.nhub; ++h) dmax = std::max(dmax, std::min(len[h], universe));
    B.fin_lg = HUB_FIN_LG;
    while (B.fin_lg < HUB_FIN_LG_MAX && ((i64)1 << (B.fin_lg - 2 + HUB_MAX_BLG)) < dmax) ++B.fin_lg;
    // LV_HUB_BUCKET_TARGET (tests only) shrinks the bucket target to exercise many buckets
    static const char *tenv = getenv("LV_HUB_BUCKET_TARGET");
    const i64 target = tenv ? atoll(tenv) : ((i64)1 << (B.fin_lg - 2));
    for (i64 h = 0; h < B.nhub; ++h) {
      const i64 distinct_max = std::min(len[h], universe);
      int lgb = 0;
      while (lgb < HUB_MAX_BLG && (target << lgb) < distinct_max) ++lgb;
      LV_REQUIRE((target << lgb) >= distinct_max, LV_ERANGE,
                 "hub row too long for the bucketed hub path (" + std::to_string(len[h]) + " entries)");
      blg[h] = lgb;
      B.max_blg = std::max(B.max_blg, lgb);
      cfirst[h] = (i64)ch.size();
      for (i64 e = 0; e < len[h]; e += HUB_CHUNK) {
        Chunk k;
        k.beg = beg[h] + e;
        k.end = beg[h] + std::min(len[h], e + HUB_CHUNK);
        k.h = (int32_t)h;
        k.pad = 0;
        ch.push_back(k);
        segoff.push_back(B.nseg);
        B.nseg += ((i64)1 << lgb) + 1;
      }
      ccount[h] = (int32_t)((i64)ch.size() - cfirst[h]);
      bfirst[h] = (i64)fit.size();
      for (int b = 0; b < (1 << lgb); ++b) fit.push_back(make_int2((int)h, b));
    }
    B.nchunks = (i64)ch.size();
    B.nfin = (i64)fit.size();
    B.chunks.alloc(c.A, B.nchunks);
    B.cfirst.alloc(c.A, B.nhub);
    B.ccount.alloc(c.A, B.nhub);
    B.blg.alloc(c.A, B.nhub);
    B.bfirst.alloc(c.A, B.nhub);
    B.segoff.alloc(c.A, B.nchunks);
    B.seg.alloc(c.A, B.nseg);
    // batches of whole hub rows whose chunk pool fits a bound (reused by every batch)
    // (LV_HUB_POOL_CHUNKS, tests only, forces small batches)
    static const char *penv = getenv("LV_HUB_POOL_CHUNKS");
    const i64 POOL_CHUNKS_MAX = penv ? std::max<i64>(1, atoll(penv))
                                     : std::max<i64>(1, ((i64)4 << 30) / (HUB_CHUNK * 16));  // ~4 GB at u64
    B.h_cfirst = cfirst;
    B.h_cfirst.push_back(B.nchunks);
    B.h_bfirst = bfirst;
    B.h_bfirst.push_back(B.nfin);
    B.batch_h.assign(1, 0);
    B.pool_chunks = 0;
    for (i64 h = 0; h < B.nhub; ++h) {
      const i64 hb0 = B.batch_h.back();
      if (h > hb0 && (h == B.ncl || B.h_cfirst[h + 1] - B.h_cfirst[hb0] > POOL_CHUNKS_MAX)) B.batch_h.push_back(h);
    }
    B.batch_h.push_back(B.nhub);
    for (size_t i = 0; i + 1 < B.batch_h.size(); ++i)
      B.pool_chunks = std::max(B.pool_chunks, B.h_cfirst[B.batch_h[i + 1]] - B.h_cfirst[B.batch_h[i]]);
    B.pent.alloc(c.A, B.pool_chunks * HUB_CHUNK);  // packed 16-byte pool entries
    B.fitem.alloc(c.A, B.nfin);
    B.part.alloc(c.A, B.nfin);
    B.emit_cur.alloc(c.A, B.nhub);
    B.overflow.alloc(c.A, 1);
    LV_CUDA(cudaMemcpyAsync(B.chunks.p, ch.data(), B.nchunks * sizeof(Chunk), cudaMemcpyHostToDevice, c.s));
    LV_CUDA(cudaMemcpyAsync(B.cfirst.p, cfirst.data(), B.nhub * sizeof(i64), cudaMemcpyHostToDevice, c.s));
    LV_CUDA(cudaMemcpyAsync(B.ccount.p, ccount.data(), B.nhub * sizeof(int32_t), cudaMemcpyHostToDevice, c.s));
    LV_CUDA(cudaMemcpyAsync(B.blg.p, blg.data(), B.nhub * sizeof(int32_t), cudaMemcpyHostToDevice, c.s));
    LV_CUDA(cudaMemcpyAsync(B.bfirst.p, bfirst.data(), B.nhub * sizeof(i64), cudaMemcpyHostToDevice, c.s));
    LV_CUDA(cudaMemcpyAsync(B.segoff.p, segoff.data(), B.nchunks * sizeof(i64), cudaMemcpyHostToDevice, c.s));
    LV_CUDA(cudaMemcpyAsync(B.fitem.p, fit.data(), B.nfin * sizeof(int2), cudaMemcpyHostToDevice, c.s));
    LV_CUDA(cudaMemsetAsync(B.emit_cur.p, 0, B.nhub * sizeof(u64), c.s));
    LV_CUDA(cudaMemsetAsync(B.overflow.p, 0, sizeof(int), c.s));
    LV_CUDA(cudaStreamSynchronize(c.s));  // host vectors go out of scope
  }
}

// ----------------------------------------------------------------- launch
template <int G, int BLOCK, int MODE, class WT, class VT>
void launch_reg(Ctx &c, KTimer *tm, const AggArgs &a, const char *tag, cudaStream_t st) {
  constexpr bool NARROW = sizeof(VT) == 4;
  // SWEEP rows <= 16: the software-pipelined kernel (measured faster; at G = 32 the plain
  // one wins).  LV_REG_PIPE=0 / 2 force plain / pipelined everywhere.
  static const int pipe_env = getenv("LV_REG_PIPE") ? atoi(getenv("LV_REG_PIPE")) : 1;
  const bool pipe = pipe_env == 2 || (pipe_env == 1 && G <= 16);
  // SWEEP rows of <= LV_THR (default 8) entries: a thread per row (k_sweep_thr; C4 level-0
  // sweep: <= 8 bin 0.35 -> 0.26 ms, <= 4 bin 0.85 -> 0.80 ms, tools/variants.sh)
  if constexpr (MODE == M_SWEEP && G <= 8) {
    static const int thr_env = getenv("LV_THR") ? atoi(getenv("LV_THR")) : 8;
    if (G <= thr_env) {
      auto kt = k_sweep_thr<G, WT>;
      const int occ_t = kernel_occ(kt, 256, 0);
      const i64 grid_t = std::min<i64>(cdiv(a.nrows, 256), (i64)c.sms * occ_t * 8);
      if (tm) tm->begin(st, tag);
      LV_LAUNCH_ON(c, st, kt, (unsigned)grid_t, 256, 0, a);
      if (tm) tm->end(st);
      return;
    }
  }
  auto kern = (MODE == M_SWEEP && pipe) ? k_sweep_reg<G, BLOCK, WT, NARROW> : k_agg_reg<G, BLOCK, MODE, WT, NARROW>;
  constexpr int GPB = BLOCK / G;
  const int occ = kernel_occ(kern, BLOCK, 0);
  i64 grid = cdiv(a.nrows, GPB);
  // the pipelined kernel at G = 8, 16 is persistent (one resident wave: many rows per
  // group keep the pipeline full; measured faster), otherwise up to 8 waves
  static const int w4 = getenv("LV_REG_WAVES4") ? atoi(getenv("LV_REG_WAVES4")) : 8;  // experiments
  i64 cap = (i64)c.sms * occ * ((MODE == M_SWEEP && pipe && G >= 8) ? 1 : (G == 4 ? w4 : 8));
  if (grid > cap) grid = cap;
  if (tm) tm->begin(st, tag);
  LV_LAUNCH_ON(c, st, kern, (unsigned)grid, BLOCK, 0, a);
  if (tm) tm->end(st);
}

template <int G, int CAP, int BLOCK, int MODE, class WT, class VT>
void launch_bin(Ctx &c, KTimer *tm, const AggArgs &a, const char *tag, cudaStream_t st) {
  auto kern = k_agg_smem<G, CAP, BLOCK, MODE, WT, VT>;
  constexpr int GPB = BLOCK / G;
  const size_t smem = smem_bytes<G, CAP, BLOCK, VT, MODE>();
  const int occ = kernel_occ(kern, BLOCK, smem);
  i64 grid = cdiv(a.nrows, GPB);
  i64 cap = (i64)c.sms * occ * 8;
  if (grid > cap) grid = cap;
  if (tm) tm->begin(st, tag);  // events on the launching stream
  LV_LAUNCH_ON(c, st, kern, (unsigned)grid, BLOCK, smem, a);
  if (tm) tm->end(st);
}

static const char *BIN_NAME[NBIN] = {"reg_g4",    "reg_g8",    "reg_g16",    "reg_g32",
                                     "tab_le128", "tab_le256", "tab_le512",  "tab_le1024",
                                     "tab_le2048", "tab_le4096", "tab_le8192", "agg_hub"};

// The sweep kernel for the table bins (lv_sweep.cuh): WARPS warps per row, CAP slots.
template <int WARPS, int CAP, class WT, int U = 4>
void launch_tab(Ctx &c, KTimer *tm, const AggArgs &a, const char *tag, cudaStream_t st, bool s64all) {
  using Cfg = TabCfg<WARPS, CAP>;
  auto kern = s64all ? k_sweep_tab<WARPS, CAP, U, WT, true> : k_sweep_tab<WARPS, CAP, U, WT, false>;
  const int occ = kernel_occ(kern, Cfg::NT, Cfg::SMEM);
  i64 grid = cdiv(a.nrows, Cfg::GPC);
  const i64 cap = (i64)c.sms * occ * 8;
  if (grid > cap) grid = cap;
  if (tm) tm->begin(st, tag);
  LV_LAUNCH_ON(c, st, kern, (unsigned)grid, Cfg::NT, Cfg::SMEM, a);
  if (tm) tm->end(st);
}

// The cluster hub kernel over hub rows [0, B.ncl) (B.clhdr, by decreasing length):
// persistent, one cluster of B.cl_cs CTAs per resident slot.
template <int CS, class WT, bool S64ALL>
void launch_hcl_cs(Ctx &c, const AggArgs &a, const Bins &B, cudaStream_t st) {
  auto kern = k_hub_cl<CS, WT, S64ALL>;
  const int act = hcl_prepare<CS, WT, S64ALL>();
  LV_REQUIRE(act > 0, LV_ECUDA, "cluster hub kernel cannot be resident");
  const i64 ncl = std::min<i64>(B.ncl, act);
  cudaLaunchAttribute at[1];
  cudaLaunchConfig_t cfg = hcl_config(CS, (unsigned)(ncl * CS), st, at);
  LV_CUDA(cudaLaunchKernelEx(&cfg, kern, a, (const RowHdr *)B.clhdr.p, B.ncl, B.overflow.p));
  c.launches++;
}
template <class WT>
void launch_hcl(Ctx &c, KTimer *tm, const AggArgs &a, const Bins &B, cudaStream_t st, bool s64all, const char *tag) {
  if (tm) tm->begin(st, tag);
  if (B.cl_cs == 16) {
    if (s64all) launch_hcl_cs<16, WT, true>(c, a, B, st);
    else launch_hcl_cs<16, WT, false>(c, a, B, st);
  } else {
    if (s64all) launch_hcl_cs<8, WT, true>(c, a, B, st);
    else launch_hcl_cs<8, WT, false>(c, a, B, st);
  }
  if (tm) tm->end(st);
}

// One pass of MODE over every bin of B.  `a` carries the common arguments.  VT is the
// shared-table value type (uint32_t only when every row sum is known to be < 2^32).
template <int MODE, class WT, class VT>
void launch_agg(Ctx &c, const Bins &B, AggArgs a, KTimer *tm = nullptr, bool s64all = false) {
  static const char *MN[3] = {"sweep", "merge", "emit"};
  u64 *ctr = a.counters;  // NBIN slots of 8 counters (one per bin) or NULL
  auto set = [&](int b) {
    a.rows = B.rows.p + B.off[b];
    a.hdr = B.hdr.p + B.off[b];
    a.nrows = B.count(b);
    a.counters = ctr ? ctr + 8 * b : nullptr;
  };
  std::string pre = std::string(MN[MODE]) + ":";
  const bool conc = c.concurrent;
  if (conc) {  // fork: side streams start after everything already queued on the handle stream
    LV_CUDA(cudaEventRecord(c.fork_ev, c.s));
    for (int i = 0; i < Ctx::NSIDE; ++i) LV_CUDA(cudaStreamWaitEvent(c.side[i], c.fork_ev, 0));
  }
  cudaStream_t hub_s = conc ? c.side[0] : c.s;
  // hub path first (longest rows), then the big bins, then the small ones
  if (B.nhub) {
    set(NSMEM);
    a.chunks = B.chunks.p;
    HubArgs hb;
    hb.cfirst = B.cfirst.p;
    hb.ccount = B.ccount.p;
    hb.blg = B.blg.p;
    hb.bfirst = B.bfirst.p;
    hb.segoff = B.segoff.p;
    hb.seg = B.seg.p;
    hb.pent = B.pent.p;
    hb.fitem = B.fitem.p;
    hb.part = B.part.p;
    hb.emit_cur = B.emit_cur.p;
    hb.overflow = B.overflow.p;
    hb.nhub = B.nhub;
    hb.nchunks = B.nchunks;
    hb.nfin = B.nfin;
    hb.fin_lg = B.fin_lg;
    const size_t acc_smem = hub_acc_smem<VT, MODE>(B.max_blg);
    const size_t fin_smem = hub_fin_smem<VT, MODE>(B.fin_lg);
    const int occ_acc = kernel_occ(k_hub_acc<MODE, WT, VT>, HUB_ACC_T, acc_smem);
    // SWEEP: the two-barrier specialisation (k_hub_fin_sw); LV_HUB_FIN_OLD=1 keeps the
    // generic kernel (A/B)
    static const bool fin_old = getenv("LV_HUB_FIN_OLD") != nullptr;
    auto fin_kern = (MODE == M_SWEEP && !fin_old) ? k_hub_fin_sw<VT> : k_hub_fin<MODE, VT>;
    const int occ_fin = kernel_occ(fin_kern, HUB_FIN_T, fin_smem);
    // SWEEP with narrow tables: the cluster kernel takes hub rows [0, ncl)
    const bool use_cl = MODE == M_SWEEP && sizeof(VT) == 4 && B.ncl > 0;
    if (MODE == M_SWEEP) B.cl_used = use_cl;
    if constexpr (MODE == M_SWEEP && sizeof(VT) == 4) {
      if (use_cl) launch_hcl<WT>(c, tm, a, B, hub_s, s64all, (pre + "hub_cl").c_str());
    }
    for (size_t bi = 0; bi + 1 < B.batch_h.size(); ++bi) {  // batches of whole hub rows
      hb.h0 = B.batch_h[bi];
      hb.h1 = B.batch_h[bi + 1];
      if (use_cl && hb.h1 <= B.ncl) continue;
      hb.c0 = B.h_cfirst[hb.h0];
      hb.c1 = B.h_cfirst[hb.h1];
      hb.f0 = B.h_bfirst[hb.h0];
      hb.f1 = B.h_bfirst[hb.h1];
      const i64 g_acc = std::min<i64>(hb.c1 - hb.c0, (i64)c.sms * occ_acc);
      const i64 g_fin = std::min<i64>(hb.f1 - hb.f0, (i64)c.sms * occ_fin);
      if (tm) tm->begin(hub_s, pre + "hub_acc");
      LV_LAUNCH_ON(c, hub_s, (k_hub_acc<MODE, WT, VT>), (unsigned)g_acc, HUB_ACC_T, acc_smem, a, hb);
      if (tm) tm->end(hub_s);
      if (tm) tm->begin(hub_s, pre + "hub_fin");
      LV_LAUNCH_ON(c, hub_s, fin_kern, (unsigned)g_fin, HUB_FIN_T, fin_smem, a, hb);
      if (tm) tm->end(hub_s);
      if (tm) tm->begin(hub_s, pre + "hub_decide");
      LV_LAUNCH_ON(c, hub_s, (k_hub_decide<MODE>), (unsigned)cdiv(hb.h1 - hb.h0, 4), 128, 0, a, hb);
      if (tm) tm->end(hub_s);
    }
  }
  // bins in decreasing length; concurrent mode spreads them over the side streams
  auto st = [&](int k) { return conc ? c.side[(k + 1) % Ctx::NSIDE] : c.s; };
  // the table bins: the sweep-specialised kernel (narrow tables), else the generic one
  static const bool old_sweep = getenv("LV_OLD_SWEEP") != nullptr;  // A/B experiments
  const bool tab = MODE == M_SWEEP && sizeof(VT) == 4 && !old_sweep;
  const std::string tg = pre;
  auto nm = [&](int b) { return tg + BIN_NAME[b]; };
  if constexpr (MODE == M_SWEEP && sizeof(VT) == 4) {
    if (tab) {
      // warps per row: measured r2 (C4 level 0; 16 -> 32 warps: 1.24 -> 1.11 ms, 2 -> 4:
      // 1.24 -> 1.02 ms, 8 -> 16 in the 4096 bin: 1.45 -> 1.49 ms)
      // edges per lane per batch (C4 level 0, CUDA events, profiles/r2a[tuvw]_sweep_variants.txt):
      // 1 in the 4097-8192 bin (1.03 -> 0.84 ms) and the 33-128 bin (0.70 -> 0.68 ms); 2 in the
      // 129-256, 513-1024 and 2049-4096 bins (0.76 -> 0.71, 1.02 -> 0.95, 1.39 -> 1.30 ms) — the
      // smaller batches keep fewer registers live and fill a row's last batch better; 4 in the
      // 1025-2048 bin (0.59 -> 0.65 ms with 2, 0.84 with 1 at level 1).
      // LV_TAB_U1 / LV_TAB_U2 (experiments): bit b = bin b with 1 / 2 edges per lane.
      static const int u2 = getenv("LV_TAB_U2") ? atoi(getenv("LV_TAB_U2")) : (32 | 128 | 512);
      static const int u1 = getenv("LV_TAB_U1") ? atoi(getenv("LV_TAB_U1")) : (16 | 1024);
#define LV_TABU(b, W_, C_, S_)                                                                \
  if (B.count(b)) {                                                                          \
    set(b);                                                                                  \
    if ((u1 >> (b)) & 1) launch_tab<W_, C_, WT, 1>(c, tm, a, nm(b).c_str(), st(S_), s64all); \
    else if ((u2 >> (b)) & 1) launch_tab<W_, C_, WT, 2>(c, tm, a, nm(b).c_str(), st(S_), s64all); \
    else launch_tab<W_, C_, WT>(c, tm, a, nm(b).c_str(), st(S_), s64all);                    \
  }
      LV_TABU(10, 32, 16384, 1)
      LV_TABU(9, 8, 8192, 0)
      LV_TABU(8, 4, 4096, 1)
      LV_TABU(7, 4, 2048, 2)
      LV_TABU(6, 1, 1024, 0)
      LV_TABU(5, 1, 512, 1)
      LV_TABU(4, 1, 256, 2)
#undef LV_TABU
    }
  }
  if (!tab) {
    if (B.count(10)) { set(10); launch_bin<1024, 16384, 1024, MODE, WT, VT>(c, tm, a, nm(10).c_str(), st(1)); }
    if (B.count(9)) { set(9); launch_bin<512, 8192, 512, MODE, WT, VT>(c, tm, a, nm(9).c_str(), st(0)); }
    if (B.count(8)) { set(8); launch_bin<256, 4096, 256, MODE, WT, VT>(c, tm, a, nm(8).c_str(), st(1)); }
    if (B.count(7)) { set(7); launch_bin<256, 4096, 256, MODE, WT, VT>(c, tm, a, nm(7).c_str(), st(2)); }
    if (B.count(6)) { set(6); launch_bin<128, 1024, 128, MODE, WT, VT>(c, tm, a, nm(6).c_str(), st(0)); }
    if (B.count(5)) { set(5); launch_bin<128, 1024, 128, MODE, WT, VT>(c, tm, a, nm(5).c_str(), st(1)); }
    if (B.count(4)) { set(4); launch_bin<32, 256, 256, MODE, WT, VT>(c, tm, a, nm(4).c_str(), st(2)); }
  }
  if (B.count(3)) { set(3); launch_reg<32, 256, MODE, WT, VT>(c, tm, a, (pre + BIN_NAME[3]).c_str(), st(1)); }
  if (B.count(2)) { set(2); launch_reg<16, 256, MODE, WT, VT>(c, tm, a, (pre + BIN_NAME[2]).c_str(), st(2)); }
  if (B.count(1)) { set(1); launch_reg<8, 256, MODE, WT, VT>(c, tm, a, (pre + BIN_NAME[1]).c_str(), st(0)); }
  if (B.count(0)) { set(0); launch_reg<4, 256, MODE, WT, VT>(c, tm, a, (pre + BIN_NAME[0]).c_str(), st(1)); }
  if (conc) {  // join: the handle stream waits for every side stream
    for (int i = 0; i < Ctx::NSIDE; ++i) {
      LV_CUDA(cudaEventRecord(c.join_ev[i], c.side[i]));
      LV_CUDA(cudaStreamWaitEvent(c.s, c.join_ev[i], 0));
    }
  }
  if (B.nhub && !c.capturing) {  // a bucket beyond its distinct-key capacity would have been dropped
    int ovf = 0;
    LV_CUDA(cudaMemcpyAsync(&ovf, B.overflow.p, sizeof(int), cudaMemcpyDeviceToHost, c.s));
    LV_CUDA(cudaStreamSynchronize(c.s));
    LV_REQUIRE(ovf == 0, LV_ECUDA, "hub bucket overflow (a hash bucket exceeded its table)");
  }
}

// s64all: every score of the pass fits int64 (2W·max δ < 2^63, checked by the caller)
template <int MODE>
void launch_agg_wt(Ctx &c, int wt, bool narrow, const Bins &B, const AggArgs &a, KTimer *tm = nullptr,
                   bool s64all = false) {
  if (narrow) {
    if (wt == WT_NONE) launch_agg<MODE, WNone, uint32_t>(c, B, a, tm, s64all);
    else if (wt == WT_U32) launch_agg<MODE, WU32, uint32_t>(c, B, a, tm, s64all);
    else launch_agg<MODE, WU64, uint32_t>(c, B, a, tm, s64all);
  } else {
    if (wt == WT_NONE) launch_agg<MODE, WNone, u64>(c, B, a, tm);
    else if (wt == WT_U32) launch_agg<MODE, WU32, u64>(c, B, a, tm);
    else launch_agg<MODE, WU64, u64>(c, B, a, tm);
  }
}

}  // namespace lv
