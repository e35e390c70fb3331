// lv_color.cuh — the distance-1 colouring heuristic (reading D29).
//
// Lu et al.'s colouring heuristic — one of "the other heuristics" the paper leaves to
// future work: colour the level graph so that no two neighbours share a
// colour, then sweep the colour classes in turn; a class decides in parallel (its
// vertices are pairwise non-adjacent, so none reads another's changing label) against
// the state the previous class committed.  This removes the Jacobi swap oscillation of
// the fully synchronous sweep (Alg. 1).
//
// Colouring: Jones–Plassmann with priorities π(v) = fmix64(v ^ 0x9E37...) keyed on the
// level graph's vertex id: a vertex whose higher-priority neighbours are all coloured
// takes the smallest colour none of them uses — exactly the greedy colouring in
// decreasing-π order (what the oracle computes sequentially), independent of schedule.
#pragma once
#include "lv_bins.cuh"

namespace lv {

__device__ __forceinline__ u64 color_prio(i64 v) {  // MurmurHash3 fmix64 (a bijection)
  u64 k = (u64)v ^ 0x9E3779B97F4A7C15ull;
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return k;
}

// Jones–Plassmann as a topological sweep of the priority DAG (edges from higher to lower
// priority), so every row is scanned a constant number of times instead of once per
// round it waits: wait[v] = number of higher-priority neighbours not yet coloured; a
// round colours its frontier (rows with wait = 0: colour = smallest colour no
// higher-priority neighbour uses — all of them final) and decrements the counters of the
// lower-priority neighbours, which join the next frontier when theirs reaches 0.  Same
// colouring as the sequential greedy in decreasing-π order; rounds = the longest
// decreasing-priority path.
// π of every row, once per colouring (saves the orig[] indirection in every scan)
__global__ void k_jp_prio(i64 n, const int32_t *__restrict__ orig, u64 *pri) {
  for (i64 v = (i64)blockIdx.x * 256 + threadIdx.x; v < n; v += (i64)gridDim.x * 256)
    pri[v] = color_prio(orig ? orig[v] : v);
}

// Rows longer than JP_LONG take a CTA each (k_jp_round_long) — a warp per 400k-entry hub
// row would serialise its round.  Frontier lists: [0] short rows, [1] long rows.
constexpr i64 JP_LONG = 1024;
constexpr int JP_CTA = 1024;
constexpr int JP_BITS = 8192;  // colours < 8192 tracked in shared memory (more: rescans)

__device__ __forceinline__ void jp_push(const i64 *rp, int32_t u, int32_t *wl_s, u64 *cnt_s, int32_t *wl_l,
                                        u64 *cnt_l) {
  if (rp[u + 1] - rp[u] > JP_LONG) wl_l[atomicAdd((unsigned long long *)cnt_l, 1ull)] = u;
  else wl_s[atomicAdd((unsigned long long *)cnt_s, 1ull)] = u;
}

__global__ void __launch_bounds__(256) k_jp_init(i64 n, const i64 *__restrict__ rp, const int32_t *__restrict__ col,
                                                 const u64 *__restrict__ pri, int32_t *wait, int32_t *wl_s,
                                                 u64 *cnt_s, int32_t *wl_l, u64 *cnt_l) {
  const int lane = threadIdx.x & 31;
  const i64 nw = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 v = (((i64)blockIdx.x * blockDim.x) + threadIdx.x) >> 5; v < n; v += nw) {
    const u64 pv = pri[v];
    int32_t c = 0;
    for (i64 k = rp[v] + lane; k < rp[v + 1]; k += 32) c += pri[col[k]] > pv;
    c = __reduce_add_sync(0xffffffffu, (uint32_t)c);
    if (lane == 0) {
      wait[v] = c;
      if (c == 0) jp_push(rp, (int32_t)v, wl_s, cnt_s, wl_l, cnt_l);
    }
  }
}

// Short rows: a warp each; 4 entries per lane in flight (the round's critical path is
// its longest row's chain of dependent loads).
constexpr int JP_U = 4;
__global__ void __launch_bounds__(256) k_jp_round(const int32_t *__restrict__ wl_in, const u64 *__restrict__ cnt_in,
                                                  const i64 *__restrict__ rp, const int32_t *__restrict__ col,
                                                  const u64 *__restrict__ pri, int32_t *color, int32_t *wait,
                                                  int32_t *wl_s, u64 *cnt_s, int32_t *wl_l, u64 *cnt_l) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const i64 nw = ((i64)gridDim.x * blockDim.x) >> 5;
  const i64 cnt = (i64)*cnt_in;
  for (i64 t = (((i64)blockIdx.x * blockDim.x) + threadIdx.x) >> 5; t < cnt; t += nw) {
    const int32_t v = wl_in[t];
    const u64 pv = pri[v];
    const i64 b = rp[v], e = rp[v + 1];
    int c = -1;
    for (int base = 0; c < 0; base += 64) {  // colour windows [base, base + 64)
      u64 m = 0;
      for (i64 k0 = b; k0 < e; k0 += 32 * JP_U) {
        int32_t u[JP_U];
        bool hi[JP_U];
#pragma unroll
        for (int j = 0; j < JP_U; ++j) {
          const i64 k = k0 + j * 32 + lane;
          u[j] = k < e ? col[k] : -1;
        }
#pragma unroll
        for (int j = 0; j < JP_U; ++j) hi[j] = u[j] >= 0 && pri[u[j]] > pv;
#pragma unroll
        for (int j = 0; j < JP_U; ++j) {
          if (u[j] < 0) continue;
          if (hi[j]) {
            const int32_t cu = __ldcg(&color[u[j]]);  // final: coloured in an earlier round
            if (cu >= base && cu < base + 64) m |= 1ull << (cu - base);
          } else if (base == 0 && atomicSub(&wait[u[j]], 1) == 1) {  // u's last higher neighbour
            jp_push(rp, u[j], wl_s, cnt_s, wl_l, cnt_l);
          }
        }
      }
      const u64 all = ((u64)__reduce_or_sync(full, (uint32_t)(m >> 32)) << 32) | __reduce_or_sync(full, (uint32_t)m);
      if (~all) c = base + __ffsll((long long)~all) - 1;
    }
    if (lane == 0) __stcg(&color[v], c);
  }
}

// Long rows: a CTA each, the used colours as a shared bitmap.
__global__ void __launch_bounds__(JP_CTA) k_jp_round_long(const int32_t *__restrict__ wl_in,
                                                          const u64 *__restrict__ cnt_in, const i64 *__restrict__ rp,
                                                          const int32_t *__restrict__ col,
                                                          const u64 *__restrict__ pri, int32_t *color,
                                                          int32_t *wait, int32_t *wl_s, u64 *cnt_s, int32_t *wl_l,
                                                          u64 *cnt_l) {
  __shared__ uint32_t bits[JP_BITS / 32];
  __shared__ int best;
  const i64 cnt = (i64)*cnt_in;
  for (i64 t = blockIdx.x; t < cnt; t += gridDim.x) {
    const int32_t v = wl_in[t];
    const u64 pv = pri[v];
    const i64 b = rp[v], e = rp[v + 1];
    int c = -1;
    for (int base = 0; c < 0; base += JP_BITS) {
      for (int i = threadIdx.x; i < JP_BITS / 32; i += JP_CTA) bits[i] = 0;
      if (threadIdx.x == 0) best = INT32_MAX;
      __syncthreads();
      for (i64 k0 = b; k0 < e; k0 += (i64)JP_CTA * JP_U) {
        int32_t u[JP_U];
        bool hi[JP_U];
#pragma unroll
        for (int j = 0; j < JP_U; ++j) {
          const i64 k = k0 + (i64)j * JP_CTA + threadIdx.x;
          u[j] = k < e ? col[k] : -1;
        }
#pragma unroll
        for (int j = 0; j < JP_U; ++j) hi[j] = u[j] >= 0 && pri[u[j]] > pv;
#pragma unroll
        for (int j = 0; j < JP_U; ++j) {
          if (u[j] < 0) continue;
          if (hi[j]) {
            const int32_t cu = __ldcg(&color[u[j]]) - base;
            if (cu >= 0 && cu < JP_BITS) atomicOr(&bits[cu >> 5], 1u << (cu & 31));
          } else if (base == 0 && atomicSub(&wait[u[j]], 1) == 1) {
            jp_push(rp, u[j], wl_s, cnt_s, wl_l, cnt_l);
          }
        }
      }
      __syncthreads();
      for (int i = threadIdx.x; i < JP_BITS / 32; i += JP_CTA)
        if (~bits[i]) atomicMin(&best, i * 32 + __ffs(~bits[i]) - 1);
      __syncthreads();
      if (best != INT32_MAX) c = base + best;
      __syncthreads();
    }
    if (threadIdx.x == 0) __stcg(&color[v], c);
  }
}

__global__ void k_fill_i32(i64 n, int32_t *a, int32_t v) {
  for (i64 i = (i64)blockIdx.x * 256 + threadIdx.x; i < n; i += (i64)gridDim.x * 256) a[i] = v;
}

// out[i] = src[idx[i]]
__global__ void k_gather_i32(i64 n, const int32_t *__restrict__ idx, const int32_t *__restrict__ src, int32_t *out) {
  for (i64 i = (i64)blockIdx.x * 256 + threadIdx.x; i < n; i += (i64)gridDim.x * 256) out[i] = src[idx[i]];
}

// class = min(colour, cap - 1) (cap > 0; reading D29); returns via max_of the largest colour
__global__ void k_cap_classes(i64 n, int32_t *color, int32_t cap) {
  for (i64 i = (i64)blockIdx.x * 256 + threadIdx.x; i < n; i += (i64)gridDim.x * 256)
    if (cap > 0 && color[i] > cap - 1) color[i] = cap - 1;
}

// Exact ΔI2 of a pass whose moving vertices may be adjacent (the capped last class of
// D29, swept synchronously): I2 = Σ_directed w_ij [C(i) = C(j)], so over the rows of the
// pass ΔI2 = Σ_{i moved} Σ_j w_ij ([C'(i) = C'(j)] − [C(i) = C(j)]) · (j moved ? 1 : 2)
// (an entry (j, i) with j unmoved is only seen from i's row).  A warp per row.
__global__ void __launch_bounds__(256) k_delta_i2(i64 nrows, const int32_t *__restrict__ rows,
                                                  const i64 *__restrict__ rp, const int32_t *__restrict__ col,
                                                  const void *w, int wt, const int32_t *__restrict__ lab0,
                                                  const int32_t *__restrict__ lab1, u64 *out) {
  const int lane = threadIdx.x & 31;
  const i64 nw = ((i64)gridDim.x * blockDim.x) >> 5;
  i64 acc = 0;
  for (i64 t = (((i64)blockIdx.x * blockDim.x) + threadIdx.x) >> 5; t < nrows; t += nw) {
    const int32_t i = rows[t];
    const int32_t a0 = lab0[i], a1 = lab1[i];
    if (a0 == a1) continue;  // warp-uniform
    for (i64 k = rp[i] + lane; k < rp[i + 1]; k += 32) {
      const int32_t j = col[k];
      const int32_t b0 = lab0[j], b1 = lab1[j];
      const i64 wk = wt == 0 ? 1 : wt == 1 ? (i64)((const uint32_t *)w)[k] : (i64)((const u64 *)w)[k];
      const i64 d = (i64)(a1 == b1) - (i64)(a0 == b0);
      acc += d * wk * (b0 != b1 ? 1 : 2);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0 && acc) atomicAdd((unsigned long long *)out, (unsigned long long)acc);
}

struct ColorArr {
  const int32_t *c;
  __device__ __forceinline__ u64 operator()(i64 i) const { return (u64)(i64)c[i]; }
};

// Degree bins of every colour class at once: one counting pass keyed by
// (class, bin), one scatter, then per class a slice copy + headers (+ hub tables) —
// instead of K full build_bins passes (9 scans each), which dominated small dense levels
// with hundreds of classes.  Row order within a (class, bin) follows the scatter's atomics:
// every consumer's result is order-independent (exact sums, total-order argmax).
__global__ void k_cls_count(i64 n, const i64 *__restrict__ rp, const int32_t *__restrict__ cls, uint32_t *cnt,
                            u64 *edges) {
  for (i64 r = (i64)blockIdx.x * 256 + threadIdx.x; r < n; r += (i64)gridDim.x * 256) {
    const i64 d = rp[r + 1] - rp[r];
    const int b = bin_of(d);
    if (b == 255) continue;
    const i64 key = (i64)cls[r] * NBIN + b;
    atomicAdd(&cnt[key], 1u);
    atomicAdd((unsigned long long *)&edges[key], (unsigned long long)d);
  }
}

__global__ void k_cls_scatter(i64 n, const i64 *__restrict__ rp, const int32_t *__restrict__ cls,
                              const i64 *__restrict__ off, uint32_t *cur, int32_t *rows) {
  for (i64 r = (i64)blockIdx.x * 256 + threadIdx.x; r < n; r += (i64)gridDim.x * 256) {
    const int b = bin_of(rp[r + 1] - rp[r]);
    if (b == 255) continue;
    const i64 key = (i64)cls[r] * NBIN + b;
    rows[off[key] + atomicAdd(&cur[key], 1u)] = (int32_t)r;
  }
}

inline void build_class_bins(Ctx &c, const i64 *rp, i64 n, const int32_t *cls, int32_t K,
                             std::vector<std::unique_ptr<Bins>> &out) {
  const size_t nk = (size_t)K * NBIN;
  Buf<uint32_t> cnt(c.A, 2 * nk);
  Buf<u64> ed(c.A, nk);
  LV_CUDA(cudaMemsetAsync(cnt.p, 0, 2 * nk * sizeof(uint32_t), c.s));
  LV_CUDA(cudaMemsetAsync(ed.p, 0, nk * sizeof(u64), c.s));
  LV_LAUNCH(c, k_cls_count, grid_for(c, n), 256, 0, n, rp, cls, cnt.p, ed.p);
  std::vector<uint32_t> hc(nk);
  std::vector<u64> he(nk);
  LV_CUDA(cudaMemcpyAsync(hc.data(), cnt.p, nk * sizeof(uint32_t), cudaMemcpyDeviceToHost, c.s));
  LV_CUDA(cudaMemcpyAsync(he.data(), ed.p, nk * sizeof(u64), cudaMemcpyDeviceToHost, c.s));
  LV_CUDA(cudaStreamSynchronize(c.s));
  std::vector<i64> off(nk + 1, 0);
  for (size_t k = 0; k < nk; ++k) off[k + 1] = off[k] + hc[k];
  Buf<i64> doff(c.A, nk + 1);
  Buf<int32_t> rows(c.A, off[nk] > 0 ? off[nk] : 1);
  LV_CUDA(cudaMemcpyAsync(doff.p, off.data(), (nk + 1) * sizeof(i64), cudaMemcpyHostToDevice, c.s));
  LV_LAUNCH(c, k_cls_scatter, grid_for(c, n), 256, 0, n, rp, cls, doff.p, cnt.p + nk, rows.p);
  for (int32_t k = 0; k < K; ++k) {
    auto B = std::make_unique<Bins>();
    B->nrows = n;
    std::vector<i64> cb(NBIN);
    i64 eb[NBIN];
    for (int b = 0; b < NBIN; ++b) {
      cb[b] = hc[(size_t)k * NBIN + b];
      eb[b] = (i64)he[(size_t)k * NBIN + b];
      B->off[b + 1] = B->off[b] + cb[b];
    }
    const i64 tot = B->off[NBIN];
    B->rows.alloc(c.A, tot > 0 ? tot : 1);
    if (tot > 0)
      LV_CUDA(cudaMemcpyAsync(B->rows.p, rows.p + off[(size_t)k * NBIN], tot * sizeof(int32_t),
                              cudaMemcpyDeviceToDevice, c.s));
    finish_bins(c, rp, n, *B, cb, eb);
    out.push_back(std::move(B));
  }
}

// Colour the n rows of (rp, col); returns the number of colours K.  ROUNDS_PER_SYNC
// rounds are queued between host checks of the frontier size (a round on an empty
// frontier is a no-op).
inline int32_t color_graph(Ctx &c, i64 n, const i64 *rp, const int32_t *col, const int32_t *orig, Buf<int32_t> &color,
                           int32_t *rounds_out = nullptr) {
  constexpr int ROUNDS_PER_SYNC = 32;
  color.alloc(c.A, n > 0 ? n : 1);
  if (n == 0) return 0;
  Buf<int32_t> wl[2][2], wait(c.A, n);  // [buffer][short, long]
  for (auto &x : wl)
    for (auto &y : x) y.alloc(c.A, n);
  Buf<u64> cnt(c.A, 4);  // [buffer * 2 + kind]
  LV_CUDA(cudaMemsetAsync(cnt.p, 0, 4 * sizeof(u64), c.s));
  const unsigned grid = (unsigned)std::min<i64>(cdiv(n, 8), (i64)c.sms * 8);
  const unsigned grid_l = (unsigned)c.sms * 2;
  Buf<u64> pri(c.A, n);
  LV_LAUNCH(c, k_jp_prio, grid_for(c, n), 256, 0, n, orig, pri.p);
  LV_LAUNCH(c, k_jp_init, grid, 256, 0, n, rp, col, pri.p, wait.p, wl[0][0].p, cnt.p, wl[0][1].p, cnt.p + 1);
  int32_t rounds = 0, cur = 0;
  for (;;) {
    for (int r = 0; r < ROUNDS_PER_SYNC; ++r) {
      const int nx = cur ^ 1;
      u64 *cs = cnt.p + 2 * nx, *cl = cnt.p + 2 * nx + 1;
      LV_CUDA(cudaMemsetAsync(cs, 0, 2 * sizeof(u64), c.s));
      LV_LAUNCH(c, k_jp_round_long, grid_l, JP_CTA, 0, wl[cur][1].p, cnt.p + 2 * cur + 1, rp, col, pri.p, color.p,
                wait.p, wl[nx][0].p, cs, wl[nx][1].p, cl);
      LV_LAUNCH(c, k_jp_round, grid, 256, 0, wl[cur][0].p, cnt.p + 2 * cur, rp, col, pri.p, color.p, wait.p,
                wl[nx][0].p, cs, wl[nx][1].p, cl);
      cur = nx;
      ++rounds;
    }
    u64 h[2] = {0, 0};
    LV_CUDA(cudaMemcpyAsync(h, cnt.p + 2 * cur, 2 * sizeof(u64), cudaMemcpyDeviceToHost, c.s));
    LV_CUDA(cudaStreamSynchronize(c.s));
    static const bool trace = getenv("LV_COLOR_TRACE") != nullptr;
    if (trace) fprintf(stderr, "jp: n=%lld rounds=%d frontier short=%llu long=%llu\n", (long long)n, rounds,
                       (unsigned long long)h[0], (unsigned long long)h[1]);
    if (h[0] == 0 && h[1] == 0) break;
    LV_REQUIRE(rounds <= n + ROUNDS_PER_SYNC, LV_ECUDA, "colouring did not converge");
  }
  if (rounds_out) *rounds_out = rounds;  // rounds issued (a multiple of ROUNDS_PER_SYNC)
  Buf<u64> t(c.A, 1);
  LV_CUDA(cudaMemsetAsync(t.p, 0, sizeof(u64), c.s));
  LV_LAUNCH(c, k_max_u64<ColorArr>, grid_for(c, n), 256, 0, ColorArr{color.p}, n, t.p);
  u64 mx = 0;
  LV_CUDA(cudaMemcpyAsync(&mx, t.p, sizeof(u64), cudaMemcpyDeviceToHost, c.s));
  LV_CUDA(cudaStreamSynchronize(c.s));
  return (int32_t)mx + 1;
}

}  // namespace lv
