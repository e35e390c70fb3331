// lv_scan.cuh — device-wide exclusive prefix sum (three-phase: tile reduce, scan of tile
// sums, tile scan).  Used for the row offsets of "Neighbor computation" (P:L271,
// "exclusive_scan"), the renumbering prefix sum (reading D18) and the
// contraction's row offsets.  Input comes from a functor so that flags and
// lengths are never materialised.
#pragma once
#include "lv_common.cuh"

namespace lv {

constexpr int SCAN_T = 256;
constexpr int SCAN_IPT = 16;
constexpr int SCAN_TILE = SCAN_T * SCAN_IPT;

template <typename T>
struct ArrayIn {
  const T *a;
  __device__ __forceinline__ T operator()(i64 i) const { return a[i]; }
};

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int l = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T t = __shfl_up_sync(0xffffffffu, v, o);
    if (l >= o) v += t;
  }
  return v;
}

// exclusive block scan of one value per thread; returns (exclusive prefix, block total)
template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T &total) {
  __shared__ T wsum[SCAN_T / 32];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  T inc = warp_incl_scan(v);
  if (l == 31) wsum[w] = inc;
  __syncthreads();
  if (w == 0) {
    T x = (l < SCAN_T / 32) ? wsum[l] : T(0);
    x = warp_incl_scan(x);
    if (l < SCAN_T / 32) wsum[l] = x;
  }
  __syncthreads();
  T pre = (w > 0 ? wsum[w - 1] : T(0)) + inc - v;
  total = wsum[SCAN_T / 32 - 1];
  __syncthreads();
  return pre;
}

template <typename T, typename F>
__global__ void __launch_bounds__(SCAN_T) k_scan_reduce(F f, i64 n, T *bsum) {
  const i64 base = (i64)blockIdx.x * SCAN_TILE;
  T s = 0;
#pragma unroll 4
  for (int k = 0; k < SCAN_IPT; ++k) {
    i64 i = base + (i64)k * SCAN_T + threadIdx.x;
    if (i < n) s += f(i);
  }
  T tot;
  block_excl_scan<T>(s, tot);
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

template <typename T, typename F>
__global__ void __launch_bounds__(SCAN_T) k_scan_tile(F f, i64 n, const T *bprefix, T *out,
                                                      int write_total) {
  __shared__ T tile[SCAN_TILE];
  const i64 base = (i64)blockIdx.x * SCAN_TILE;
#pragma unroll 4
  for (int k = 0; k < SCAN_IPT; ++k) {
    int j = k * SCAN_T + threadIdx.x;
    i64 i = base + j;
    tile[j] = (i < n) ? f(i) : T(0);
  }
  __syncthreads();
  T v[SCAN_IPT];
  T s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_IPT; ++k) {
    v[k] = tile[threadIdx.x * SCAN_IPT + k];
    s += v[k];
  }
  T tot;
  T run = block_excl_scan<T>(s, tot) + (bprefix ? bprefix[blockIdx.x] : T(0));
#pragma unroll
  for (int k = 0; k < SCAN_IPT; ++k) {
    tile[threadIdx.x * SCAN_IPT + k] = run;
    run += v[k];
  }
  __syncthreads();
#pragma unroll 4
  for (int k = 0; k < SCAN_IPT; ++k) {
    int j = k * SCAN_T + threadIdx.x;
    i64 i = base + j;
    if (i < n) out[i] = tile[j];
  }
  if (write_total && blockIdx.x == gridDim.x - 1 && threadIdx.x == SCAN_T - 1)
    out[n] = run;  // last thread's running value = grand total
}

template <typename T>
__global__ void k_set_scalar(T *p, T v) { *p = v; }

// out[0..n) = exclusive prefix of f; if write_total, out[n] = total (out holds n+1).
template <typename T, typename F>
void exclusive_scan(Ctx &c, F f, i64 n, T *out, bool write_total) {
  if (n <= 0) {
    if (write_total) LV_LAUNCH(c, k_set_scalar<T>, 1, 1, 0, out, T(0));
    return;
  }
  const i64 nb = cdiv(n, SCAN_TILE);
  if (nb == 1) {
    LV_LAUNCH(c, (k_scan_tile<T, F>), 1, SCAN_T, 0, f, n, (const T *)nullptr, out, (int)write_total);
    return;
  }
  Buf<T> bsum(c.A, nb), bpre(c.A, nb);
  LV_LAUNCH(c, (k_scan_reduce<T, F>), (unsigned)nb, SCAN_T, 0, f, n, bsum.p);
  exclusive_scan<T, ArrayIn<T>>(c, ArrayIn<T>{bsum.p}, nb, bpre.p, false);
  LV_LAUNCH(c, (k_scan_tile<T, F>), (unsigned)nb, SCAN_T, 0, f, n, (const T *)bpre.p, out, (int)write_total);
}

// Device-wide sum into *out (u64), via scan-reduce blocks + atomics.
template <typename F>
__global__ void __launch_bounds__(256) k_sum_u64(F f, i64 n, u64 *out) {
  u64 s = 0;
  for (i64 i = (i64)blockIdx.x * 256 + threadIdx.x; i < n; i += (i64)gridDim.x * 256) s += f(i);
  s = block_sum_u64<256>(s);
  if (threadIdx.x == 0 && s) atomicAdd(out, s);
}

// Device-wide max of non-negative values into *out (u64).
template <typename F>
__global__ void __launch_bounds__(256) k_max_u64(F f, i64 n, u64 *out) {
  u64 m = 0;
  for (i64 i = (i64)blockIdx.x * 256 + threadIdx.x; i < n; i += (i64)gridDim.x * 256) {
    const u64 x = (u64)f(i);
    m = x > m ? x : m;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const u64 y = __shfl_xor_sync(0xffffffffu, m, o);
    m = y > m ? y : m;
  }
  if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

// Device-wide sum of squares of non-negative i64 values (exact 128-bit) into out[0]=lo,out[1]=hi.
template <typename F>
__global__ void __launch_bounds__(256) k_sumsq_u128(F f, i64 n, u64 *out) {
  u64 hi = 0, lo = 0;
  for (i64 i = (i64)blockIdx.x * 256 + threadIdx.x; i < n; i += (i64)gridDim.x * 256) {
    u64 x = (u64)f(i);
    u128 sq = (u128)x * x;
    add128(hi, lo, (u64)(sq >> 64), (u64)sq);
  }
  // warp reduce of 128-bit values
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    u64 ohi = __shfl_xor_sync(0xffffffffu, hi, o), olo = __shfl_xor_sync(0xffffffffu, lo, o);
    add128(hi, lo, ohi, olo);
  }
  if ((threadIdx.x & 31) == 0 && (hi | lo)) atomic_add128(out, out + 1, hi, lo);
}

}  // namespace lv
