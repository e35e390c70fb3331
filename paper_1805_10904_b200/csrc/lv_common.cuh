// lv_common.cuh — shared plumbing of liblouvain (sm_100a): error handling, the device
// allocator, launch accounting and small device helpers (warp/block reductions).
// Nothing here implements a step of the method; see lv_agg.cuh / lv_graph.cuh.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <string>
#include <vector>

#include "louvain.h"

namespace lv {

typedef unsigned long long u64;
typedef long long i64;
typedef __int128 i128;
typedef unsigned __int128 u128;

struct Error {
  int code;
  std::string msg;
};

#define LV_CUDA(x)                                                                          \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess)                                                                  \
      throw ::lv::Error{LV_ECUDA, std::string(#x) + " -> " + cudaGetErrorString(e_) +       \
                                      " @" + __FILE__ + ":" + std::to_string(__LINE__)};    \
  } while (0)

#define LV_REQUIRE(cond, code, msg)                      \
  do {                                                   \
    if (!(cond)) throw ::lv::Error{(code), (msg)};      \
  } while (0)

// ------------------------------------------------------------------ device memory
struct Alloc {
  louvain_alloc_fn a = nullptr;
  louvain_free_fn f = nullptr;
  void *ctx = nullptr;
  cudaStream_t s = nullptr;
  size_t live = 0, peak = 0;

  void *get(size_t bytes) {
    if (bytes == 0) bytes = 16;
    bytes = (bytes + 255) & ~size_t(255);
    void *p = nullptr;
    if (a) {
      p = a(ctx, bytes, (void *)s);
      if (!p) {
        size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        throw Error{LV_ENOMEM, "device allocation hook failed (" + std::to_string(bytes) + " B; library live " +
                                   std::to_string(live) + " B, peak " + std::to_string(peak) + " B; device free " +
                                   std::to_string(fr) + " of " + std::to_string(tot) + " B)"};
      }
    } else {
      cudaError_t e = cudaMallocAsync(&p, bytes, s);
      if (e != cudaSuccess) {  // freed blocks may be fragmented in the pool: trim it, retry once
        cudaGetLastError();
        int dev = 0;
        cudaGetDevice(&dev);
        cudaMemPool_t pool;
        cudaStreamSynchronize(s);
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
        e = cudaMallocAsync(&p, bytes, s);
      }
      if (e != cudaSuccess) {
        cudaGetLastError();
        size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        throw Error{LV_ENOMEM, "cudaMallocAsync(" + std::to_string(bytes) + ") failed: " + cudaGetErrorString(e) +
                                   " (library live " + std::to_string(live) + " B, peak " + std::to_string(peak) +
                                   " B; device free " + std::to_string(fr) + " of " + std::to_string(tot) + " B)"};
      }
    }
    live += bytes;
    if (live > peak) peak = live;
    static const bool trace = getenv("LV_TRACE_ALLOC") != nullptr;
    if (trace && bytes >= ((size_t)256 << 20))
      fprintf(stderr, "[lv alloc] %.2f GB -> live %.2f GB\n", bytes / 1e9, live / 1e9);
    return p;
  }
  void put(void *p, size_t bytes) {
    if (!p) return;
    if (bytes == 0) bytes = 16;
    bytes = (bytes + 255) & ~size_t(255);
    live -= bytes;
    static const bool trace = getenv("LV_TRACE_ALLOC") != nullptr;
    if (trace && bytes >= ((size_t)256 << 20))
      fprintf(stderr, "[lv free ] %.2f GB -> live %.2f GB\n", bytes / 1e9, live / 1e9);
    if (f) f(ctx, p, bytes, (void *)s);
    else cudaFreeAsync(p, s);
  }
};

// RAII device buffer (stream-ordered).
template <typename T>
struct Buf {
  T *p = nullptr;
  size_t n = 0;
  Alloc *A = nullptr;
  Buf() {}
  Buf(Alloc &al, size_t count) { alloc(al, count); }
  void alloc(Alloc &al, size_t count) {
    release();
    A = &al;
    n = count;
    p = (T *)al.get(count * sizeof(T));
  }
  void release() {
    if (p && A) A->put(p, n * sizeof(T));
    p = nullptr;
    n = 0;
  }
  ~Buf() { release(); }
  Buf(const Buf &) = delete;
  Buf &operator=(const Buf &) = delete;
  Buf(Buf &&o) noexcept : p(o.p), n(o.n), A(o.A) { o.p = nullptr; o.n = 0; }
  Buf &operator=(Buf &&o) noexcept {
    if (this != &o) {
      release();
      p = o.p; n = o.n; A = o.A;
      o.p = nullptr; o.n = 0;
    }
    return *this;
  }
  T *get() const { return p; }
};

// Execution context: device, stream, allocator, launch accounting.
struct Ctx {
  int device = 0;
  int sms = 148;
  cudaStream_t s = nullptr;  // the handle's stream: every public call is ordered on it
  Alloc A;
  i64 launches = 0;
  // fork/join pool for independent kernels of one pass (degree bins run concurrently)
  static constexpr int NSIDE = 4;
  cudaStream_t side[NSIDE] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t fork_ev = nullptr, join_ev[NSIDE] = {nullptr, nullptr, nullptr, nullptr};
  bool concurrent = false;
  bool capturing = false;  // a CUDA-graph capture is open on s: no host syncs may be issued
  void init_side() {
    for (int i = 0; i < NSIDE; ++i) {
      if (cudaStreamCreateWithFlags(&side[i], cudaStreamNonBlocking) != cudaSuccess) return;
      cudaEventCreateWithFlags(&join_ev[i], cudaEventDisableTiming);
    }
    cudaEventCreateWithFlags(&fork_ev, cudaEventDisableTiming);
    concurrent = true;
  }
  void free_side() {
    for (int i = 0; i < NSIDE; ++i) {
      if (side[i]) cudaStreamDestroy(side[i]);
      if (join_ev[i]) cudaEventDestroy(join_ev[i]);
    }
    if (fork_ev) cudaEventDestroy(fork_ev);
    concurrent = false;
  }
};

#define LV_LAUNCH(ctx, kern, grid, block, smem, ...)                          \
  do {                                                                        \
    kern<<<(grid), (block), (smem), (ctx).s>>>(__VA_ARGS__);                  \
    (ctx).launches++;                                                         \
    LV_CUDA(cudaGetLastError());                                              \
  } while (0)

#define LV_LAUNCH_ON(ctx, strm, kern, grid, block, smem, ...)                 \
  do {                                                                        \
    kern<<<(grid), (block), (smem), (strm)>>>(__VA_ARGS__);                   \
    (ctx).launches++;                                                         \
    LV_CUDA(cudaGetLastError());                                              \
  } while (0)

inline i64 cdiv(i64 a, i64 b) { return (a + b - 1) / b; }

// ------------------------------------------------------------------ device helpers
__device__ __forceinline__ u64 warp_sum_u64(u64 v, unsigned mask = 0xffffffffu) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o);
  return v;
}

// exact 128-bit add of (hi,lo) pairs
__device__ __forceinline__ void add128(u64 &hi, u64 &lo, u64 ohi, u64 olo) {
  u64 nlo = lo + olo;
  hi = hi + ohi + (nlo < lo ? 1ull : 0ull);
  lo = nlo;
}

// Atomically add a 128-bit unsigned value (hi,lo) into two u64 words (order-free exact).
__device__ __forceinline__ void atomic_add128(u64 *dst_lo, u64 *dst_hi, u64 hi, u64 lo) {
  u64 old = atomicAdd(dst_lo, lo);
  u64 carry = (old + lo < old) ? 1ull : 0ull;
  if (hi + carry) atomicAdd(dst_hi, hi + carry);
}

// Block-wide sum of a u64 (all threads call; result valid in every thread).
template <int BLOCK>
__device__ __forceinline__ u64 block_sum_u64(u64 v) {
  __shared__ u64 red[BLOCK / 32];
  v = warp_sum_u64(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  u64 t = 0;
#pragma unroll
  for (int i = 0; i < BLOCK / 32; ++i) t += red[i];
  return t;
}

// ---- shared memory through 32-bit shared-window addresses.  Generic-pointer atomics on
// shared data make the compiler re-derive the CTA's shared window (S2UR SR_CgaCtaId,
// ULEA, ...) at every access; these take the address once.
__device__ __forceinline__ uint32_t saddr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ int32_t lds_i32(uint32_t a) {
  int32_t v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ int32_t cas_s32(uint32_t a, int32_t cmp, int32_t val) {
  int32_t old;
  asm volatile("atom.shared.cas.b32 %0, [%1], %2, %3;" : "=r"(old) : "r"(a), "r"(cmp), "r"(val) : "memory");
  return old;
}
__device__ __forceinline__ uint32_t atom_add_s32(uint32_t a, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(a), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void red_add_s32(uint32_t a, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// ---- L2 eviction-priority hints (PTX createpolicy + ld.global.L2::cache_hint).
// Streams read once (row_ptr, col, w) are marked evict_first so they do not push the
// randomly gathered arrays (labels, deg_C) out of the 126 MB L2; those are evict_last.
__device__ __forceinline__ u64 l2_policy_first() {
  u64 p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ u64 l2_policy_last() {
  u64 p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ int32_t ld_stream(const int32_t *a, u64 pol) {
  int32_t v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ uint32_t ld_stream(const uint32_t *a, u64 pol) {
  uint32_t v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ u64 ld_stream(const u64 *a, u64 pol) {
  u64 v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.b64 %0, [%1], %2;" : "=l"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ i64 ld_stream(const i64 *a, u64 pol) {
  i64 v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.b64 %0, [%1], %2;" : "=l"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ int32_t ld_keep(const int32_t *a, u64 pol) {
  int32_t v;
  asm("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ i64 ld_keep(const i64 *a, u64 pol) {
  i64 v;
  asm("ld.global.nc.L2::cache_hint.b64 %0, [%1], %2;" : "=l"(v) : "l"(a), "l"(pol));
  return v;
}

}  // namespace lv
