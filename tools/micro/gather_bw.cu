// Microbenchmark: random 4-byte / 8-byte gathers from arrays of various sizes (L2-resident
// to HBM-resident), to measure the achievable random-sector throughput on this B200 —
// the real ceiling of the label / deg_C gathers on the local-move path.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void gather32(const int* __restrict__ idx, const int* __restrict__ src, long long n, int* out) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  int acc = 0;
  for (; i < n; i += (long long)gridDim.x * blockDim.x) acc += __ldg(&src[__ldg(&idx[i])]);
  if (acc == 0x7fffffff) out[0] = acc;
}
__global__ void gather64(const int* __restrict__ idx, const long long* __restrict__ src, long long n, long long* out) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long acc = 0;
  for (; i < n; i += (long long)gridDim.x * blockDim.x) acc += __ldg(&src[__ldg(&idx[i])]);
  if (acc == 0x7fffffffffffLL) out[0] = acc;
}
__global__ void fill_idx(int* idx, long long n, unsigned range, unsigned seed) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    unsigned x = (unsigned)i * 2654435761u ^ seed; x ^= x >> 15; x *= 2246822519u; x ^= x >> 13; x *= 3266489917u; x ^= x >> 16;
    idx[i] = (int)(((unsigned long long)x * range) >> 32);
  }
}
int main() {
  const long long n = 1ll << 28;  // 268M gathers
  int *idx, *out; cudaMalloc(&idx, n * 4); cudaMalloc(&out, 16);
  long long sizes_mb[] = {32, 64, 128, 256, 1024, 4096};
  for (long long mb : sizes_mb) {
    for (int w = 4; w <= 8; w += 4) {
      long long elems = mb * (1 << 20) / w;
      void* src; cudaMalloc(&src, mb << 20); cudaMemset(src, 1, mb << 20);
      fill_idx<<<148 * 16, 256>>>(idx, n, (unsigned)elems, 12345);
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        if (w == 4) gather32<<<148 * 16, 256>>>(idx, (int*)src, n, out);
        else gather64<<<148 * 16, 256>>>(idx, (long long*)src, n, (long long*)out);
        cudaEventRecord(b); cudaEventSynchronize(b);
      }
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("array %5lld MB  elem %dB: %.3f ms  %.1f G gathers/s  idx-stream %.0f GB/s  sector-equiv %.0f GB/s\n",
             mb, w, ms, n / ms / 1e6, n * 4.0 / ms / 1e6, n * 32.0 / ms / 1e6);
      cudaFree(src);
    }
  }
  return 0;
}
