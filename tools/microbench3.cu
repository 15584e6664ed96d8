// Microbenchmark: random CSR probes whose targets stay inside a sliding window
// of the table (queries pre-grouped by level-1 bin), i.e. can the table slice of
// one level-1 bin be probed straight from L2 instead of staging it in smem?
//   per query: h = bucket inside the current window; a = off[h], e = off[h+1];
//   count edges[a..e) == key; write the count.  Table: 2^28 buckets, degree 1.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/microbench3 tools/microbench3.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t fmix(uint32_t h) {
  h ^= h >> 16; h *= 0x85EBCA6Bu; h ^= h >> 13; h *= 0xC2B2AE35u; h ^= h >> 16; return h;
}

__global__ void k_init(uint32_t* off, uint32_t* edges, uint32_t* q, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += gridDim.x * blockDim.x) {
    off[i] = i;
    if (i < n) { edges[i] = fmix(i + 1); q[i] = fmix(i * 7 + 3); }
  }
}

// QPT queries per thread in flight; W = window buckets (power of two)
template <int QPT>
__global__ void __launch_bounds__(512) k_probe(const uint32_t* __restrict__ off, const uint32_t* __restrict__ edges,
                                               const uint32_t* __restrict__ q, uint32_t* __restrict__ out, uint32_t n,
                                               uint32_t wbits) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t i0 = blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += QPT * stride) {
    uint32_t key[QPT], h[QPT], a[QPT], e[QPT];
#pragma unroll
    for (int k = 0; k < QPT; k++) {
      const uint32_t i = i0 + k * stride;
      key[k] = i < n ? __ldcs(q + i) : 0u;
      h[k] = ((i >> wbits) << wbits) | (fmix(key[k]) & ((1u << wbits) - 1));
      if (h[k] >= n) h[k] = n - 1;
    }
#pragma unroll
    for (int k = 0; k < QPT; k++) {
      a[k] = off[h[k]];
      e[k] = off[h[k] + 1];
    }
#pragma unroll
    for (int k = 0; k < QPT; k++) {
      const uint32_t i = i0 + k * stride;
      uint32_t c = 0;
      for (uint32_t t = a[k]; t < e[k]; t++) c += edges[t] == key[k];
      if (i < n) __stcs(out + i, c);
    }
  }
}

int main() {
  const uint32_t n = 1u << 28;
  uint32_t *off, *edges, *q, *out;
  CK(cudaMalloc(&off, (size_t)(n + 1) * 4));
  CK(cudaMalloc(&edges, (size_t)n * 4));
  CK(cudaMalloc(&q, (size_t)n * 4));
  CK(cudaMalloc(&out, (size_t)n * 4));
  k_init<<<148 * 8, 512>>>(off, edges, q, n);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int sms = 148;
  for (int wbits : {16, 18, 19, 20, 21, 22, 23, 24, 28}) {
    for (int occ : {2, 4}) {
      float best = 1e9;
      for (int rep = 0; rep < 4; rep++) {
        cudaEventRecord(a);
        k_probe<8><<<sms * occ, 512>>>(off, edges, q, out, n, wbits);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      // algorithmic bytes: q read + out write + off 4 B + edges 4 B per query
      printf("window 2^%d buckets (%5.1f MB table slice) ctas/SM %d: %.3f ms  %.1f G q/s  alg %.0f GB/s\n", wbits,
             (double)(8ull << wbits) / 1e6, occ, best, n / best / 1e6, 16.0 * n / best / 1e6);
    }
  }
  CK(cudaGetLastError());
  return 0;
}
