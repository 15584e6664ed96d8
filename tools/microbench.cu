// Microbenchmarks that size the HashGraph kernel design on B200 (sm_100a):
// streaming copy/read bandwidth, random global atomics (L2-resident vs HBM),
// random scattered 4-B stores, shared-memory histogram atomics.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/microbench tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t fmix(uint32_t h) {
  h ^= h >> 16; h *= 0x85EBCA6Bu; h ^= h >> 13; h *= 0xC2B2AE35u; h ^= h >> 16; return h;
}

__global__ void k_copy(const uint4* __restrict__ a, uint4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
__global__ void k_read(const uint4* __restrict__ a, size_t n, uint32_t* out) {
  uint32_t s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) { uint4 v = a[i]; s ^= v.x ^ v.y ^ v.z ^ v.w; }
  if (s == 0x12345678) *out = s;
}
// random global atomics: mode 0 = RED (no return), 1 = ATOM with return used
template <int MODE>
__global__ void k_gatomic(uint32_t* arr, uint32_t mask, size_t nops, uint32_t* out) {
  uint32_t s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nops; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t h = fmix((uint32_t)i * 2654435761u + 7) & mask;
    if (MODE == 0) atomicAdd(arr + h, 1u); else s += atomicAdd(arr + h, 1u);
  }
  if (MODE == 1 && s == 0x12345678) *out = s;
}
__global__ void k_scatter(uint32_t* arr, uint32_t mask, size_t nops) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nops; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t h = fmix((uint32_t)i * 2654435761u + 7) & mask;
    arr[h] = (uint32_t)i;
  }
}
// shared-memory histogram, BINS bins; MODE 0 = RED, 1 = return used, 2 = match_any aggregated
template <int BINS, int MODE>
__global__ void k_shist(size_t nops, uint32_t* out) {
  extern __shared__ uint32_t hist[];
  for (int i = threadIdx.x; i < BINS; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  uint32_t s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nops; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t h = fmix((uint32_t)i) & (BINS - 1);
    if (MODE == 0) atomicAdd(hist + h, 1u);
    else if (MODE == 1) s += atomicAdd(hist + h, 1u);
    else {
      unsigned m = __match_any_sync(__activemask(), h);
      int leader = __ffs(m) - 1;
      if ((threadIdx.x & 31) == leader) atomicAdd(hist + h, __popc(m));
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = hist[0] + s;
}

template <typename F>
float timeit(F f, int reps = 5) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; r++) {
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int l2 = 0; cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
  printf("device %s SMs %d L2 %d MB smemPerBlockOptin %zu\n", p.name, p.multiProcessorCount, l2 >> 20, p.sharedMemPerBlockOptin);
  int sms = p.multiProcessorCount;
  size_t bytes = 1ull << 30;
  uint4 *a, *b; uint32_t* out;
  CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes)); CK(cudaMalloc(&out, 1 << 20));
  cudaMemset(a, 1, bytes); cudaMemset(b, 0, bytes);
  size_t n16 = bytes / 16;
  for (int per : {4, 8, 16}) {
    float ms = timeit([&] { k_copy<<<sms * per, 256>>>(a, b, n16); });
    printf("copy 1GiB grid=%dx148: %.3f ms  %.1f GB/s (r+w)\n", per, ms, 2.0 * bytes / ms / 1e6);
    ms = timeit([&] { k_read<<<sms * per, 256>>>(a, n16, out); });
    printf("read 1GiB grid=%dx148: %.3f ms  %.1f GB/s\n", per, ms, 1.0 * bytes / ms / 1e6);
  }
  size_t nops = 1ull << 28;
  uint32_t* arr = (uint32_t*)b;
  for (int lg : {14, 20, 22, 24, 25, 26, 28}) {
    uint32_t mask = (1u << lg) - 1;
    float ms0 = timeit([&] { k_gatomic<0><<<sms * 16, 256>>>(arr, mask, nops, out); }, 3);
    float ms1 = timeit([&] { k_gatomic<1><<<sms * 16, 256>>>(arr, mask, nops, out); }, 3);
    float ms2 = timeit([&] { k_scatter<<<sms * 16, 256>>>(arr, mask, nops); }, 3);
    printf("random 4B ops into %6.1f MB: RED %.2f Gop/s  ATOM %.2f Gop/s  STORE %.2f Gop/s\n",
           (4.0 * (1u << lg)) / 1e6, nops / ms0 / 1e6, nops / ms1 / 1e6, nops / ms2 / 1e6);
  }
  size_t sops = 1ull << 30;
  {
    cudaFuncSetAttribute(k_shist<4096, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    float m0 = timeit([&] { k_shist<4096, 0><<<sms * 4, 512, 4096 * 4>>>(sops, out); }, 3);
    float m1 = timeit([&] { k_shist<4096, 1><<<sms * 4, 512, 4096 * 4>>>(sops, out); }, 3);
    float m2 = timeit([&] { k_shist<4096, 2><<<sms * 4, 512, 4096 * 4>>>(sops, out); }, 3);
    printf("smem hist 4096 bins: RED %.1f  ATOM %.1f  MATCH %.1f Gop/s chip\n", sops / m0 / 1e6, sops / m1 / 1e6, sops / m2 / 1e6);
    cudaFuncSetAttribute(k_shist<16384, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    cudaFuncSetAttribute(k_shist<16384, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    m0 = timeit([&] { k_shist<16384, 0><<<sms * 2, 1024, 16384 * 4>>>(sops, out); }, 3);
    m1 = timeit([&] { k_shist<16384, 1><<<sms * 2, 1024, 16384 * 4>>>(sops, out); }, 3);
    printf("smem hist 16384 bins: RED %.1f  ATOM %.1f Gop/s chip\n", sops / m0 / 1e6, sops / m1 / 1e6);
  }
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  printf("done\n");
  return 0;
}
