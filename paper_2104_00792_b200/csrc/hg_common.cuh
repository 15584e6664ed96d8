// hg_common.cuh -- shared device/host helpers for libhashgraph_b200 (sm_100a).
//
// Hash family (hashing.py:77-114): murmur32 = fmix32(key ^ seed) mod V,
// identity = key mod V.  64-bit keys (an extension; the reference truncates to
// uint32 at core.py:84-88) use the Murmur3 fmix64 finalizer.  The reduction
// mod V is exact: a mask for powers of two, Lemire's fastmod (M = 2^64/V + 1,
// exact for every 32-bit numerator) otherwise.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/hashgraph_b200.h"

namespace hg {

// --------------------------------------------------------------------------- errors

int set_error(int code, const char* fmt, ...);
int cuda_error(cudaError_t e, const char* where);

// Per-launch bookkeeping: launch counter and optional CUDA-event timing.
void note_launch_begin(const char* name, cudaStream_t s);
void note_launch_end(cudaStream_t s);

#define HG_CHECK_CUDA(expr)                                        \
  do {                                                             \
    cudaError_t _e = (expr);                                       \
    if (_e != cudaSuccess) return ::hg::cuda_error(_e, #expr);     \
  } while (0)

// Opt a kernel into dynamic shared memory: once per call site and device the
// kernel's limit is raised to the device's opt-in maximum (a permission, not
// an allocation: each launch still asks for its own size), so call sites of
// the same kernel never lower each other's limit.  The driver call costs
// microseconds, which adds up over the many small builds of virtual shards.
int smem_optin_max();
template <typename F>
cudaError_t smem_raise_limit(F kernel) {
  cudaFuncAttributes fa{};
  cudaError_t e = cudaFuncGetAttributes(&fa, kernel);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              smem_optin_max() - (int)fa.sharedSizeBytes);
}
#define HG_SET_SMEM(kernel, bytes)                                                                   \
  do {                                                                                               \
    static std::atomic<bool> _hg_smem_done[16];                                                      \
    int _hg_dev = 0;                                                                                 \
    HG_CHECK_CUDA(cudaGetDevice(&_hg_dev));                                                          \
    if ((int)(bytes) > ::hg::smem_optin_max())                                                       \
      return ::hg::set_error(HG_ERR_CONFIG, "kernel needs %d bytes of shared memory", (int)(bytes)); \
    if (_hg_dev >= 16 || !_hg_smem_done[_hg_dev].load(std::memory_order_acquire)) {                  \
      HG_CHECK_CUDA(::hg::smem_raise_limit(kernel));                                                 \
      if (_hg_dev < 16) _hg_smem_done[_hg_dev].store(true, std::memory_order_release);               \
    }                                                                                                \
  } while (0)

// Launch a kernel with bookkeeping; returns from the enclosing function on a
// launch error.
#define HG_LAUNCH(name, kernel, grid, block, smem, stream, ...)             \
  do {                                                                     \
    ::hg::note_launch_begin(name, stream);                                 \
    kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);            \
    cudaError_t _e = cudaGetLastError();                                   \
    ::hg::note_launch_end(stream);                                         \
    if (_e != cudaSuccess) return ::hg::cuda_error(_e, name);              \
  } while (0)

// --------------------------------------------------------------------------- hashing

struct HashParams {
  uint64_t v;      // hash range (>= 1)
  uint64_t magic;  // fastmod multiplier, valid when mode == kFastmod
  uint64_t mask;   // v - 1, valid when mode == kMask
  uint64_t magic64;  // floor((2^64 - 1) / v): Barrett reduction of 64-bit mixed values
  uint32_t seed;
  int kind;        // 0 murmur, 1 identity
  int mode;        // kMask / kFastmod / kNone / kGeneric64
  uint32_t m32;    // kFastmod, 32-bit values: Granlund-Montgomery multiplier for floor(x / v)
  uint32_t sh2;    // ... and its second shift (the first is 1)
};

enum { kMask = 0, kFastmod = 1, kNone = 2, kGeneric64 = 3 };

inline HashParams make_hash_params(int kind, uint32_t seed, uint64_t v, int key_bits) {
  HashParams hp{};
  hp.v = v;
  hp.seed = seed;
  hp.kind = kind;
  hp.magic64 = UINT64_MAX / v;
  if ((v & (v - 1)) == 0) {
    hp.mode = kMask;
    hp.mask = v - 1;
  } else if (key_bits == 32 && v > 0xFFFFFFFFull) {
    hp.mode = kNone;  // every 32-bit mixed value is already < v
  } else if (v <= 0xFFFFFFFFull) {
    hp.mode = kFastmod;
    hp.magic = UINT64_MAX / v + 1;
    // floor(x / v) = (t + ((x - t) >> 1)) >> (l - 1), t = umulhi(x, m32), for
    // every 32-bit x (v not a power of two here, so 2 < v < 2^32 and l >= 2)
    int l = 0;
    while ((1ull << l) < v) l++;
    hp.m32 = (uint32_t)((((1ull << l) - v) << 32) / v + 1);
    hp.sh2 = (uint32_t)(l - 1);
  } else {
    hp.mode = kGeneric64;
  }
  return hp;
}

__host__ __device__ __forceinline__ uint32_t fmix32(uint32_t h) {
  h ^= h >> 16;
  h *= 0x85EBCA6Bu;
  h ^= h >> 13;
  h *= 0xC2B2AE35u;
  h ^= h >> 16;
  return h;
}

__host__ __device__ __forceinline__ uint64_t fmix64(uint64_t h) {
  h ^= h >> 33;
  h *= 0xFF51AFD7ED558CCDull;
  h ^= h >> 33;
  h *= 0xC4CEB9FE1A85EC53ull;
  h ^= h >> 33;
  return h;
}

__device__ __forceinline__ uint32_t fastmod_u32(uint32_t x, uint64_t magic, uint32_t d) {
  uint64_t low = magic * (uint64_t)x;
  return (uint32_t)__umul64hi(low, (uint64_t)d);
}

// x mod d for 32-bit x and a non-power-of-two d < 2^32 by division with an
// invariant multiplier (Granlund & Montgomery): two integer multiplies and
// five ALU operations, where Lemire's 64-bit fastmod issues five wide
// multiplies (the multiply pipe is what the build kernels' hashing waits on).
__host__ __device__ __forceinline__ uint32_t mod_gm32(uint32_t x, uint32_t m, uint32_t sh2, uint32_t d) {
#ifdef __CUDA_ARCH__
  const uint32_t t = __umulhi(x, m);
#else
  const uint32_t t = (uint32_t)(((uint64_t)x * m) >> 32);
#endif
  const uint32_t q = (t + ((x - t) >> 1)) >> sh2;
  return x - q * d;
}

// x mod d for any 64-bit x: q = floor(x * m / 2^64) with m = floor((2^64-1)/d)
// undershoots floor(x/d) by at most 2, so two conditional subtractions finish.
__device__ __forceinline__ uint64_t barrett_mod64(uint64_t x, uint64_t m, uint64_t d) {
  const uint64_t q = __umul64hi(x, m);
  uint64_t r = x - q * d;
  if (r >= d) r -= d;
  if (r >= d) r -= d;
  return r;
}

__device__ __forceinline__ uint64_t mix_key(uint32_t key, const HashParams& hp) {
  return hp.kind == HG_KIND_IDENTITY ? (uint64_t)key : (uint64_t)fmix32(key ^ hp.seed);
}
__device__ __forceinline__ uint64_t mix_key(uint64_t key, const HashParams& hp) {
  return hp.kind == HG_KIND_IDENTITY ? key : fmix64(key ^ (uint64_t)hp.seed);
}

// hash(key) mod v, general (any v).
template <typename K>
__device__ __forceinline__ uint64_t hash_mod(K key, const HashParams& hp) {
  uint64_t x = mix_key(key, hp);
  switch (hp.mode) {
    case kMask:
      return x & hp.mask;
    case kNone:
      return x;
    case kFastmod:
      if (sizeof(K) == 4) return mod_gm32((uint32_t)x, hp.m32, hp.sh2, (uint32_t)hp.v);
      return barrett_mod64(x, hp.magic64, hp.v);
    default:
      return barrett_mod64(x, hp.magic64, hp.v);
  }
}

// Compile-time specialised hasher: MODE fixes the reduction (kMask, kFastmod,
// kNone, kGeneric64) so the hot loops carry no per-key dispatch.
template <typename K, int MODE, int KIND = HG_KIND_MURMUR32>
struct Hasher {
  using Key = K;
  static __device__ __forceinline__ uint64_t mix(K key, const HashParams& hp) {
    if constexpr (KIND == HG_KIND_IDENTITY) {
      return (uint64_t)key;
    } else if constexpr (sizeof(K) == 4) {
      return (uint64_t)fmix32((uint32_t)key ^ hp.seed);
    } else {
      return fmix64((uint64_t)key ^ (uint64_t)hp.seed);
    }
  }
  static __device__ __forceinline__ uint32_t bucket(K key, const HashParams& hp) {
    const uint64_t x = mix(key, hp);
    if constexpr (MODE == kMask) {
      return (uint32_t)(x & hp.mask);
    } else if constexpr (MODE == kNone) {
      return (uint32_t)x;
    } else if constexpr (MODE == kFastmod && sizeof(K) == 4) {
      return mod_gm32((uint32_t)x, hp.m32, hp.sh2, (uint32_t)hp.v);
    } else {
      return (uint32_t)barrett_mod64(x, hp.magic64, hp.v);
    }
  }
};

// Bucket id for builds/queries: v <= 2^32 is enforced on the host, so the
// result fits uint32.
template <typename K>
__device__ __forceinline__ uint32_t bucket_of(K key, const HashParams& hp) {
  return (uint32_t)hash_mod(key, hp);
}

// Exact floor division of a hash value by a bin size (fastdiv for 32-bit h).
struct DivParams {
  uint64_t d;
  uint64_t magic;
  int shift;  // >= 0 when d is a power of two
};

inline DivParams make_div_params(uint64_t d) {
  DivParams p{};
  p.d = d;
  p.shift = -1;
  if ((d & (d - 1)) == 0) {
    int s = 0;
    while ((1ull << s) < d) s++;
    p.shift = s;
  } else {
    p.magic = UINT64_MAX / d + 1;
  }
  return p;
}

__device__ __forceinline__ uint64_t div_by(uint64_t h, const DivParams& p) {
  if (p.shift >= 0) return h >> p.shift;
  if (h <= 0xFFFFFFFFull && p.d <= 0xFFFFFFFFull) return __umul64hi(p.magic, h);
  return h / p.d;
}

// --------------------------------------------------------------------------- TMA (1-D bulk copies)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

// Order this thread's generic-proxy shared-memory accesses before later
// async-proxy (TMA) accesses of the same memory.
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// One thread: expect `bytes` on `bar` and start a global->shared bulk copy
// (16-byte aligned addresses, size a multiple of 16).
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// shared -> global bulk store (16-byte aligned, size multiple of 16), bulk-group completion
__device__ __forceinline__ void tma_store_1d(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_store_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// the smem source of this thread's committed bulk stores may be reused
__device__ __forceinline__ void tma_store_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void tma_store_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Add `bytes` of expected transactions to the barrier's current phase (no arrive).
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// global -> shared bulk copy that completes transactions on `bar` (caller accounts the bytes)
__device__ __forceinline__ void tma_load_1d_tx(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// --------------------------------------------------------------------------- misc

// bar.sync on a named barrier shared by `count` threads (a multiple of 32)
__device__ __forceinline__ void named_barrier_sync(int id, uint32_t count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

inline int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

// opt-in dynamic shared memory per CTA (227 KB on sm_100)
inline int max_dyn_smem() {
  static int bytes = 0;
  if (!bytes) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&bytes, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (bytes <= 0) bytes = 232448;
  }
  return bytes;
}

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Simple bump allocator over a caller-provided workspace.
struct Workspace {
  char* base;
  size_t cap;
  size_t used;
  template <typename T>
  T* take(size_t count) {
    used = align_up(used, 256);
    T* p = reinterpret_cast<T*>(base + used);
    used += count * sizeof(T);
    return p;
  }
  bool ok() const { return used <= cap; }
};

}  // namespace hg
