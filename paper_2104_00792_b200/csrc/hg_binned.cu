// hg_binned.cu -- the binned HashGraph build and query for sm_100a (v3).
//
// Green's cache-blocked HashGraph build ("first assigns each
// hash value to one of B_L bins ... B_L is small enough to fit in the cache")
// mapped onto B200 shared memory.  The hash range [0, V) is cut into FINE
// bins of 2^s consecutive buckets, sized so one fine bin's keys (~16K) plus
// its counters fit in the shared memory of one of the two CTAs an SM runs.
// Keys reach their fine bin through at most two partition levels of <= 128
// sub-bins each, so every (tile, sub-bin) run written to HBM is ~128 keys or
// longer: HBM sees long coalesced streams, all random accesses hit smem.
//
//   A   k_hist          per-CTA level-1 counts + global fine-bin histogram
//       k_colscan       per-(CTA, level-1 bin) write bases
//       k_starts        fine/level-1 starts, level-2 tile table, big-bin list
//   P1  k_part1         CTA chunk, 8K-key tiles: per-warp smem-atomic ranks,
//                       smem staging, one contiguous run per bin
//   P2  k_part2         the same over each level-1 bin, claiming fine-bin space
//   C   k_local_build   one CTA per fine bin: count, scan, place in smem,
//                       write offsets + edges (bins above the smem capacity:
//                       k_big_count / k_big_place, hg_bigbin.cuh)
//   Q   k_local_probe   one CTA per fine bin (plus extra work items for hot
//                       bins): the table's CSR slice staged in smem, deep
//                       buckets sorted, the bin's queries probe it
//                       (IntersectArray); slices above the smem capacity:
//                       k_ht_* (hg_bigbin.cuh)
//   R   k_unpart<2,1>   query answers back to input order: each tile's runs
//                       are pulled into smem and read back through a u16 map
//
// Results equal Alg. 1's: offsets exact, every bucket the
// same multiset (core.py:12-14 leaves the in-bucket order unspecified).
#include "hg_binned.cuh"

namespace hg {

constexpr int kT = 512;          // threads per CTA; two CTAs per SM
constexpr int kW = kT / 32;      // warps per CTA
constexpr int kSub = 128;        // level-2 fan-out (fine bins per level-1 bin) up to 32768 fine bins
constexpr int kSubMax = 256;     // ... and up to 65536 (e.g. 2^30 keys at C = 1 on one GPU): runs half as long
constexpr int kMaxBins = 256;    // bins one partition tile can split into (8-bit bin ids)
constexpr uint32_t kMaxFine = kSubMax * kMaxBins;  // 65536

template <typename K>
struct TileShape {
  static constexpr int kTile = sizeof(K) == 4 ? 8192 : 4096;  // 32 KB staged
  static constexpr int kKPT = kTile / kT;                     // 16 / 8 keys per thread
};

template <typename K>
struct LocalShape {
  static constexpr int kKPT = sizeof(K) == 4 ? 38 : 19;
  static constexpr uint32_t kCap = kKPT * kT;  // keys per fine bin the probe stages in smem
};

#ifndef HG_BUILD_KPT32
#define HG_BUILD_KPT32 38
#endif
// keys per fine bin the local build holds in smem (bins above it: hg_bigbin.cuh)
template <typename K>
struct BuildShape {
  static constexpr uint32_t kCap = (sizeof(K) == 4 ? HG_BUILD_KPT32 : 19) * kT;
};


static int ceil_log2(uint32_t x) {
  int b = 0;
  while ((1u << b) < x) b++;
  return b;
}

// ~0.85 of the local stages' capacity per fine bin on average
static int pick_s(uint64_t n, uint64_t v, int key_bits) {
  const double per_bucket = v ? (double)n / (double)v : 1.0;
  const double target = key_bits == 32 ? 17000.0 : 8500.0;
  int s = 14;
  while (s > 6 && per_bucket * (double)(1ull << s) > target) s--;
  return s;
}

// n_table sizes the fine bins (a bin's table keys must fit smem); n sizes the chunks.
bool binned_layout(uint64_t n_table, uint64_t n, uint64_t v, int key_bits, BinLayout* L) {
  if (v > (1ull << 32)) return false;
  const int s = pick_s(n_table, v, key_bits);
  const uint64_t F = (v + (1ull << s) - 1) >> s;
  if (F > kMaxFine) return false;
  L->s = s;
  L->nfine = (uint32_t)F;
  L->two_level = F > (uint64_t)kSub;
  L->sub = F > (uint64_t)kSub * kMaxBins ? kSubMax : kSub;
  L->group = L->two_level ? L->sub : 1;
  L->nb1 = (uint32_t)((F + L->group - 1) / L->group);
  L->bits1 = ceil_log2(L->nb1);
  L->shift1 = s + (L->two_level ? ceil_log2(L->sub) : 0);
  L->tile = key_bits == 32 ? 8192u : 4096u;  // == TileShape<K>::kTile
  L->grid = (uint32_t)num_sms() * 2;
  const uint64_t per = (n + L->grid - 1) / L->grid;
  L->chunk = (per + L->tile - 1) / L->tile * L->tile;
  if (L->chunk == 0) L->chunk = L->tile;
  L->ntiles1 = (n + L->tile - 1) / L->tile;
  L->max_tiles2 = L->ntiles1 + L->nb1 + 1;
  return true;
}

template <typename H>
using KeyOf = typename H::Key;

template <typename H>
__device__ __forceinline__ uint32_t fine_of(typename H::Key key, const HashParams& hp, int s) {
  return H::bucket(key, hp) >> s;
}

// --------------------------------------------------------------------------- block helpers

// In-place exclusive scan of n (<= 32 * blockDim) uint32 in smem; returns total.
__device__ uint32_t block_exscan(uint32_t* a, uint32_t n) {
  __shared__ uint32_t s_w[32];
  const uint32_t per = (n + blockDim.x - 1) / blockDim.x;
  const uint32_t lo = threadIdx.x * per, hi = min(lo + per, n);
  uint32_t sum = 0;
  for (uint32_t i = lo; i < hi; i++) sum += a[i];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) s_w[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < nw ? s_w[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) s_w[lane] = w;
  }
  __syncthreads();
  uint32_t run = (warp ? s_w[warp - 1] : 0u) + inc - sum;
  const uint32_t total = s_w[nw - 1];
  for (uint32_t i = lo; i < hi; i++) {
    uint32_t x = a[i];
    a[i] = run;
    run += x;
  }
  __syncthreads();
  return total;
}

// Exclusive scan of n uint32 in smem (in place), warp-row layout (no bank
// conflicts); `base` is added to every output.  Returns the total.
__device__ uint32_t block_exscan_rows(uint32_t* a, uint32_t n, uint32_t base) {
  __shared__ uint32_t s_w[32];
  __shared__ uint32_t s_total;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint32_t seg = ((n + nw - 1) / nw + 31) & ~31u;
  const uint32_t w0 = warp * seg, w1 = min(w0 + seg, n);
  uint32_t part = 0;
  for (uint32_t i = w0 + lane; i < w1; i += 32) part += a[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  if (lane == 0) s_w[warp] = part;
  __syncthreads();
  if (warp == 0) {
    const uint32_t x = lane < nw ? s_w[lane] : 0u;
    uint32_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane < nw) s_w[lane] = inc - x;
    if (lane == 31) s_total = inc;
  }
  __syncthreads();
  const uint32_t total = s_total;
  uint32_t carry = base + s_w[warp];
  for (uint32_t r = w0; r < w1; r += 32) {
    const uint32_t i = r + lane;
    const uint32_t x = i < w1 ? a[i] : 0u;
    uint32_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (i < w1) a[i] = carry + inc - x;
    carry += __shfl_sync(0xffffffffu, inc, 31);
  }
  __syncthreads();
  return total;
}

// Block-wide exclusive scan of one value per thread (any blockDim <= 1024);
// returns the exclusive prefix, `total` gets the block sum.  Three barriers.
template <typename T>
__device__ __forceinline__ T block_scan_excl(T x, T& total) {
  __shared__ T s_ws[33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  T inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) s_ws[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const T w = lane < nw ? s_ws[lane] : T(0);
    T wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    s_ws[lane] = wi - w;
    if (lane == 31) s_ws[32] = wi;
  }
  __syncthreads();
  const T r = s_ws[warp] + inc - x;
  total = s_ws[32];
  __syncthreads();
  return r;
}

// Index j with pre[j] <= x < pre[j + 1] (pre ascending, pre[0] = 0, n entries + end).
__device__ __forceinline__ uint32_t upper_index(const uint32_t* pre, uint32_t n, uint32_t x) {
  uint32_t a = 0, z = n;
  while (z - a > 1) {
    const uint32_t m = (a + z) >> 1;
    if (pre[m] <= x) a = m; else z = m;
  }
  return a;
}

__device__ __forceinline__ uint32_t get16(const uint32_t* p, uint32_t k) { return (p[k >> 1] >> ((k & 1) * 16)) & 0xFFFFu; }

// Tile loads: full 16-byte-aligned tiles use 128-bit loads (element of key k
// = ((k / VPL) * kT + tid) * VPL + k % VPL); ragged tiles use k * kT + tid.
template <typename K>
__device__ __forceinline__ uint32_t tile_elem(int k, bool vec) {
  constexpr int VPL = 16 / sizeof(K);
  return vec ? (uint32_t)(((k / VPL) * kT + threadIdx.x) * VPL + k % VPL) : (uint32_t)(k * kT + threadIdx.x);
}

template <typename K, int KPT>
__device__ __forceinline__ bool load_tile(const K* __restrict__ src, uint32_t m, K (&kv)[KPT]) {
  constexpr int VPL = 16 / sizeof(K);
  const bool vec = (m == (uint32_t)KPT * kT) && ((reinterpret_cast<uintptr_t>(src) & 15) == 0);
  if (vec) {
    const uint4* p = reinterpret_cast<const uint4*>(src);
#pragma unroll
    for (int l = 0; l < KPT / VPL; l++) {
      uint4 q = __ldcs(p + l * kT + threadIdx.x);
      const K* qk = reinterpret_cast<const K*>(&q);
#pragma unroll
      for (int j = 0; j < VPL; j++) kv[l * VPL + j] = qk[j];
    }
  } else {
#pragma unroll
    for (int k = 0; k < KPT; k++) {
      const uint32_t e = k * kT + threadIdx.x;
      kv[k] = e < m ? src[e] : K(0);
    }
  }
  return vec;
}

// --------------------------------------------------------------------------- pass A

template <bool kSplit>
__device__ __forceinline__ void hist_add_t(uint32_t* s_h, uint32_t f_lo, uint32_t nf, uint32_t f) {
  if (!kSplit) atomicAdd(s_h + f, 1u);
  else if (f - f_lo < nf) atomicAdd(s_h + f - f_lo, 1u);
}
#define hist_add(...) hist_add_t<kSplit>(__VA_ARGS__)

// kSplit (more than kHistMax fine bins): this launch counts only fine bins
// [f_lo, f_lo + nf) (one smem counter each); the caller launches once per range.
constexpr uint32_t kHistMax = 32768;

template <typename H, bool kSplit>
__global__ void __launch_bounds__(kT)
k_hist(const KeyOf<H>* __restrict__ keys, uint64_t n, HashParams hp, int s, uint32_t nfine, uint32_t group, uint32_t nb1,
       uint64_t chunk, uint32_t* __restrict__ M, uint32_t* __restrict__ fine_cnt, uint32_t f_lo, uint32_t nf) {
  using K = typename H::Key;
  extern __shared__ uint32_t s_h[];
  if (!kSplit) {
    f_lo = 0;
    nf = nfine;
  }
  for (uint32_t i = threadIdx.x; i < nf; i += blockDim.x) s_h[i] = 0;
  __syncthreads();
  uint64_t lo = (uint64_t)blockIdx.x * chunk;
  const uint64_t hi = min(n, lo + chunk);
  {
    // keys that are a view at an offset (e.g. one virtual shard's rows): the
    // < 16 / sizeof(K) keys before the next 16-byte boundary one by one, the
    // rest with vector loads
    const uint32_t mis = (uint32_t)(reinterpret_cast<uintptr_t>(keys + lo) & 15);
    if (mis && (mis % sizeof(K)) == 0 && lo < hi) {
      const uint64_t head = min(hi - lo, (uint64_t)((16 - mis) / sizeof(K)));
      if (threadIdx.x < head) hist_add(s_h, f_lo, nf, fine_of<H>(keys[lo + threadIdx.x], hp, s));
      lo += head;
    }
  }
  if (sizeof(K) == 8 && lo < hi && ((reinterpret_cast<uintptr_t>(keys + lo) & 15) == 0)) {
    const uint4* p = reinterpret_cast<const uint4*>(keys + lo);
    const uint64_t nv = (hi - lo) / 2;
    uint64_t i = threadIdx.x;
    constexpr int U = 8;  // 16-byte loads in flight per thread (two keys each)
    for (; i + (U - 1) * blockDim.x < nv; i += U * blockDim.x) {
      uint4 q[U];
#pragma unroll
      for (int u = 0; u < U; u++) q[u] = __ldcs(p + i + u * blockDim.x);
#pragma unroll
      for (int u = 0; u < U; u++) {
        const K* qk = reinterpret_cast<const K*>(&q[u]);
        hist_add(s_h, f_lo, nf, fine_of<H>(qk[0], hp, s));
        hist_add(s_h, f_lo, nf, fine_of<H>(qk[1], hp, s));
      }
    }
    for (; i < nv; i += blockDim.x) {
      uint4 q = __ldcs(p + i);
      const K* qk = reinterpret_cast<const K*>(&q);
      hist_add(s_h, f_lo, nf, fine_of<H>(qk[0], hp, s));
      hist_add(s_h, f_lo, nf, fine_of<H>(qk[1], hp, s));
    }
    for (uint64_t j = lo + nv * 2 + threadIdx.x; j < hi; j += blockDim.x) hist_add(s_h, f_lo, nf, fine_of<H>(keys[j], hp, s));
  } else if (sizeof(K) == 4 && lo < hi && ((reinterpret_cast<uintptr_t>(keys + lo) & 15) == 0)) {
    const uint4* p = reinterpret_cast<const uint4*>(keys + lo);
    const uint64_t nv = (hi - lo) / 4;
    uint64_t i = threadIdx.x;
    for (; i + 3 * blockDim.x < nv; i += 4 * blockDim.x) {
      uint4 q[4];
#pragma unroll
      for (int u = 0; u < 4; u++) q[u] = __ldcs(p + i + u * blockDim.x);
#pragma unroll
      for (int u = 0; u < 4; u++) {
        hist_add(s_h, f_lo, nf, fine_of<H>((K)q[u].x, hp, s));
        hist_add(s_h, f_lo, nf, fine_of<H>((K)q[u].y, hp, s));
        hist_add(s_h, f_lo, nf, fine_of<H>((K)q[u].z, hp, s));
        hist_add(s_h, f_lo, nf, fine_of<H>((K)q[u].w, hp, s));
      }
    }
    for (; i < nv; i += blockDim.x) {
      uint4 q = __ldcs(p + i);
      hist_add(s_h, f_lo, nf, fine_of<H>((K)q.x, hp, s));
      hist_add(s_h, f_lo, nf, fine_of<H>((K)q.y, hp, s));
      hist_add(s_h, f_lo, nf, fine_of<H>((K)q.z, hp, s));
      hist_add(s_h, f_lo, nf, fine_of<H>((K)q.w, hp, s));
    }
    for (uint64_t j = lo + nv * 4 + threadIdx.x; j < hi; j += blockDim.x) hist_add(s_h, f_lo, nf, fine_of<H>(keys[j], hp, s));
  } else {
    for (uint64_t j = lo + threadIdx.x; j < hi; j += blockDim.x) hist_add(s_h, f_lo, nf, fine_of<H>(keys[j], hp, s));
  }
  __syncthreads();
  uint32_t* row = M + (uint64_t)blockIdx.x * nb1;
  for (uint32_t c = f_lo / group + threadIdx.x; c < nb1 && c * group < f_lo + nf; c += blockDim.x) {
    uint32_t sum = 0;
    const uint32_t f1 = min((c + 1) * group, nfine);
    for (uint32_t f = c * group; f < f1; f++) sum += s_h[f - f_lo];
    row[c] = sum;
  }
  for (uint32_t f = threadIdx.x; f < nf; f += blockDim.x)
    if (s_h[f]) atomicAdd(fine_cnt + f_lo + f, s_h[f]);
}

#undef hist_add

// One CTA per level-1 bin: exclusive prefix down its column of per-CTA counts
// (in place).  All G loads are in flight at once; a thread-per-bin serial walk
// was 296 dependent loads long.
__global__ void __launch_bounds__(1024) k_colscan(uint32_t* __restrict__ M, uint32_t G, uint32_t nb1) {
  extern __shared__ uint32_t s_col[];  // G
  const uint32_t b = blockIdx.x;
  for (uint32_t g = threadIdx.x; g < G; g += blockDim.x) s_col[g] = M[(uint64_t)g * nb1 + b];
  __syncthreads();
  block_exscan(s_col, G);
  for (uint32_t g = threadIdx.x; g < G; g += blockDim.x) M[(uint64_t)g * nb1 + b] = s_col[g];
}

// One CTA: fine starts (F+1), level-1 starts (nb1+1), level-2 tile prefix
// (nb1+1; tp[nb1] = level-2 tile count), fine cursors (= fine starts), the
// list of fine bins above `cap` keys (build only: big_list[0, big_count[0])
// the medium ones, big_list[nfine - 1 - j], j < big_count[1], the ones above
// kHugeBin keys) with the huge ones' prefix of `big_chunk`-key chunks (big_cp,
// nhuge + 1) and zeroed per-bin chunk-completion counters (big_done[j] and
// big_done[nfine + 1 + j]), and `nzero` zeroed words at `zero` (the query's
// plan).
constexpr uint32_t kHugeBin = 1u << 16;  // oversized bins above this are built by many CTAs in chunks

constexpr uint32_t kStartsChunk = 32768;  // fine bins k_starts scans per smem round

__global__ void __launch_bounds__(1024)
k_starts(const uint32_t* __restrict__ fine_cnt, uint32_t nfine, uint32_t group, uint32_t nb1, uint32_t tile,
         uint32_t cap, uint32_t* __restrict__ fine_start, uint32_t* __restrict__ c_start, uint32_t* __restrict__ tp,
         uint32_t* __restrict__ fine_cursor, uint32_t* __restrict__ big_list, uint32_t* __restrict__ big_count,
         uint32_t big_chunk, uint32_t* __restrict__ big_cp, uint32_t* __restrict__ big_done, uint32_t* __restrict__ zero,
         uint32_t nzero) {
  for (uint32_t i = threadIdx.x; i < nzero; i += blockDim.x) zero[i] = 0;
  extern __shared__ uint32_t s_a[];  // min(nfine, kStartsChunk)
  __shared__ uint32_t s_t[kMaxBins + 1];
  __shared__ uint32_t s_big, s_huge;
  if (threadIdx.x == 0) s_big = s_huge = 0;
  __syncthreads();
  // fine bins in rounds of kStartsChunk (a level-1 bin never straddles two:
  // group divides the round); the scan carries across rounds
  uint32_t carry = 0;
  for (uint32_t base = 0; base < nfine; base += kStartsChunk) {
    const uint32_t len = min(kStartsChunk, nfine - base);
    for (uint32_t i = threadIdx.x; i < len; i += blockDim.x) {
      const uint32_t t = fine_cnt[base + i];
      s_a[i] = t;
      // oversized bins: medium ones from the front of the list, huge ones
      // (> kHugeBin keys, built in chunks by many CTAs) from the back
      if (t > kHugeBin && big_cp) big_list[nfine - 1 - atomicAdd(&s_huge, 1u)] = base + i;
      else if (t > cap) big_list[atomicAdd(&s_big, 1u)] = base + i;
    }
    __syncthreads();
    const uint32_t tot = block_exscan_rows(s_a, len, carry);  // warp-row layout: no bank conflicts
    for (uint32_t i = threadIdx.x; i < len; i += blockDim.x) {
      fine_start[base + i] = s_a[i];
      fine_cursor[base + i] = s_a[i];
    }
    for (uint32_t c = base / group + threadIdx.x; c < nb1 && c * group < base + len; c += blockDim.x)
      c_start[c] = s_a[c * group - base];
    carry += tot;
    __syncthreads();
  }
  const uint32_t total = carry;
  if (threadIdx.x == 0) {
    fine_start[nfine] = total;
    c_start[nb1] = total;
    big_count[0] = s_big;
    big_count[1] = s_huge;
  }
  __syncthreads();  // c_start (global, this CTA's writes) complete
  for (uint32_t c = threadIdx.x; c < nb1; c += blockDim.x) s_t[c] = (c_start[c + 1] - c_start[c] + tile - 1) / tile;
  __syncthreads();
  const uint32_t ntiles = block_exscan(s_t, nb1);
  for (uint32_t c = threadIdx.x; c < nb1; c += blockDim.x) tp[c] = s_t[c];
  if (threadIdx.x == 0) tp[nb1] = ntiles;
  // oversized bins (hg_bigbin.cuh): chunk prefix, completion counters
  const uint32_t nbig = s_huge;
  if (big_cp == nullptr || nbig == 0) return;
  uint32_t ccarry = 0;
  for (uint32_t base = 0; base < nbig; base += blockDim.x) {
    const uint32_t j = base + threadIdx.x;
    uint32_t c = 0;
    if (j < nbig) {
      const uint32_t f = big_list[nfine - 1 - j];
      c = (fine_start[f + 1] - fine_start[f] + big_chunk - 1) / big_chunk;
    }
    uint32_t tot;
    const uint32_t e = block_scan_excl<uint32_t>(c, tot);
    if (j < nbig) big_cp[j] = ccarry + e;
    ccarry += tot;
  }
  if (threadIdx.x == 0) big_cp[nbig] = ccarry;
  for (uint32_t j = threadIdx.x; j < nbig; j += blockDim.x) {
    big_done[j] = 0;              // k_big_count
    big_done[nfine + 1 + j] = 0;  // k_big_place
  }
}

// --------------------------------------------------------------------------- partition

// Runs are staged in smem at positions congruent (mod 4 elements) to their
// global destination, so the aligned body of every run leaves with one TMA
// bulk store: bin b's run starts at pt[b] = toff[b] + 8b + 4 + ((dst[b] - toff[b]) & 3).
// The 5..11 slots between runs also leave room for the 16-byte-aligned
// superset of every run (<= 3 slots either side, never overlapping the next
// run's superset), so the unpartition pulls each run back with one bulk copy
// and no per-element head/tail loads.
constexpr uint32_t kPadMod = 4;                  // alignment unit (elements)
constexpr uint32_t kPadRun = 8;                  // staged slots reserved per bin
constexpr uint32_t kPadTotal = kPadRun * kMaxBins + 2 * kPadMod;  // staged size over the tile

template <typename K>
struct PartSmem {
  K raw[TileShape<K>::kTile + 16 / sizeof(K)];              // TMA landing buffer (next tile)
  K staged[TileShape<K>::kTile + kPadTotal];  // runs, padded for alignment
  uint32_t wcnt[kW][kMaxBins];  // per-warp counts -> per-warp slot bases
  uint32_t toff[kMaxBins + 1];  // tile offsets per bin (unpadded)
  uint32_t pt[kMaxBins];        // padded staged start per bin
  uint32_t dst[kMaxBins];       // global write base per bin
  uint32_t tp[kMaxBins + 1];    // level-2 tile prefix (P2 only)
  uint32_t cs[kMaxBins + 1];    // level-1 bin starts (P2 only): locating a tile needs no global load
  alignas(8) uint64_t bar;  // TMA load barrier
};

__device__ __forceinline__ uint32_t pad_start(uint32_t toff, uint32_t b, uint32_t dst) {
  return toff + kPadRun * b + kPadMod + ((dst - toff) & (kPadMod - 1));
}

// Rank a register tile by bin: one atomic on the warp's private bin counter
// per key (rank kept in registers), then a per-bin prefix over warps.  On
// return s.toff holds the tile offsets (s.toff[nb] = tile size), s.pt each
// run's padded staged start (congruent to s.dst[b] mod 4) and s.wcnt[w][b]
// warp w's first staged slot in bin b.
//
// claims != nullptr (level 2): each bin's space is claimed (atomicAdd on
// claims[b]) as soon as the bin's total is known, and the answer lands in
// s.dst[b] after the bin scan, so the atomic's latency overlaps the scan.
//
// after_count() runs right after the counting barrier (every thread has
// finished reading the tile's raw keys by then): the caller lands the next
// tile there, with no barrier of its own.
struct NoOp {
  __device__ void operator()() const {}
};

template <typename K, int KPT, bool kFull, typename F = NoOp>
__device__ __forceinline__ void rank_tile(PartSmem<K>& s, const uint32_t (&bp)[KPT / 4], uint32_t (&rk)[KPT / 2],
                                          uint32_t m, uint32_t nb, uint32_t* __restrict__ claims = nullptr,
                                          F after_count = F()) {
  constexpr bool vec = kFull;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t b = lane; b < nb; b += 32) s.wcnt[warp][b] = 0;
  __syncwarp();
#pragma unroll
  for (int k = 0; k < KPT; k++) {
    const uint32_t b = (bp[k >> 2] >> ((k & 3) * 8)) & 0xFFu;
    uint32_t r = 0;
    if (kFull || tile_elem<K>(k, vec) < m) r = atomicAdd(&s.wcnt[warp][b], 1u);
    if (k & 1) rk[k >> 1] |= r << 16; else rk[k >> 1] = r;
  }
  __syncthreads();
  after_count();
  // Per-bin prefix over warps and the scan over bins, by the warps that own
  // bins only (thread b = bin b), synchronised with a named barrier among
  // them: the rest of the CTA waits at one barrier instead of four.
  __shared__ uint32_t s_bw[kMaxBins / 32];
  const uint32_t nbw = (nb + 31) / 32;  // warps that own bins (CTA-uniform)
  if ((uint32_t)warp < nbw) {
    const uint32_t b = threadIdx.x;
    uint32_t run = 0, d = 0;
    if (b < nb) {
#pragma unroll
      for (int w = 0; w < kW; w++) {
        const uint32_t c = s.wcnt[w][b];
        s.wcnt[w][b] = run;
        run += c;
      }
      if (claims && run) d = atomicAdd(claims + b, run);
    }
    uint32_t inc = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) s_bw[warp] = inc;
    named_barrier_sync(1, nbw * 32);
    uint32_t base = 0;
    for (int w = 0; w < warp; w++) base += s_bw[w];
    if (b < nb) {
      const uint32_t toff_b = base + inc - run;
      s.toff[b] = toff_b;
      if (b == nb - 1) s.toff[nb] = base + inc;
      if (claims) s.dst[b] = d;
      else d = s.dst[b];
      // padded staged start of the run; the warps' offsets become absolute slots
      const uint32_t p = pad_start(toff_b, b, d);
      s.pt[b] = p;
#pragma unroll
      for (int w = 0; w < kW; w++) s.wcnt[w][b] += p;
    }
  }
  __syncthreads();
}

// Stage every key at its padded slot; pmap (optional) gets the slot.
template <typename K, int KPT, bool kFull>
__device__ __forceinline__ void place_tile(PartSmem<K>& s, const K (&kv)[KPT], const uint32_t (&bp)[KPT / 4],
                                           const uint32_t (&rk)[KPT / 2], uint32_t m, uint16_t* __restrict__ pmap) {
  constexpr bool vec = kFull;
  constexpr int VPL = 16 / sizeof(K);  // consecutive elements per thread in the vector mapping
  const int warp = threadIdx.x >> 5;
  uint32_t sl[VPL];
#pragma unroll
  for (int k = 0; k < KPT; k++) {
    const uint32_t e = tile_elem<K>(k, vec);
    if (kFull || e < m) {
      const uint32_t b = (bp[k >> 2] >> ((k & 3) * 8)) & 0xFFu;
      const uint32_t slot = s.wcnt[warp][b] + ((rk[k >> 1] >> ((k & 1) * 16)) & 0xFFFFu);
      s.staged[slot] = kv[k];
      if (kFull) {
        sl[k % VPL] = slot;
        if (pmap && k % VPL == VPL - 1) {  // VPL consecutive u16 slots -> one store
          if (VPL == 4)
            *reinterpret_cast<uint2*>(pmap + e - 3) = make_uint2(sl[0] | (sl[1 % VPL] << 16), sl[2 % VPL] | (sl[3 % VPL] << 16));
          else
            *reinterpret_cast<uint32_t*>(pmap + e - 1) = sl[0] | (sl[1 % VPL] << 16);
        }
      } else if (pmap) {
        pmap[e] = (uint16_t)slot;
      }
    }
  }
  fence_proxy_async();  // staged (generic writes) -> TMA bulk-store reads
  __syncthreads();
}

// One thread per bin: the unaligned head/tail (< 4 keys each) with plain
// stores, the aligned body with one TMA bulk store.
template <typename K>
__device__ __forceinline__ void store_runs(const PartSmem<K>& s, uint32_t nb, K* __restrict__ out) {
  if (threadIdx.x < nb) {
    const uint32_t b = threadIdx.x;
    const uint32_t cnt = s.toff[b + 1] - s.toff[b];
    if (cnt) {
      const uint32_t g = s.dst[b], p = s.pt[b];
      const uint32_t h = min(cnt, (kPadMod - (g & (kPadMod - 1))) & (kPadMod - 1));
      const uint32_t body = (cnt - h) & ~(kPadMod - 1);
      for (uint32_t i = 0; i < h; i++) out[g + i] = s.staged[p + i];
      if (body) {
        tma_store_1d(out + g + h, s.staged + p + h, body * (uint32_t)sizeof(K));
        tma_store_commit();
      }
      for (uint32_t i = h + body; i < cnt; i++) out[g + i] = s.staged[p + i];
    }
  }
}

// Level 1: CTA chunk tiles, bin = bucket >> shift1, deterministic bases
// (column-scanned per-CTA counts).  Query mode also records the u16 staged
// slot of every key (pmap) and each tile's offsets (meta, nb+1 words).
template <typename H, bool kQuery>
__global__ void __launch_bounds__(kT, 2)
k_part1(const KeyOf<H>* __restrict__ keys, uint64_t n, HashParams hp, int shift1, int bits1, uint32_t nb1, uint64_t chunk,
        const uint32_t* __restrict__ M, const uint32_t* __restrict__ c_start, KeyOf<H>* __restrict__ out,
        uint16_t* __restrict__ pmap, uint32_t* __restrict__ meta) {
  using K = typename H::Key;
  using TS = TileShape<K>;
  constexpr int KPT = TS::kKPT;
  constexpr int VPL = 16 / sizeof(K);
  extern __shared__ __align__(128) unsigned char s_raw[];
  PartSmem<K>& s = *reinterpret_cast<PartSmem<K>*>(s_raw);
  const uint64_t lo = (uint64_t)blockIdx.x * chunk;
  const uint64_t hi = min(n, lo + chunk);
  const uint32_t* row = M + (uint64_t)blockIdx.x * nb1;
  if (threadIdx.x < nb1) s.dst[threadIdx.x] = c_start[threadIdx.x] + row[threadIdx.x];
  // full tiles stream through one TMA buffer: tile i+1 lands while tile i is ranked
  const bool tma = (reinterpret_cast<uintptr_t>(keys) & 15) == 0;
  if (threadIdx.x == 0) {
    mbar_init(&s.bar, 1);
    fence_proxy_async();
  }
  __syncthreads();
  uint32_t parity = 0;
  if (threadIdx.x == 0 && tma && lo + TS::kTile <= hi) tma_load_1d(s.raw, keys + lo, TS::kTile * sizeof(K), &s.bar);
  for (uint64_t t0 = lo; t0 < hi; t0 += TS::kTile) {
    const uint32_t m = (uint32_t)min((uint64_t)TS::kTile, hi - t0);
    K kv[KPT];
    bool vec;
    if (tma && m == (uint32_t)TS::kTile) {
      mbar_wait(&s.bar, parity);
      parity ^= 1;
      const uint4* r4 = reinterpret_cast<const uint4*>(s.raw);
#pragma unroll
      for (int l = 0; l < KPT / VPL; l++) {
        uint4 q = r4[l * kT + threadIdx.x];
        const K* qk = reinterpret_cast<const K*>(&q);
#pragma unroll
        for (int j = 0; j < VPL; j++) kv[l * VPL + j] = qk[j];
      }
      vec = true;
    } else {
      vec = load_tile<K, KPT>(keys + t0, m, kv);
    }
    uint32_t bp[KPT / 4];
#pragma unroll
    for (int k = 0; k < KPT; k++) {
      const uint32_t b = (uint32_t)(H::bucket(kv[k], hp) >> shift1);
      if ((k & 3) == 0) bp[k >> 2] = 0;
      bp[k >> 2] |= (b & 0xFFu) << ((k & 3) * 8);
    }
    if (threadIdx.x < nb1) tma_store_wait_read();  // previous tile's runs have left smem (before placement)
    fence_proxy_async();                            // raw reads ordered before the next tile's TMA write
    auto prefetch = [&] {
      if (threadIdx.x == 0 && tma && t0 + 2 * TS::kTile <= hi)
        tma_load_1d(s.raw, keys + t0 + TS::kTile, TS::kTile * sizeof(K), &s.bar);
    };
    uint32_t rk[KPT / 2];
    if (vec) rank_tile<K, KPT, true>(s, bp, rk, m, nb1, nullptr, prefetch);
    else rank_tile<K, KPT, false>(s, bp, rk, m, nb1, nullptr, prefetch);
    if (vec) place_tile<K, KPT, true>(s, kv, bp, rk, m, kQuery ? pmap + t0 : nullptr);
    else place_tile<K, KPT, false>(s, kv, bp, rk, m, kQuery ? pmap + t0 : nullptr);
    if (kQuery)
      for (uint32_t i = threadIdx.x; i <= nb1; i += blockDim.x) meta[(t0 / TS::kTile) * (nb1 + 1) + i] = s.toff[i];
    store_runs<K>(s, nb1, out);
    if (threadIdx.x < nb1) s.dst[threadIdx.x] += s.toff[threadIdx.x + 1] - s.toff[threadIdx.x];
  }
  if (threadIdx.x < nb1) tma_store_wait_all();
}

// Level 2: tiles of each level-1 bin, sub-bin = fine & 127, space claimed per
// (tile, fine bin) from the fine cursors.  Query mode records pmap (indexed in
// level-1 order) and meta = [128 claims | 129 tile offsets] per tile.  Tiles
// start anywhere, so the TMA copy starts at the 16-byte boundary below the
// tile (the input buffer carries 16 bytes of tail padding).
template <typename H, bool kQuery, uint32_t sub>  // sub = level-2 fan-out (128 or 256), compile-time
__global__ void __launch_bounds__(kT, 2)
k_part2(const KeyOf<H>* __restrict__ in, HashParams hp, int s_log, uint32_t nb1, const uint32_t* __restrict__ c_start,
        const uint32_t* __restrict__ tp_g, uint32_t* __restrict__ fine_cursor, KeyOf<H>* __restrict__ out,
        uint16_t* __restrict__ pmap, uint32_t* __restrict__ meta, uint32_t c_lo = 0, uint32_t c_hi = 0xFFFFFFFFu) {
  using K = typename H::Key;
  using TS = TileShape<K>;
  constexpr int KPT = TS::kKPT;
  constexpr uint32_t VPL = 16 / sizeof(K);
  extern __shared__ __align__(128) unsigned char s_raw[];
  PartSmem<K>& s = *reinterpret_cast<PartSmem<K>*>(s_raw);
  for (uint32_t i = threadIdx.x; i <= nb1; i += blockDim.x) {
    s.tp[i] = tp_g[i];
    s.cs[i] = c_start[i];
  }
  if (threadIdx.x == 0) {
    mbar_init(&s.bar, 1);
    fence_proxy_async();
  }
  __syncthreads();
  const uint32_t ntiles = s.tp[min(c_hi, nb1)];  // level-1 bins [c_lo, c_hi): tiles [tp[c_lo], tp[c_hi])
  const uint32_t tfirst = s.tp[min(c_lo, nb1)] + blockIdx.x;
  // thread 0 locates a tile (binary search over the level-2 tile prefix plus
  // two c_start loads) when it issues the tile's TMA, one tile ahead, and
  // leaves (bin, first element, size) in smem: no global latency at the top
  // of a tile
  __shared__ uint32_t s_loc[3];
  __shared__ uint32_t s_cur[3];  // the current tile's (bin, first, size), re-read after ranking: fewer live registers
  auto locate_issue = [&](uint32_t t) {
    uint32_t a = 0, z = nb1;  // level-1 bin c: tp[c] <= t < tp[c+1]
    while (z - a > 1) {
      const uint32_t mid = (a + z) >> 1;
      if (s.tp[mid] <= t) a = mid; else z = mid;
    }
    const uint32_t t0 = s.cs[a] + (t - s.tp[a]) * TS::kTile;
    const uint32_t m = min((uint32_t)TS::kTile, s.cs[a + 1] - t0);
    s_loc[0] = a;
    s_loc[1] = t0;
    s_loc[2] = m;
    const uint32_t a0 = t0 & ~(VPL - 1);
    const uint32_t bytes = ((t0 - a0 + m) * (uint32_t)sizeof(K) + 15) & ~15u;
    tma_load_1d(s.raw, in + a0, bytes, &s.bar);
  };
  uint32_t parity = 0;
  if (threadIdx.x == 0 && tfirst < ntiles) locate_issue(tfirst);
  __syncthreads();  // s_loc of the first tile (later ones are ordered by the tile loop's barriers)
  for (uint32_t t = tfirst; t < ntiles; t += gridDim.x) {
    const uint32_t c = s_loc[0], t0 = s_loc[1], m = s_loc[2];
    if (!kQuery && threadIdx.x == 0) {  // build: re-read after ranking (measured: fewer spills); query: registers
      s_cur[0] = c;
      s_cur[1] = t0;
      s_cur[2] = m;
    }
    mbar_wait(&s.bar, parity);
    parity ^= 1;
    const uint32_t sh = t0 & (VPL - 1);
    K kv[KPT];
#pragma unroll
    for (int k = 0; k < KPT; k++) {
      const uint32_t e = k * kT + threadIdx.x;
      kv[k] = e < m ? s.raw[sh + e] : K(0);
    }
    uint32_t bp[KPT / 4];
#pragma unroll
    for (int k = 0; k < KPT; k++) {
      const uint32_t b = (uint32_t)(H::bucket(kv[k], hp) >> s_log) & (sub - 1);
      if ((k & 3) == 0) bp[k >> 2] = 0;
      bp[k >> 2] |= b << ((k & 3) * 8);
    }
    if (threadIdx.x < sub) tma_store_wait_read();
    fence_proxy_async();
    __syncthreads();  // raw and s_loc consumed by every thread
    if (threadIdx.x == 0 && t + gridDim.x < ntiles) locate_issue(t + gridDim.x);
    uint32_t rk[KPT / 2];
    rank_tile<K, KPT, false>(s, bp, rk, kQuery ? m : s_cur[2], sub, fine_cursor + (kQuery ? c : s_cur[0]) * sub);
    if (kQuery) {
      if (threadIdx.x < sub) meta[(uint64_t)t * (2 * sub + 1) + threadIdx.x] = s.dst[threadIdx.x];
      for (uint32_t i = threadIdx.x; i <= sub; i += blockDim.x) meta[(uint64_t)t * (2 * sub + 1) + sub + i] = s.toff[i];
    }
    place_tile<K, KPT, false>(s, kv, bp, rk, kQuery ? m : s_cur[2], kQuery ? pmap + t0 : nullptr);
    store_runs<K>(s, sub, out);
  }
  if (threadIdx.x < sub) tma_store_wait_all();
}

// Reverse of a partition level for per-query uint32 values.  Level 2: tiles
// from the level-2 tile table, run bases from meta; level 1: each CTA replays
// its chunk's tiles with cursors from the column-scanned counts.  Each run is
// pulled back into its padded staged slot range (TMA for the aligned body),
// then out[i] = staged[pmap[i]].  Two staging buffers: tile i+1's runs are in
// flight (meta read, bulk loads issued) while tile i is gathered.
constexpr uint32_t kUnpStaged = 8192 + kPadTotal;

template <int kLevel>
__global__ void __launch_bounds__(kT, 2)
k_unpart(const uint32_t* __restrict__ vals, uint32_t* __restrict__ out, const uint16_t* __restrict__ pmap,
         const uint32_t* __restrict__ meta, uint32_t sub, uint32_t nb, uint32_t tile, uint64_t n, uint64_t chunk,
         const uint32_t* __restrict__ M, const uint32_t* __restrict__ c_start, const uint32_t* __restrict__ tp_g) {
  constexpr int VPT = 8192 / kT;  // gathered values per thread (tile <= 8192)
  constexpr uint32_t TO = kMaxBins + 1;
  extern __shared__ __align__(128) unsigned char s_raw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(s_raw);                 // 2
  uint32_t* staged = reinterpret_cast<uint32_t*>(s_raw + 16);         // 2 x kUnpStaged
  uint32_t* toff = staged + 2 * kUnpStaged;                           // 2 x (kMaxBins + 1)
  uint32_t* base = toff + 2 * TO;                                     // 2 x kMaxBins
  uint32_t* tps = base + 2 * kMaxBins;                                // kMaxBins + 1
  const uint32_t nbb = kLevel == 1 ? nb : sub;
  uint64_t lo = 0, hi = 0;
  uint32_t ntiles = 0;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    fence_proxy_async();
  }
  if (kLevel == 1) {
    lo = (uint64_t)blockIdx.x * chunk;
    hi = min(n, lo + chunk);
    ntiles = hi > lo ? (uint32_t)((hi - lo + tile - 1) / tile) : 0u;
  } else {
    for (uint32_t i = threadIdx.x; i <= nb; i += blockDim.x) tps[i] = tp_g[i];
  }
  __syncthreads();
  if (kLevel == 2) {
    const uint32_t tot = tps[nb];
    ntiles = tot > blockIdx.x ? (tot - blockIdx.x + gridDim.x - 1) / gridDim.x : 0u;
  }
  if (ntiles == 0) return;
  // this CTA's i-th tile: first element, size, index into meta
  auto tile_of = [&](uint32_t i, uint64_t& t0, uint32_t& m, uint64_t& tix) {
    if (kLevel == 1) {
      t0 = lo + (uint64_t)i * tile;
      m = (uint32_t)min((uint64_t)tile, hi - t0);
      tix = t0 / tile;
    } else {
      const uint32_t t = blockIdx.x + i * gridDim.x;
      uint32_t a = 0, z = nb;
      while (z - a > 1) {
        const uint32_t mid = (a + z) >> 1;
        if (tps[mid] <= t) a = mid; else z = mid;
      }
      t0 = c_start[a] + (t - tps[a]) * tile;
      m = min(tile, c_start[a + 1] - (uint32_t)t0);
      tix = t;
    }
  };
  // Per tile, thread x <= nbb holds its meta words in registers one tile
  // ahead: level 1 the run offset toff[x]; level 2 the claim base[x] and
  // toff[x].  They are loaded from global memory while the previous tile is
  // gathered and only stored to smem (no global latency) before the barrier.
  auto meta_load = [&](uint64_t tix, uint32_t& r0, uint32_t& r1) {
    const uint32_t x = threadIdx.x;
    if (kLevel == 1) {
      if (x <= nb) r0 = meta[tix * (nb + 1) + x];
    } else {
      if (x < sub) r1 = meta[tix * (2 * sub + 1) + x];
      if (x <= sub) r0 = meta[tix * (2 * sub + 1) + sub + x];
    }
  };
  // registers -> buffer bf; level-1 bases chain from the previous tile (bf ^ 1)
  auto meta_store = [&](uint32_t i, int bf, uint32_t r0, uint32_t r1) {
    const uint32_t x = threadIdx.x;
    if (kLevel == 1) {
      if (x <= nb) toff[bf * TO + x] = r0;
      if (x < nb) {
        const uint32_t pb = (bf ^ 1) * TO;
        base[bf * kMaxBins + x] = i == 0 ? c_start[x] + M[(uint64_t)blockIdx.x * nb + x]
                                         : base[(bf ^ 1) * kMaxBins + x] + toff[pb + x + 1] - toff[pb + x];
      }
    } else {
      if (x < sub) base[bf * kMaxBins + x] = r1;
      if (x <= sub) toff[bf * TO + x] = r0;
    }
  };
  // one thread per bin: the run's 16-byte-aligned superset in one bulk copy
  // (the padding absorbs the <= 3 extra slots on each side; `vals` carries
  // 16 bytes of tail padding)
  auto issue = [&](int bf) {
    if (threadIdx.x < nbb) {
      const uint32_t b = threadIdx.x;
      const uint32_t cnt = toff[bf * TO + b + 1] - toff[bf * TO + b];
      if (cnt) {
        uint32_t* st = staged + bf * kUnpStaged;
        const uint32_t g = base[bf * kMaxBins + b];
        const uint32_t p = pad_start(toff[bf * TO + b], b, g);
        const uint32_t g0 = g & ~(kPadMod - 1), g1 = (g + cnt + kPadMod - 1) & ~(kPadMod - 1);
        mbar_expect_tx(bar + bf, (g1 - g0) * 4);
        tma_load_1d_tx(st + p - (g - g0), vals + g0, (g1 - g0) * 4, bar + bf);
      }
    }
  };
  uint64_t t0c, t0n = 0, tix;
  uint32_t mc, mn = 0;
  uint32_t r0 = 0, r1 = 0;  // meta of the next tile (it + 1), in flight
  tile_of(0, t0c, mc, tix);
  meta_load(tix, r0, r1);
  meta_store(0, 0, r0, r1);
  __syncthreads();
  issue(0);
  __syncthreads();
  if (threadIdx.x == 0) mbar_arrive(bar);
  if (ntiles > 1) {
    tile_of(1, t0n, mn, tix);
    meta_load(tix, r0, r1);
  }
  for (uint32_t it = 0; it < ntiles; it++) {
    const int cur = it & 1, nxt = cur ^ 1;
    const bool more = it + 1 < ntiles;
    const uint32_t* st = staged + cur * kUnpStaged;
    const bool vec = kLevel == 1 && mc == tile && tile == (uint32_t)VPT * kT;
    // position maps of tile it load while tile it+1's runs are requested
    uint4 pm4[VPT / 8];
    uint32_t pm[VPT];
    if (vec) {
      const uint4* p4 = reinterpret_cast<const uint4*>(pmap + t0c);
#pragma unroll
      for (int k = 0; k < VPT / 8; k++) pm4[k] = p4[k * kT + threadIdx.x];
    } else {
#pragma unroll
      for (int k = 0; k < VPT; k++) {
        const uint32_t i = k * kT + threadIdx.x;
        pm[k] = i < mc ? pmap[t0c + i] : 0u;
      }
    }
    if (more) meta_store(it + 1, nxt, r0, r1);
    __syncthreads();
    if (more) issue(nxt);
    uint64_t t0nn = 0;
    uint32_t mnn = 0;
    if (it + 2 < ntiles) {  // look ahead: tile it+2's position and meta load during this gather
      tile_of(it + 2, t0nn, mnn, tix);
      meta_load(tix, r0, r1);
    }
    mbar_wait(bar + cur, (it >> 1) & 1);
    if (vec) {
      // full level-1 tiles are 16-byte aligned: 8 slots per 16-byte load,
      // 4 values per 16-byte store
      uint4* o4 = reinterpret_cast<uint4*>(out + t0c);
#pragma unroll
      for (int k = 0; k < VPT / 8; k++) {
        const uint32_t w[4] = {pm4[k].x, pm4[k].y, pm4[k].z, pm4[k].w};
        const uint32_t c = k * kT + threadIdx.x;
        o4[2 * c] = make_uint4(st[w[0] & 0xFFFFu], st[w[0] >> 16], st[w[1] & 0xFFFFu], st[w[1] >> 16]);
        o4[2 * c + 1] = make_uint4(st[w[2] & 0xFFFFu], st[w[2] >> 16], st[w[3] & 0xFFFFu], st[w[3] >> 16]);
      }
    } else {
#pragma unroll
      for (int k = 0; k < VPT; k++) {
        const uint32_t i = k * kT + threadIdx.x;
        if (i < mc) out[t0c + i] = st[pm[k]];
      }
    }
    fence_proxy_async();  // generic reads of this buffer before the next bulk writes into it
    __syncthreads();      // buffer cur free; tile it+1's expect_tx all posted
    if (more && threadIdx.x == 0) mbar_arrive(bar + nxt);
    t0c = t0n;
    mc = mn;
    t0n = t0nn;
    mn = mnn;
  }
}

// Forward of a partition level for per-key uint32 values (the inverse of
// k_unpart): each tile's values (input order; level 1 with vals == nullptr:
// the input index itself) go to their staged slots through the recorded u16
// position map -- the staging layout k_part1 / k_part2 used for the keys, so
// every run's aligned body leaves with one TMA bulk store -- with no hashing
// or ranking.  build_traced uses it to carry input indices to the grouped
// order.  The next tile's map, values and metadata load during this tile's
// stores.
template <int kLevel>
__global__ void __launch_bounds__(kT, 2)
k_repart(const uint32_t* __restrict__ vals, uint32_t* __restrict__ out, const uint16_t* __restrict__ pmap,
         const uint32_t* __restrict__ meta, uint32_t sub, uint32_t nb, uint32_t tile, uint64_t n, uint64_t chunk,
         const uint32_t* __restrict__ M, const uint32_t* __restrict__ c_start, const uint32_t* __restrict__ tp_g) {
  constexpr int VPT = 8192 / kT;  // values per thread (tile <= 8192)
  extern __shared__ __align__(128) unsigned char s_raw[];
  uint32_t* staged = reinterpret_cast<uint32_t*>(s_raw);  // kUnpStaged
  __shared__ uint32_t toff[kMaxBins + 1], base[kMaxBins], tps[kMaxBins + 1];
  const uint32_t nbb = kLevel == 1 ? nb : sub;
  uint64_t lo = 0, hi = 0;
  uint32_t ntiles;
  if (kLevel == 1) {
    lo = (uint64_t)blockIdx.x * chunk;
    hi = min(n, lo + chunk);
    ntiles = hi > lo ? (uint32_t)((hi - lo + tile - 1) / tile) : 0u;
  } else {
    for (uint32_t i = threadIdx.x; i <= nb; i += blockDim.x) tps[i] = tp_g[i];
    __syncthreads();
    const uint32_t tot = tps[nb];
    ntiles = tot > blockIdx.x ? (tot - blockIdx.x + gridDim.x - 1) / gridDim.x : 0u;
  }
  auto tile_of = [&](uint32_t it, uint64_t& t0, uint32_t& m, uint64_t& tix) {
    if (kLevel == 1) {
      t0 = lo + (uint64_t)it * tile;
      m = (uint32_t)min((uint64_t)tile, hi - t0);
      tix = t0 / tile;
    } else {
      const uint32_t t = blockIdx.x + it * gridDim.x;
      uint32_t a = 0, z = nb;
      while (z - a > 1) {
        const uint32_t mid = (a + z) >> 1;
        if (tps[mid] <= t) a = mid; else z = mid;
      }
      t0 = c_start[a] + (t - tps[a]) * tile;
      m = min(tile, c_start[a + 1] - (uint32_t)t0);
      tix = t;
    }
  };
  // per-thread registers of a tile: its map slots, values and (threads <= nbb) meta words
  uint32_t pm[VPT], vv[VPT], r0 = 0, r1 = 0;
  uint64_t t0 = 0, tix = 0;
  uint32_t m = 0;
  auto load = [&](uint32_t it) {
    tile_of(it, t0, m, tix);
    if (kLevel == 1 && vals == nullptr && m == tile && tile == (uint32_t)VPT * kT) {
      // full level-1 tiles are 16-byte aligned: 8 slots per 16-byte map load,
      // each thread owning 8 consecutive elements per load (any element ->
      // thread mapping works: every value carries its own slot)
      const uint4* p4 = reinterpret_cast<const uint4*>(pmap + t0);
#pragma unroll
      for (int k = 0; k < VPT / 8; k++) {
        const uint4 w4 = p4[k * kT + threadIdx.x];
        const uint32_t w[4] = {w4.x, w4.y, w4.z, w4.w};
        const uint32_t e0 = 8 * (k * kT + threadIdx.x);
#pragma unroll
        for (int j = 0; j < 8; j++) {
          pm[8 * k + j] = (w[j / 2] >> ((j & 1) * 16)) & 0xFFFFu;
          vv[8 * k + j] = (uint32_t)t0 + e0 + j;
        }
      }
    } else {
#pragma unroll
      for (int k = 0; k < VPT; k++) {
        const uint32_t i = k * kT + threadIdx.x;
        pm[k] = i < m ? (uint32_t)pmap[t0 + i] : 0u;
        vv[k] = i < m ? (vals ? vals[t0 + i] : (uint32_t)(t0 + i)) : 0u;
      }
    }
    const uint32_t x = threadIdx.x;
    if (kLevel == 1) {
      if (x <= nb) r0 = meta[tix * (nb + 1) + x];
    } else {
      if (x <= sub) r0 = meta[tix * (2 * sub + 1) + sub + x];
      if (x < sub) r1 = meta[tix * (2 * sub + 1) + x];
    }
  };
  if (ntiles) load(0);
  for (uint32_t it = 0; it < ntiles; it++) {
    const uint32_t mc = m;
    if (threadIdx.x < nbb) tma_store_wait_read();  // the previous tile's runs have left staged
    __syncthreads();
    const uint32_t x = threadIdx.x;
    if (kLevel == 1) {
      if (x < nb) base[x] = it == 0 ? c_start[x] + M[(uint64_t)blockIdx.x * nb + x] : base[x] + toff[x + 1] - toff[x];
    } else if (x < sub) {
      base[x] = r1;
    }
    __syncthreads();  // (level 1: base chained from the previous tile's toff before toff is replaced)
    if (x <= nbb) toff[x] = r0;
#pragma unroll
    for (int k = 0; k < VPT; k++)
      if (k * kT + threadIdx.x < mc) staged[pm[k]] = vv[k];
    fence_proxy_async();  // staged (generic writes) -> TMA bulk-store reads
    __syncthreads();
    if (it + 1 < ntiles) load(it + 1);  // next tile's loads fly during the stores
    if (threadIdx.x < nbb) {
      const uint32_t b = threadIdx.x;
      const uint32_t c0 = toff[b], cnt = toff[b + 1] - c0, g = base[b];
      if (cnt) {
        const uint32_t p = pad_start(c0, b, g);
        const uint32_t h = min(cnt, (kPadMod - (g & (kPadMod - 1))) & (kPadMod - 1));
        const uint32_t body = (cnt - h) & ~(kPadMod - 1);
        for (uint32_t i = 0; i < h; i++) out[g + i] = staged[p + i];
        if (body) {
          tma_store_1d(out + g + h, staged + p + h, body * 4u);
          tma_store_commit();
        }
        for (uint32_t i = h + body; i < cnt; i++) out[g + i] = staged[p + i];
      }
    }
  }
  if (threadIdx.x < nbb) tma_store_wait_all();
}

// --------------------------------------------------------------------------- C: local build

// Exclusive scan of the nb packed-u16 bucket counters of a 1024-thread CTA
// (8 consecutive words = 16 buckets per thread, nb <= 16384), in place, and
// the bin's offsets (lo + start) written 16 per thread as 16-byte stores.
__device__ __forceinline__ void scan_c16_offsets(uint32_t* c16, uint32_t nb, uint32_t lo, uint32_t* __restrict__ off) {
  __shared__ uint32_t s_w[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t nwords = (nb + 1) / 2;
  const uint32_t w0 = threadIdx.x * 8;
  uint32_t x[8];
  if (w0 + 8 <= nwords) {
    const uint4 a = reinterpret_cast<const uint4*>(c16)[2 * threadIdx.x];
    const uint4 b = reinterpret_cast<const uint4*>(c16)[2 * threadIdx.x + 1];
    x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w; x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
  } else {
#pragma unroll
    for (int k = 0; k < 8; k++) x[k] = w0 + k < nwords ? c16[w0 + k] : 0u;
  }
  uint32_t sum = 0;
#pragma unroll
  for (int k = 0; k < 8; k++) sum += (x[k] & 0xFFFFu) + (x[k] >> 16);
  uint32_t inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) s_w[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const uint32_t t = s_w[lane];
    uint32_t ti = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, ti, o);
      if (lane >= o) ti += y;
    }
    s_w[lane] = ti - t;
  }
  __syncthreads();
  uint32_t run = s_w[warp] + inc - sum;
  uint32_t o[16];
#pragma unroll
  for (int k = 0; k < 8; k++) {
    const uint32_t p0 = run, p1 = run + (x[k] & 0xFFFFu);
    run = p1 + (x[k] >> 16);
    x[k] = (p0 & 0xFFFFu) | (p1 << 16);
    o[2 * k] = lo + p0;
    o[2 * k + 1] = lo + p1;
  }
  if (w0 + 8 <= nwords) {
    reinterpret_cast<uint4*>(c16)[2 * threadIdx.x] = make_uint4(x[0], x[1], x[2], x[3]);
    reinterpret_cast<uint4*>(c16)[2 * threadIdx.x + 1] = make_uint4(x[4], x[5], x[6], x[7]);
  } else {
#pragma unroll
    for (int k = 0; k < 8; k++)
      if (w0 + k < nwords) c16[w0 + k] = x[k];
  }
  const uint32_t b0 = threadIdx.x * 16;
  if (b0 + 16 <= nb) {
    uint4* o4 = reinterpret_cast<uint4*>(off + b0);
#pragma unroll
    for (int k = 0; k < 4; k++) o4[k] = make_uint4(o[4 * k], o[4 * k + 1], o[4 * k + 2], o[4 * k + 3]);
  } else {
#pragma unroll
    for (int k = 0; k < 16; k++)
      if (b0 + k < nb) off[b0 + k] = o[k];
  }
  __syncthreads();
}

template <typename K>
struct LocalPShape {
  static constexpr int kThreads = 1024;
  static constexpr int kVPL = 16 / sizeof(K);
  static constexpr uint32_t kCap = BuildShape<K>::kCap;                      // keys per bin in smem
  static constexpr uint32_t kChunks = (kCap + 2 * kVPL - 2) / kVPL;          // 16-byte chunks a bin spans
  static constexpr int kCPT = (kChunks + kThreads - 1) / kThreads;           // chunks per thread
  static constexpr uint32_t kElems = kChunks * kVPL;
  __host__ __device__ static size_t c16_bytes(int s) { return (((size_t)1 << s) / 2 * 4 + 127) & ~(size_t)127; }
  static size_t smem(int s) { return c16_bytes(s) + 2 * (size_t)kChunks * 16; }
};

// kTrace (build_traced / build_query_table): also positions[p] = a2[g] (the
// input index of grouped key g, from k_repart) for the slot p each grouped key
// lands in.
template <typename H, bool kTrace = false>
__global__ void __launch_bounds__(1024, 1)
k_local_build_p(const KeyOf<H>* src, const uint32_t* __restrict__ fine_start, uint32_t nfine, HashParams hp, int s,
                uint64_t v, uint32_t* __restrict__ offsets, KeyOf<H>* edges, const uint32_t* __restrict__ a2 = nullptr,
                uint32_t* __restrict__ positions = nullptr, uint32_t f_lo = 0,
                uint32_t f_hi = 0xFFFFFFFFu) {
  f_hi = min(f_hi, nfine);  // this launch builds fine bins [f_lo, f_hi)
  using K = typename H::Key;
  using PS = LocalPShape<K>;
  constexpr int NT = PS::kThreads;
  constexpr uint32_t VPL = PS::kVPL;
  constexpr int CPT = PS::kCPT;
  constexpr uint32_t kCap = PS::kCap;
  extern __shared__ __align__(128) unsigned char s_raw[];
  __shared__ alignas(8) uint64_t s_bar;
  const uint32_t S = 1u << s;
  uint32_t* c16 = reinterpret_cast<uint32_t*>(s_raw);                 // S/2 words of packed u16 counters
  K* raw = reinterpret_cast<K*>(s_raw + PS::c16_bytes(s));            // next bin's keys (TMA)
  K* staged = raw + PS::kElems;                                       // this bin's edges, chunk-aligned to global
  if (blockIdx.x == 0 && threadIdx.x == 0) offsets[v] = fine_start[nfine];
  // bins above kCap belong to k_big_count / k_big_place; the bucket counters
  // (the offsets slice) of those above kHugeBin are zeroed here
  auto next_small = [&](uint32_t f) -> uint32_t {
    uint32_t sz;
    while (f < f_hi && (sz = fine_start[f + 1] - fine_start[f]) > kCap) {
      if (sz > kHugeBin) {
        const uint64_t fb = (uint64_t)f << s;
        const uint32_t nbz = (uint32_t)min((uint64_t)S, v - fb);
        for (uint32_t l = threadIdx.x; l < nbz; l += NT) offsets[fb + l] = 0;
      }
      f += gridDim.x;
    }
    return f;
  };
  // bin f's keys [lo, hi) land at raw[lo - lo_al ...] with one bulk copy of
  // their 16-byte-aligned superset (the few keys of the neighbouring bins it
  // brings along are never read).  Only the array's last bin, whose superset
  // would run past the end, copies the aligned part and loads the < VPL keys
  // after it by threads 0..VPL-1.
  auto fetch = [&](uint32_t f) {
    if (threadIdx.x >= VPL) return;  // threads 0..VPL-1 only: short-lived registers
    const uint32_t lo = fine_start[f], hi = fine_start[f + 1];
    const uint32_t lo_al = lo & ~(VPL - 1), hi_up = (hi + VPL - 1) & ~(VPL - 1);
    const uint32_t hi_cp = hi_up <= fine_start[nfine] ? hi_up : hi & ~(VPL - 1);
    if (threadIdx.x == 0) {
      const uint32_t bytes = hi_cp > lo_al ? (hi_cp - lo_al) * (uint32_t)sizeof(K) : 0u;
      if (bytes) tma_load_1d(raw, src + lo_al, bytes, &s_bar);
      else mbar_arrive(&s_bar);
    }
    const uint32_t g = hi_cp + threadIdx.x;
    if (g >= lo && g < hi) raw[g - lo_al] = src[g];
  };
  uint32_t f = next_small(f_lo + blockIdx.x);
  if (threadIdx.x == 0) {
    mbar_init(&s_bar, 1);
    fence_proxy_async();
  }
  __syncthreads();
  if (f < f_hi) fetch(f);
  // tail keys written by threads 0..VPL-1 (only for the array's last bin) are
  // visible after this barrier; later fetches are ordered by a bin's barriers
  __syncthreads();
  uint32_t parity = 0;
  while (f < f_hi) {
    const uint32_t lo = fine_start[f], hi = fine_start[f + 1];
    const uint32_t cnt = hi - lo;
    const uint32_t lo_al = lo & ~(VPL - 1), sh = lo - lo_al;
    const uint32_t nch = (sh + cnt + VPL - 1) / VPL;
    const uint64_t first = (uint64_t)f << s;
    const uint32_t nb = (uint32_t)min((uint64_t)S, v - first);
    const uint32_t fn = next_small(f + gridDim.x);
    mbar_wait(&s_bar, parity);
    parity ^= 1;
    K kv[CPT * VPL];
    const uint4* raw4 = reinterpret_cast<const uint4*>(raw);
#pragma unroll
    for (int i = 0; i < CPT; i++) {
      const uint32_t c = i * NT + threadIdx.x;
      uint4 q = make_uint4(0, 0, 0, 0);
      if (c < nch) q = raw4[c];
      const K* qk = reinterpret_cast<const K*>(&q);
#pragma unroll
      for (int j = 0; j < (int)VPL; j++) kv[i * VPL + j] = qk[j];
    }
    for (uint32_t i = threadIdx.x; i < ((nb + 1) / 2 + 3) / 4; i += NT)  // 16-byte stores (c16 is 128-byte padded)
      reinterpret_cast<uint4*>(c16)[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();  // raw consumed, counters zero
    if (fn < f_hi) fetch(fn);
    // count: the atomic's old value is the key's rank inside its bucket.
    // Only the first and last chunk of a bin can be partial, so validity is
    // decided per chunk and full chunks run branch-free.  u32 keys keep only
    // the rank (packed u16, two per register) and re-hash the bucket at
    // placement: 20 keys per thread plus (bucket, rank) words spilled at 64
    // registers; u64 keys (10 per thread) keep (bucket << 16 | rank) -- their
    // re-hash (fmix64) costs more than it saves.
    constexpr bool kRehash = sizeof(K) == 4;
    constexpr int NK = CPT * (int)VPL;
    constexpr int NW = kRehash ? (NK + 1) / 2 : NK;  // rank words
    uint32_t rk[NW];
#pragma unroll
    for (int i = 0; i < NW; i++) rk[i] = 0;
    auto count_key = [&](K key, int k) {
      const uint32_t l = H::bucket(key, hp) - (uint32_t)first;
      const uint32_t sft = (l & 1) * 16;
      const uint32_t r = (atomicAdd(c16 + (l >> 1), 1u << sft) >> sft) & 0xFFFFu;
      if (kRehash) rk[k >> 1] |= r << ((k & 1) * 16);
      else rk[k] = (l << 16) | r;
    };
#pragma unroll
    for (int i = 0; i < CPT; i++) {
      const uint32_t c = i * NT + threadIdx.x;
      const uint32_t e0 = c * VPL;
      if (c < nch) {
        if (e0 >= sh && e0 + VPL <= sh + cnt) {
#pragma unroll
          for (int j = 0; j < (int)VPL; j++) count_key(kv[i * VPL + j], i * VPL + j);
        } else {
#pragma unroll
          for (int j = 0; j < (int)VPL; j++)
            if (e0 + j - sh < cnt) count_key(kv[i * VPL + j], i * VPL + j);
        }
      }
    }
    __syncthreads();
    scan_c16_offsets(c16, nb, lo, offsets + first);
    if (threadIdx.x == 0) tma_store_wait_read();  // the previous bin's edges have left staged
    __syncthreads();
    K* stg = staged + sh;
    auto place_key = [&](K key, int k) {
      uint32_t rel;
      if (kRehash) {
        const uint32_t l = H::bucket(key, hp) - (uint32_t)first;
        rel = get16(c16, l) + ((rk[k >> 1] >> ((k & 1) * 16)) & 0xFFFFu);
      } else {
        rel = get16(c16, rk[k] >> 16) + (rk[k] & 0xFFFFu);
      }
      stg[rel] = key;
      if (kTrace) {  // the slot replaces the rank: the positions pass needs no re-hash or counter load
        if (kRehash) {
          const int sft = (k & 1) * 16;
          rk[k >> 1] = (rk[k >> 1] & ~(0xFFFFu << sft)) | (rel << sft);
        } else {
          rk[k] = rel;
        }
      }
    };
#pragma unroll
    for (int i = 0; i < CPT; i++) {
      const uint32_t c = i * NT + threadIdx.x;
      const uint32_t e0 = c * VPL;
      if (c < nch) {
        if (e0 >= sh && e0 + VPL <= sh + cnt) {
#pragma unroll
          for (int j = 0; j < (int)VPL; j++) place_key(kv[i * VPL + j], i * VPL + j);
        } else {
#pragma unroll
          for (int j = 0; j < (int)VPL; j++)
            if (e0 + j - sh < cnt) place_key(kv[i * VPL + j], i * VPL + j);
        }
      }
    }
    fence_proxy_async();
    __syncthreads();
    // edges: aligned body by one bulk store, head and tail (< VPL each) by threads
    const uint32_t g0 = min(hi, (lo + VPL - 1) & ~(VPL - 1));
    const uint32_t g1 = max(g0, hi & ~(VPL - 1));
    if (threadIdx.x == 0 && g1 > g0) {
      tma_store_1d(edges + g0, staged + (g0 - lo_al), (g1 - g0) * (uint32_t)sizeof(K));
      tma_store_commit();
    }
    if (threadIdx.x < VPL) {
      const uint32_t gh = lo + threadIdx.x;
      if (gh < g0) edges[gh] = staged[gh - lo_al];
      const uint32_t gt = g1 + threadIdx.x;
      if (gt < hi) edges[gt] = staged[gt - lo_al];
    }
    if (kTrace) {
      // positions through the same staging buffer once the edges have left
      // it: slot rel of the bin gets a2[g] of the key placed there, then one
      // bulk store (u32 view, 16-byte congruent to positions + lo)
      if (threadIdx.x == 0) tma_store_wait_read();
      __syncthreads();
      uint32_t* st32 = reinterpret_cast<uint32_t*>(staged) + (lo & 3u);
      auto place_pos = [&](K key, int k, uint32_t a) {
        (void)key;
        const uint32_t rel = kRehash ? (rk[k >> 1] >> ((k & 1) * 16)) & 0xFFFFu : rk[k];  // slot from the edges pass
        st32[rel] = a;
      };
#pragma unroll
      for (int i = 0; i < CPT; i++) {
        const uint32_t c = i * NT + threadIdx.x;
        const uint32_t e0 = c * VPL;
        if (c < nch) {
          // the chunk's carried indices in one vector load (a2 is padded
          // past n, and lo_al + e0 is VPL-aligned)
          uint32_t av[VPL];
          if (VPL == 4) {
            const uint4 x = __ldcs(reinterpret_cast<const uint4*>(a2 + lo_al + e0));
            av[0] = x.x;
            av[1 % VPL] = x.y;
            av[2 % VPL] = x.z;
            av[3 % VPL] = x.w;
          } else {
            const uint2 x = __ldcs(reinterpret_cast<const uint2*>(a2 + lo_al + e0));
            av[0] = x.x;
            av[1 % VPL] = x.y;
          }
#pragma unroll
          for (int j = 0; j < (int)VPL; j++)
            if (e0 + j - sh < cnt) place_pos(kv[i * VPL + j], i * VPL + j, av[j]);
        }
      }
      fence_proxy_async();
      __syncthreads();
      const uint32_t p0 = min(hi, (lo + 3) & ~3u), p1 = max(p0, hi & ~3u);
      if (threadIdx.x == 0 && p1 > p0) {
        tma_store_1d(positions + p0, st32 + (p0 - lo), (p1 - p0) * 4u);
        tma_store_commit();
      }
      if (threadIdx.x < 4) {
        const uint32_t gh = lo + threadIdx.x;
        if (gh < p0) positions[gh] = st32[gh - lo];
        const uint32_t gt = p1 + threadIdx.x;
        if (gt < hi) positions[gt] = st32[gt - lo];
      }
    }
    f = fn;
  }
  if (threadIdx.x == 0) tma_store_wait_all();
}

// Fine bins above the smem capacity (high-duplicate inputs) are built by
// k_big_count / k_big_place (hg_bigbin.cuh).

// --------------------------------------------------------------------------- Q: probe

__device__ __forceinline__ void flush_agg(uint64_t matched, uint64_t total, uint64_t comps, unsigned long long* agg) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    matched += __shfl_xor_sync(0xffffffffu, matched, o);
    total += __shfl_xor_sync(0xffffffffu, total, o);
    comps += __shfl_xor_sync(0xffffffffu, comps, o);
  }
  if ((threadIdx.x & 31) == 0 && (matched | total | comps)) {
    atomicAdd(agg + 0, (unsigned long long)matched);
    atomicAdd(agg + 1, (unsigned long long)total);
    atomicAdd(agg + 2, (unsigned long long)comps);
  }
}

#ifndef HG_PROBE_QPT
#define HG_PROBE_QPT 4
#endif
#ifndef HG_PROBE_QPT64
#define HG_PROBE_QPT64 8
#endif
#ifndef HG_TAIL_UNROLL
#define HG_TAIL_UNROLL 4  // (experiment knob: unroll of the probe's linear tail)
#endif
constexpr int kTailUnroll = HG_TAIL_UNROLL;
#ifndef HG_PROBE_NOFULL
#define HG_PROBE_NOFULL 0  // experiment: one batch variant (bounds-checked) instead of two
#endif
// queries per thread per probe batch (the next batch is prefetched); 64-bit
// keys use fewer: their unrolled batch loop otherwise overflows the
// instruction cache and the register file
template <typename K>
struct ProbeQ {
  static constexpr int kQPT = sizeof(K) == 4 ? HG_PROBE_QPT : HG_PROBE_QPT64;
};

// Query slot k of a probe batch starting at q0 (a multiple of QVec<K>):
// 32-bit keys -- each thread owns groups of 4 consecutive queries, so a group
// loads with one 16-byte load and its counts leave with one 16-byte store;
// 64-bit keys -- one query per slot, strided by the CTA (2-key groups measured
// slower: their extra live registers spill).
template <typename K>
struct QVec {
  static constexpr int kV = sizeof(K) == 4 ? 4 : 1;
};
template <typename K>
__device__ __forceinline__ uint32_t qslot(uint32_t q0, int k) {
  constexpr int VPL = QVec<K>::kV;
  return q0 + (uint32_t)(k / VPL) * (VPL * kT) + VPL * threadIdx.x + (uint32_t)(k % VPL);
}

// The batch at q0 of the bin's queries [qlo, qhi) (slots outside read as 0).
template <typename K>
__device__ __forceinline__ void load_queries(const K* __restrict__ qpart, uint32_t q0, uint32_t qlo, uint32_t qhi,
                                             K (&qv)[ProbeQ<K>::kQPT]) {
  constexpr int QPT = ProbeQ<K>::kQPT;
  constexpr int VPL = QVec<K>::kV;
#pragma unroll
  for (int g = 0; g < QPT / VPL; g++) {
    const uint32_t j0 = qslot<K>(q0, g * VPL);
    if (VPL == 4 && j0 >= qlo && j0 + VPL <= qhi) {
      const uint4 x = __ldcs(reinterpret_cast<const uint4*>(qpart + j0));
      const K* xk = reinterpret_cast<const K*>(&x);
#pragma unroll
      for (int e = 0; e < VPL; e++) qv[g * VPL + e] = xk[e];
    } else if (VPL == 1) {  // (batches start at qlo)
      qv[g] = j0 < qhi ? __ldcs(qpart + j0) : K(0);
    } else {
#pragma unroll
      for (int e = 0; e < VPL; e++) qv[g * VPL + e] = (j0 + e >= qlo && j0 + e < qhi) ? __ldcs(qpart + j0 + e) : K(0);
    }
  }
}

// ---- small per-CTA map for deep buckets (high-duplicate inputs)
// Bucket depth classes of the shared-memory probe.  d <= 4: four branch-free
// slots; d <= kLinDeg: the slots plus a short warp-uniform linear tail;
// d <= kSortMax: the bucket is sorted in smem at staging and the count is
// upper_bound - lower_bound (O(log d) per query, like the reference's
// searchsorted, query.py:104-117); deeper: the per-bin key -> count map.
constexpr uint32_t kLinDeg = 16;
constexpr uint32_t kSortMax = 1024;
constexpr uint32_t kBigDeg = kSortMax;  // buckets deeper than this use the map
constexpr uint32_t kMapSlots = 256;     // open addressing, power of two
enum : uint32_t { kBinSort = 1, kBinMap = 2 };  // depth classes present in a bin

template <typename K>
struct BigMap {
  K key[kMapSlots];
  uint32_t cnt[kMapSlots];
  uint32_t state[kMapSlots];  // 0 empty, 1 claiming, 2 ready
  uint32_t full;
};

template <typename K>
__device__ __forceinline__ void map_clear(BigMap<K>& m) {
  for (uint32_t i = threadIdx.x; i < kMapSlots; i += blockDim.x) {
    m.state[i] = 0;
    m.cnt[i] = 0;
  }
  if (threadIdx.x == 0) m.full = 0;
}

template <typename K>
__device__ __forceinline__ uint32_t map_slot(K key) {
  return (uint32_t)(fmix64((uint64_t)key) & (kMapSlots - 1));
}

// Slot keys are written and read with atomics while the map is being built
// (the state word publishes them; racecheck-clean), plainly after the
// building barrier.
__device__ __forceinline__ void key_store(uint32_t* p, uint32_t k) { atomicExch(p, k); }
__device__ __forceinline__ void key_store(uint64_t* p, uint64_t k) {
  atomicExch(reinterpret_cast<unsigned long long*>(p), (unsigned long long)k);
}
__device__ __forceinline__ uint32_t key_load(uint32_t* p) { return atomicOr(p, 0u); }
__device__ __forceinline__ uint64_t key_load(uint64_t* p) {
  return atomicOr(reinterpret_cast<unsigned long long*>(p), 0ull);
}

// Add `add` occurrences of `key` (per lane; a slot is claimed with CAS and
// published once its key is written).
template <typename K>
__device__ __forceinline__ void map_add_n(BigMap<K>& m, K key, uint32_t add) {
  uint32_t i = map_slot(key);
  for (uint32_t probe = 0; probe < kMapSlots; probe++, i = (i + 1) & (kMapSlots - 1)) {
    uint32_t st = atomicCAS(&m.state[i], 0u, 1u);
    if (st == 0) {  // claimed an empty slot
      key_store(&m.key[i], key);
      __threadfence_block();
      atomicExch(&m.state[i], 2u);
      atomicAdd(&m.cnt[i], add);
      return;
    }
    while (st == 1) st = atomicAdd(&m.state[i], 0u);  // another thread is publishing this slot
    __threadfence_block();
    if (key_load(&m.key[i]) == key) {
      atomicAdd(&m.cnt[i], add);
      return;
    }
  }
  m.full = 1;
}

template <typename K>
__device__ __noinline__ uint32_t map_count(const BigMap<K>& m, K key) {
  uint32_t i = map_slot(key);
  for (uint32_t probe = 0; probe < kMapSlots; probe++, i = (i + 1) & (kMapSlots - 1)) {
    if (m.state[i] == 0) return 0;
    if (m.key[i] == key) return m.cnt[i];
  }
  return 0;
}

#include "hg_bigbin.cuh"

// The bin's queries against the staged slice, 16 per thread per batch (the
// loads were issued first), in phases so the hashes, offset loads and slot
// loads of all 16 queries overlap: (1) hash + both u16 offsets, packed; (2)
// IntersectArray count over the bucket.  Four slots run without a branch (the
// slice buffer is padded so te[a + 3] is always readable); queries are
// size-biased towards deep buckets (~9% see more than four keys at C = 1, i.e.
// almost every warp), so the rest runs as a warp-uniform loop to the warp's
// deepest bucket rather than a divergent per-lane loop.  Buckets deeper than
// kBigDeg are answered from the map (one warp-uniform check per batch).
// One batch (QPT queries per thread): kFull -- every query slot of the batch
// is valid, so no bounds checks; bin_flags -- which depth classes the bin has
// (known from staging): only then are queries checked for the sorted search
// or the map.
// Count of q in the sorted bucket te[a, a + d): lower and upper bound by
// binary search (two independent chains, floor(log2 d) + 1 steps).  Per lane
// and out of line, like map_count: only the few lanes whose bucket is in the
// sorted class pay for it, and the probe's unrolled batch loop stays small
// enough for the instruction cache.
template <typename K>
__device__ __noinline__ uint32_t sorted_count(const K* te, uint32_t a, uint32_t d, K q) {
  uint32_t lb = a, ln = d, ub = a, un = d;
  while (ln | un) {
    const uint32_t hl = ln >> 1, hu = un >> 1;
    const K xl = te[lb + hl], xu = te[ub + hu];
    if (ln) {
      if (xl < q) {
        lb += hl + 1;
        ln -= hl + 1;
      } else {
        ln = hl;
      }
    }
    if (un) {
      if (!(q < xu)) {
        ub += hu + 1;
        un -= hu + 1;
      } else {
        un = hu;
      }
    }
  }
  return ub - lb;
}

template <typename H, bool kFull>
__device__ __forceinline__ void probe_batch(uint32_t q0, uint32_t qlo, uint32_t qhi, const HashParams& hp, uint32_t first,
                                            const uint16_t* off16, const KeyOf<H>* te, const BigMap<KeyOf<H>>& map,
                                            bool overflow, uint32_t bin_flags, uint32_t* __restrict__ mult_bo,
                                            const KeyOf<H> (&qv)[ProbeQ<KeyOf<H>>::kQPT], uint32_t& m32, uint32_t& t32,
                                            uint32_t& d32) {
  using K = typename H::Key;
  constexpr int QPT = ProbeQ<K>::kQPT;
  constexpr int VPL = QVec<K>::kV;
  auto valid = [&](int k) {
    const uint32_t j = qslot<K>(q0, k);
    return kFull || ((VPL == 1 || j >= qlo) && j < qhi);  // (VPL == 1: batches start at qlo)
  };
  // query slots this batch can fill (whole groups of VPL)
  const uint32_t kmax = kFull ? (uint32_t)QPT : (qhi - q0 + VPL * kT - 1) / (VPL * kT) * VPL;
  uint32_t ae[QPT];
#pragma unroll
  for (int k = 0; k < QPT; k++) {
    ae[k] = 0;
    if (!kFull && (uint32_t)k >= kmax) continue;
    if (valid(k)) {
      const uint32_t l = H::bucket(qv[k], hp) - first;
      ae[k] = (uint32_t)off16[l] | ((uint32_t)off16[l + 1] << 16);
    }
  }
  bool deep = false;
  if (bin_flags & kBinMap) {
#pragma unroll
    for (int k = 0; k < QPT; k++) deep |= (ae[k] >> 16) - (ae[k] & 0xFFFFu) > kBigDeg;
  }
  const bool use_map = __any_sync(0xffffffffu, deep) && !overflow;
  // slots answered after the batch by the sorted search or the map (one call
  // site each, outside the unrolled loop: the loop stays small enough for the
  // instruction cache and no registers are saved around calls inside it)
  uint32_t rare = 0;
  constexpr bool kVecOut = sizeof(K) == 4;  // (64-bit keys: registers are short, counts stored one by one)
  uint32_t cv[kVecOut ? QPT : 1];
#pragma unroll
  for (int k = 0; k < QPT; k++) {
    if (!kFull && (uint32_t)k >= kmax) break;
    const K q = qv[k];
    const uint32_t a = ae[k] & 0xFFFFu, d = (ae[k] >> 16) - a;
    const bool mapped = use_map && d > kBigDeg;
    const bool srt = (bin_flags & kBinSort) && d > kLinDeg && d <= kSortMax;
    const K e0 = te[a], e1 = te[a + 1], e2 = te[a + 2], e3 = te[a + 3];
    uint32_t c = (uint32_t)((d > 0) & (e0 == q)) + (uint32_t)((d > 1) & (e1 == q)) +
                 (uint32_t)((d > 2) & (e2 == q)) + (uint32_t)((d > 3) & (e3 == q));
    const uint32_t dmax = __reduce_max_sync(0xffffffffu, mapped || srt ? 0u : d);
#pragma unroll kTailUnroll
    for (uint32_t t = 4; t < dmax; t++) {
      const bool in = t < d;
      const K x = in ? te[a + t] : K(0);
      c += (uint32_t)(in & (x == q));
    }
    if (kVecOut) cv[k % (kVecOut ? QPT : 1)] = c;
    if (valid(k)) {
      d32 += d;
      if (mapped || srt) {
        rare |= 1u << k;
      } else {
        if (!kVecOut) mult_bo[qslot<K>(q0, k)] = c;
        m32 += (c != 0);
        t32 += c;
      }
    }
  }
  if (!kVecOut) {
  } else if (kFull && rare == 0) {  // VPL consecutive counts per store
#pragma unroll
    for (int g = 0; g < QPT / VPL; g++) {
      uint32_t* p = mult_bo + qslot<K>(q0, g * VPL);
      *reinterpret_cast<uint4*>(p) = make_uint4(cv[(g * VPL) % QPT], cv[(g * VPL + 1) % QPT], cv[(g * VPL + 2) % QPT],
                                                cv[(g * VPL + 3) % QPT]);
    }
  } else {
#pragma unroll
    for (int k = 0; k < QPT; k++)
      if (valid(k) && !((rare >> k) & 1u)) mult_bo[qslot<K>(q0, k)] = cv[k % (kVecOut ? QPT : 1)];
  }
  while (rare) {
    const int k = __ffs(rare) - 1;
    rare &= rare - 1;
    K q = qv[0];
    uint32_t e = ae[0];
#pragma unroll
    for (int i = 1; i < QPT; i++)
      if (i == k) {
        q = qv[i];
        e = ae[i];
      }
    const uint32_t a = e & 0xFFFFu, d = (e >> 16) - a;
    const uint32_t c = d > kBigDeg ? map_count(map, q) : sorted_count<K>(te, a, d, q);
    mult_bo[qslot<K>(q0, k)] = c;
    m32 += (c != 0);
    t32 += c;
  }
}

template <typename H>
__device__ __forceinline__ void probe_queries_smem(const KeyOf<H>* __restrict__ qpart, uint32_t qlo, uint32_t qhi,
                                                   const HashParams& hp, uint32_t first, const uint16_t* off16,
                                                   const KeyOf<H>* te, const BigMap<KeyOf<H>>& map, bool overflow,
                                                   uint32_t bin_flags, uint32_t* __restrict__ mult_bo,
                                                   KeyOf<H> (&qv)[ProbeQ<KeyOf<H>>::kQPT], uint64_t& matched, uint64_t& total,
                                                   uint64_t& comps) {
  using K = typename H::Key;
  constexpr int QPT = ProbeQ<K>::kQPT;
  constexpr uint32_t B = QPT * kT;
  K qn[QPT];  // the next batch, in flight while this one is probed
  const uint32_t qa = qlo & ~((uint32_t)QVec<K>::kV - 1);  // batches start at a group boundary
  for (uint32_t q0 = qa; q0 < qhi; q0 += B) {
    if (q0 != qa) {
#pragma unroll
      for (int k = 0; k < QPT; k++) qv[k] = qn[k];  // (the first batch was loaded before staging)
    }
    if (q0 + B < qhi) load_queries<K>(qpart, q0 + B, qlo, qhi, qn);
    uint32_t m32 = 0, t32 = 0, d32 = 0;
    if (!HG_PROBE_NOFULL && q0 >= qlo && qhi - q0 >= B)
      probe_batch<H, true>(q0, qlo, qhi, hp, first, off16, te, map, overflow, bin_flags, mult_bo, qv, m32, t32, d32);
    else
      probe_batch<H, false>(q0, qlo, qhi, hp, first, off16, te, map, overflow, bin_flags, mult_bo, qv, m32, t32, d32);
    matched += m32;
    total += t32;
    comps += d32;
  }
}

// Sort one bucket of d keys (kLinDeg < d <= kSortMax) in smem, by one warp.
// d <= 32: a register bitonic network over shuffles (the all-ones sentinel
// pads to 32 and sorts last).  Larger: the bitonic network in place with the
// mirror form of each merge, so every comparator is ascending and the
// virtual +inf elements past d never move (pairs reaching past d are skipped).
template <typename K>
__device__ __forceinline__ void warp_sort_bucket(K* p, uint32_t d, int lane) {
  if (d <= 32) {
    K x = (uint32_t)lane < d ? p[lane] : ~K(0);
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
      for (int j = k >> 1; j > 0; j >>= 1) {
        const K y = __shfl_xor_sync(0xffffffffu, x, j);
        const bool up = (lane & k) == 0, lower = (lane & j) == 0;
        x = (lower == up) ? (y < x ? y : x) : (y < x ? x : y);
      }
    }
    if ((uint32_t)lane < d) p[lane] = x;
    __syncwarp();
    return;
  }
  const uint32_t P = 1u << (32 - __clz(d - 1));
  for (uint32_t k = 2; k <= P; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      const int lj = __ffs(j) - 1;
      for (uint32_t t = lane; t < P / 2; t += 32) {
        const uint32_t blk = t >> lj, x = t & (j - 1);
        uint32_t lo, hi;
        if (j == (k >> 1)) {
          lo = blk * k + x;
          hi = blk * k + k - 1 - x;
        } else {
          lo = blk * 2 * j + x;
          hi = lo + j;
        }
        if (hi < d) {
          const K u = p[lo], w = p[hi];
          if (w < u) {
            p[lo] = w;
            p[hi] = u;
          }
        }
      }
      __syncwarp();
    }
  }
}

// Shared-memory probe work item = (fine bin, chunk of <= kProbeChunk of its
// queries): CTA f takes bin f's first chunk, CTAs past nfine the further
// chunks of hot bins (k_probe_plan); bins whose table slice exceeds kCap take
// the hash-table path (hg_bigbin.cuh).  The table's CSR slice (uint16 local
// offsets + edges) is staged in smem; the queries probe it with
// IntersectArray semantics (count of equal keys in the bucket, PAPER.md:62-72;
// comparisons += bucket degree, query.py:153-155) and write counts in
// partitioned order.  Hot bins split into several items, so a skewed query
// set does not serialise on one SM.
template <typename H>
__global__ void __launch_bounds__(kT, 2)
k_local_probe(const uint32_t* __restrict__ t_off, const KeyOf<H>* __restrict__ t_edges, const KeyOf<H>* __restrict__ qpart,
              const uint32_t* __restrict__ q_start, uint32_t nfine, const uint32_t* __restrict__ item_x,
              unsigned long long* __restrict__ plan, uint32_t* __restrict__ big_bin, HashParams hp, int s, uint64_t v,
              uint32_t* __restrict__ mult_bo, unsigned long long* __restrict__ agg) {
  using K = typename H::Key;
  constexpr uint32_t VPL = 16 / sizeof(K);
  extern __shared__ __align__(128) unsigned char s_raw[];
  __shared__ alignas(8) uint64_t s_bar;
  __shared__ uint32_t s_flags;
  constexpr uint32_t kCap = LocalShape<K>::kCap;
  const uint32_t S = 1u << s;
  uint16_t* off16 = reinterpret_cast<uint16_t*>(s_raw);                        // S + 1 (+ pad to 8)
  K* tedges = reinterpret_cast<K*>(s_raw + ((2 * (S + 8) + 15) & ~15u));       // VPL + kCap + 8
  BigMap<K>& map = *reinterpret_cast<BigMap<K>*>(reinterpret_cast<unsigned char*>(tedges) + (kCap + 8) * sizeof(K));
  uint32_t f = blockIdx.x, c = 0;  // CTA f: the first chunk of bin f's queries
  if (f >= nfine) {                // further chunks of hot bins
    const uint32_t x = f - nfine;
    if (x >= plan[kPlanItems]) return;
    f = item_x[2 * x];
    c = item_x[2 * x + 1];
  }
  const uint32_t qlo = q_start[f] + c * kProbeChunk;
  uint32_t qhi = min(q_start[f + 1], qlo + kProbeChunk);
  if (qlo >= qhi) return;
  K qv[ProbeQ<K>::kQPT];
  load_queries<K>(qpart, qlo & ~((uint32_t)QVec<K>::kV - 1), qlo, qhi, qv);  // first batch in flight during staging
  const uint64_t first = (uint64_t)f << s;
  const uint32_t nb = (uint32_t)min((uint64_t)S, v - first);
  const uint32_t tlo = t_off[first], thi = t_off[first + nb];
  const uint32_t tn = thi - tlo;
  if (tn > kCap) {  // medium slice: key -> count map; else (or too many distinct keys) the hash-table path
    if (tn <= 4 * kCap && probe_slice_map<H>(t_edges, t_off, tlo, thi, qpart, qlo, qhi, hp, s_raw, mult_bo, agg)) return;
    if (tn <= 4 * kCap && c == 0 && threadIdx.x == 0) {  // k_probe_plan left it to the probe: hand it over
      big_bin[atomicAdd(plan + kPlanBig, 1ull)] = f;
      atomicAdd(plan + kPlanBigT, (unsigned long long)tn);
      atomicAdd(plan + kPlanBigQ, (unsigned long long)(q_start[f + 1] - q_start[f]));
    }
    return;
  }
  // edges: one TMA bulk copy of the 16-byte chunks from the boundary below
  // tlo (tedges[sh + j] = edge tlo + j) lands while the offsets convert
  const uint32_t a0 = tlo & ~(VPL - 1);
  const uint32_t sh = tlo - a0;
  const uint32_t ebytes = tn ? ((thi - a0) * (uint32_t)sizeof(K) + 15u) & ~15u : 0u;
  if (threadIdx.x == 0) {
    s_flags = 0;
    if (ebytes) {
      mbar_init(&s_bar, 1);
      fence_proxy_async();
      tma_load_1d(tedges, t_edges + a0, ebytes, &s_bar);
    }
  }
  map_clear(map);
  {
    // offsets: 4 per 16-byte load (first is a multiple of 2^s), stored as u16
    // relative to tlo, three loads in flight per thread; the bin's depth
    // classes (sorted / map) are flagged on the way
    const uint4* o4 = reinterpret_cast<const uint4*>(t_off + first);
    uint32_t flags = 0;
    constexpr int R = 3;
    for (uint32_t w0 = threadIdx.x; 4 * w0 <= nb; w0 += R * blockDim.x) {
      uint4 x[R];
      uint32_t nx[R];
#pragma unroll
      for (int r = 0; r < R; r++) {
        const uint32_t w = w0 + r * blockDim.x, i0 = 4 * w;
        x[r] = make_uint4(0, 0, 0, 0);
        nx[r] = 0;
        if (i0 + 4 <= nb) {
          x[r] = o4[w];
          nx[r] = t_off[first + i0 + 4];
        } else if (i0 <= nb) {
          uint32_t t[4] = {0, 0, 0, 0};
          for (uint32_t e = 0; i0 + e <= nb; e++) t[e] = t_off[first + i0 + e];
          x[r] = make_uint4(t[0], t[1], t[2], t[3]);
        }
      }
#pragma unroll
      for (int r = 0; r < R; r++) {
        const uint32_t w = w0 + r * blockDim.x, i0 = 4 * w;
        if (i0 > nb) break;
        // degrees of buckets i0..i0+3 (only those below nb exist)
        const uint32_t dg[4] = {i0 + 1 <= nb ? x[r].y - x[r].x : 0u, i0 + 2 <= nb ? x[r].z - x[r].y : 0u,
                                i0 + 3 <= nb ? x[r].w - x[r].z : 0u, i0 + 4 <= nb ? nx[r] - x[r].w : 0u};
#pragma unroll
        for (int e = 0; e < 4; e++) {
          flags |= dg[e] > kBigDeg ? (uint32_t)kBinMap : 0u;
          flags |= (dg[e] > kLinDeg && dg[e] <= kSortMax) ? (uint32_t)kBinSort : 0u;
        }
        const uint32_t lo2 = ((x[r].x - tlo) & 0xFFFFu) | ((x[r].y - tlo) << 16);
        const uint32_t hi2 = ((x[r].z - tlo) & 0xFFFFu) | ((x[r].w - tlo) << 16);
        reinterpret_cast<uint2*>(off16)[w] = make_uint2(lo2, hi2);
      }
    }
    __syncthreads();  // s_flags initialised
    flags = __reduce_or_sync(0xffffffffu, flags);
    if (flags && (threadIdx.x & 31) == 0) atomicOr(&s_flags, flags);
    if (threadIdx.x == 0 && ebytes) mbar_wait(&s_bar, 0);
  }
  __syncthreads();
  const uint32_t bin_flags = s_flags;
  K* te = tedges + sh;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (bin_flags & kBinSort) {
    // every warp scans its share of the buckets and sorts the ones in the
    // sorted class, one at a time (buckets are disjoint between warps)
    const uint32_t per = ((nb + nw - 1) / nw + 31) & ~31u;
    const uint32_t b1 = min(nb, (uint32_t)(warp + 1) * per);
    for (uint32_t b0 = warp * per; b0 < b1; b0 += 32) {
      const uint32_t l = b0 + lane;
      uint32_t a = 0, d = 0;
      if (l < b1) {
        a = off16[l];
        d = (uint32_t)off16[l + 1] - a;
      }
      uint32_t m = __ballot_sync(0xffffffffu, d > kLinDeg && d <= kSortMax);
      while (m) {
        const int src = __ffs(m) - 1;
        m &= m - 1;
        warp_sort_bucket<K>(te + __shfl_sync(0xffffffffu, a, src), __shfl_sync(0xffffffffu, d, src), lane);
      }
    }
    __syncthreads();
  }
  // Buckets deeper than kBigDeg (high-duplicate inputs) are answered from a
  // small smem map key -> occurrences, built once per bin, instead of an
  // O(degree) scan per query (the map was cleared before staging).
  if (bin_flags & kBinMap) {
    // All warps walk the slice's edges (warp w owns a contiguous range of
    // 32-edge rows; lane j sees every 32nd edge of it).  Each lane counts runs
    // of equal keys and adds a run to the map when its key changes, so a deep
    // bucket holding one repeated key costs a few map updates spread over the
    // whole CTA instead of one warp-serial update per 32 keys.
    const uint32_t rows = (tn + 31) / 32;
    const uint32_t per = (rows + nw - 1) / nw;
    const uint32_t r1 = min(rows, (uint32_t)(warp + 1) * per);
    K cur = K(0);
    uint32_t run = 0;
    bool cur_deep = false;
    for (uint32_t r = (uint32_t)warp * per; r < r1; r++) {
      const uint32_t t = r * 32 + lane;
      if (t >= tn) break;
      const K key = te[t];
      if (run == 0 || key != cur) {
        if (run && cur_deep) map_add_n(map, cur, run);
        cur = key;
        run = 0;
        const uint32_t l = H::bucket(key, hp) - (uint32_t)first;
        cur_deep = (uint32_t)off16[l + 1] - off16[l] > kBigDeg;
      }
      run++;
    }
    if (run && cur_deep) map_add_n(map, cur, run);
  }
  __syncthreads();
  const bool overflow = map.full != 0;
  uint64_t matched = 0, total = 0, comps = 0;
#if defined(HG_EXP_PROBE) && HG_EXP_PROBE == 3  // timing experiment (tools/build_variant.py): first batch only
  qhi = min(qhi, qlo + ProbeQ<K>::kQPT * kT);
#endif
  probe_queries_smem<H>(qpart, qlo, qhi, hp, (uint32_t)first, off16, te, map, overflow, bin_flags, mult_bo, qv, matched,
                        total, comps);
  if (agg) flush_agg(matched, total, comps, agg);
}

// --------------------------------------------------------------------------- host drivers

static size_t part_smem(int key_bits) {
  return key_bits == 32 ? sizeof(PartSmem<uint32_t>) : sizeof(PartSmem<uint64_t>);
}
static size_t probe_smem(int s, int key_bits) {
  return (size_t)((2 * ((1u << s) + 8) + 15) & ~15u) +
         (key_bits == 32 ? (LocalShape<uint32_t>::kCap + 8) * 4 + sizeof(BigMap<uint32_t>)
                         : (LocalShape<uint64_t>::kCap + 8) * 8 + sizeof(BigMap<uint64_t>));
}
static size_t unpart_smem() { return (2 * kUnpStaged + 2 * (kMaxBins + 1) + 2 * kMaxBins + kMaxBins + 1) * 4 + 16; }

// Hash-table slots the query reserves for oversized bins: a bin exceeds the
// smem capacity only if the table has more keys than that capacity; the
// device sizes the live table to >= 2x the keys of the bins that take it.
static uint64_t ht_slots(uint64_t n_table, int key_bits) {
  const uint64_t cap = key_bits == 32 ? LocalShape<uint32_t>::kCap : LocalShape<uint64_t>::kCap;
  if (n_table <= cap) return 0;
  uint64_t c = 1024;
  while (c < 2 * n_table) c <<= 1;
  return c;
}

struct PartOut {
  const void* grouped;  // keys grouped by fine bin at fine_start positions
  void* out1;           // level-1 buffer (n keys of workspace)
  uint32_t* big_cp;     // build: oversized-bin chunk prefix (nfine + 1)
  uint32_t* big_done;   // build: their chunk-completion counters (2 x nfine)
  uint32_t* plan32;     // query: the probe plan words (zeroed by k_starts)
  uint32_t* fine_cursor;
  uint32_t* M;
  uint32_t* fine_start;
  uint32_t* c_start;
  uint32_t* tp;
  uint32_t* big_list;
  uint32_t* big_count;
  uint16_t* pmap1;
  uint16_t* pmap2;
  uint32_t* meta1;
  uint32_t* meta2;
};

// Partition modes: kPartBuild (keys grouped straight into the table's edges,
// oversized-bin lists), kPartQuery (position maps + run metadata for the way
// back, the probe plan), kPartTraced (build_traced: both maps and lists; the
// grouped keys stay in workspace and the maps outlive the call as the trace).
enum PartMode { kPartBuild, kPartQuery, kPartTraced };

// Carve the partition's buffers out of the workspace (also used to re-derive
// a trace's pointers from its workspace: same order, same sizes).
template <typename K>
static void part_alloc(uint64_t n, const BinLayout& L, PartMode mode, K* final_out, Workspace& ws, PartOut* po,
                       uint32_t** fine_cnt, uint32_t** fine_cursor, K** out2) {
  const bool maps = mode != kPartBuild, lists = mode != kPartQuery;
  *fine_cnt = ws.take<uint32_t>(L.nfine + 1);
  po->fine_start = ws.take<uint32_t>(L.nfine + 1);
  *fine_cursor = ws.take<uint32_t>(L.nfine + 1);
  po->big_list = ws.take<uint32_t>(L.nfine + 1);
  po->c_start = ws.take<uint32_t>(L.nb1 + 1);
  po->tp = ws.take<uint32_t>(L.nb1 + 1);
  po->big_count = ws.take<uint32_t>(64);
  po->M = ws.take<uint32_t>((size_t)L.grid * L.nb1);
  po->big_cp = lists ? ws.take<uint32_t>(L.nfine + 1) : nullptr;
  po->big_done = lists ? ws.take<uint32_t>(2 * (size_t)L.nfine + 2) : nullptr;
  po->plan32 = mode == kPartQuery ? ws.take<uint32_t>(2 * kPlanWords) : nullptr;
  K* out1 = ws.take<K>(n + 16 / sizeof(K));  // + tail padding for k_part2's TMA
  po->out1 = out1;
  po->pmap1 = po->pmap2 = nullptr;
  po->meta1 = po->meta2 = nullptr;
  if (maps) {
    *out2 = L.two_level ? ws.take<K>(n) : nullptr;
    po->pmap1 = ws.take<uint16_t>(n);
    po->pmap2 = L.two_level ? ws.take<uint16_t>(n) : nullptr;
    po->meta1 = ws.take<uint32_t>(L.ntiles1 * (L.nb1 + 1));
    po->meta2 = L.two_level ? ws.take<uint32_t>(L.max_tiles2 * (2 * L.sub + 1)) : nullptr;
  } else {
    *out2 = final_out;
  }
  po->grouped = L.two_level ? (const void*)*out2 : (const void*)out1;
}

// The probe stage's buffers (queries grouped by fine bin -> counts in the
// same order), carved after the partition's.
struct ProbeBufs {
  uint32_t* mult_bo;   // counts in grouped order (+ tail padding for k_unpart's aligned run copies)
  uint32_t* item_x;    // extra probe work items (bin, chunk) of hot bins
  uint32_t* big_bin;   // hash-table bins, their table-key / query prefixes
  uint32_t* big_t;
  uint32_t* big_q;
  void* hk;            // hash table keys / counts (ht_slots(n_table))
  uint32_t* hc;
  uint32_t max_extra;
  uint64_t hs;
};

template <typename K>
static void probe_alloc(uint64_t q, const BinLayout& L, uint64_t n_table, Workspace& ws, ProbeBufs* pb) {
  pb->mult_bo = ws.take<uint32_t>(q + 4);
  pb->max_extra = (uint32_t)(q / kProbeChunk + 1);
  pb->item_x = ws.take<uint32_t>(2 * (size_t)pb->max_extra);
  pb->big_bin = ws.take<uint32_t>(L.nfine + 1);
  pb->big_t = ws.take<uint32_t>(L.nfine + 1);
  pb->big_q = ws.take<uint32_t>(L.nfine + 1);
  pb->hs = ht_slots(n_table, sizeof(K) * 8);
  pb->hk = ws.take<K>(pb->hs);
  pb->hc = ws.take<uint32_t>(pb->hs);
}

// Workspace of a binned pass, by a dry run of the same carve-up the pass
// performs (mode: kPartBuild / kPartQuery / kPartTraced; the query adds its
// probe buffers, the traced build the carried input indices).
template <typename K>
static size_t ws_dry_run(uint64_t n, const BinLayout& L, PartMode mode, uint64_t n_table) {
  Workspace w{nullptr, ~(size_t)0, 0};
  PartOut po{};
  uint32_t *fc, *fcur;
  K* out2;
  part_alloc<K>(n, L, mode, nullptr, w, &po, &fc, &fcur, &out2);
  if (mode == kPartQuery) {
    ProbeBufs pb;
    probe_alloc<K>(n, L, n_table, w, &pb);
  } else if (mode == kPartTraced) {
    w.take<uint32_t>(n + 4);  // carried input indices (a2)
  }
  return w.used + 4096;
}

size_t binned_ws_bytes(uint64_t n, const BinLayout& L, int key_bits, int mode, uint64_t n_table) {
  return key_bits == 32 ? ws_dry_run<uint32_t>(n, L, (PartMode)mode, n_table)
                        : ws_dry_run<uint64_t>(n, L, (PartMode)mode, n_table);
}

// Passes A + P1 (+ P2).  Build mode with two levels writes the fine-grouped
// keys into `final_out`; otherwise they stay in workspace buffers.
template <typename H>
static int run_partition(const KeyOf<H>* keys, uint64_t n, const HashParams& hp, const BinLayout& L, uint32_t cap,
                         PartMode mode, KeyOf<H>* final_out, Workspace& ws, cudaStream_t st, PartOut* po,
                         bool skip_part2 = false) {
  using K = KeyOf<H>;
  const bool query = mode != kPartBuild;  // position maps + metadata
  uint32_t *fine_cnt, *fine_cursor;
  K* out2;
  part_alloc<K>(n, L, mode, final_out, ws, po, &fine_cnt, &fine_cursor, &out2);
  K* out1 = (K*)po->out1;
  if (!ws.ok()) return set_error(HG_ERR_CONFIG, "binned workspace too small (%zu < %zu)", ws.cap, ws.used);
  HG_CHECK_CUDA(cudaMemsetAsync(fine_cnt, 0, 4 * (size_t)L.nfine, st));
  if (L.nfine <= kHistMax) {
    const size_t smA = (size_t)L.nfine * 4;
    HG_SET_SMEM((k_hist<H, false>), (int)smA);
    HG_LAUNCH("hg_hist", (k_hist<H, false>), L.grid, kT, smA, st, keys, n, hp, L.s, L.nfine, L.group, L.nb1, L.chunk,
              po->M, fine_cnt, 0u, L.nfine);
  } else {  // more fine bins than one smem histogram holds: one pass per range
    const size_t smA = (size_t)kHistMax * 4;
    HG_SET_SMEM((k_hist<H, true>), (int)smA);
    for (uint32_t f_lo = 0; f_lo < L.nfine; f_lo += kHistMax)
      HG_LAUNCH("hg_hist", (k_hist<H, true>), L.grid, kT, smA, st, keys, n, hp, L.s, L.nfine, L.group, L.nb1, L.chunk,
                po->M, fine_cnt, f_lo, std::min<uint32_t>(kHistMax, L.nfine - f_lo));
  }
  HG_LAUNCH("hg_colscan", k_colscan, L.nb1, (L.grid + 31) / 32 * 32 > 1024 ? 1024 : (L.grid + 31) / 32 * 32,
            (size_t)L.grid * 4, st, po->M, L.grid, L.nb1);
  const size_t smS = (size_t)std::min<uint32_t>(L.nfine, kStartsChunk) * 4;
  HG_SET_SMEM((k_starts), (int)smS);
  HG_LAUNCH("hg_starts", k_starts, 1, 1024, smS, st, fine_cnt, L.nfine, L.group, L.nb1, L.tile, cap, po->fine_start,
            po->c_start, po->tp, fine_cursor, po->big_list, po->big_count, (uint32_t)BigShape<K>::kChunk, po->big_cp,
            po->big_done, po->plan32, po->plan32 ? (uint32_t)(2 * kPlanWords) : 0u);
  const size_t smP = part_smem(sizeof(K) * 8);
  if (query) {
    HG_SET_SMEM((k_part1<H, true>), (int)smP);
    HG_LAUNCH("hg_part1_q", (k_part1<H, true>), L.grid, kT, smP, st, keys, n, hp, L.shift1, L.bits1, L.nb1, L.chunk,
              po->M, po->c_start, out1, po->pmap1, po->meta1);
  } else {
    HG_SET_SMEM((k_part1<H, false>), (int)smP);
    HG_LAUNCH("hg_part1", (k_part1<H, false>), L.grid, kT, smP, st, keys, n, hp, L.shift1, L.bits1, L.nb1, L.chunk,
              po->M, po->c_start, out1, nullptr, nullptr);
  }
  po->fine_cursor = fine_cursor;
  if (L.two_level && !skip_part2) {
    auto part2 = [&](auto kern, const char* name, uint16_t* pm, uint32_t* mt) -> int {
      HG_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smP));  // (kern is a runtime pointer: no per-site cache)
      HG_LAUNCH(name, kern, L.grid, kT, smP, st, out1, hp, L.s, L.nb1, po->c_start, po->tp, fine_cursor, out2, pm, mt,
                0u, 0xFFFFFFFFu);
      return HG_OK;
    };
    int rc2;
    if (query)
      rc2 = L.sub == kSub ? part2(k_part2<H, true, kSub>, "hg_part2_q", po->pmap2, po->meta2)
                          : part2(k_part2<H, true, kSubMax>, "hg_part2_q", po->pmap2, po->meta2);
    else
      rc2 = L.sub == kSub ? part2(k_part2<H, false, kSub>, "hg_part2", nullptr, nullptr)
                          : part2(k_part2<H, false, kSubMax>, "hg_part2", nullptr, nullptr);
    if (rc2) return rc2;
  }
  return HG_OK;
}

// positions != nullptr: build_traced -- the partition also records its
// position maps (kPartTraced), k_repart carries every key's input index to
// the grouped order, and the local build writes positions[p].
// The workspace then holds the trace hg_intersect_tables reuses.
template <typename H>
static int build_impl(const KeyOf<H>* keys, uint64_t n, const HashParams& hp, uint64_t v, const BinLayout& L, uint32_t* offsets,
                      KeyOf<H>* edges, Workspace& ws, cudaStream_t st, uint32_t* positions = nullptr) {
  using K = KeyOf<H>;
  const bool traced = positions != nullptr;
  // experiment (HG_GROUPED=G): level-2 partition and local build alternate
  // over groups of G level-1 bins, so the local build reads its bins while
  // they are still in L2
  static const int groups = getenv("HG_GROUPED") ? atoi(getenv("HG_GROUPED")) : 0;
  const bool grouped_sched = groups > 0 && !traced && L.two_level;
  PartOut po{};
  int rc = run_partition<H>(keys, n, hp, L, BuildShape<K>::kCap, traced ? kPartTraced : kPartBuild, edges, ws, st, &po,
                            grouped_sched);
  if (rc) return rc;
  if (grouped_sched) {
    const size_t smP = part_smem(sizeof(K) * 8), smC = LocalPShape<K>::smem(L.s);
    HG_SET_SMEM((k_local_build_p<H>), (int)smC);
    auto kp2 = L.sub == kSub ? k_part2<H, false, kSub> : k_part2<H, false, kSubMax>;
    HG_CHECK_CUDA(cudaFuncSetAttribute(kp2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smP));
    for (uint32_t c0 = 0; c0 < L.nb1; c0 += groups) {
      const uint32_t c1 = std::min<uint32_t>(L.nb1, c0 + groups);
      HG_LAUNCH("hg_part2", kp2, L.grid, kT, smP, st, (const K*)po.out1, hp, L.s, L.nb1, po.c_start, po.tp,
                po.fine_cursor, edges, nullptr, nullptr, c0, c1);
      HG_LAUNCH("hg_local_build", k_local_build_p<H>, num_sms(), LocalPShape<K>::kThreads, smC, st, (const K*)edges,
                po.fine_start, L.nfine, hp, L.s, v, offsets, edges, nullptr, nullptr, c0 * L.sub, c1 * L.sub);
    }
  }
  uint32_t* a2 = nullptr;
  if (traced) {
    a2 = ws.take<uint32_t>(n + 4);
    if (!ws.ok()) return set_error(HG_ERR_CONFIG, "binned workspace too small for a traced build");
    const size_t smR = (size_t)kUnpStaged * 4;
    HG_SET_SMEM((k_repart<1>), (int)smR);
    uint32_t* a1 = L.two_level ? reinterpret_cast<uint32_t*>(po.out1) : a2;  // level-1 keys are dead after part2
    HG_LAUNCH("hg_repart1", k_repart<1>, L.grid, kT, smR, st, nullptr, a1, po.pmap1, po.meta1, L.sub, L.nb1, L.tile, n,
              L.chunk, po.M, po.c_start, po.tp);
    if (L.two_level) {
      HG_SET_SMEM((k_repart<2>), (int)smR);
      HG_LAUNCH("hg_repart2", k_repart<2>, L.grid, kT, smR, st, a1, a2, po.pmap2, po.meta2, L.sub, L.nb1, L.tile, n,
                L.chunk, po.M, po.c_start, po.tp);
    }
  }
  const K* grouped = (const K*)po.grouped;  // build: == edges (two levels) or the level-1 buffer; traced: workspace
  const size_t smC = LocalPShape<K>::smem(L.s);
  if (traced) {
    HG_SET_SMEM((k_local_build_p<H, true>), (int)smC);
    HG_LAUNCH("hg_local_build_traced", (k_local_build_p<H, true>), num_sms(), LocalPShape<K>::kThreads, smC, st, grouped,
              po.fine_start, L.nfine, hp, L.s, v, offsets, edges, a2, positions);
  } else if (!grouped_sched) {
    HG_SET_SMEM((k_local_build_p<H>), (int)smC);
    HG_LAUNCH("hg_local_build", k_local_build_p<H>, num_sms(), LocalPShape<K>::kThreads, smC, st, grouped, po.fine_start,
              L.nfine, hp, L.s, v, offsets, edges, nullptr, nullptr);
  }
  // oversized fine bins (hg_bigbin.cuh), in chunks over the whole grid: with
  // two levels (untraced) their keys sit in edges (in place), so the count
  // pass copies them to the free level-1 buffer and placement reads them
  // from there
  const int copy = (L.two_level && !traced) ? 1 : 0;
  K* src = copy ? (K*)po.out1 : (K*)grouped;
  const size_t smBig = (size_t)(1u << L.s) * 4;
  HG_SET_SMEM((k_big_count<H>), (int)smBig);
  const uint32_t* huge_list = po.big_list + L.nfine - 1;  // grows downwards (k_starts)
  HG_LAUNCH("hg_big_count", k_big_count<H>, num_sms(), 1024, smBig, st, grouped, (K*)po.out1, copy, po.fine_start,
            po.big_list, huge_list, po.big_count, po.big_cp, po.big_done, hp, L.s, v, offsets, edges, a2, positions);
  HG_SET_SMEM((k_big_place<H>), (int)smBig);
  HG_LAUNCH("hg_big_place", k_big_place<H>, num_sms(), 1024, smBig, st, (const K*)src, po.fine_start, huge_list,
            po.big_count, po.big_cp, po.big_done + L.nfine + 1, hp, L.s, v, offsets, edges, a2, positions);
  return HG_OK;
}

// The probe of queries already grouped by fine bin (q_start: F + 1 bin
// starts): shared-memory probe items, then the hash-table path.  `plan`
// (kPlanWords) must be zero.  Counts land in pb.mult_bo in grouped order.
template <typename H>
static int probe_stage(const uint32_t* t_off, const KeyOf<H>* t_edges, const KeyOf<H>* qpart, const uint32_t* q_start,
                       uint64_t q, const HashParams& hp, uint64_t v, const BinLayout& L, unsigned long long* plan,
                       ProbeBufs& pb, uint64_t* agg, cudaStream_t st) {
  using K = KeyOf<H>;
  (void)q;
  HG_LAUNCH("hg_probe_plan", k_probe_plan, (L.nfine + 255) / 256, 256, 0, st, t_off, q_start, L.nfine, L.s, v,
            LocalShape<K>::kCap, pb.item_x, pb.big_bin, plan);
  const size_t smQ = probe_smem(L.s, sizeof(K) * 8);
  HG_SET_SMEM((k_local_probe<H>), (int)smQ);
  HG_LAUNCH("hg_local_probe", k_local_probe<H>, L.nfine + pb.max_extra, kT, smQ, st, t_off, t_edges, qpart, q_start,
            L.nfine, pb.item_x, plan, pb.big_bin, hp, L.s, v, pb.mult_bo, reinterpret_cast<unsigned long long*>(agg));
  if (pb.hs) {  // oversized table slices: key -> count hash table over the whole grid
    K* hk = (K*)pb.hk;
    HG_LAUNCH("hg_ht_prep", k_ht_prep<K>, num_sms() * 4, 256, 0, st, plan, pb.big_bin, t_off, q_start, L.s, v, pb.big_t,
              pb.big_q, hk, pb.hc);
    HG_LAUNCH("hg_ht_insert", k_ht_insert<H>, num_sms() * 2, kHtT, 0, st, t_off, t_edges, L.s, v, pb.big_bin, pb.big_t,
              plan, hk, pb.hc);
    HG_LAUNCH("hg_ht_lookup", k_ht_lookup<H>, num_sms() * 2, kHtT, 0, st, qpart, q_start, t_off, hp, L.s, v, pb.big_bin,
              pb.big_q, plan, hk, pb.hc, pb.mult_bo, reinterpret_cast<unsigned long long*>(agg));
  }
  return HG_OK;
}

template <typename H>
static int query_impl(const uint32_t* t_off, const KeyOf<H>* t_edges, uint64_t n_table, const KeyOf<H>* queries, uint64_t q,
                      const HashParams& hp, uint64_t v, const BinLayout& L, uint32_t* mult, uint64_t* agg, Workspace& ws,
                      cudaStream_t st, cudaEvent_t split) {
  using K = KeyOf<H>;
  PartOut po{};
  int rc = run_partition<H>(queries, q, hp, L, 0xFFFFFFFFu, kPartQuery, nullptr, ws, st, &po);
  if (rc) return rc;
  if (split) HG_CHECK_CUDA(cudaEventRecord(split, st));  // query-side grouping done (intersect_timed's split)
  ProbeBufs pb;
  probe_alloc<K>(q, L, n_table, ws, &pb);
  if (!ws.ok()) return set_error(HG_ERR_CONFIG, "binned workspace too small");
  rc = probe_stage<H>(t_off, t_edges, (const K*)po.grouped, po.fine_start, q, hp, v, L, reinterpret_cast<unsigned long long*>(po.plan32), pb,
                      agg, st);
  if (rc) return rc;
  uint32_t* mult_bo = pb.mult_bo;
  const size_t smR = unpart_smem();
  uint32_t* level1_vals = reinterpret_cast<uint32_t*>(po.out1);  // level-1 keys are dead by now
  if (L.two_level) {
    HG_SET_SMEM((k_unpart<2>), (int)smR);
    HG_LAUNCH("hg_unpart2", k_unpart<2>, L.grid, kT, smR, st, mult_bo, level1_vals, po.pmap2, po.meta2, L.sub, L.nb1, L.tile,
              q, L.chunk, po.M, po.c_start, po.tp);
  } else {
    level1_vals = mult_bo;
  }
  HG_SET_SMEM((k_unpart<1>), (int)smR);
  HG_LAUNCH("hg_unpart1", k_unpart<1>, L.grid, kT, smR, st, level1_vals, mult, po.pmap1, po.meta1, L.sub, L.nb1, L.tile, q,
            L.chunk, po.M, po.c_start, po.tp);
  return HG_OK;
}

// --------------------------------------------------------------------------- two-step query (query.py:84-179)

__global__ void k_qstart(const uint32_t* __restrict__ q_off, uint32_t nfine, int s, uint64_t v, uint32_t* __restrict__ q_start) {
  const uint32_t f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f <= nfine) q_start[f] = q_off[min((uint64_t)f << s, v)];
}

// Probe-layout bin starts from a trace grouped at a finer or equal layout
// (fine bins nest: bin f of shift s_p is bins [f << d, (f + 1) << d) of shift
// s_p - d, in the same ascending order).
__global__ void k_qstart_nested(const uint32_t* __restrict__ fs, uint32_t nfine_t, uint32_t nfine_p, int d,
                                uint32_t* __restrict__ q_start) {
  const uint32_t f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f <= nfine_p) q_start[f] = fs[min((uint64_t)f << d, (uint64_t)nfine_t)];
}

__global__ void k_scatter_pos(const uint32_t* __restrict__ src, const uint32_t* __restrict__ pos, uint64_t n,
                              uint32_t* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[__ldcs(pos + i)] = __ldcs(src + i);
}

// intersect_tables (query.py:120-179) over a query table that is already
// grouped by bucket, so no partition runs.  With the trace of the hg_build
// that produced the query table with positions, the probe reads the trace's
// grouped query keys -- exactly what hg_query's partition leaves (grouped by
// fine bin, in the order the position maps undo) -- and the counts go back to
// query order through the maps (k_unpart x 2), as in the fused query: at the
// table's probe layout when the trace's fine bins nest in it, else at the
// trace's own coarser layout (slices above the smem capacity take the map /
// hash-table paths).  Without a trace (foreign positions) the query table's
// fine-bin slices are probed and the counts scatter through positions.
template <typename H>
static int tables_impl(const uint32_t* t_off, const KeyOf<H>* t_edges, uint64_t n_table, const uint32_t* q_off,
                       const KeyOf<H>* q_edges, const uint32_t* positions, uint64_t q, const HashParams& hp, uint64_t v,
                       const BinLayout& Lp, const BinLayout* Lt, void* trace, size_t trace_bytes, uint32_t* mult,
                       uint64_t* agg, Workspace& ws, cudaStream_t st) {
  using K = KeyOf<H>;
  uint32_t* q_start = ws.take<uint32_t>(Lp.nfine + 1);
  unsigned long long* plan = ws.take<unsigned long long>(kPlanWords);
  ProbeBufs pb;
  probe_alloc<K>(q, Lp, n_table, ws, &pb);  // (a coarser trace layout has fewer fine bins: these fit it too)
  uint32_t* level1 = ws.take<uint32_t>(q + 4);
  if (!ws.ok()) return set_error(HG_ERR_CONFIG, "intersect_tables workspace too small (%zu < %zu)", ws.cap, ws.used);
  HG_CHECK_CUDA(cudaMemsetAsync(plan, 0, kPlanWords * 8, st));
  if (!trace) {
    HG_LAUNCH("hg_qstart", k_qstart, (Lp.nfine + 256) / 256, 256, 0, st, q_off, Lp.nfine, Lp.s, v, q_start);
    int rc = probe_stage<H>(t_off, t_edges, q_edges, q_start, q, hp, v, Lp, plan, pb, agg, st);
    if (rc) return rc;
    HG_LAUNCH("hg_scatter_pos", k_scatter_pos, num_sms() * 8, 256, 0, st, pb.mult_bo, positions, q, mult);
    return HG_OK;
  }
  // re-derive the trace's buffers: the same carve-up as the traced build
  PartOut tpo{};
  {
    Workspace tw{(char*)trace, trace_bytes, 0};
    uint32_t *fc, *fcur;
    K* out2;
    part_alloc<K>(q, *Lt, kPartTraced, nullptr, tw, &tpo, &fc, &fcur, &out2);
    tw.take<uint32_t>(q + 4);  // a2
    if (!tw.ok()) return set_error(HG_ERR_CONFIG, "trace buffer too small (%zu < %zu)", tw.cap, tw.used);
  }
  const BinLayout& L = *Lt;
  int rc;
  if (L.s <= Lp.s) {
    HG_LAUNCH("hg_qstart", k_qstart_nested, (Lp.nfine + 256) / 256, 256, 0, st, tpo.fine_start, L.nfine, Lp.nfine,
              Lp.s - L.s, q_start);
    rc = probe_stage<H>(t_off, t_edges, (const K*)tpo.grouped, q_start, q, hp, v, Lp, plan, pb, agg, st);
  } else {
    rc = probe_stage<H>(t_off, t_edges, (const K*)tpo.grouped, tpo.fine_start, q, hp, v, L, plan, pb, agg, st);
  }
  if (rc) return rc;
  uint32_t* vals = pb.mult_bo;  // counts in grouped order
  const size_t smR = unpart_smem();
  uint32_t* l1 = vals;
  if (L.two_level) {
    HG_SET_SMEM((k_unpart<2>), (int)smR);
    HG_LAUNCH("hg_unpart2", k_unpart<2>, L.grid, kT, smR, st, vals, level1, tpo.pmap2, tpo.meta2, L.sub, L.nb1, L.tile, q,
              L.chunk, tpo.M, tpo.c_start, tpo.tp);
    l1 = level1;
  }
  HG_SET_SMEM((k_unpart<1>), (int)smR);
  HG_LAUNCH("hg_unpart1", k_unpart<1>, L.grid, kT, smR, st, l1, mult, tpo.pmap1, tpo.meta1, L.sub, L.nb1, L.tile, q, L.chunk,
            tpo.M, tpo.c_start, tpo.tp);
  return HG_OK;
}

size_t binned_tables_ws_bytes(uint64_t q, const BinLayout& Lp, int key_bits, uint64_t n_table) {
  Workspace w{nullptr, ~(size_t)0, 0};
  w.take<uint32_t>(Lp.nfine + 1);
  w.take<unsigned long long>(kPlanWords);
  ProbeBufs pb;
  if (key_bits == 32) probe_alloc<uint32_t>(q, Lp, n_table, w, &pb);
  else probe_alloc<uint64_t>(q, Lp, n_table, w, &pb);
  w.take<uint32_t>(q + 4);
  return w.used + 4096;
}

// Host dispatch to the compile-time hasher (reduction mode x hash kind).
template <typename K, int KIND, typename F>
static int with_mode(const HashParams& hp, F&& f) {
  switch (hp.mode) {
    case kMask:
      return f(Hasher<K, kMask, KIND>{});
    case kNone:
      if constexpr (sizeof(K) == 4) return f(Hasher<K, kNone, KIND>{});
      [[fallthrough]];
    case kFastmod:
      if constexpr (sizeof(K) == 4) return f(Hasher<K, kFastmod, KIND>{});
      [[fallthrough]];
    default:
      return f(Hasher<K, kGeneric64, KIND>{});
  }
}

template <typename K, typename F>
static int with_hasher(const HashParams& hp, F&& f) {
  if (hp.kind == HG_KIND_IDENTITY) return with_mode<K, HG_KIND_IDENTITY>(hp, f);
  return with_mode<K, HG_KIND_MURMUR32>(hp, f);
}

template <typename K>
int binned_build(const K* keys, uint64_t n, const HashParams& hp, uint64_t v, const BinLayout& L, uint32_t* offsets,
                 K* edges, Workspace& ws, cudaStream_t st, uint32_t* positions) {
  return with_hasher<K>(hp, [&](auto h) {
    return build_impl<decltype(h)>(keys, n, hp, v, L, offsets, edges, ws, st, positions);
  });
}

template <typename K>
int binned_tables(const uint32_t* t_off, const K* t_edges, uint64_t n_table, const uint32_t* q_off, const K* q_edges,
                  const uint32_t* positions, uint64_t q, const HashParams& hp, uint64_t v, const BinLayout& Lp,
                  const BinLayout* Lt, void* trace, size_t trace_bytes, uint32_t* mult, uint64_t* agg, Workspace& ws,
                  cudaStream_t st) {
  return with_hasher<K>(hp, [&](auto h) {
    return tables_impl<decltype(h)>(t_off, t_edges, n_table, q_off, q_edges, positions, q, hp, v, Lp, Lt, trace,
                                    trace_bytes, mult, agg, ws, st);
  });
}

template <typename K>
int binned_query(const uint32_t* t_off, const K* t_edges, uint64_t n_table, const K* queries, uint64_t q,
                 const HashParams& hp, uint64_t v, const BinLayout& L, uint32_t* mult, uint64_t* agg, Workspace& ws,
                 cudaStream_t st, cudaEvent_t split) {
  return with_hasher<K>(hp, [&](auto h) {
    return query_impl<decltype(h)>(t_off, t_edges, n_table, queries, q, hp, v, L, mult, agg, ws, st, split);
  });
}

template int binned_build<uint32_t>(const uint32_t*, uint64_t, const HashParams&, uint64_t, const BinLayout&,
                                    uint32_t*, uint32_t*, Workspace&, cudaStream_t, uint32_t*);
template int binned_build<uint64_t>(const uint64_t*, uint64_t, const HashParams&, uint64_t, const BinLayout&,
                                    uint32_t*, uint64_t*, Workspace&, cudaStream_t, uint32_t*);
template int binned_tables<uint32_t>(const uint32_t*, const uint32_t*, uint64_t, const uint32_t*, const uint32_t*,
                                     const uint32_t*, uint64_t, const HashParams&, uint64_t, const BinLayout&,
                                     const BinLayout*, void*, size_t, uint32_t*, uint64_t*, Workspace&, cudaStream_t);
template int binned_tables<uint64_t>(const uint32_t*, const uint64_t*, uint64_t, const uint32_t*, const uint64_t*,
                                     const uint32_t*, uint64_t, const HashParams&, uint64_t, const BinLayout&,
                                     const BinLayout*, void*, size_t, uint32_t*, uint64_t*, Workspace&, cudaStream_t);
template int binned_query<uint32_t>(const uint32_t*, const uint32_t*, uint64_t, const uint32_t*, uint64_t,
                                    const HashParams&, uint64_t, const BinLayout&, uint32_t*, uint64_t*, Workspace&,
                                    cudaStream_t, cudaEvent_t);
template int binned_query<uint64_t>(const uint32_t*, const uint64_t*, uint64_t, const uint64_t*, uint64_t,
                                    const HashParams&, uint64_t, const BinLayout&, uint32_t*, uint64_t*, Workspace&,
                                    cudaStream_t, cudaEvent_t);

}  // namespace hg
