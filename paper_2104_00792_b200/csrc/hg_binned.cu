// hg_binned.cu -- the v2 "binned" HashGraph build and query (sm_100a).
//
// Green's cache-blocked HashGraph build ("first assigns each
// hash value to one of B_L bins ... B_L is small enough to fit in the cache")
// mapped onto B200 shared memory.  The hash range [0, V) is cut into bins of
// S = 2^s consecutive buckets, sized so one bin's keys plus its S counters fit
// in one CTA's shared memory (<= 227 KB).  Every global-memory access is then
// a coalesced stream; all random accesses (counting, ranking, placing) hit
// shared memory.
//
//   pass A  k_bin_count      per-CTA bin histogram of a contiguous input chunk
//   pass A' k_bin_colscan    per-(CTA, bin) exclusive prefix down each column
//           k_bin_starts     bin start offsets + list of oversized bins
//   pass B  k_partition      tile-by-tile partition by bin, staged in smem so
//                            each bin's run is written contiguously; cursors
//                            persist per CTA (no global atomics); optional
//                            slot map (input index -> partitioned slot)
//   pass C  k_local_build    one CTA per bin: count (packed u16 smem atomics),
//                            scan, place in smem, write offsets+edges coalesced
//           k_local_probe    one CTA per bin: table bin CSR staged in smem,
//                            the bin's queries probe it (IntersectArray)
//   pass D  k_unpartition    per-query values back to input order (replays pass B's
//                            tiles, stages each tile's bin runs in smem)
//   slow    k_local_build_big / k_local_probe_big for bins above smem capacity
//
// The result equals Alg. 1's: offsets exact, each bucket
// the same multiset (core.py:12-14 leaves the in-bucket order unspecified).
#include "hg_common.cuh"

namespace hg {

constexpr int kBT = 1024;                 // threads per CTA in the binned kernels
constexpr int kMaxBinsLog = 13;           // bins per pass B (smem cursors)
constexpr int kSLog = 15;                 // max buckets per bin
constexpr uint32_t kProbeCap = 38 * 1024; // table keys per bin handled in smem (pass C probe)

struct BinLayout {
  int s;           // log2 buckets per bin
  uint32_t nbins;  // ceil(v / 2^s)
  uint32_t tile;   // pass B tile (keys)
  uint32_t grid;   // CTAs of pass A / B (one chunk each)
  uint64_t chunk;  // keys per chunk (multiple of tile)
};

// Choose s so a bin holds ~2^15 keys: S * n / v ~= 32768.
static int pick_s(uint64_t n, uint64_t v) {
  double per_bucket = v ? (double)n / (double)v : 1.0;
  int s = kSLog;
  while (s > 8 && per_bucket * (double)(1ull << s) > 36000.0) s--;
  return s;
}

// n_table sizes the bins (a bin's table keys must fit shared memory); n_items
// (keys being partitioned) sizes the per-CTA chunks.
bool binned_layout(uint64_t n_table, uint64_t n, uint64_t v, int key_bits, BinLayout* L) {
  if (v > (1ull << 32)) return false;
  int s = pick_s(n_table, v);
  uint64_t nb = (v + (1ull << s) - 1) >> s;
  if (nb > (1ull << kMaxBinsLog)) return false;
  L->s = s;
  L->nbins = (uint32_t)nb;
  L->tile = key_bits == 32 ? 32768u : 16384u;  // == TileShape<K>::kTile
  L->grid = (uint32_t)num_sms();
  uint64_t per = (n + L->grid - 1) / L->grid;
  L->chunk = (per + L->tile - 1) / L->tile * L->tile;
  if (L->chunk == 0) L->chunk = L->tile;
  return true;
}

template <typename K>
__device__ __forceinline__ uint32_t bin_of(K key, const HashParams& hp, int s) {
  return bucket_of(key, hp) >> s;
}

// In-place exclusive scan of n (<= 16 * blockDim) uint32 values in smem.
// Returns the total to every thread.  Caller syncs before (data ready).
__device__ uint32_t block_exscan(uint32_t* a, uint32_t n) {
  __shared__ uint32_t s_w[32];
  const uint32_t per = (n + blockDim.x - 1) / blockDim.x;
  const uint32_t lo = threadIdx.x * per;
  const uint32_t hi = min(lo + per, n);
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

// Same for n packed uint16 counters stored two per word (word i holds values
// 2i (low half) and 2i+1 (high half)); totals must stay below 65536.
__device__ uint32_t block_exscan_u16(uint32_t* w16, uint32_t nvals) {
  __shared__ uint32_t s_w[32];
  const uint32_t nwords = (nvals + 1) / 2;
  const uint32_t per = (nwords + blockDim.x - 1) / blockDim.x;
  const uint32_t lo = threadIdx.x * per;
  const uint32_t hi = min(lo + per, nwords);
  uint32_t sum = 0;
  for (uint32_t i = lo; i < hi; i++) {
    uint32_t x = w16[i];
    sum += (x & 0xFFFFu) + (x >> 16);
  }
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
    uint32_t x = w16[i];
    uint32_t a = run, b = run + (x & 0xFFFFu);
    w16[i] = (a & 0xFFFFu) | (b << 16);
    run = b + (x >> 16);
  }
  __syncthreads();
  return total;
}

// --------------------------------------------------------------------------- pass A

template <typename K>
__global__ void __launch_bounds__(kBT)
k_bin_count(const K* __restrict__ keys, uint64_t n, HashParams hp, int s, uint32_t nbins, uint64_t chunk,
            uint32_t* __restrict__ M) {
  extern __shared__ uint32_t s_cnt[];
  for (uint32_t i = threadIdx.x; i < nbins; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  const uint64_t lo = (uint64_t)blockIdx.x * chunk;
  const uint64_t hi = min(n, lo + chunk);
  if (sizeof(K) == 4 && lo < hi && ((reinterpret_cast<uintptr_t>(keys + lo) & 15) == 0)) {
    const uint4* p = reinterpret_cast<const uint4*>(keys + lo);
    const uint64_t nv = (hi - lo) / 4;
    for (uint64_t i = threadIdx.x; i < nv; i += blockDim.x) {
      uint4 q = __ldcs(p + i);
      atomicAdd(s_cnt + bin_of((K)q.x, hp, s), 1u);
      atomicAdd(s_cnt + bin_of((K)q.y, hp, s), 1u);
      atomicAdd(s_cnt + bin_of((K)q.z, hp, s), 1u);
      atomicAdd(s_cnt + bin_of((K)q.w, hp, s), 1u);
    }
    for (uint64_t i = lo + nv * 4 + threadIdx.x; i < hi; i += blockDim.x) atomicAdd(s_cnt + bin_of(keys[i], hp, s), 1u);
  } else {
    for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) atomicAdd(s_cnt + bin_of(keys[i], hp, s), 1u);
  }
  __syncthreads();
  uint32_t* row = M + (uint64_t)blockIdx.x * nbins;
  for (uint32_t i = threadIdx.x; i < nbins; i += blockDim.x) row[i] = s_cnt[i];
}

// Thread per bin: exclusive prefix of the bin's counts over CTAs (in place);
// the column total goes to totals[b].
__global__ void k_bin_colscan(uint32_t* __restrict__ M, uint32_t G, uint32_t nbins, uint32_t* __restrict__ totals) {
  uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nbins) return;
  uint32_t run = 0;
  for (uint32_t g = 0; g < G; g++) {
    uint32_t c = M[(uint64_t)g * nbins + b];
    M[(uint64_t)g * nbins + b] = run;
    run += c;
  }
  totals[b] = run;
}

// One CTA: bin starts (exclusive scan of totals, bin_start[nbins] = total) and
// the list of bins whose key count exceeds `cap`.
__global__ void __launch_bounds__(kBT)
k_bin_starts(const uint32_t* __restrict__ totals, uint32_t nbins, uint32_t cap, uint32_t* __restrict__ bin_start,
             uint32_t* __restrict__ big_list, uint32_t* __restrict__ big_count) {
  extern __shared__ uint32_t s_a[];
  __shared__ uint32_t s_big;
  if (threadIdx.x == 0) s_big = 0;
  for (uint32_t i = threadIdx.x; i < nbins; i += blockDim.x) {
    uint32_t t = totals[i];
    s_a[i] = t;
    if (big_list && t > cap) big_list[atomicAdd(&s_big, 1u)] = i;
  }
  __syncthreads();
  uint32_t total = block_exscan(s_a, nbins);
  for (uint32_t i = threadIdx.x; i < nbins; i += blockDim.x) bin_start[i] = s_a[i];
  if (threadIdx.x == 0) {
    bin_start[nbins] = total;
    if (big_count) *big_count = s_big;
  }
}

// --------------------------------------------------------------------------- register tiles

// A CTA tile of TILE keys held in registers, KPT = TILE / kBT per thread.
// Full, 16-byte-aligned tiles load with 128-bit vector loads (element k of a
// thread is ((k / VPL) * kBT + tid) * VPL + k % VPL); ragged tiles load
// element k * kBT + tid.  Both mappings are coalesced.
template <typename K>
struct TileShape {
  static constexpr int kTile = sizeof(K) == 4 ? 32768 : 16384;
  static constexpr int kKPT = kTile / kBT;
  static constexpr int kVPL = 16 / sizeof(K);
};

template <typename K, int KPT>
__device__ __forceinline__ uint32_t tile_elem(int k, bool vec) {
  constexpr int VPL = 16 / sizeof(K);
  return vec ? (uint32_t)(((k / VPL) * kBT + threadIdx.x) * VPL + k % VPL) : (uint32_t)(k * kBT + threadIdx.x);
}

template <typename K, int KPT>
__device__ __forceinline__ bool load_tile(const K* __restrict__ src, uint32_t m, K (&kv)[KPT]) {
  constexpr int VPL = 16 / sizeof(K);
  const bool vec = (m == (uint32_t)KPT * kBT) && ((reinterpret_cast<uintptr_t>(src) & 15) == 0);
  if (vec) {
    const uint4* p = reinterpret_cast<const uint4*>(src);
#pragma unroll
    for (int l = 0; l < KPT / VPL; l++) {
      uint4 q = __ldcs(p + l * kBT + threadIdx.x);
      const K* qk = reinterpret_cast<const K*>(&q);
#pragma unroll
      for (int j = 0; j < VPL; j++) kv[l * VPL + j] = qk[j];
    }
  } else {
#pragma unroll
    for (int k = 0; k < KPT; k++) {
      uint32_t e = k * kBT + threadIdx.x;
      kv[k] = e < m ? src[e] : K(0);
    }
  }
  return vec;
}

__device__ __forceinline__ uint32_t get16(const uint32_t* p, int k) { return (p[k >> 1] >> ((k & 1) * 16)) & 0xFFFFu; }
__device__ __forceinline__ void set16(uint32_t* p, int k, uint32_t v) {
  if (k & 1) p[k >> 1] = (p[k >> 1] & 0xFFFFu) | (v << 16);
  else p[k >> 1] = (p[k >> 1] & 0xFFFF0000u) | (v & 0xFFFFu);
}

// Inclusive max-scan of n (<= 32 * blockDim) uint32 in smem, in place.
__device__ void block_maxscan(uint32_t* a, uint32_t n) {
  __shared__ uint32_t s_w[32];
  const uint32_t per = (n + blockDim.x - 1) / blockDim.x;
  const uint32_t lo = threadIdx.x * per, hi = min(lo + per, n);
  uint32_t mx = 0;
  for (uint32_t i = lo; i < hi; i++) mx = max(mx, a[i]);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t inc = mx;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc = max(inc, y);
  }
  if (lane == 31) s_w[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < nw ? s_w[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w = max(w, y);
    }
    if (lane < nw) s_w[lane] = w;
  }
  __syncthreads();
  uint32_t run = warp ? s_w[warp - 1] : 0u;
  uint32_t y = __shfl_up_sync(0xffffffffu, inc, 1);
  if (lane > 0) run = max(run, y);
  for (uint32_t i = lo; i < hi; i++) {
    run = max(run, a[i]);
    a[i] = run;
  }
  __syncthreads();
}

// --------------------------------------------------------------------------- pass B

// Partition a CTA's contiguous chunk tile by tile.  Per tile: bins of the
// register-held keys -> smem histogram -> tile offsets -> keys staged in smem
// grouped by bin -> each bin's run written contiguously at the CTA's cursor.
// kSlot also records, per input key, its staged position inside its tile
// (pmap, uint16), which the reverse pass uses to restore query order.
template <typename K, bool kSlot>
__global__ void __launch_bounds__(kBT, 1)
k_partition(const K* __restrict__ keys, uint64_t n, HashParams hp, int s, uint32_t nbins, uint64_t chunk,
            const uint32_t* __restrict__ M, const uint32_t* __restrict__ bin_start, K* __restrict__ out,
            uint16_t* __restrict__ pmap) {
  using TS = TileShape<K>;
  constexpr int KPT = TS::kKPT;
  extern __shared__ __align__(16) unsigned char s_raw[];
  uint32_t* R = reinterpret_cast<uint32_t*>(s_raw);  // tile counts -> offsets -> running
  uint32_t* cur = R + nbins + 1;                     // per-bin output cursor
  K* staged = reinterpret_cast<K*>(s_raw + (((2 * nbins + 1) * 4 + 15) & ~15u));
  const uint64_t lo = (uint64_t)blockIdx.x * chunk;
  const uint64_t hi = min(n, lo + chunk);
  const uint32_t* row = M + (uint64_t)blockIdx.x * nbins;
  for (uint32_t b = threadIdx.x; b < nbins; b += blockDim.x) cur[b] = bin_start[b] + row[b];

  for (uint64_t t0 = lo; t0 < hi; t0 += TS::kTile) {
    const uint32_t m = (uint32_t)min((uint64_t)TS::kTile, hi - t0);
    for (uint32_t b = threadIdx.x; b < nbins; b += blockDim.x) R[b] = 0;
    K kv[KPT];
    const bool vec = load_tile<K, KPT>(keys + t0, m, kv);
    uint32_t bp[KPT / 2];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < KPT; k++) {
      const bool ok = tile_elem<K, KPT>(k, vec) < m;
      const uint32_t b = ok ? bin_of(kv[k], hp, s) : 0xFFFFu;
      if (k & 1) bp[k >> 1] |= b << 16; else bp[k >> 1] = b;
      if (ok) atomicAdd(R + b, 1u);
    }
    __syncthreads();
    block_exscan(R, nbins);
    for (uint32_t b = threadIdx.x; b < nbins; b += blockDim.x) cur[b] -= R[b];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < KPT; k++) {
      const uint32_t b = get16(bp, k);
      if (b != 0xFFFFu) {
        const uint32_t slot = atomicAdd(R + b, 1u);
        staged[slot] = kv[k];
        if (kSlot) pmap[t0 + tile_elem<K, KPT>(k, vec)] = (uint16_t)slot;
      }
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < m; j += blockDim.x) {
      const K key = staged[j];
      out[cur[bin_of(key, hp, s)] + j] = key;
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < nbins; b += blockDim.x) cur[b] += R[b];
  }
}

// Reverse of k_partition for per-query values: CTA g replays its chunk's
// tiles (same tiling, same cursors), rebuilds each tile's bin runs, pulls the
// runs of `vals_bo` (bin-ordered) into smem staged order, and writes
// out[i] = staged[pmap[i]] in input order.  Every global access is coalesced
// per run or per tile.
template <typename K>
__global__ void __launch_bounds__(kBT, 1)
k_unpartition(const K* __restrict__ keys, uint64_t n, HashParams hp, int s, uint32_t nbins, uint64_t chunk,
              const uint32_t* __restrict__ M, const uint32_t* __restrict__ bin_start,
              const uint32_t* __restrict__ vals_bo, const uint16_t* __restrict__ pmap, uint32_t* __restrict__ out) {
  using TS = TileShape<K>;
  constexpr int KPT = TS::kKPT;
  constexpr int VPT = 32768 / kBT;  // staged values per thread (u32 tile of up to 32K)
  extern __shared__ __align__(16) unsigned char s_raw[];
  uint32_t* R = reinterpret_cast<uint32_t*>(s_raw);
  uint32_t* cur = R + nbins + 1;
  uint32_t* staged = reinterpret_cast<uint32_t*>(s_raw + (((2 * nbins + 1) * 4 + 15) & ~15u));
  const uint64_t lo = (uint64_t)blockIdx.x * chunk;
  const uint64_t hi = min(n, lo + chunk);
  const uint32_t* row = M + (uint64_t)blockIdx.x * nbins;
  for (uint32_t b = threadIdx.x; b < nbins; b += blockDim.x) cur[b] = bin_start[b] + row[b];

  for (uint64_t t0 = lo; t0 < hi; t0 += TS::kTile) {
    const uint32_t m = (uint32_t)min((uint64_t)TS::kTile, hi - t0);
    for (uint32_t b = threadIdx.x; b < nbins; b += blockDim.x) R[b] = 0;
    for (uint32_t j = threadIdx.x; j < m; j += blockDim.x) staged[j] = 0;
    K kv[KPT];
    const bool vec = load_tile<K, KPT>(keys + t0, m, kv);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < KPT; k++)
      if (tile_elem<K, KPT>(k, vec) < m) atomicAdd(R + bin_of(kv[k], hp, s), 1u);
    __syncthreads();
    const uint32_t total = block_exscan(R, nbins);
    if (threadIdx.x == 0) R[nbins] = total;
    for (uint32_t b = threadIdx.x; b < nbins; b += blockDim.x) cur[b] -= R[b];
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < nbins; b += blockDim.x)
      if (R[b + 1] > R[b]) staged[R[b]] = b;  // run starts
    __syncthreads();
    block_maxscan(staged, m);  // staged[j] = bin of staged position j
    uint32_t v[VPT];
#pragma unroll
    for (int k = 0; k < VPT; k++) {
      const uint32_t j = k * kBT + threadIdx.x;
      v[k] = j < m ? vals_bo[cur[staged[j]] + j] : 0u;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < VPT; k++) {
      const uint32_t j = k * kBT + threadIdx.x;
      if (j < m) staged[j] = v[k];
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < m; j += blockDim.x) out[t0 + j] = staged[pmap[t0 + j]];
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < nbins; b += blockDim.x) cur[b] += R[b + 1];
  }
}

// --------------------------------------------------------------------------- pass C: build

template <typename K>
struct BuildShape {
  static constexpr int kKPT = sizeof(K) == 4 ? 38 : 19;
  static constexpr uint32_t kCap = kKPT * kBT;
};

// One CTA per bin: the bin's keys (<= kCap) are held in registers; counting
// and ranking use packed uint16 smem counters (one atomic each), offsets and
// edges leave as coalesced streams.
template <typename K>
__global__ void __launch_bounds__(kBT, 1)
k_local_build(const K* __restrict__ part, const uint32_t* __restrict__ bin_start, uint32_t nbins, HashParams hp,
              int s, uint64_t v, uint32_t* __restrict__ offsets, K* __restrict__ edges) {
  constexpr int KPT = BuildShape<K>::kKPT;
  extern __shared__ __align__(16) unsigned char s_raw[];
  const uint32_t S = 1u << s;
  uint32_t* c16 = reinterpret_cast<uint32_t*>(s_raw);  // S/2 packed u16 counters
  K* staged = reinterpret_cast<K*>(c16 + S / 2);
  const uint32_t b = blockIdx.x;
  const uint32_t lo = bin_start[b], hi = bin_start[b + 1];
  const uint32_t cnt = hi - lo;
  const uint64_t first = (uint64_t)b << s;
  const uint32_t nb = (uint32_t)min((uint64_t)S, v - first);
  if (b == nbins - 1 && threadIdx.x == 0) offsets[v] = hi;
  if (cnt > (uint32_t)KPT * kBT) return;  // k_local_build_big owns this bin
  K kv[KPT];
#pragma unroll
  for (int k = 0; k < KPT; k++) {
    const uint32_t j = k * kBT + threadIdx.x;
    kv[k] = j < cnt ? part[lo + j] : K(0);
  }
  for (uint32_t i = threadIdx.x; i < (nb + 1) / 2; i += blockDim.x) c16[i] = 0;
  __syncthreads();
#pragma unroll
  for (int k = 0; k < KPT; k++) {
    if (k * kBT + threadIdx.x < cnt) {
      const uint32_t l = bucket_of(kv[k], hp) - (uint32_t)first;
      atomicAdd(c16 + (l >> 1), 1u << ((l & 1) * 16));
    }
  }
  __syncthreads();
  block_exscan_u16(c16, nb);
  for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) offsets[first + i] = lo + get16(c16, i);
  __syncthreads();
#pragma unroll
  for (int k = 0; k < KPT; k++) {
    if (k * kBT + threadIdx.x < cnt) {
      const uint32_t l = bucket_of(kv[k], hp) - (uint32_t)first;
      const uint32_t sh = (l & 1) * 16;
      const uint32_t old = atomicAdd(c16 + (l >> 1), 1u << sh);
      staged[(old >> sh) & 0xFFFFu] = kv[k];
    }
  }
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < cnt; j += blockDim.x) edges[lo + j] = staged[j];
}

// Oversized bins: global-memory counters (one S-sized scratch per CTA).
template <typename K>
__global__ void __launch_bounds__(kBT)
k_local_build_big(const K* __restrict__ part, const uint32_t* __restrict__ bin_start, const uint32_t* __restrict__ big_list,
                  const uint32_t* __restrict__ big_count, HashParams hp, int s, uint64_t v, uint32_t* __restrict__ scratch,
                  uint32_t* __restrict__ offsets, K* __restrict__ edges) {
  const uint32_t S = 1u << s;
  uint32_t* cnt = scratch + (uint64_t)blockIdx.x * S;
  __shared__ uint32_t s_w[32];
  for (uint32_t k = blockIdx.x; k < *big_count; k += gridDim.x) {
    const uint32_t b = big_list[k];
    const uint32_t lo = bin_start[b], hi = bin_start[b + 1];
    const uint64_t first = (uint64_t)b << s;
    const uint32_t nb = (uint32_t)min((uint64_t)S, v - first);
    for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) cnt[i] = 0;
    __syncthreads();
    for (uint32_t j = lo + threadIdx.x; j < hi; j += blockDim.x)
      atomicAdd(cnt + (bucket_of(part[j], hp) - (uint32_t)first), 1u);
    __syncthreads();
    const uint32_t per = (nb + blockDim.x - 1) / blockDim.x;
    const uint32_t a0 = threadIdx.x * per, a1 = min(a0 + per, nb);
    uint32_t sum = 0;
    for (uint32_t i = a0; i < a1; i++) sum += cnt[i];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint32_t inc = sum;
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      uint32_t w = lane < nw ? s_w[lane] : 0u;
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      if (lane < nw) s_w[lane] = w;
    }
    __syncthreads();
    uint32_t run = lo + (warp ? s_w[warp - 1] : 0u) + inc - sum;
    for (uint32_t i = a0; i < a1; i++) {
      uint32_t x = cnt[i];
      cnt[i] = run;
      offsets[first + i] = run;
      run += x;
    }
    __syncthreads();
    for (uint32_t j = lo + threadIdx.x; j < hi; j += blockDim.x) {
      K key = part[j];
      uint32_t slot = atomicAdd(cnt + (bucket_of(key, hp) - (uint32_t)first), 1u);
      edges[slot] = key;
    }
    __syncthreads();
  }
}

// --------------------------------------------------------------------------- pass C: probe

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

// One CTA per bin: the table's CSR slice for the bin (local uint16 offsets +
// edges) is staged in smem; the bin's queries (register batches) probe it
// with IntersectArray semantics (count of equal keys in the bucket,
// PAPER.md:62-72) and write their counts in bin order.  Table slices above the
// smem capacity are probed in global memory instead.
template <typename K>
__global__ void __launch_bounds__(kBT, 1)
k_local_probe(const uint32_t* __restrict__ t_off, const K* __restrict__ t_edges, const K* __restrict__ qpart,
              const uint32_t* __restrict__ qbin_start, HashParams hp, int s, uint64_t v, uint32_t cap,
              uint32_t* __restrict__ mult_bo, unsigned long long* __restrict__ agg) {
  constexpr int QPT = 16;
  extern __shared__ __align__(16) unsigned char s_raw[];
  const uint32_t S = 1u << s;
  uint16_t* off16 = reinterpret_cast<uint16_t*>(s_raw);
  K* tedges = reinterpret_cast<K*>(s_raw + ((2 * (S + 1) + 15) & ~15u));
  const uint32_t b = blockIdx.x;
  const uint32_t qlo = qbin_start[b], qhi = qbin_start[b + 1];
  if (qlo == qhi) return;
  const uint64_t first = (uint64_t)b << s;
  const uint32_t nb = (uint32_t)min((uint64_t)S, v - first);
  const uint32_t tlo = t_off[first], thi = t_off[first + nb];
  const bool in_smem = thi - tlo <= cap;
  if (in_smem) {
    for (uint32_t i0 = 0; i0 <= nb; i0 += 8 * kBT) {
      uint32_t x[8];
#pragma unroll
      for (int k = 0; k < 8; k++) {
        uint32_t i = i0 + k * kBT + threadIdx.x;
        x[k] = i <= nb ? t_off[first + i] : 0u;
      }
#pragma unroll
      for (int k = 0; k < 8; k++) {
        uint32_t i = i0 + k * kBT + threadIdx.x;
        if (i <= nb) off16[i] = (uint16_t)(x[k] - tlo);
      }
    }
    for (uint32_t j0 = 0; j0 < thi - tlo; j0 += 8 * kBT) {
      K x[8];
#pragma unroll
      for (int k = 0; k < 8; k++) {
        uint32_t j = j0 + k * kBT + threadIdx.x;
        x[k] = j < thi - tlo ? t_edges[tlo + j] : K(0);
      }
#pragma unroll
      for (int k = 0; k < 8; k++) {
        uint32_t j = j0 + k * kBT + threadIdx.x;
        if (j < thi - tlo) tedges[j] = x[k];
      }
    }
  }
  __syncthreads();
  uint64_t matched = 0, total = 0, comps = 0;
  for (uint32_t q0 = qlo; q0 < qhi; q0 += QPT * kBT) {
    K qv[QPT];
#pragma unroll
    for (int k = 0; k < QPT; k++) {
      uint32_t j = q0 + k * kBT + threadIdx.x;
      qv[k] = j < qhi ? qpart[j] : K(0);
    }
#pragma unroll
    for (int k = 0; k < QPT; k++) {
      uint32_t j = q0 + k * kBT + threadIdx.x;
      if (j < qhi) {
        const K q = qv[k];
        const uint32_t h = bucket_of(q, hp);
        uint32_t a, e, c = 0;
        if (in_smem) {
          const uint32_t l = h - (uint32_t)first;
          a = off16[l];
          e = off16[l + 1];
          for (uint32_t t = a; t < e; t++) c += (tedges[t] == q);
        } else {
          a = t_off[h];
          e = t_off[h + 1];
          for (uint32_t t = a; t < e; t++) c += (t_edges[t] == q);
        }
        mult_bo[j] = c;
        matched += (c != 0);
        total += c;
        comps += e - a;
      }
    }
  }
  if (agg) flush_agg(matched, total, comps, agg);
}

// --------------------------------------------------------------------------- host drivers

static size_t partition_smem(const BinLayout& L, int key_bits) {
  return (size_t)(((2 * L.nbins + 1) * 4 + 15) & ~15u) + (size_t)32768 * 4;  // staged: 32K u32 / 16K u64
  (void)key_bits;
}
static uint32_t caps_for(int key_bits, uint32_t cap) { return key_bits == 32 ? cap : cap / 2; }

static size_t build_smem(const BinLayout& L, int key_bits) {
  return (size_t)(1u << L.s) / 2 * 4 + (size_t)(key_bits == 32 ? BuildShape<uint32_t>::kCap * 4 : BuildShape<uint64_t>::kCap * 8);
}
static size_t probe_smem(const BinLayout& L, int key_bits) {
  return (size_t)((2 * ((1u << L.s) + 1) + 15) & ~15u) + (size_t)caps_for(key_bits, kProbeCap) * (key_bits / 8);
}

size_t binned_ws_bytes(uint64_t n, const BinLayout& L, int key_bits, bool query) {
  size_t kb = key_bits / 8;
  size_t b = 0;
  b += align_up((size_t)L.grid * L.nbins * 4, 256);  // M
  b += align_up((size_t)L.nbins * 4, 256);           // totals
  b += align_up((size_t)(L.nbins + 1) * 4, 256);     // bin starts
  b += align_up((size_t)L.nbins * 4, 256) + 256;     // big list + count
  b += align_up(n * kb, 256);                        // partitioned keys
  if (query) b += align_up(n * 2, 256) + align_up(n * 4, 256);  // pmap + bin-ordered multiplicities
  else b += align_up((size_t)num_sms() * (1u << L.s) * 4, 256);  // big-bin scratch
  return b + 1024;
}

struct PartitionOut {
  void* part;
  uint32_t* M;
  uint32_t* bin_start;
  uint32_t* big_list;
  uint32_t* big_count;
  uint16_t* pmap;
};

template <typename K>
static int run_partition(const K* keys, uint64_t n, const HashParams& hp, const BinLayout& L, uint32_t cap,
                         bool want_pmap, Workspace& ws, cudaStream_t st, PartitionOut* po) {
  uint32_t* M = ws.take<uint32_t>((size_t)L.grid * L.nbins);
  uint32_t* totals = ws.take<uint32_t>(L.nbins);
  po->M = M;
  po->bin_start = ws.take<uint32_t>(L.nbins + 1);
  po->big_list = ws.take<uint32_t>(L.nbins);
  po->big_count = ws.take<uint32_t>(64);
  K* part = ws.take<K>(n);
  po->part = part;
  po->pmap = want_pmap ? ws.take<uint16_t>(n) : nullptr;
  if (!ws.ok()) return set_error(HG_ERR_CONFIG, "binned workspace too small (%zu < %zu)", ws.cap, ws.used);
  size_t smA = (size_t)L.nbins * 4;
  HG_CHECK_CUDA(cudaFuncSetAttribute(k_bin_count<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smA));
  HG_LAUNCH("hg_bin_count", k_bin_count<K>, L.grid, kBT, smA, st, keys, n, hp, L.s, L.nbins, L.chunk, M);
  HG_LAUNCH("hg_bin_colscan", k_bin_colscan, (L.nbins + 255) / 256, 256, 0, st, M, L.grid, L.nbins, totals);
  HG_CHECK_CUDA(cudaFuncSetAttribute(k_bin_starts, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smA));
  HG_LAUNCH("hg_bin_starts", k_bin_starts, 1, kBT, smA, st, totals, L.nbins, cap, po->bin_start, po->big_list,
            po->big_count);
  size_t smB = partition_smem(L, sizeof(K) * 8);
  if (want_pmap) {
    HG_CHECK_CUDA(cudaFuncSetAttribute(k_partition<K, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smB));
    HG_LAUNCH("hg_partition_slot", (k_partition<K, true>), L.grid, kBT, smB, st, keys, n, hp, L.s, L.nbins, L.chunk, M,
              po->bin_start, part, po->pmap);
  } else {
    HG_CHECK_CUDA(cudaFuncSetAttribute(k_partition<K, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smB));
    HG_LAUNCH("hg_partition", (k_partition<K, false>), L.grid, kBT, smB, st, keys, n, hp, L.s, L.nbins, L.chunk, M,
              po->bin_start, part, po->pmap);
  }
  return HG_OK;
}

template <typename K>
int binned_build(const K* keys, uint64_t n, const HashParams& hp, uint64_t v, const BinLayout& L, uint32_t* offsets,
                 K* edges, Workspace& ws, cudaStream_t st) {
  const uint32_t cap = BuildShape<K>::kCap;
  PartitionOut po{};
  int rc = run_partition<K>(keys, n, hp, L, cap, false, ws, st, &po);
  if (rc) return rc;
  uint32_t* scratch = ws.take<uint32_t>((size_t)num_sms() * (1u << L.s));
  if (!ws.ok()) return set_error(HG_ERR_CONFIG, "binned workspace too small");
  size_t smC = build_smem(L, sizeof(K) * 8);
  HG_CHECK_CUDA(cudaFuncSetAttribute(k_local_build<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smC));
  HG_LAUNCH("hg_local_build", k_local_build<K>, L.nbins, kBT, smC, st, (const K*)po.part, po.bin_start, L.nbins, hp,
            L.s, v, offsets, edges);
  HG_LAUNCH("hg_local_build_big", k_local_build_big<K>, num_sms(), kBT, 0, st, (const K*)po.part, po.bin_start,
            po.big_list, po.big_count, hp, L.s, v, scratch, offsets, edges);
  return HG_OK;
}

template <typename K>
int binned_query(const uint32_t* t_off, const K* t_edges, const K* queries, uint64_t q, const HashParams& hp,
                 uint64_t v, const BinLayout& L, uint32_t* mult, uint64_t* agg, Workspace& ws, cudaStream_t st) {
  PartitionOut po{};
  int rc = run_partition<K>(queries, q, hp, L, 0xFFFFFFFFu, true, ws, st, &po);
  if (rc) return rc;
  uint32_t* mult_bo = ws.take<uint32_t>(q);
  if (!ws.ok()) return set_error(HG_ERR_CONFIG, "binned workspace too small");
  const uint32_t cap = caps_for(sizeof(K) * 8, kProbeCap);
  size_t smC = probe_smem(L, sizeof(K) * 8);
  HG_CHECK_CUDA(cudaFuncSetAttribute(k_local_probe<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smC));
  HG_LAUNCH("hg_local_probe", k_local_probe<K>, L.nbins, kBT, smC, st, t_off, t_edges, (const K*)po.part, po.bin_start,
            hp, L.s, v, cap, mult_bo, reinterpret_cast<unsigned long long*>(agg));
  size_t smR = partition_smem(L, 32);
  HG_CHECK_CUDA(cudaFuncSetAttribute(k_unpartition<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smR));
  HG_LAUNCH("hg_unpartition", k_unpartition<K>, L.grid, kBT, smR, st, queries, q, hp, L.s, L.nbins, L.chunk, po.M,
            po.bin_start, mult_bo, po.pmap, mult);
  return HG_OK;
}

template int binned_build<uint32_t>(const uint32_t*, uint64_t, const HashParams&, uint64_t, const BinLayout&,
                                    uint32_t*, uint32_t*, Workspace&, cudaStream_t);
template int binned_build<uint64_t>(const uint64_t*, uint64_t, const HashParams&, uint64_t, const BinLayout&,
                                    uint32_t*, uint64_t*, Workspace&, cudaStream_t);
template int binned_query<uint32_t>(const uint32_t*, const uint32_t*, const uint32_t*, uint64_t, const HashParams&,
                                    uint64_t, const BinLayout&, uint32_t*, uint64_t*, Workspace&, cudaStream_t);
template int binned_query<uint64_t>(const uint32_t*, const uint64_t*, const uint64_t*, uint64_t, const HashParams&,
                                    uint64_t, const BinLayout&, uint32_t*, uint64_t*, Workspace&, cudaStream_t);

}  // namespace hg
