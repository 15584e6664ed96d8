// hg_shard.cu -- the partitioned (multi-shard) phases and small utilities.
//
//   k_bin_hist     Phase 1 global-bin histogram   (multishard.py:371-377, 286-289)
//   k_split_plan   split search                   (multishard.py:249-263)
//   k_reorg_*      Phase 2 stable per-destination CSR (multishard.py:294-318)
//   k_scatter_u32  positional merge               (multishard.py:523)
//   k_generate     SplitMix64 workload            (workload.py:63-85)
#include "hg_common.cuh"

namespace hg {

constexpr int kT = 256;

static inline int grid_cap(uint64_t n, int per_sm) {
  uint64_t b = (n + kT - 1) / kT;
  uint64_t cap = (uint64_t)num_sms() * per_sm;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

// --------------------------------------------------------------------------- Phase 1

// Shared-memory histogram over the BINS_G global bins (BINS_G <= smem_bins),
// flushed once per CTA with 64-bit atomics.  Falls back to global atomics for
// very large bin counts (smem_bins == 0).
template <typename K>
__global__ void k_bin_hist(const K* __restrict__ keys, uint64_t n, HashParams hp, DivParams bin,
                           uint32_t bins_g, int use_smem, unsigned long long* __restrict__ out) {
  extern __shared__ uint32_t s_hist[];
  if (use_smem) {
    for (uint32_t i = threadIdx.x; i < bins_g; i += blockDim.x) s_hist[i] = 0;
    __syncthreads();
  }
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t b = (uint32_t)div_by(hash_mod(keys[i], hp), bin);
    if (use_smem)
      atomicAdd(s_hist + b, 1u);
    else
      atomicAdd(out + b, 1ull);
  }
  if (use_smem) {
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < bins_g; i += blockDim.x)
      if (s_hist[i]) atomicAdd(out + i, (unsigned long long)s_hist[i]);
  }
}

// One CTA: inclusive prefix over the bin counts, then for r = 1..P-1 the
// lower bound of r * floor(N/P), plus one (multishard.py:257-262).
__global__ void k_split_plan(const unsigned long long* __restrict__ counts, uint64_t bins_g,
                             uint64_t total, uint32_t shards, long long* __restrict__ splits) {
  __shared__ unsigned long long s_part[1024];
  const int t = threadIdx.x, nt = blockDim.x;
  const uint64_t per = (bins_g + nt - 1) / nt;
  const uint64_t lo = (uint64_t)t * per;
  const uint64_t hi = lo + per < bins_g ? lo + per : bins_g;
  unsigned long long sum = 0;
  for (uint64_t i = lo; i < hi; i++) sum += counts[i];
  s_part[t] = sum;
  __syncthreads();
  // Hillis-Steele inclusive scan over nt partial sums (nt <= 1024)
  for (int o = 1; o < nt; o <<= 1) {
    unsigned long long y = t >= o ? s_part[t - o] : 0ull;
    __syncthreads();
    s_part[t] += y;
    __syncthreads();
  }
  const unsigned long long excl = s_part[t] - sum;
  const uint64_t quota = total / shards;
  if (t == 0) {
    splits[0] = 0;
    splits[shards] = (long long)bins_g;
  }
  if (lo < hi) {
    for (uint32_t r = 1; r < shards; r++) {
      const unsigned long long target = (unsigned long long)r * quota;
      // this chunk holds the first index whose inclusive prefix reaches target?
      if (excl + sum >= target && (lo == 0 || excl < target)) {
        unsigned long long run = excl;
        uint64_t i = lo;
        for (; i < hi; i++) {
          run += counts[i];
          if (run >= target) break;
        }
        splits[r] = (long long)(i + 1);
      }
    }
  }
  // targets beyond the total are impossible ((P-1)*floor(N/P) <= N); nothing else to do
}

// --------------------------------------------------------------------------- Phase 2

constexpr int kReorgWarps = 8;
constexpr int kReorgPerLane = 8;
constexpr int kReorgTile = kReorgWarps * 32 * kReorgPerLane;  // 2048 keys per tile

// destination shard of a bin: #{d in 1..P-1 : splits[d] <= bin}, i.e.
// searchsorted(boundaries, h, 'right') - 1 with boundaries = splits * bin_size
// (multishard.py:107-113); equal splits route to the later shard.
__device__ __forceinline__ uint32_t dest_of_bin(uint64_t bin, const long long* s_splits, uint32_t shards) {
  uint32_t lo = 1, hi = shards;  // first d in [1, P) with splits[d] > bin
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if ((uint64_t)s_splits[mid] <= bin) lo = mid + 1; else hi = mid;
  }
  return lo - 1;
}

// Count pass: per-tile destination counts into tile_counts[tile * P + d]; sum
// of (dest + 1) into steps (the linear-scan cost model, multishard.py:300-307).
template <typename K>
__global__ void __launch_bounds__(kReorgWarps * 32)
k_reorg_count(const K* __restrict__ keys, uint64_t n, HashParams hp, DivParams bin,
              const long long* __restrict__ splits, uint32_t shards, uint32_t* __restrict__ tile_counts,
              unsigned long long* __restrict__ steps) {
  extern __shared__ unsigned char s_raw[];
  long long* s_splits = reinterpret_cast<long long*>(s_raw);
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(s_splits + shards + 1);
  for (uint32_t i = threadIdx.x; i <= shards; i += blockDim.x) s_splits[i] = splits[i];
  for (uint32_t i = threadIdx.x; i < shards; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * kReorgTile;
  unsigned long long st = 0;
  for (int j = threadIdx.x; j < kReorgTile; j += blockDim.x) {
    uint64_t i = base + j;
    if (i < n) {
      uint32_t d = dest_of_bin(div_by(hash_mod(keys[i], hp), bin), s_splits, shards);
      atomicAdd(s_cnt + d, 1u);
      st += d + 1;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) st += __shfl_xor_sync(0xffffffffu, st, o);
  if ((threadIdx.x & 31) == 0 && st && steps) atomicAdd(steps, st);
  __syncthreads();
  for (uint32_t d = threadIdx.x; d < shards; d += blockDim.x)
    tile_counts[(uint64_t)blockIdx.x * shards + d] = s_cnt[d];
}

// Column scan: for destination d (one CTA each), exclusive prefix of the
// per-tile counts in tile order; the column total goes to totals[d].
__global__ void k_reorg_scan(uint32_t* __restrict__ tile_counts, uint64_t tiles, uint32_t shards,
                             unsigned long long* __restrict__ totals) {
  __shared__ unsigned long long s_w[32];
  __shared__ unsigned long long s_carry;
  const uint32_t d = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (uint64_t b0 = 0; b0 < tiles; b0 += blockDim.x) {
    uint64_t t = b0 + threadIdx.x;
    unsigned long long x = t < tiles ? tile_counts[t * shards + d] : 0ull;
    unsigned long long inc = x;
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      unsigned long long w = lane < nw ? s_w[lane] : 0ull;
      for (int o = 1; o < 32; o <<= 1) {
        unsigned long long y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      if (lane < nw) s_w[lane] = w;
    }
    __syncthreads();
    unsigned long long excl = s_carry + (warp ? s_w[warp - 1] : 0ull) + inc - x;
    if (t < tiles) tile_counts[t * shards + d] = (uint32_t)excl;
    __syncthreads();
    if (threadIdx.x == 0) s_carry += s_w[nw - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) totals[d] = s_carry;
}

__global__ void k_reorg_rows(const unsigned long long* __restrict__ totals, uint32_t shards,
                             unsigned long long* __restrict__ row_offsets) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned long long run = 0;
    row_offsets[0] = 0;
    for (uint32_t d = 0; d < shards; d++) {
      run += totals[d];
      row_offsets[d + 1] = run;
    }
  }
}

// Place pass: stable within a tile (warp w owns keys [w*256, (w+1)*256) of
// the tile, processed in 32-key rounds in index order; ranks inside a round
// come from ballots per distinct destination).
template <typename K>
__global__ void __launch_bounds__(kReorgWarps * 32)
k_reorg_place(const K* __restrict__ keys, uint64_t n, HashParams hp, DivParams bin,
              const long long* __restrict__ splits, uint32_t shards,
              const uint32_t* __restrict__ tile_base, const unsigned long long* __restrict__ row_offsets,
              K* __restrict__ grouped, uint32_t* __restrict__ order) {
  extern __shared__ unsigned char s_raw[];
  long long* s_splits = reinterpret_cast<long long*>(s_raw);
  unsigned long long* s_base = reinterpret_cast<unsigned long long*>(s_splits + shards + 1);
  uint32_t* s_wcnt = reinterpret_cast<uint32_t*>(s_base + shards);  // [warps][shards]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t i = threadIdx.x; i <= shards; i += blockDim.x) s_splits[i] = splits[i];
  for (uint32_t i = threadIdx.x; i < shards; i += blockDim.x)
    s_base[i] = row_offsets[i] + tile_base[(uint64_t)blockIdx.x * shards + i];
  for (uint32_t i = threadIdx.x; i < kReorgWarps * shards; i += blockDim.x) s_wcnt[i] = 0;
  __syncthreads();

  const uint64_t wbase = (uint64_t)blockIdx.x * kReorgTile + (uint64_t)warp * 32 * kReorgPerLane;
  K kv[kReorgPerLane];
  uint32_t dv[kReorgPerLane];
#pragma unroll
  for (int r = 0; r < kReorgPerLane; r++) {
    uint64_t i = wbase + r * 32 + lane;
    dv[r] = 0xffffffffu;
    if (i < n) {
      kv[r] = keys[i];
      dv[r] = dest_of_bin(div_by(hash_mod(kv[r], hp), bin), s_splits, shards);
      atomicAdd(s_wcnt + warp * shards + dv[r], 1u);
    }
  }
  __syncthreads();
  // exclusive prefix over warps, per destination
  for (uint32_t d = threadIdx.x; d < shards; d += blockDim.x) {
    uint32_t run = 0;
    for (int w = 0; w < kReorgWarps; w++) {
      uint32_t c = s_wcnt[w * shards + d];
      s_wcnt[w * shards + d] = run;
      run += c;
    }
  }
  __syncthreads();
  uint32_t* my = s_wcnt + warp * shards;  // running per-destination cursor of this warp
#pragma unroll
  for (int r = 0; r < kReorgPerLane; r++) {
    const uint32_t d = dv[r];
    uint32_t active = __ballot_sync(0xffffffffu, d != 0xffffffffu);
    uint32_t slot_rank = 0, slot_d = d;
    while (active) {
      const int leader = __ffs(active) - 1;
      const uint32_t d0 = __shfl_sync(0xffffffffu, d, leader);
      const uint32_t m = __ballot_sync(0xffffffffu, d == d0) & active;
      uint32_t cur = my[d0];
      if (d == d0) slot_rank = cur + __popc(m & lanemask_lt());
      __syncwarp();
      if (lane == leader) my[d0] = cur + __popc(m);
      __syncwarp();
      active &= ~m;
    }
    if (d != 0xffffffffu) {
      unsigned long long slot = s_base[slot_d] + slot_rank;
      grouped[slot] = kv[r];
      if (order) order[slot] = (uint32_t)(wbase + r * 32 + lane);
    }
  }
}

// --------------------------------------------------------------------------- utilities

__global__ void k_scatter_u32(const uint32_t* __restrict__ src, const uint32_t* __restrict__ order, uint64_t n,
                              uint32_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[order[i]] = src[i];
}

__global__ void k_widen_u32(const uint32_t* __restrict__ src, uint64_t n, long long* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = (long long)src[i];
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t seed, uint64_t idx) {
  uint64_t z = seed + (idx + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void k_generate32(uint64_t seed, uint64_t start, uint64_t count, uint64_t mask, uint32_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = (uint32_t)((splitmix64(seed, start + i) & mask) + 1);
}

__global__ void k_generate64(uint64_t seed, uint64_t start, uint64_t count, uint64_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = splitmix64(seed, start + i);
}

static int check_hash(int key_bits, int kind, uint64_t v) {
  if (key_bits != 32 && key_bits != 64) return set_error(HG_ERR_CONFIG, "key_bits must be 32 or 64, got %d", key_bits);
  if (kind != HG_KIND_MURMUR32 && kind != HG_KIND_IDENTITY) return set_error(HG_ERR_CONFIG, "unknown hash kind %d", kind);
  if (v < 1) return set_error(HG_ERR_CONFIG, "hash range must be >= 1");
  return HG_OK;
}

}  // namespace hg

using namespace hg;

extern "C" {

int hg_bin_histogram(const void* keys, uint64_t n, int key_bits, int kind, uint32_t seed, uint64_t hash_range,
                     uint64_t bins_g, uint64_t bin_size, uint64_t* bin_counts, void* stream) {
  int rc = check_hash(key_bits, kind, hash_range);
  if (rc) return rc;
  if (bins_g < 1 || bin_size < 1) return set_error(HG_ERR_CONFIG, "bins_g and bin_size must be >= 1");
  if (bins_g > 0xFFFFFFFFull) return set_error(HG_ERR_CONFIG, "bins_g too large");
  if (!n) return HG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  HashParams hp = make_hash_params(kind, seed, hash_range, key_bits);
  DivParams dp = make_div_params(bin_size);
  const uint64_t smem = 4 * bins_g;
  int use_smem = smem <= 200 * 1024;
  int grid = use_smem ? num_sms() : grid_cap(n, 16);
  if (use_smem) {
    if (key_bits == 32)
      HG_CHECK_CUDA(cudaFuncSetAttribute(k_bin_hist<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    else
      HG_CHECK_CUDA(cudaFuncSetAttribute(k_bin_hist<uint64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  }
  size_t dyn = use_smem ? smem : 0;
  if (key_bits == 32)
    HG_LAUNCH("hg_bin_hist", k_bin_hist<uint32_t>, grid, 1024, dyn, s, (const uint32_t*)keys, n, hp, dp,
              (uint32_t)bins_g, use_smem, (unsigned long long*)bin_counts);
  else
    HG_LAUNCH("hg_bin_hist", k_bin_hist<uint64_t>, grid, 1024, dyn, s, (const uint64_t*)keys, n, hp, dp,
              (uint32_t)bins_g, use_smem, (unsigned long long*)bin_counts);
  return HG_OK;
}

int hg_split_plan(const uint64_t* bin_counts, uint64_t bins_g, uint64_t total_keys, uint32_t shards, int64_t* splits,
                  void* stream) {
  if (shards < 1) return set_error(HG_ERR_CONFIG, "shard count must be >= 1");
  if (bins_g < shards) return set_error(HG_ERR_CONFIG, "bins_g=%llu is less than shard count %u", (unsigned long long)bins_g, shards);
  cudaStream_t s = (cudaStream_t)stream;
  HG_LAUNCH("hg_split_plan", k_split_plan, 1, 1024, 0, s, (const unsigned long long*)bin_counts, bins_g, total_keys,
            shards, (long long*)splits);
  return HG_OK;
}

size_t hg_reorganize_workspace_size(uint64_t n, uint32_t shards) {
  uint64_t tiles = (n + kReorgTile - 1) / kReorgTile;
  return align_up(4 * tiles * (uint64_t)shards, 256) + align_up(8 * (uint64_t)shards, 256) + 512;
}

int hg_reorganize(const void* keys, uint64_t n, int key_bits, int kind, uint32_t seed, uint64_t hash_range,
                  uint64_t bin_size, const int64_t* splits, uint32_t shards, uint64_t* row_offsets, void* grouped,
                  uint32_t* order, uint64_t* search_steps, void* workspace, size_t workspace_bytes, void* stream) {
  int rc = check_hash(key_bits, kind, hash_range);
  if (rc) return rc;
  if (shards < 1 || shards > 4096) return set_error(HG_ERR_CONFIG, "shard count must be in [1, 4096], got %u", shards);
  if (bin_size < 1) return set_error(HG_ERR_CONFIG, "bin_size must be >= 1");
  if (n >= (1ull << 32)) return set_error(HG_ERR_CONFIG, "a shard holds fewer than 2^32 keys");
  cudaStream_t s = (cudaStream_t)stream;
  uint64_t tiles = (n + kReorgTile - 1) / kReorgTile;
  Workspace ws{(char*)workspace, workspace_bytes, 0};
  uint32_t* tile_counts = ws.take<uint32_t>(tiles * shards);
  unsigned long long* totals = ws.take<unsigned long long>(shards);
  if (!ws.ok()) return set_error(HG_ERR_CONFIG, "reorganize workspace too small");
  if (!n) {
    HG_CHECK_CUDA(cudaMemsetAsync(row_offsets, 0, 8 * ((uint64_t)shards + 1), s));
    return HG_OK;
  }
  HashParams hp = make_hash_params(kind, seed, hash_range, key_bits);
  DivParams dp = make_div_params(bin_size);
  size_t smem_c = 8 * (shards + 1) + 4 * shards;
  size_t smem_p = 8 * (shards + 1) + 8 * shards + 4 * kReorgWarps * shards;
  if (key_bits == 32) {
    HG_LAUNCH("hg_reorg_count", k_reorg_count<uint32_t>, (unsigned)tiles, kReorgWarps * 32, smem_c, s,
              (const uint32_t*)keys, n, hp, dp, (const long long*)splits, shards, tile_counts,
              (unsigned long long*)search_steps);
  } else {
    HG_LAUNCH("hg_reorg_count", k_reorg_count<uint64_t>, (unsigned)tiles, kReorgWarps * 32, smem_c, s,
              (const uint64_t*)keys, n, hp, dp, (const long long*)splits, shards, tile_counts,
              (unsigned long long*)search_steps);
  }
  HG_LAUNCH("hg_reorg_scan", k_reorg_scan, shards, 1024, 0, s, tile_counts, tiles, shards, totals);
  HG_LAUNCH("hg_reorg_rows", k_reorg_rows, 1, 32, 0, s, totals, shards, (unsigned long long*)row_offsets);
  if (key_bits == 32) {
    HG_LAUNCH("hg_reorg_place", k_reorg_place<uint32_t>, (unsigned)tiles, kReorgWarps * 32, smem_p, s,
              (const uint32_t*)keys, n, hp, dp, (const long long*)splits, shards, tile_counts,
              (const unsigned long long*)row_offsets, (uint32_t*)grouped, order);
  } else {
    HG_LAUNCH("hg_reorg_place", k_reorg_place<uint64_t>, (unsigned)tiles, kReorgWarps * 32, smem_p, s,
              (const uint64_t*)keys, n, hp, dp, (const long long*)splits, shards, tile_counts,
              (const unsigned long long*)row_offsets, (uint64_t*)grouped, order);
  }
  return HG_OK;
}

int hg_scatter_u32(const uint32_t* src, const uint32_t* order, uint64_t n, uint32_t* out, void* stream) {
  if (!n) return HG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  HG_LAUNCH("hg_scatter_u32", k_scatter_u32, grid_cap(n, 16), kT, 0, s, src, order, n, out);
  return HG_OK;
}

int hg_widen_u32(const uint32_t* src, uint64_t n, int64_t* out, void* stream) {
  if (!n) return HG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  HG_LAUNCH("hg_widen_u32", k_widen_u32, grid_cap(n, 16), kT, 0, s, src, n, (long long*)out);
  return HG_OK;
}

int hg_generate(uint64_t seed, uint64_t start, uint64_t count, int k, int key_bits, void* out, void* stream) {
  if (key_bits != 32 && key_bits != 64) return set_error(HG_ERR_CONFIG, "key_bits must be 32 or 64");
  if (key_bits == 32 && (k < 1 || k > 32)) return set_error(HG_ERR_CONFIG, "k must be in [1, 32], got %d", k);
  if (!count) return HG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (key_bits == 32) {
    uint64_t mask = k == 64 ? ~0ull : ((1ull << k) - 1);
    HG_LAUNCH("hg_generate", k_generate32, grid_cap(count, 16), kT, 0, s, seed, start, count, mask, (uint32_t*)out);
  } else {
    HG_LAUNCH("hg_generate", k_generate64, grid_cap(count, 16), kT, 0, s, seed, start, count, (uint64_t*)out);
  }
  return HG_OK;
}

}  // extern "C"
