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
__device__ __forceinline__ void bin_hist_add(K key, const HashParams& hp, const DivParams& bin, int use_smem,
                                             uint32_t* s_hist, unsigned long long* out) {
  const uint32_t b = (uint32_t)div_by(hash_mod(key, hp), bin);
  if (use_smem) atomicAdd(s_hist + b, 1u);
  else atomicAdd(out + b, 1ull);
}

// 16-byte loads, four in flight per thread (the loop is latency-bound with
// one scalar load per iteration).
template <typename K>
__global__ void __launch_bounds__(1024) k_bin_hist(const K* __restrict__ keys, uint64_t n, HashParams hp, DivParams bin,
                                                   uint32_t bins_g, int use_smem, unsigned long long* __restrict__ out) {
  constexpr int VPL = 16 / sizeof(K);
  extern __shared__ uint32_t s_hist[];
  if (use_smem) {
    for (uint32_t i = threadIdx.x; i < bins_g; i += blockDim.x) s_hist[i] = 0;
    __syncthreads();
  }
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t done = 0;
  if ((reinterpret_cast<uintptr_t>(keys) & 15) == 0) {
    const uint4* p = reinterpret_cast<const uint4*>(keys);
    const uint64_t nv = n / VPL;
    for (uint64_t v = tid; v < nv; v += 4 * stride) {
      uint4 q[4];
#pragma unroll
      for (int u = 0; u < 4; u++) q[u] = v + u * stride < nv ? __ldcs(p + v + u * stride) : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int u = 0; u < 4; u++) {
        if (v + u * stride >= nv) break;
        const K* qk = reinterpret_cast<const K*>(&q[u]);
#pragma unroll
        for (int j = 0; j < VPL; j++) bin_hist_add(qk[j], hp, bin, use_smem, s_hist, out);
      }
    }
    done = nv * VPL;
  }
  for (uint64_t i = done + tid; i < n; i += stride) bin_hist_add(keys[i], hp, bin, use_smem, s_hist, out);
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
constexpr int kReorgPerLane = 16;
constexpr int kReorgTile = kReorgWarps * 32 * kReorgPerLane;  // 4096 keys per tile

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
  K kv[kReorgPerLane];  // all loads in flight before any hashing
#pragma unroll
  for (int r = 0; r < kReorgPerLane; r++) {
    const uint64_t i = base + r * blockDim.x + threadIdx.x;
    kv[r] = i < n ? keys[i] : K(0);
  }
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int r = 0; r < kReorgPerLane; r++) {
    const bool ok = base + r * blockDim.x + threadIdx.x < n;
    const uint32_t d = ok ? dest_of_bin(div_by(hash_mod(kv[r], hp), bin), s_splits, shards) : 0xffffffffu;
    const uint32_t peers = __match_any_sync(0xffffffffu, d);  // one atomic per destination per round
    if (ok && (peers & lt) == 0) atomicAdd(s_cnt + d, (uint32_t)__popc(peers));
    st += ok ? d + 1 : 0u;
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
//
// kPeer: Phase 2 and Phase 3 fused -- each key is stored straight into its
// destination rank's receive buffer (dest_ptrs[d], peer memory mapped over
// NVLink / NVSwitch) at dest_base[d] + (its stable rank in row d); `order`
// still records the input index at the local grouped position.
//
// kGather (hg_reorganize_gather): the same stable slots, read instead of
// written -- gout[i] = gvals[slot of input key i] returns per-row values to
// input order with coalesced stores (a scatter through `order` writes each
// row's values at 1/P density across the whole output).
template <typename K, bool kPeer, bool kGather = false>
__global__ void __launch_bounds__(kReorgWarps * 32)
k_reorg_place(const K* __restrict__ keys, uint64_t n, HashParams hp, DivParams bin,
              const long long* __restrict__ splits, uint32_t shards,
              const uint32_t* __restrict__ tile_base, const unsigned long long* __restrict__ row_offsets,
              K* __restrict__ grouped, uint32_t* __restrict__ order,
              const unsigned long long* __restrict__ dest_ptrs, const unsigned long long* __restrict__ dest_base,
              const uint32_t* __restrict__ gvals = nullptr, uint32_t* __restrict__ gout = nullptr) {
  extern __shared__ unsigned char s_raw[];
  long long* s_splits = reinterpret_cast<long long*>(s_raw);
  unsigned long long* s_base = reinterpret_cast<unsigned long long*>(s_splits + shards + 1);
  unsigned long long* s_rbase = s_base + shards;                      // kPeer: remote slot base per row
  uint32_t* s_wcnt = reinterpret_cast<uint32_t*>(s_rbase + (kPeer ? shards : 0));  // [warps][shards]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t i = threadIdx.x; i <= shards; i += blockDim.x) s_splits[i] = splits[i];
  for (uint32_t i = threadIdx.x; i < shards; i += blockDim.x) {
    const uint32_t tb = tile_base[(uint64_t)blockIdx.x * shards + i];
    s_base[i] = row_offsets[i] + tb;
    if (kPeer) s_rbase[i] = dest_base[i] + tb;
  }
  for (uint32_t i = threadIdx.x; i < kReorgWarps * shards; i += blockDim.x) s_wcnt[i] = 0;
  __syncthreads();

  const uint64_t wbase = (uint64_t)blockIdx.x * kReorgTile + (uint64_t)warp * 32 * kReorgPerLane;
  const uint32_t lt = lanemask_lt();
  uint32_t* my = s_wcnt + warp * shards;  // this warp's per-destination counts, then cursors
  K kv[kReorgPerLane];
  uint32_t dv[kReorgPerLane];
#pragma unroll
  for (int r = 0; r < kReorgPerLane; r++) {
    const uint64_t i = wbase + r * 32 + lane;
    kv[r] = i < n ? keys[i] : K(0);
  }
  // count: lanes of a round with the same destination (match_any) are
  // counted once by their lowest lane; the warp owns its row, so the
  // increments need no atomics
#pragma unroll
  for (int r = 0; r < kReorgPerLane; r++) {
    const bool ok = wbase + r * 32 + lane < n;
    dv[r] = ok ? dest_of_bin(div_by(hash_mod(kv[r], hp), bin), s_splits, shards) : 0xffffffffu;
    const uint32_t peers = __match_any_sync(0xffffffffu, dv[r]);
    if (ok && (peers & lt) == 0) my[dv[r]] += __popc(peers);
    __syncwarp();
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
  // place: a round's lanes with the same destination take consecutive slots
  // in lane order after the warp's cursor (stable: rounds, then lanes, in
  // input order)
  unsigned long long gsl[kGather ? kReorgPerLane : 1];
#pragma unroll
  for (int r = 0; r < kReorgPerLane; r++) {
    const uint32_t d = dv[r];
    const bool ok = d != 0xffffffffu;
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    const uint32_t cur = ok ? my[d] : 0u;
    __syncwarp();
    if (ok && (peers & lt) == 0) my[d] = cur + __popc(peers);
    __syncwarp();
    if (ok) {
      const uint32_t rank = cur + __popc(peers & lt);
      const unsigned long long slot = s_base[d] + rank;
      if (kGather) {
        gsl[r % (kGather ? kReorgPerLane : 1)] = slot;  // loaded after the loop: all rounds' gathers in flight at once
      } else {
        if (kPeer) reinterpret_cast<K*>(dest_ptrs[d])[s_rbase[d] + rank] = kv[r];
        else grouped[slot] = kv[r];
        if (order) order[slot] = (uint32_t)(wbase + r * 32 + lane);
      }
    }
  }
  if (kGather) {
    uint32_t gv[kGather ? kReorgPerLane : 1];
#pragma unroll
    for (int r = 0; r < kReorgPerLane; r++)
      if (dv[r] != 0xffffffffu) gv[r % (kGather ? kReorgPerLane : 1)] = __ldcs(gvals + gsl[r % (kGather ? kReorgPerLane : 1)]);
#pragma unroll
    for (int r = 0; r < kReorgPerLane; r++)
      if (dv[r] != 0xffffffffu) gout[wbase + r * 32 + lane] = gv[r % (kGather ? kReorgPerLane : 1)];
  }
  if (kPeer) __threadfence_system();  // peer stores ordered before the barrier that publishes them
}

// Routing without a count pass (the distributed build and query): per tile,
// each key's destination and its rank among the warp's keys for that
// destination (match_any), per-warp prefix, then ONE global claim per
// (tile, destination) on cursors[d]; the key goes to slot dest_base[d] +
// claim (peer memory, kPeer) or row_offsets[d] + claim (local grouped
// buffer), and order[row_offsets[d] + claim] = its input index.  Each warp
// round writes a contiguous run per destination.  Rows hold the right keys
// but not in input order (claims race), which the local build and the
// positional query merge do not need; the reference-order API
// (hg_reorganize) keeps the stable two-pass kernels.  (Staging the tile in
// smem to write one run per destination measured slower.)
//
// MAXP > 0 (P <= MAXP, the GPU count of a node): ranks come from one ballot
// per destination per round with warp-uniform running counts in registers --
// no smem traffic or warp syncs per round; MAXP == 0 uses match_any.
template <typename K, bool kPeer, int MAXP>
__global__ void __launch_bounds__(kReorgWarps * 32)
k_route_claim(const K* __restrict__ keys, uint64_t n, HashParams hp, DivParams bin, const long long* __restrict__ splits,
              uint32_t shards, const unsigned long long* __restrict__ row_offsets,
              const unsigned long long* __restrict__ dest_ptrs, const unsigned long long* __restrict__ dest_base,
              K* __restrict__ grouped, uint32_t* __restrict__ order, unsigned long long* __restrict__ cursors) {
  extern __shared__ unsigned char s_raw[];
  long long* s_splits = reinterpret_cast<long long*>(s_raw);
  unsigned long long* s_tb = reinterpret_cast<unsigned long long*>(s_splits + shards + 1);  // claim base per d
  uint32_t* s_wcnt = reinterpret_cast<uint32_t*>(s_tb + shards);                              // [warps][shards]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t lt = lanemask_lt();
  for (uint32_t i = threadIdx.x; i <= shards; i += blockDim.x) s_splits[i] = splits[i];
  for (uint32_t i = threadIdx.x; i < kReorgWarps * shards; i += blockDim.x) s_wcnt[i] = 0;
  const uint64_t wbase = (uint64_t)blockIdx.x * kReorgTile + (uint64_t)warp * 32 * kReorgPerLane;
  K kv[kReorgPerLane];
#pragma unroll
  for (int r = 0; r < kReorgPerLane; r++) {
    const uint64_t i = wbase + r * 32 + lane;
    kv[r] = i < n ? keys[i] : K(0);
  }
  __syncthreads();
  uint32_t* my = s_wcnt + warp * shards;
  uint32_t dr[kReorgPerLane];  // destination << 16 | rank inside the warp's keys for it (or ~0)
  if (MAXP > 0) {
    uint32_t cnt[MAXP > 0 ? MAXP : 1];
#pragma unroll
    for (int dd = 0; dd < MAXP; dd++) cnt[dd] = 0;
#pragma unroll
    for (int r = 0; r < kReorgPerLane; r++) {
      const bool ok = wbase + r * 32 + lane < n;
      const uint32_t d = ok ? (shards == 1 ? 0u : dest_of_bin(div_by(hash_mod(kv[r], hp), bin), s_splits, shards))
                            : 0xffffffffu;
      uint32_t rank = 0;
#pragma unroll
      for (int dd = 0; dd < MAXP; dd++) {
        if ((uint32_t)dd < shards) {
          const uint32_t m = __ballot_sync(0xffffffffu, d == (uint32_t)dd);
          if (d == (uint32_t)dd) rank = cnt[dd] + __popc(m & lt);
          cnt[dd] += __popc(m);
        }
      }
      dr[r] = ok ? (d << 16) | rank : 0xffffffffu;
    }
    if (lane == 0) {
#pragma unroll
      for (int dd = 0; dd < MAXP; dd++)
        if ((uint32_t)dd < shards) my[dd] = cnt[dd];
    }
  } else {
#pragma unroll
    for (int r = 0; r < kReorgPerLane; r++) {
      const bool ok = wbase + r * 32 + lane < n;
      const uint32_t d = ok ? dest_of_bin(div_by(hash_mod(kv[r], hp), bin), s_splits, shards) : 0xffffffffu;
      const uint32_t peers = __match_any_sync(0xffffffffu, d);
      const uint32_t cur = ok ? my[d] : 0u;
      __syncwarp();
      if (ok && (peers & lt) == 0) my[d] = cur + __popc(peers);
      __syncwarp();
      dr[r] = ok ? (d << 16) | (cur + __popc(peers & lt)) : 0xffffffffu;
    }
  }
  __syncthreads();
  __shared__ uint32_t s_cnt[MAXP > 0 ? MAXP : 1], s_toff[MAXP > 0 ? MAXP : 1];
  for (uint32_t d = threadIdx.x; d < shards; d += blockDim.x) {
    uint32_t run = 0;
    for (int w = 0; w < kReorgWarps; w++) {
      const uint32_t c = s_wcnt[w * shards + d];
      s_wcnt[w * shards + d] = run;
      run += c;
    }
    s_tb[d] = run ? atomicAdd(cursors + d, (unsigned long long)run) : 0ull;
    if (MAXP > 0) s_cnt[d] = run;
  }
  __syncthreads();
  if (MAXP > 0) {
    // P <= 8: the tile's keys are staged destination-major in smem and every
    // destination's run leaves as consecutive lanes' stores (full 32-byte
    // sectors on NVLink / HBM) instead of one scattered store per key
    K* st_k = reinterpret_cast<K*>(s_wcnt + kReorgWarps * shards);
    uint32_t* st_o = reinterpret_cast<uint32_t*>(st_k + kReorgTile);
    if (threadIdx.x == 0) {
      uint32_t acc = 0;
      for (uint32_t d = 0; d < shards; d++) {
        s_toff[d] = acc;
        acc += s_cnt[d];
      }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kReorgPerLane; r++) {
      if (dr[r] == 0xffffffffu) continue;
      const uint32_t d = dr[r] >> 16;
      const uint32_t slot = s_toff[d] + my[d] + (dr[r] & 0xFFFFu);
      st_k[slot] = kv[r];
      if (order) st_o[slot] = (uint32_t)(wbase + r * 32 + lane);
    }
    __syncthreads();
    const uint32_t total = s_toff[shards - 1] + s_cnt[shards - 1];
    for (uint32_t i = threadIdx.x; i < total; i += blockDim.x) {  // consecutive threads: consecutive slots of a run
      uint32_t d = 0;
#pragma unroll
      for (int dd = 1; dd < MAXP; dd++)
        if ((uint32_t)dd < shards && i >= s_toff[dd]) d = dd;
      const unsigned long long c = s_tb[d] + (i - s_toff[d]);
      if (kPeer) reinterpret_cast<K*>(dest_ptrs[d])[dest_base[d] + c] = st_k[i];
      else grouped[row_offsets[d] + c] = st_k[i];
      if (order) order[row_offsets[d] + c] = st_o[i];
    }
  } else {
#pragma unroll
    for (int r = 0; r < kReorgPerLane; r++) {
      if (dr[r] == 0xffffffffu) continue;
      const uint32_t d = dr[r] >> 16;
      const unsigned long long c = s_tb[d] + my[d] + (dr[r] & 0xFFFFu);
      if (kPeer) reinterpret_cast<K*>(dest_ptrs[d])[dest_base[d] + c] = kv[r];
      else grouped[row_offsets[d] + c] = kv[r];
      if (order) order[row_offsets[d] + c] = (uint32_t)(wbase + r * 32 + lane);
    }
  }
  if (kPeer) __threadfence_system();
}

// Reverse exchange over peer memory: element i of this rank's receive order
// belongs to sender s with recv_bounds[s] <= i < recv_bounds[s+1]; its value
// goes to sender s's buffer back_ptrs[s] at back_base[s] + (i - recv_bounds[s])
// (the sender's grouped position of that key).  Contiguous per sender, so the
// peer stores coalesce.
__global__ void k_return_peers(const uint32_t* __restrict__ vals, uint64_t n, const unsigned long long* __restrict__ recv_bounds,
                               const unsigned long long* __restrict__ back_ptrs,
                               const unsigned long long* __restrict__ back_base, uint32_t shards) {
  extern __shared__ unsigned long long s_rb[];  // recv_bounds (P+1), back_base (P), back_ptrs (P)
  for (uint32_t i = threadIdx.x; i <= shards; i += blockDim.x) s_rb[i] = recv_bounds[i];
  for (uint32_t i = threadIdx.x; i < shards; i += blockDim.x) {
    s_rb[shards + 1 + i] = back_base[i];
    s_rb[2 * shards + 1 + i] = back_ptrs[i];
  }
  __syncthreads();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t lo = 0, hi = shards;  // last s with recv_bounds[s] <= i
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (s_rb[mid] <= i) lo = mid; else hi = mid;
    }
    reinterpret_cast<uint32_t*>(s_rb[2 * shards + 1 + lo])[s_rb[shards + 1 + lo] + (i - s_rb[lo])] = vals[i];
  }
}

// --------------------------------------------------------------------------- utilities

__global__ void k_scatter_u32(const uint32_t* __restrict__ src, const uint32_t* __restrict__ order, uint64_t n,
                              uint32_t* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += 4 * stride) {
    uint32_t o[4], v[4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const uint64_t j = i + u * stride;
      o[u] = j < n ? __ldcs(order + j) : 0u;
      v[u] = j < n ? __ldcs(src + j) : 0u;
    }
#pragma unroll
    for (int u = 0; u < 4; u++)
      if (i + u * stride < n) out[o[u]] = v[u];
  }
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

// Count pass + column scan + row offsets; tile bases stay in the workspace for
// the place pass (hg_reorganize or hg_reorganize_place_peers).
static int reorg_count(const void* keys, uint64_t n, int key_bits, const HashParams& hp, const DivParams& dp,
                       const int64_t* splits, uint32_t shards, uint64_t* row_offsets, uint64_t* search_steps,
                       uint32_t* tile_counts, unsigned long long* totals, cudaStream_t s) {
  const uint64_t tiles = (n + kReorgTile - 1) / kReorgTile;
  const size_t smem_c = 8 * (shards + 1) + 4 * shards;
  if (key_bits == 32)
    HG_SET_SMEM((k_reorg_count<uint32_t>), (int)smem_c);
  else
    HG_SET_SMEM((k_reorg_count<uint64_t>), (int)smem_c);
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
  return HG_OK;
}

template <bool kPeer>
static int reorg_place(const void* keys, uint64_t n, int key_bits, const HashParams& hp, const DivParams& dp,
                       const int64_t* splits, uint32_t shards, const uint32_t* tile_counts, const uint64_t* row_offsets,
                       void* grouped, uint32_t* order, const uint64_t* dest_ptrs, const uint64_t* dest_base,
                       cudaStream_t s) {
  const uint64_t tiles = (n + kReorgTile - 1) / kReorgTile;
  const size_t smem_p = 8 * (shards + 1) + 8 * shards * (kPeer ? 2 : 1) + 4 * kReorgWarps * shards;
  const auto* ro = (const unsigned long long*)row_offsets;
  const auto* dp_ = (const unsigned long long*)dest_ptrs;
  const auto* db = (const unsigned long long*)dest_base;
  // up to 224 KB at 4096 shards (reorg_check bounds the shard count by the opt-in limit)
  if (key_bits == 32)
    HG_SET_SMEM((k_reorg_place<uint32_t, kPeer>), (int)smem_p);
  else
    HG_SET_SMEM((k_reorg_place<uint64_t, kPeer>), (int)smem_p);
  if (key_bits == 32) {
    HG_LAUNCH("hg_reorg_place", (k_reorg_place<uint32_t, kPeer>), (unsigned)tiles, kReorgWarps * 32, smem_p, s,
              (const uint32_t*)keys, n, hp, dp, (const long long*)splits, shards, tile_counts, ro, (uint32_t*)grouped,
              order, dp_, db);
  } else {
    HG_LAUNCH("hg_reorg_place", (k_reorg_place<uint64_t, kPeer>), (unsigned)tiles, kReorgWarps * 32, smem_p, s,
              (const uint64_t*)keys, n, hp, dp, (const long long*)splits, shards, tile_counts, ro, (uint64_t*)grouped,
              order, dp_, db);
  }
  return HG_OK;
}

// Per-row values back to input order (kGather): the tile bases of the
// count pass that produced row_offsets are still in the workspace.
static int reorg_gather(const void* keys, uint64_t n, int key_bits, const HashParams& hp, const DivParams& dp,
                        const int64_t* splits, uint32_t shards, const uint32_t* tile_counts, const uint64_t* row_offsets,
                        const uint32_t* vals, uint32_t* out, cudaStream_t s) {
  const uint64_t tiles = (n + kReorgTile - 1) / kReorgTile;
  const size_t smem_p = 8 * (shards + 1) + 8 * shards + 4 * kReorgWarps * shards;
  const auto* ro = (const unsigned long long*)row_offsets;
  if (key_bits == 32) {
    HG_SET_SMEM((k_reorg_place<uint32_t, false, true>), (int)smem_p);
    HG_LAUNCH("hg_reorg_gather", (k_reorg_place<uint32_t, false, true>), (unsigned)tiles, kReorgWarps * 32, smem_p, s,
              (const uint32_t*)keys, n, hp, dp, (const long long*)splits, shards, tile_counts, ro, nullptr, nullptr,
              nullptr, nullptr, vals, out);
  } else {
    HG_SET_SMEM((k_reorg_place<uint64_t, false, true>), (int)smem_p);
    HG_LAUNCH("hg_reorg_gather", (k_reorg_place<uint64_t, false, true>), (unsigned)tiles, kReorgWarps * 32, smem_p, s,
              (const uint64_t*)keys, n, hp, dp, (const long long*)splits, shards, tile_counts, ro, nullptr, nullptr,
              nullptr, nullptr, vals, out);
  }
  return HG_OK;
}

static int reorg_check(int key_bits, int kind, uint64_t hash_range, uint32_t shards, uint64_t bin_size, uint64_t n) {
  int rc = check_hash(key_bits, kind, hash_range);
  if (rc) return rc;
  if (shards < 1 || shards > 4096) return set_error(HG_ERR_CONFIG, "shard count must be in [1, 4096], got %u", shards);
  // k_reorg_place's peer variant stages 8 (P+1) + 16 P + 4 * warps * P bytes of shared memory
  const size_t need = 8 * ((size_t)shards + 1) + 16 * (size_t)shards + 4 * (size_t)kReorgWarps * shards;
  if (need > (size_t)max_dyn_smem())
    return set_error(HG_ERR_CONFIG, "%u shards need %zu bytes of shared memory per CTA (limit %d)", shards, need, max_dyn_smem());
  if (bin_size < 1) return set_error(HG_ERR_CONFIG, "bin_size must be >= 1");
  if (n >= (1ull << 32)) return set_error(HG_ERR_CONFIG, "a shard holds fewer than 2^32 keys");
  return HG_OK;
}

// hg_route's launch: the ballot-ranked kernel sized to the shard count when
// it is a node's GPU count (<= 8), the match_any kernel beyond.
template <typename K, bool kPeer>
static int route_launch(const K* keys, uint64_t n, const HashParams& hp, const DivParams& dp, const long long* sp,
                        uint32_t shards, const unsigned long long* ro, const unsigned long long* dpt,
                        const unsigned long long* db, K* grouped, uint32_t* order, unsigned long long* cur,
                        uint64_t tiles, size_t smem, cudaStream_t s) {
  auto go = [&](auto kern) -> int {
    HG_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));  // runtime pointer
    HG_LAUNCH("hg_route", kern, (unsigned)tiles, kReorgWarps * 32, smem, s, keys, n, hp, dp, sp, shards, ro, dpt, db,
              grouped, order, cur);
    return HG_OK;
  };
  if (shards == 1) return go(k_route_claim<K, kPeer, 1>);
  if (shards == 2) return go(k_route_claim<K, kPeer, 2>);
  if (shards <= 4) return go(k_route_claim<K, kPeer, 4>);
  if (shards <= 8) return go(k_route_claim<K, kPeer, 8>);
  return go(k_route_claim<K, kPeer, 0>);
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
      HG_SET_SMEM((k_bin_hist<uint32_t>), (int)smem);
    else
      HG_SET_SMEM((k_bin_hist<uint64_t>), (int)smem);
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
  int rc = reorg_check(key_bits, kind, hash_range, shards, bin_size, n);
  if (rc) return rc;
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
  rc = reorg_count(keys, n, key_bits, hp, dp, splits, shards, row_offsets, search_steps, tile_counts, totals, s);
  if (rc) return rc;
  return reorg_place<false>(keys, n, key_bits, hp, dp, splits, shards, tile_counts, row_offsets, grouped, order,
                            nullptr, nullptr, s);
}

int hg_reorganize_gather(const void* keys, uint64_t n, int key_bits, int kind, uint32_t seed, uint64_t hash_range,
                         uint64_t bin_size, const int64_t* splits, uint32_t shards, const uint64_t* row_offsets,
                         const uint32_t* vals, uint32_t* out, const void* workspace, size_t workspace_bytes,
                         void* stream) {
  int rc = reorg_check(key_bits, kind, hash_range, shards, bin_size, n);
  if (rc) return rc;
  if (!n) return HG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  uint64_t tiles = (n + kReorgTile - 1) / kReorgTile;
  Workspace ws{(char*)const_cast<void*>(workspace), workspace_bytes, 0};
  const uint32_t* tile_counts = ws.take<uint32_t>(tiles * shards);  // the carve-up of hg_reorganize
  if (!ws.ok()) return set_error(HG_ERR_CONFIG, "reorganize workspace too small");
  HashParams hp = make_hash_params(kind, seed, hash_range, key_bits);
  DivParams dp = make_div_params(bin_size);
  return reorg_gather(keys, n, key_bits, hp, dp, splits, shards, tile_counts, row_offsets, vals, out, s);
}

int hg_reorganize_count(const void* keys, uint64_t n, int key_bits, int kind, uint32_t seed, uint64_t hash_range,
                        uint64_t bin_size, const int64_t* splits, uint32_t shards, uint64_t* row_offsets,
                        uint64_t* search_steps, void* workspace, size_t workspace_bytes, void* stream) {
  int rc = reorg_check(key_bits, kind, hash_range, shards, bin_size, n);
  if (rc) return rc;
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
  return reorg_count(keys, n, key_bits, hp, dp, splits, shards, row_offsets, search_steps, tile_counts, totals, s);
}

int hg_reorganize_place_peers(const void* keys, uint64_t n, int key_bits, int kind, uint32_t seed,
                              uint64_t hash_range, uint64_t bin_size, const int64_t* splits, uint32_t shards,
                              const uint64_t* row_offsets, const uint64_t* dest_ptrs, const uint64_t* dest_base,
                              uint32_t* order, void* workspace, size_t workspace_bytes, void* stream) {
  int rc = reorg_check(key_bits, kind, hash_range, shards, bin_size, n);
  if (rc) return rc;
  if (!n) return HG_OK;
  if (!dest_ptrs || !dest_base) return set_error(HG_ERR_CONFIG, "dest_ptrs and dest_base are required");
  cudaStream_t s = (cudaStream_t)stream;
  uint64_t tiles = (n + kReorgTile - 1) / kReorgTile;
  Workspace ws{(char*)workspace, workspace_bytes, 0};
  uint32_t* tile_counts = ws.take<uint32_t>(tiles * shards);
  if (!ws.ok()) return set_error(HG_ERR_CONFIG, "reorganize workspace too small");
  HashParams hp = make_hash_params(kind, seed, hash_range, key_bits);
  DivParams dp = make_div_params(bin_size);
  return reorg_place<true>(keys, n, key_bits, hp, dp, splits, shards, tile_counts, row_offsets, nullptr, order,
                           dest_ptrs, dest_base, s);
}

int hg_route(const void* keys, uint64_t n, int key_bits, int kind, uint32_t seed, uint64_t hash_range,
             uint64_t bin_size, const int64_t* splits, uint32_t shards, const uint64_t* row_offsets,
             const uint64_t* dest_ptrs, const uint64_t* dest_base, void* grouped, uint32_t* order, uint64_t* cursors,
             void* stream) {
  int rc = reorg_check(key_bits, kind, hash_range, shards, bin_size, n);
  if (rc) return rc;
  if (shards > 65535) return set_error(HG_ERR_CONFIG, "hg_route supports at most 65535 shards");
  cudaStream_t s = (cudaStream_t)stream;
  HG_CHECK_CUDA(cudaMemsetAsync(cursors, 0, 8 * (size_t)shards, s));
  if (!n) return HG_OK;
  const bool peer = dest_ptrs != nullptr;
  if (peer && !dest_base) return set_error(HG_ERR_CONFIG, "dest_base is required with dest_ptrs");
  if (!peer && !grouped) return set_error(HG_ERR_CONFIG, "grouped is required without dest_ptrs");
  HashParams hp = make_hash_params(kind, seed, hash_range, key_bits);
  DivParams dp = make_div_params(bin_size);
  const uint64_t tiles = (n + kReorgTile - 1) / kReorgTile;
  size_t smem = 8 * (shards + 1) + 8 * (size_t)shards + 4 * (size_t)kReorgWarps * shards;
  if (shards <= 8) smem = (smem + 15) / 16 * 16 + (size_t)kReorgTile * (key_bits / 8 + 4);  // staged keys + input indices
  if (smem > 200 * 1024) return set_error(HG_ERR_CONFIG, "too many shards for hg_route (%u)", shards);
  const auto* ro = (const unsigned long long*)row_offsets;
  const auto* dpt = (const unsigned long long*)dest_ptrs;
  const auto* db = (const unsigned long long*)dest_base;
  auto* cur = (unsigned long long*)cursors;
  const auto* sp = (const long long*)splits;
  if (key_bits == 32) {
    if (peer) return route_launch<uint32_t, true>((const uint32_t*)keys, n, hp, dp, sp, shards, ro, dpt, db, (uint32_t*)grouped, order, cur, tiles, smem, s);
    return route_launch<uint32_t, false>((const uint32_t*)keys, n, hp, dp, sp, shards, ro, dpt, db, (uint32_t*)grouped, order, cur, tiles, smem, s);
  }
  if (peer) return route_launch<uint64_t, true>((const uint64_t*)keys, n, hp, dp, sp, shards, ro, dpt, db, (uint64_t*)grouped, order, cur, tiles, smem, s);
  return route_launch<uint64_t, false>((const uint64_t*)keys, n, hp, dp, sp, shards, ro, dpt, db, (uint64_t*)grouped, order, cur, tiles, smem, s);
}

int hg_return_peers(const uint32_t* vals, uint64_t n, const uint64_t* recv_bounds, const uint64_t* back_ptrs,
                    const uint64_t* back_base, uint32_t shards, void* stream) {
  if (shards < 1 || shards > 4096) return set_error(HG_ERR_CONFIG, "shard count must be in [1, 4096], got %u", shards);
  // k_reorg_place's peer variant stages 8 (P+1) + 16 P + 4 * warps * P bytes of shared memory
  const size_t need = 8 * ((size_t)shards + 1) + 16 * (size_t)shards + 4 * (size_t)kReorgWarps * shards;
  if (need > (size_t)max_dyn_smem())
    return set_error(HG_ERR_CONFIG, "%u shards need %zu bytes of shared memory per CTA (limit %d)", shards, need, max_dyn_smem());
  if (!n) return HG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  HG_LAUNCH("hg_return_peers", k_return_peers, grid_cap(n, 8), kT, 8 * (3 * (size_t)shards + 1), s, vals, n,
            (const unsigned long long*)recv_bounds, (const unsigned long long*)back_ptrs,
            (const unsigned long long*)back_base, shards);
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
