// hg_bigbin.cuh -- fine bins too large for shared memory (high-duplicate and
// skewed inputs).  Part of hg_binned.cu (textually included inside its
// namespace hg, after its block helpers); split out for size.
//
// A fine bin holds more than kCap keys only when many keys share few buckets:
// all-identical keys, Zipf-like hot keys, or a hash range far below the key
// count (acceptance c05/c06 sweep the duplicate rate, test_acceptance.py:
// 160-196; the paper claims build throughput flat across it).
// Such a bin must not serialise on one SM, so both sides work in chunks that
// every CTA of the grid shares:
//
//   build   k_starts     lists the oversized bins: medium (<= kHugeBin keys)
//                        and huge ones, the huge ones' chunk prefix
//           k_local_build_p  zeroes the huge bins' bucket counters (= their
//                        offsets slice)
//           k_big_count  medium bin: one CTA counts, scans and places it
//                        (smem counters, two passes over its keys);
//                        huge-bin chunk: smem counts, one global add per
//                        bucket; the CTA finishing a bin's last chunk turns
//                        its counts into bucket starts
//           k_big_place  huge-bin chunk: smem ranks, one global claim per
//                        bucket, keys stored at claim + rank; the CTA
//                        finishing a bin's last chunk shifts the claimed ends
//                        to starts
//   query   k_probe_plan per fine bin: extra probe work items for hot bins,
//                        the list of bins whose table slice is oversized
//           k_ht_prep    key -> count hash table for those bins (cleared),
//                        their table-key / query prefixes
//           k_ht_insert  their table keys, runs and warp peers aggregated
//           k_ht_lookup  their queries: count from the table, comparisons
//                        from the bucket degree (query.py:153-155)
// ============================================================================ build

template <typename K>
struct BigShape {
  static constexpr int kThreads = 1024;
  static constexpr int kKPT = sizeof(K) == 4 ? 16 : 8;  // keys per thread per chunk (registers)
  static constexpr uint32_t kChunk = kKPT * kThreads;
};

// Locate chunk k: bin index j, fine bin f, key range [lo, hi), chunks of j.
__device__ __forceinline__ void big_chunk(uint32_t k, uint32_t nbig, uint32_t CH, const uint32_t* __restrict__ big_cp,
                                          const uint32_t* __restrict__ huge_list, const uint32_t* __restrict__ fine_start,
                                          uint32_t* s_loc) {
  if (threadIdx.x == 0) {
    const uint32_t j = upper_index(big_cp, nbig, k);
    const uint32_t f = *(huge_list - j);  // the huge list grows downwards
    const uint32_t lo = fine_start[f] + (k - big_cp[j]) * CH;
    s_loc[0] = f;
    s_loc[1] = lo;
    s_loc[2] = min(fine_start[f + 1], lo + CH);
    s_loc[3] = j;
    s_loc[4] = big_cp[j + 1] - big_cp[j];
  }
  __syncthreads();
}

// True in every thread of the CTA that completed the last of `nchunks`
// chunks of bin j (done[j] counts completed chunks; zeroed by k_starts).
// The CTA's global writes and atomics are fenced before the count, and the
// winner fences again before it reads the others' results.
__device__ __forceinline__ bool last_chunk(uint32_t* done, uint32_t j, uint32_t nchunks) {
  __shared__ uint32_t s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(done + j, 1u) == nchunks - 1;
    if (s_last) __threadfence();
  }
  __syncthreads();
  return s_last != 0;
}

// Per chunk: count keys per bucket in smem (lanes of a warp that hit the same
// bucket share one atomic), then add the nonzero counters to the bin's global
// counters (its offsets slice, zeroed by k_local_build_p).  The CTA that
// completes a bin's last chunk scans the counts into bucket starts.  `copy`
// (two partition levels: the grouped keys sit in `edges`) also copies the
// chunk to `dst` so placement can overwrite edges.
// A medium oversized bin [lo, hi) (kCap < keys <= kHugeBin), whole, by one
// CTA: smem counters for its 2^s buckets, a counting pass (lanes of a warp
// that hit the same bucket share one atomic; `copy` also copies the keys to
// `dst`), the scan into offsets, and a placing pass whose atomics return each
// key's slot.
template <typename H>
__device__ __forceinline__ void big_medium(const KeyOf<H>* __restrict__ src, KeyOf<H>* __restrict__ dst, int copy,
                                           uint32_t lo, uint32_t hi, uint64_t first, const HashParams& hp, int s,
                                           uint64_t v, uint32_t* cnt, uint32_t* __restrict__ offsets,
                                           KeyOf<H>* __restrict__ edges, const uint32_t* __restrict__ a2,
                                           uint32_t* __restrict__ positions) {
  using K = KeyOf<H>;
  const uint32_t nb = (uint32_t)min((uint64_t)1 << s, v - first);
  const uint32_t lt = lanemask_lt();
  for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  constexpr int U = BigShape<K>::kKPT;  // keys per thread per round (a bin of <= kChunk keys: one round)
  const uint32_t step = U * blockDim.x;
  for (uint32_t r0 = lo; r0 < hi; r0 += step) {
    K kv[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint32_t e = r0 + u * blockDim.x + threadIdx.x;
      kv[u] = e < hi ? src[e] : K(0);
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint32_t e = r0 + u * blockDim.x + threadIdx.x;
      const bool ok = e < hi;
      if (ok && copy) dst[e] = kv[u];
      const uint32_t l = ok ? H::bucket(kv[u], hp) - (uint32_t)first : 0xFFFFFFFFu;
      const uint32_t peers = __match_any_sync(0xffffffffu, l);
      if (ok && (peers & lt) == 0) atomicAdd(cnt + l, (uint32_t)__popc(peers));
    }
  }
  __syncthreads();
  block_exscan_rows(cnt, nb, lo);
  for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) offsets[first + i] = cnt[i];
  __syncthreads();
  const K* from = copy ? dst : src;
  for (uint32_t r0 = lo; r0 < hi; r0 += step) {
    K kv[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint32_t e = r0 + u * blockDim.x + threadIdx.x;
      kv[u] = e < hi ? from[e] : K(0);
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      const bool ok = r0 + u * blockDim.x + threadIdx.x < hi;
      const uint32_t l = ok ? H::bucket(kv[u], hp) - (uint32_t)first : 0xFFFFFFFFu;
      const uint32_t peers = __match_any_sync(0xffffffffu, l);
      uint32_t b0 = 0;
      if (ok && (peers & lt) == 0) b0 = atomicAdd(cnt + l, (uint32_t)__popc(peers));
      b0 = __shfl_sync(0xffffffffu, b0, __ffs(peers) - 1);
      if (ok) {
        const uint32_t slot = b0 + __popc(peers & lt);
        edges[slot] = kv[u];
        if (a2) {  // traced build
          const uint32_t e = r0 + u * blockDim.x + threadIdx.x;
          positions[slot] = a2[e];
        }
      }
    }
  }
  __syncthreads();
}

template <typename H>
__global__ void __launch_bounds__(1024) k_big_count(const KeyOf<H>* __restrict__ src, KeyOf<H>* __restrict__ dst, int copy,
                                                    const uint32_t* __restrict__ fine_start, const uint32_t* __restrict__ big_list,
                                                    const uint32_t* __restrict__ huge_list,
                                                    const uint32_t* __restrict__ big_count, const uint32_t* __restrict__ big_cp,
                                                    uint32_t* __restrict__ done, HashParams hp, int s, uint64_t v,
                                                    uint32_t* __restrict__ offsets, KeyOf<H>* __restrict__ edges,
                                                    const uint32_t* __restrict__ a2, uint32_t* __restrict__ positions) {
  using K = KeyOf<H>;
  using BS = BigShape<K>;
  extern __shared__ uint32_t cnt[];  // 2^s
  __shared__ uint32_t s_loc[5];
  const uint32_t nmed = big_count[0], nbig = big_count[1];
  const uint32_t nch = nbig ? big_cp[nbig] : 0u;
  const uint32_t lt = lanemask_lt();
  for (uint32_t k = blockIdx.x; k < nmed; k += gridDim.x) {
    const uint32_t f = big_list[k];
    big_medium<H>(src, dst, copy, fine_start[f], fine_start[f + 1], (uint64_t)f << s, hp, s, v, cnt, offsets, edges, a2,
                  positions);
  }
  for (uint32_t k = blockIdx.x; k < nch; k += gridDim.x) {
    big_chunk(k, nbig, BS::kChunk, big_cp, huge_list, fine_start, s_loc);
    const uint32_t f = s_loc[0], lo = s_loc[1], hi = s_loc[2], j = s_loc[3], nck = s_loc[4];
    const uint64_t first = (uint64_t)f << s;
    const uint32_t nb = (uint32_t)min((uint64_t)1 << s, v - first);
    for (uint32_t l = threadIdx.x; l < nb; l += blockDim.x) cnt[l] = 0;
    __syncthreads();
    K kv[BS::kKPT];
#pragma unroll
    for (int u = 0; u < BS::kKPT; u++) {
      const uint32_t e = lo + u * BS::kThreads + threadIdx.x;
      kv[u] = e < hi ? src[e] : K(0);
    }
#pragma unroll
    for (int u = 0; u < BS::kKPT; u++) {
      const uint32_t e = lo + u * BS::kThreads + threadIdx.x;
      const bool ok = e < hi;
      if (ok && copy) dst[e] = kv[u];
      const uint32_t l = ok ? H::bucket(kv[u], hp) - (uint32_t)first : 0xFFFFFFFFu;
      const uint32_t peers = __match_any_sync(0xffffffffu, l);
      if (ok && (peers & lt) == 0) atomicAdd(cnt + l, (uint32_t)__popc(peers));
    }
    __syncthreads();
    for (uint32_t l = threadIdx.x; l < nb; l += blockDim.x)
      if (cnt[l]) atomicAdd(offsets + first + l, cnt[l]);
    if (last_chunk(done, j, nck)) {
      for (uint32_t l = threadIdx.x; l < nb; l += blockDim.x) cnt[l] = __ldcg(offsets + first + l);
      __syncthreads();
      block_exscan_rows(cnt, nb, fine_start[f]);
      for (uint32_t l = threadIdx.x; l < nb; l += blockDim.x) offsets[first + l] = cnt[l];
    }
    __syncthreads();
  }
}

// Per chunk: ranks from smem counters (warp peers share one atomic), one
// global claim per nonzero bucket (the offsets slice is the cursor), then
// every key stored at claim + rank; in-bucket order is free (core.py:12-14).
// After a bin's last chunk every cursor holds its bucket's end = the next
// bucket's start; the CTA that completed it shifts them back by one bucket.
template <typename H>
__global__ void __launch_bounds__(1024) k_big_place(const KeyOf<H>* __restrict__ src, const uint32_t* __restrict__ fine_start,
                                                    const uint32_t* __restrict__ huge_list, const uint32_t* __restrict__ big_count,
                                                    const uint32_t* __restrict__ big_cp, uint32_t* __restrict__ done,
                                                    HashParams hp, int s, uint64_t v, uint32_t* __restrict__ offsets,
                                                    KeyOf<H>* __restrict__ edges, const uint32_t* __restrict__ a2,
                                                    uint32_t* __restrict__ positions) {
  using K = KeyOf<H>;
  using BS = BigShape<K>;
  extern __shared__ uint32_t cnt[];  // 2^s
  __shared__ uint32_t s_loc[5];
  const uint32_t nbig = big_count[1];
  if (nbig == 0) return;
  const uint32_t nch = big_cp[nbig];
  const uint32_t lt = lanemask_lt();
  for (uint32_t k = blockIdx.x; k < nch; k += gridDim.x) {
    big_chunk(k, nbig, BS::kChunk, big_cp, huge_list, fine_start, s_loc);
    const uint32_t f = s_loc[0], lo = s_loc[1], hi = s_loc[2], j = s_loc[3], nck = s_loc[4];
    const uint64_t first = (uint64_t)f << s;
    const uint32_t nb = (uint32_t)min((uint64_t)1 << s, v - first);
    for (uint32_t l = threadIdx.x; l < nb; l += blockDim.x) cnt[l] = 0;
    __syncthreads();
    K kv[BS::kKPT];
    uint32_t lr[BS::kKPT];  // bucket << 15 | rank (bucket < 2^14, rank < kChunk <= 2^14)
#pragma unroll
    for (int u = 0; u < BS::kKPT; u++) {
      const uint32_t e = lo + u * BS::kThreads + threadIdx.x;
      kv[u] = e < hi ? src[e] : K(0);
    }
#pragma unroll
    for (int u = 0; u < BS::kKPT; u++) {
      const uint32_t e = lo + u * BS::kThreads + threadIdx.x;
      const bool ok = e < hi;
      const uint32_t l = ok ? H::bucket(kv[u], hp) - (uint32_t)first : 0xFFFFFFFFu;
      const uint32_t peers = __match_any_sync(0xffffffffu, l);
      uint32_t b0 = 0;
      if (ok && (peers & lt) == 0) b0 = atomicAdd(cnt + l, (uint32_t)__popc(peers));
      b0 = __shfl_sync(0xffffffffu, b0, __ffs(peers) - 1);
      lr[u] = ok ? (l << 15) | (b0 + __popc(peers & lt)) : 0xFFFFFFFFu;
    }
    __syncthreads();
    for (uint32_t l = threadIdx.x; l < nb; l += blockDim.x) {
      const uint32_t c = cnt[l];
      if (c) cnt[l] = atomicAdd(offsets + first + l, c);
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < BS::kKPT; u++)
      if (lr[u] != 0xFFFFFFFFu) {
        const uint32_t slot = cnt[lr[u] >> 15] + (lr[u] & 0x7FFFu);
        edges[slot] = kv[u];
        if (a2) {  // traced build
          const uint32_t e = lo + u * BS::kThreads + threadIdx.x;
          positions[slot] = a2[e];
        }
      }
    if (last_chunk(done, j, nck)) {
      for (uint32_t l = threadIdx.x; l < nb; l += blockDim.x) cnt[l] = __ldcg(offsets + first + l);
      __syncthreads();
      for (uint32_t l = threadIdx.x; l < nb; l += blockDim.x) offsets[first + l] = l ? cnt[l - 1] : fine_start[f];
    }
    __syncthreads();
  }
}

// ============================================================================ query

// plan words (uint64, zeroed by k_starts): extra probe items, hash-table bins,
// their table keys, their queries, hash-table capacity, all-ones-key count
enum : int { kPlanItems = 0, kPlanBig, kPlanBigT, kPlanBigQ, kPlanCap, kPlanOnes, kPlanWords };
constexpr uint32_t kProbeChunk = 32768;  // queries per shared-memory probe work item

// One thread per fine bin f with queries (tn table keys, qn queries).  A bin
// whose table slice fits smem (or a medium slice, <= 4 kCap keys: the slice
// map) is probed by CTA f (its first kProbeChunk queries) plus one extra work
// item per further chunk (item = the pair f, c); a larger slice goes to the
// hash-table path (big_bin list; k_local_probe adds medium slices with too
// many distinct keys).  List order is free: every consumer works from the
// lists as written.
__global__ void k_probe_plan(const uint32_t* __restrict__ t_off, const uint32_t* __restrict__ q_start, uint32_t nfine,
                             int s, uint64_t v, uint32_t cap, uint32_t* __restrict__ item_x, uint32_t* __restrict__ big_bin,
                             unsigned long long* __restrict__ plan) {
  const uint32_t f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= nfine) return;
  const uint32_t qn = q_start[f + 1] - q_start[f];
  if (qn == 0) return;
  const uint32_t tn = t_off[min((uint64_t)(f + 1) << s, v)] - t_off[(uint64_t)f << s];
  if (tn > 4 * cap) {  // above kMapSlice = 4 kCap: the slice is too long to stream per work item
    big_bin[atomicAdd(plan + kPlanBig, 1ull)] = f;
    atomicAdd(plan + kPlanBigT, (unsigned long long)tn);
    atomicAdd(plan + kPlanBigQ, (unsigned long long)qn);
  } else if (qn > kProbeChunk) {
    const uint32_t k = (qn + kProbeChunk - 1) / kProbeChunk;
    const uint32_t base = (uint32_t)atomicAdd(plan + kPlanItems, (unsigned long long)(k - 1));
    for (uint32_t c = 1; c < k; c++) {  // item = (bin, chunk) word pair
      item_x[2 * (base + c - 1)] = f;
      item_x[2 * (base + c - 1) + 1] = c;
    }
  }
}

// slot hash of the key -> count tables (independent of the bucket hash)
__device__ __forceinline__ uint64_t ht_slot_mix(uint64_t key) {
  return fmix64(key * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull);
}

__device__ __forceinline__ uint32_t cas_key(uint32_t* p, uint32_t cmp, uint32_t val) { return atomicCAS(p, cmp, val); }
__device__ __forceinline__ uint64_t cas_key(uint64_t* p, uint64_t cmp, uint64_t val) {
  return atomicCAS(reinterpret_cast<unsigned long long*>(p), (unsigned long long)cmp, (unsigned long long)val);
}

// ---- medium table slices (kCap < keys <= kMapSlice): the probe CTA cannot
// stage the slice, but high-duplicate slices (few distinct keys, e.g. C3) fit
// a key -> count map in shared memory, built by streaming the slice (its
// equal keys are adjacent: a bucket's keys are contiguous in the CSR) and
// answering every query with one lookup.  A slice with more distinct keys
// than half the map goes to the global hash table instead.
template <typename K>
struct SliceMapShape {
  static constexpr uint32_t kSlots = sizeof(K) == 4 ? 8192 : 4096;  // fits the probe's smem at any s
};

template <typename K>
__device__ __forceinline__ uint32_t smap_slot(K key) {
  return (uint32_t)ht_slot_mix((uint64_t)key);
}

// Add `add` occurrences of key (all-ones key counted in *ones); false once the
// map holds more than M / 2 distinct keys (the caller flags overflow and stops
// streaming).
template <typename K>
__device__ __forceinline__ bool smap_add(K* mk, uint32_t* mc, uint32_t* claimed, uint32_t* ones, K key, uint32_t add) {
  constexpr uint32_t M = SliceMapShape<K>::kSlots;
  if (key == ~K(0)) {
    atomicAdd(ones, add);
    return true;
  }
  // too many distinct keys: give up early (the caller's final check agrees:
  // claimed only grows, so every work item of the bin decides the same way)
  if (*(volatile uint32_t*)claimed > M / 2) return false;
  uint32_t i = smap_slot(key) & (M - 1);
  // claimed <= M/2 + one pending claim per thread < M here: an empty slot exists
  for (uint32_t probe = 0; probe < M; probe++, i = (i + 1) & (M - 1)) {
    K cur = mk[i];
    if (cur == ~K(0)) {
      cur = cas_key(mk + i, ~K(0), key);
      if (cur == ~K(0)) {
        atomicAdd(claimed, 1u);
        cur = key;
      }
    }
    if (cur == key) {
      atomicAdd(mc + i, add);
      return true;
    }
  }
  return false;
}

template <typename K>
__device__ __forceinline__ uint32_t smap_count(const K* mk, const uint32_t* mc, uint32_t ones, K key) {
  constexpr uint32_t M = SliceMapShape<K>::kSlots;
  if (key == ~K(0)) return ones;
  uint32_t i = smap_slot(key) & (M - 1);
  for (uint32_t probe = 0; probe < M; probe++, i = (i + 1) & (M - 1)) {
    const K cur = mk[i];
    if (cur == key) return mc[i];
    if (cur == ~K(0)) return 0;
  }
  return 0;
}

// The probe of one work item over a medium slice [tlo, thi) of fine bin f.
// Returns false (nothing written) when the slice has too many distinct keys;
// the first chunk's CTA then hands the bin to the hash-table path.
template <typename H>
__device__ __noinline__ bool probe_slice_map(const KeyOf<H>* __restrict__ t_edges, const uint32_t* __restrict__ t_off,
                                             uint32_t tlo, uint32_t thi, const KeyOf<H>* __restrict__ qpart,
                                             uint32_t qlo, uint32_t qhi, const HashParams& hp, unsigned char* smem,
                                             uint32_t* __restrict__ mult_bo, unsigned long long* __restrict__ agg) {
  using K = KeyOf<H>;
  constexpr uint32_t M = SliceMapShape<K>::kSlots;
  K* mk = reinterpret_cast<K*>(smem);
  uint32_t* mc = reinterpret_cast<uint32_t*>(smem + M * sizeof(K));
  __shared__ uint32_t s_claimed, s_ones, s_full;
  for (uint32_t i = threadIdx.x; i < M; i += blockDim.x) {
    mk[i] = ~K(0);
    mc[i] = 0;
  }
  if (threadIdx.x == 0) s_claimed = s_ones = s_full = 0;
  __syncthreads();
  // warp w streams a contiguous range of 32-key rows, 8 rows in flight; each
  // lane counts runs of equal keys and adds a run when its key changes
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint32_t tn = thi - tlo;
  const uint32_t rows = (tn + 31) / 32;
  const uint32_t per = (rows + nw - 1) / nw;
  const uint32_t r0 = warp * per, r1 = min(rows, r0 + per);
  K cur = K(0);
  uint32_t run = 0;
  bool ok = true;
  for (uint32_t r = r0; r < r1 && __all_sync(0xffffffffu, ok); r += 8) {
    K kv[8];
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const uint32_t t = (r + u) * 32 + lane;
      kv[u] = (r + u < r1 && t < tn) ? __ldcs(t_edges + tlo + t) : K(0);
    }
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const uint32_t t = (r + u) * 32 + lane;
      if (r + u < r1 && t < tn) {
        if (run && kv[u] != cur) {
          ok &= smap_add(mk, mc, &s_claimed, &s_ones, cur, run);
          run = 0;
        }
        cur = kv[u];
        run++;
      }
    }
  }
  if (run) ok &= smap_add(mk, mc, &s_claimed, &s_ones, cur, run);
  if (!ok) s_full = 1;
  __syncthreads();
  if (s_full || s_claimed > M / 2) return false;
  const uint32_t ones = s_ones;
  uint64_t matched = 0, total = 0, comps = 0;
  for (uint32_t q0 = qlo; q0 < qhi; q0 += 4 * blockDim.x) {
    K qv[4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const uint32_t j = q0 + u * blockDim.x + threadIdx.x;
      qv[u] = j < qhi ? __ldcs(qpart + j) : K(0);
    }
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const uint32_t j = q0 + u * blockDim.x + threadIdx.x;
      if (j < qhi) {
        const uint32_t h = H::bucket(qv[u], hp);
        const uint32_t c = smap_count(mk, mc, ones, qv[u]);
        mult_bo[j] = c;
        matched += c != 0;
        total += c;
        comps += t_off[(uint64_t)h + 1] - t_off[h];
      }
    }
  }
  if (agg) flush_agg(matched, total, comps, agg);
  return true;
}

template <typename K>
__device__ __forceinline__ uint64_t ht_slot(K key) {
  return ht_slot_mix((uint64_t)key);
}

__device__ __forceinline__ unsigned long long ht_capacity(unsigned long long keys) {
  if (!keys) return 0;
  unsigned long long c = 1024;
  while (c < 2 * keys) c <<= 1;
  return c;
}

// Clear the hash table (capacity = pow2 >= 2x the keys of the hash-table
// bins); CTA 0 also writes the per-bin table-key / query prefixes.
template <typename K>
__global__ void k_ht_prep(unsigned long long* __restrict__ plan, const uint32_t* __restrict__ big_bin,
                          const uint32_t* __restrict__ t_off, const uint32_t* __restrict__ q_start, int s, uint64_t v,
                          uint32_t* __restrict__ big_t, uint32_t* __restrict__ big_q, K* __restrict__ hk,
                          uint32_t* __restrict__ hc) {
  const uint32_t nbig = (uint32_t)plan[kPlanBig];
  if (nbig == 0) return;
  const unsigned long long cap = ht_capacity(plan[kPlanBigT]);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cap; i += (uint64_t)gridDim.x * blockDim.x) {
    hk[i] = ~K(0);
    hc[i] = 0;
  }
  if (blockIdx.x != 0) return;
  if (threadIdx.x == 0) plan[kPlanCap] = cap;
  uint32_t ct = 0, cq = 0;
  for (uint32_t base = 0; base < nbig; base += blockDim.x) {
    const uint32_t j = base + threadIdx.x;
    uint32_t tn = 0, qn = 0;
    if (j < nbig) {
      const uint32_t f = big_bin[j];
      tn = t_off[min((uint64_t)(f + 1) << s, v)] - t_off[(uint64_t)f << s];
      qn = q_start[f + 1] - q_start[f];
    }
    uint32_t tt, tq;
    const uint32_t et = block_scan_excl<uint32_t>(tn, tt);
    const uint32_t eq = block_scan_excl<uint32_t>(qn, tq);
    if (j < nbig) {
      big_t[j] = ct + et;
      big_q[j] = cq + eq;
    }
    ct += tt;
    cq += tq;
  }
  if (threadIdx.x == 0) {
    big_t[nbig] = ct;
    big_q[nbig] = cq;
  }
}

// Add `add` occurrences of `key`.  The all-ones key is the empty marker and is
// counted in plan[kPlanOnes] instead.  Slots never return to empty, so a
// stale read of an empty slot is settled by the CAS.
template <typename K>
__device__ __forceinline__ void ht_add(K* hk, uint32_t* hc, uint64_t cap, K key, uint32_t add, unsigned long long* ones) {
  if (key == ~K(0)) {
    atomicAdd(ones, (unsigned long long)add);
    return;
  }
  uint64_t i = ht_slot(key) & (cap - 1);
  for (;;) {
    K cur = hk[i];
    if (cur == ~K(0)) {
      cur = cas_key(hk + i, ~K(0), key);
      if (cur == ~K(0)) cur = key;
    }
    if (cur == key) {
      atomicAdd(hc + i, add);
      return;
    }
    i = (i + 1) & (cap - 1);
  }
}

template <typename K>
__device__ __forceinline__ uint32_t ht_count(const K* hk, const uint32_t* hc, uint64_t cap, K key, uint32_t ones) {
  if (key == ~K(0)) return ones;
  uint64_t i = ht_slot(key) & (cap - 1);
  for (;;) {
    const K cur = hk[i];
    if (cur == key) return hc[i];
    if (cur == ~K(0)) return 0;
    i = (i + 1) & (cap - 1);
  }
}

constexpr int kHtT = 512;
constexpr int kHtKPT = 8;  // consecutive keys per thread: runs of equal keys are merged before inserting

// Table keys of the hash-table bins.  Each CTA takes chunks of kHtT * kHtKPT
// flattened keys; a bin holds more than `cap` >= one chunk of keys, so a chunk
// spans at most two bins.
template <typename H>
__global__ void __launch_bounds__(kHtT) k_ht_insert(const uint32_t* __restrict__ t_off, const KeyOf<H>* __restrict__ t_edges,
                                                    int s, uint64_t v, const uint32_t* __restrict__ big_bin,
                                                    const uint32_t* __restrict__ big_t, unsigned long long* __restrict__ plan,
                                                    KeyOf<H>* __restrict__ hk, uint32_t* __restrict__ hc) {
  using K = KeyOf<H>;
  constexpr uint32_t CH = kHtT * kHtKPT;
  const uint32_t nbig = (uint32_t)plan[kPlanBig];
  if (nbig == 0) return;
  const uint32_t total = (uint32_t)plan[kPlanBigT];
  const uint64_t cap = plan[kPlanCap];
  __shared__ uint32_t s_j;
  // (64-bit chunk cursor: totals can approach 2^32 and the stride must not wrap)
  for (uint64_t c0 = (uint64_t)blockIdx.x * CH; c0 < total; c0 += (uint64_t)gridDim.x * CH) {
    if (threadIdx.x == 0) s_j = upper_index(big_t, nbig, (uint32_t)c0);
    __syncthreads();
    const uint32_t j0 = s_j;
    __syncthreads();
    const uint64_t e0 = c0 + threadIdx.x * kHtKPT;
    K cur = K(0);
    uint32_t run = 0;
    for (int u = 0; u < kHtKPT; u++) {
      const uint32_t e = (uint32_t)min(e0 + u, (uint64_t)total);  // (== total: past the end)
      bool flush = false;
      K key = K(0);
      if (e < total) {
        const uint32_t j = e >= big_t[j0 + 1] ? j0 + 1 : j0;  // j0 < nbig
        const uint32_t tb = t_off[min((uint64_t)big_bin[j] << s, v)];
        key = t_edges[tb + (e - big_t[j])];
        if (run && key != cur) flush = true;
      }
      // flush the finished run (warp peers with the same key merge into one add)
      const uint32_t fm = __ballot_sync(0xffffffffu, flush);
      if (flush) {
        const uint32_t peers = __match_any_sync(fm, cur);
        const uint32_t sum = __reduce_add_sync(peers, run);
        if ((peers & lanemask_lt()) == 0) ht_add(hk, hc, cap, cur, sum, plan + kPlanOnes);
        run = 0;
      }
      if (e < total) {
        cur = key;
        run++;
      }
    }
    const bool last = run != 0;
    const uint32_t lm = __ballot_sync(0xffffffffu, last);
    if (last) {
      const uint32_t peers = __match_any_sync(lm, cur);
      const uint32_t sum = __reduce_add_sync(peers, run);
      if ((peers & lanemask_lt()) == 0) ht_add(hk, hc, cap, cur, sum, plan + kPlanOnes);
    }
  }
}

// Queries of the hash-table bins, flattened; results go to the bin-ordered
// multiplicities like the shared-memory probe's.
template <typename H>
__global__ void __launch_bounds__(kHtT) k_ht_lookup(const KeyOf<H>* __restrict__ qpart, const uint32_t* __restrict__ q_start,
                                                    const uint32_t* __restrict__ t_off, HashParams hp, int s, uint64_t v,
                                                    const uint32_t* __restrict__ big_bin, const uint32_t* __restrict__ big_q,
                                                    const unsigned long long* __restrict__ plan, const KeyOf<H>* __restrict__ hk,
                                                    const uint32_t* __restrict__ hc, uint32_t* __restrict__ mult_bo,
                                                    unsigned long long* __restrict__ agg) {
  using K = KeyOf<H>;
  constexpr uint32_t CH = kHtT * 4;
  const uint32_t nbig = (uint32_t)plan[kPlanBig];
  if (nbig == 0) return;
  const uint32_t total = (uint32_t)plan[kPlanBigQ];
  const uint64_t cap = plan[kPlanCap];
  const uint32_t ones = (uint32_t)plan[kPlanOnes];
  __shared__ uint32_t s_j[2];
  uint64_t matched = 0, tot = 0, comps = 0;
  for (uint64_t c0 = (uint64_t)blockIdx.x * CH; c0 < total; c0 += (uint64_t)gridDim.x * CH) {
    if (threadIdx.x == 0) s_j[0] = upper_index(big_q, nbig, (uint32_t)c0);
    if (threadIdx.x == 1) s_j[1] = upper_index(big_q, nbig, (uint32_t)(min((uint64_t)total, c0 + CH) - 1));
    __syncthreads();
    const uint32_t ja = s_j[0], jz = s_j[1];
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const uint64_t e64 = c0 + u * kHtT + threadIdx.x;
      const uint32_t e = (uint32_t)e64;
      if (e64 < total) {
        uint32_t a = ja, z = jz + 1;  // big_q[a] <= e < big_q[z]
        while (z - a > 1) {
          const uint32_t m = (a + z) >> 1;
          if (big_q[m] <= e) a = m; else z = m;
        }
        const uint32_t pos = q_start[big_bin[a]] + (e - big_q[a]);
        const K q = qpart[pos];
        const uint32_t h = H::bucket(q, hp);
        const uint32_t c = ht_count(hk, hc, cap, q, ones);
        mult_bo[pos] = c;
        matched += c != 0;
        tot += c;
        comps += t_off[(uint64_t)h + 1] - t_off[h];
      }
    }
  }
  flush_agg(matched, tot, comps, agg);
}
