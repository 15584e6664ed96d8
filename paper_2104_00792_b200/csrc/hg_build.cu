// hg_build.cu -- single-shard HashGraph build and query (v1 "direct" path).
//
// Paper Alg. 1 realised as three sm_100a kernels:
//   k_count : hash -> atomicAdd(counter[h])          (core.py:97  np.bincount)
//   k_scan  : single-pass decoupled look-back scan   (core.py:98-99 np.cumsum)
//   k_place : hash -> slot = atomicAdd(cursor[h]) -> edges[slot] = key
//                                                    (core.py:100-101 argsort+gather)
// and the IntersectArray query (query.py:120-179) as k_intersect.
#include <algorithm>
#include <cstdlib>

#include "hg_binned.cuh"

namespace hg {

constexpr int kThreads = 256;

inline int grid_for(uint64_t n, int per_sm = 16) {
  uint64_t blocks = (n + kThreads - 1) / kThreads;
  uint64_t cap = (uint64_t)num_sms() * per_sm;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return (int)blocks;
}

// --------------------------------------------------------------------------- hash

template <typename K, typename O>
__global__ void k_hash(const K* __restrict__ keys, uint64_t n, HashParams hp, O* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = (O)hash_mod(keys[i], hp);
}

// --------------------------------------------------------------------------- count

template <typename K>
__global__ void k_count(const K* __restrict__ keys, uint64_t n, HashParams hp,
                        uint32_t* __restrict__ counts) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    atomicAdd(counts + bucket_of(keys[i], hp), 1u);
}

// --------------------------------------------------------------------------- scan

constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;  // 4096
constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagInc = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 62) - 1;

// Exclusive scan of counts[0..v) into offsets[0..v] (offsets[v] = total);
// counts is overwritten with the exclusive prefix so it can serve as the
// placement cursor.  Tiles are ordered by an atomic ticket, so look-back only
// ever waits on tiles that are already running (forward progress).
__global__ void __launch_bounds__(kScanThreads)
k_scan(uint32_t* __restrict__ counts, uint64_t v, uint32_t* __restrict__ offsets,
       uint64_t* __restrict__ status, uint32_t* __restrict__ ticket) {
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_warp[kScanThreads / 32];
  __shared__ uint64_t s_prefix;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t base = tile * kScanTile + (uint64_t)threadIdx.x * kScanItems;

  uint32_t x[kScanItems];
  if (base + kScanItems <= v && (base & 3) == 0) {
    const uint4* p = reinterpret_cast<const uint4*>(counts + base);
#pragma unroll
    for (int j = 0; j < kScanItems / 4; j++) {
      uint4 q = p[j];
      x[4 * j] = q.x; x[4 * j + 1] = q.y; x[4 * j + 2] = q.z; x[4 * j + 3] = q.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < kScanItems; j++) x[j] = (base + j < v) ? counts[base + j] : 0u;
  }
  uint32_t tsum = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; j++) tsum += x[j];

  // warp inclusive scan of per-thread sums
  uint32_t inc = tsum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) s_warp[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < kScanThreads / 32 ? s_warp[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < kScanThreads / 32) s_warp[lane] = w;  // inclusive warp totals
  }
  __syncthreads();
  const uint32_t tile_total = s_warp[kScanThreads / 32 - 1];
  const uint32_t warp_excl = warp ? s_warp[warp - 1] : 0u;

  // decoupled look-back by warp 0
  if (warp == 0) {
    volatile unsigned long long* st = reinterpret_cast<volatile unsigned long long*>(status);
    uint64_t prefix = 0;
    if (tile == 0) {
      if (lane == 0) st[0] = kFlagInc | tile_total;
    } else {
      if (lane == 0) st[tile] = kFlagAgg | tile_total;
      int64_t p = (int64_t)tile - 1 - lane;
      while (true) {
        uint64_t s = 0;
        if (p >= 0) {
          do { s = st[p]; } while ((s >> 62) == 0);
        } else {
          s = kFlagInc;  // before tile 0: an inclusive zero
        }
        uint32_t inc_mask = __ballot_sync(0xffffffffu, (s >> 62) == 2);
        if (inc_mask) {
          int stop = __ffs(inc_mask) - 1;  // nearest inclusive predecessor
          uint64_t val = lane <= stop ? (s & kValMask) : 0ull;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
          prefix += val;
          break;
        }
        uint64_t val = s & kValMask;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
        prefix += val;
        p -= 32;
      }
      if (lane == 0) st[tile] = kFlagInc | ((prefix + tile_total) & kValMask);
    }
    if (lane == 0) s_prefix = prefix;
  }
  __syncthreads();
  uint32_t run = (uint32_t)s_prefix + warp_excl + (inc - tsum);
  uint32_t y[kScanItems];
#pragma unroll
  for (int j = 0; j < kScanItems; j++) {
    y[j] = run;
    run += x[j];
  }
  if (base + kScanItems <= v && (base & 3) == 0) {
    uint4* pc = reinterpret_cast<uint4*>(counts + base);
#pragma unroll
    for (int j = 0; j < kScanItems / 4; j++) pc[j] = make_uint4(y[4 * j], y[4 * j + 1], y[4 * j + 2], y[4 * j + 3]);
#pragma unroll
    for (int j = 0; j < kScanItems; j++) offsets[base + j] = y[j];
  } else {
#pragma unroll
    for (int j = 0; j < kScanItems; j++)
      if (base + j < v) {
        counts[base + j] = y[j];
        offsets[base + j] = y[j];
      }
  }
  if (base < v && v <= base + kScanItems) offsets[v] = run;  // grand total
}

// --------------------------------------------------------------------------- place

template <typename K>
__global__ void k_place(const K* __restrict__ keys, uint64_t n, HashParams hp,
                        uint32_t* __restrict__ cursor, K* __restrict__ edges,
                        uint32_t* __restrict__ positions) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    K key = keys[i];
    uint32_t slot = atomicAdd(cursor + bucket_of(key, hp), 1u);
    edges[slot] = key;
    if (positions) positions[slot] = (uint32_t)i;
  }
}

// --------------------------------------------------------------------------- intersect

// One thread per query-table slot j: count equal keys in the table bucket the
// slot's key hashes to (IntersectArray, PAPER.md:62-72 / query.py:62-81) and
// scatter the count to the query's input position (query.py:164).
// comparisons = sum_j deg_a(bucket(j)) == sum_h deg_a(h) * deg_b(h).
template <typename K>
__global__ void k_intersect(const uint32_t* __restrict__ off_a, const K* __restrict__ edges_a,
                            const K* __restrict__ edges_b, const uint32_t* __restrict__ pos_b,
                            uint64_t n_b, HashParams hp, uint32_t* __restrict__ mult,
                            unsigned long long* __restrict__ agg) {
  uint64_t matched = 0, total = 0, comps = 0;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n_b;
       j += (uint64_t)gridDim.x * blockDim.x) {
    K q = edges_b[j];
    const uint64_t h = hash_mod(q, hp);  // 64-bit: h + 1 == 2^32 when v == 2^32
    uint32_t lo = off_a[h], hi = off_a[h + 1];
    uint32_t c = 0;
    for (uint32_t t = lo; t < hi; t++) c += (edges_a[t] == q);
    mult[pos_b ? pos_b[j] : j] = c;
    matched += (c != 0);
    total += c;
    comps += hi - lo;
  }
  if (agg) {
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
}

// --------------------------------------------------------------------------- host

static int check_common(uint64_t n, int key_bits, int kind, uint64_t v) {
  if (key_bits != 32 && key_bits != 64) return set_error(HG_ERR_CONFIG, "key_bits must be 32 or 64, got %d", key_bits);
  if (kind != HG_KIND_MURMUR32 && kind != HG_KIND_IDENTITY) return set_error(HG_ERR_CONFIG, "unknown hash kind %d", kind);
  if (v < 1) return set_error(HG_ERR_CONFIG, "hash range must be >= 1, got %llu", (unsigned long long)v);
  if (v > (1ull << 32)) return set_error(HG_ERR_CONFIG, "device tables support hash ranges up to 2^32, got %llu", (unsigned long long)v);
  if (n >= (1ull << 32)) return set_error(HG_ERR_CONFIG, "a device table holds fewer than 2^32 keys, got %llu", (unsigned long long)n);
  return HG_OK;
}

size_t build_ws_bytes(uint64_t n, uint64_t v, int key_bits) {
  (void)n;
  (void)key_bits;
  uint64_t tiles = (v + kScanTile - 1) / kScanTile;
  return align_up(4 * v, 256) + align_up(8 * tiles, 256) + 256 + 1024;
}

template <typename K>
int build_impl(const K* keys, uint64_t n, HashParams hp, uint64_t v, uint32_t* offsets, K* edges,
               uint32_t* positions, Workspace& ws, cudaStream_t s) {
  uint64_t tiles = (v + kScanTile - 1) / kScanTile;
  uint32_t* counts = ws.take<uint32_t>(v);
  uint64_t* status = ws.take<uint64_t>(tiles);
  uint32_t* ticket = ws.take<uint32_t>(64);
  if (!ws.ok()) return set_error(HG_ERR_CONFIG, "workspace too small (%zu < %zu)", ws.cap, ws.used);
  HG_CHECK_CUDA(cudaMemsetAsync(counts, 0, 4 * v, s));
  HG_CHECK_CUDA(cudaMemsetAsync(status, 0, 8 * tiles, s));
  HG_CHECK_CUDA(cudaMemsetAsync(ticket, 0, 4, s));
  if (n) HG_LAUNCH("hg_count", k_count<K>, grid_for(n), kThreads, 0, s, keys, n, hp, counts);
  HG_LAUNCH("hg_scan", k_scan, (unsigned)tiles, kScanThreads, 0, s, counts, v, offsets, status, ticket);
  if (n) HG_LAUNCH(positions ? "hg_place_pos" : "hg_place", k_place<K>, grid_for(n), kThreads, 0, s, keys, n, hp,
                   counts, edges, positions);
  return HG_OK;
}

template <typename K>
int intersect_impl(const uint32_t* off_a, const K* edges_a, const K* edges_b, const uint32_t* pos_b,
                   uint64_t n_b, HashParams hp, uint32_t* mult, uint64_t* agg, cudaStream_t s) {
  if (!n_b) return HG_OK;
  HG_LAUNCH("hg_intersect", k_intersect<K>, grid_for(n_b), kThreads, 0, s, off_a, edges_a, edges_b, pos_b,
            n_b, hp, mult, reinterpret_cast<unsigned long long*>(agg));
  return HG_OK;
}

constexpr uint64_t kBinnedMin = 1ull << 16;  // below this the 3-kernel direct path wins

static bool use_binned(uint64_t n_table, uint64_t n, uint64_t v, int key_bits, BinLayout* L) {
  if (n < kBinnedMin) return false;
  // the binned kernels step 32-bit key cursors by up to 2^20 past a bin's
  // start; the last 2^20 indices below 2^32 stay on the direct path
  if (n > (1ull << 32) - (1ull << 20) || n_table > (1ull << 32) - (1ull << 20)) return false;
  if (getenv("HG_FORCE_DIRECT")) return false;
  return binned_layout(n_table, n, v, key_bits, L);
}

}  // namespace hg

using namespace hg;

extern "C" {

int hg_hash(const void* keys, uint64_t n, int key_bits, int kind, uint32_t seed, uint64_t v, void* out,
            int out_bits, void* stream) {
  if (key_bits != 32 && key_bits != 64) return set_error(HG_ERR_CONFIG, "key_bits must be 32 or 64");
  if (kind != HG_KIND_MURMUR32 && kind != HG_KIND_IDENTITY) return set_error(HG_ERR_CONFIG, "unknown hash kind %d", kind);
  if (v < 1) return set_error(HG_ERR_CONFIG, "hash range must be >= 1");
  if (out_bits != 32 && out_bits != 64) return set_error(HG_ERR_CONFIG, "out_bits must be 32 or 64");
  if (out_bits == 32 && (v > (1ull << 32)) && key_bits == 64)
    return set_error(HG_ERR_CONFIG, "32-bit output cannot hold hashes of range %llu", (unsigned long long)v);
  if (!n) return HG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  HashParams hp = make_hash_params(kind, seed, v, key_bits);
  if (key_bits == 32) {
    if (out_bits == 32)
      HG_LAUNCH("hg_hash", (k_hash<uint32_t, uint32_t>), grid_for(n), kThreads, 0, s, (const uint32_t*)keys, n, hp, (uint32_t*)out);
    else
      HG_LAUNCH("hg_hash", (k_hash<uint32_t, uint64_t>), grid_for(n), kThreads, 0, s, (const uint32_t*)keys, n, hp, (uint64_t*)out);
  } else {
    if (out_bits == 32)
      HG_LAUNCH("hg_hash", (k_hash<uint64_t, uint32_t>), grid_for(n), kThreads, 0, s, (const uint64_t*)keys, n, hp, (uint32_t*)out);
    else
      HG_LAUNCH("hg_hash", (k_hash<uint64_t, uint64_t>), grid_for(n), kThreads, 0, s, (const uint64_t*)keys, n, hp, (uint64_t*)out);
  }
  return HG_OK;
}

size_t hg_build_workspace_size(uint64_t n, uint64_t v, int key_bits) {
  size_t b = build_ws_bytes(n, v, key_bits);
  BinLayout L;
  if (use_binned(n, n, v, key_bits, &L)) b = std::max(b, binned_ws_bytes(n, L, key_bits, kWsBuild));
  return b;
}

size_t hg_build_traced_workspace_size(uint64_t n, uint64_t v, int key_bits) {
  size_t b = build_ws_bytes(n, v, key_bits);
  BinLayout L;
  if (use_binned(n, n, v, key_bits, &L)) b = std::max(b, binned_ws_bytes(n, L, key_bits, kWsTraced));
  return b;
}

int hg_build(const void* keys, uint64_t n, int key_bits, int kind, uint32_t seed, uint64_t v, uint32_t* offsets,
             void* edges, uint32_t* positions, void* workspace, size_t workspace_bytes, void* stream) {
  int rc = check_common(n, key_bits, kind, v);
  if (rc) return rc;
  Workspace ws{(char*)workspace, workspace_bytes, 0};
  HashParams hp = make_hash_params(kind, seed, v, key_bits);
  cudaStream_t s = (cudaStream_t)stream;
  BinLayout L;
  // positions (build_traced): the binned path when the workspace holds its trace
  if (use_binned(n, n, v, key_bits, &L) &&
      (positions == nullptr || binned_ws_bytes(n, L, key_bits, kWsTraced) <= workspace_bytes)) {
    if (key_bits == 32)
      return binned_build<uint32_t>((const uint32_t*)keys, n, hp, v, L, offsets, (uint32_t*)edges, ws, s, positions);
    return binned_build<uint64_t>((const uint64_t*)keys, n, hp, v, L, offsets, (uint64_t*)edges, ws, s, positions);
  }
  if (key_bits == 32)
    return build_impl<uint32_t>((const uint32_t*)keys, n, hp, v, offsets, (uint32_t*)edges, positions, ws, s);
  return build_impl<uint64_t>((const uint64_t*)keys, n, hp, v, offsets, (uint64_t*)edges, positions, ws, s);
}

int hg_intersect(const uint32_t* offsets_a, const void* edges_a, const uint32_t* offsets_b, const void* edges_b,
                 const uint32_t* positions_b, uint64_t n_b, int key_bits, int kind, uint32_t seed, uint64_t v,
                 uint32_t* mult, uint64_t* agg, void* stream) {
  (void)offsets_b;
  int rc = check_common(n_b, key_bits, kind, v);
  if (rc) return rc;
  HashParams hp = make_hash_params(kind, seed, v, key_bits);
  cudaStream_t s = (cudaStream_t)stream;
  if (key_bits == 32)
    return intersect_impl<uint32_t>(offsets_a, (const uint32_t*)edges_a, (const uint32_t*)edges_b, positions_b, n_b,
                                    hp, mult, agg, s);
  return intersect_impl<uint64_t>(offsets_a, (const uint64_t*)edges_a, (const uint64_t*)edges_b, positions_b, n_b,
                                  hp, mult, agg, s);
}

size_t hg_query_workspace_size(uint64_t q, uint64_t v, uint64_t n_table, int key_bits) {
  size_t kb = key_bits / 8;
  size_t b = align_up(4 * (v + 1), 256) + align_up(kb * q, 256) + align_up(4 * q, 256) + build_ws_bytes(q, v, key_bits) + 1024;
  BinLayout L;
  if (use_binned(n_table, q, v, key_bits, &L)) b = std::max(b, binned_ws_bytes(q, L, key_bits, kWsQuery, n_table));
  return b;
}

static int query_entry(const uint32_t* offsets_a, const void* edges_a, uint64_t n_a, const void* queries, uint64_t q,
                       int key_bits, int kind, uint32_t seed, uint64_t v, uint32_t* mult, uint64_t* agg,
                       void* workspace, size_t workspace_bytes, void* stream, cudaEvent_t split) {
  int rc = check_common(q, key_bits, kind, v);
  if (rc) return rc;
  Workspace ws{(char*)workspace, workspace_bytes, 0};
  HashParams hp = make_hash_params(kind, seed, v, key_bits);
  cudaStream_t s = (cudaStream_t)stream;
  BinLayout L;
  if (use_binned(n_a, q, v, key_bits, &L) && binned_ws_bytes(q, L, key_bits, kWsQuery, n_a) <= workspace_bytes) {
    if (key_bits == 32)
      return binned_query<uint32_t>(offsets_a, (const uint32_t*)edges_a, n_a, (const uint32_t*)queries, q, hp, v, L,
                                    mult, agg, ws, s, split);
    return binned_query<uint64_t>(offsets_a, (const uint64_t*)edges_a, n_a, (const uint64_t*)queries, q, hp, v, L,
                                  mult, agg, ws, s, split);
  }
  size_t kb = key_bits / 8;
  uint32_t* qoff = ws.take<uint32_t>(v + 1);
  void* qedges = ws.take<char>(kb * q);
  uint32_t* qpos = ws.take<uint32_t>(q);
  Workspace rest{ws.base + align_up(ws.used, 256), ws.cap > align_up(ws.used, 256) ? ws.cap - align_up(ws.used, 256) : 0, 0};
  if (!ws.ok()) return set_error(HG_ERR_CONFIG, "query workspace too small");
  if (key_bits == 32) {
    rc = build_impl<uint32_t>((const uint32_t*)queries, q, hp, v, qoff, (uint32_t*)qedges, qpos, rest, s);
    if (rc) return rc;
    if (split) HG_CHECK_CUDA(cudaEventRecord(split, s));
    return intersect_impl<uint32_t>(offsets_a, (const uint32_t*)edges_a, (const uint32_t*)qedges, qpos, q, hp, mult, agg, s);
  }
  rc = build_impl<uint64_t>((const uint64_t*)queries, q, hp, v, qoff, (uint64_t*)qedges, qpos, rest, s);
  if (rc) return rc;
  if (split) HG_CHECK_CUDA(cudaEventRecord(split, s));
  return intersect_impl<uint64_t>(offsets_a, (const uint64_t*)edges_a, (const uint64_t*)qedges, qpos, q, hp, mult, agg, s);
}

int hg_query(const uint32_t* offsets_a, const void* edges_a, uint64_t n_a, const void* queries, uint64_t q,
             int key_bits, int kind, uint32_t seed, uint64_t v, uint32_t* mult, uint64_t* agg, void* workspace,
             size_t workspace_bytes, void* stream) {
  return query_entry(offsets_a, edges_a, n_a, queries, q, key_bits, kind, seed, v, mult, agg, workspace,
                     workspace_bytes, stream, nullptr);
}

int hg_query_timed(const uint32_t* offsets_a, const void* edges_a, uint64_t n_a, const void* queries, uint64_t q,
                   int key_bits, int kind, uint32_t seed, uint64_t v, uint32_t* mult, uint64_t* agg, void* workspace,
                   size_t workspace_bytes, void* split_event, void* stream) {
  return query_entry(offsets_a, edges_a, n_a, queries, q, key_bits, kind, seed, v, mult, agg, workspace,
                     workspace_bytes, stream, (cudaEvent_t)split_event);
}

size_t hg_intersect_tables_workspace_size(uint64_t n_b, uint64_t v, uint64_t n_a, int key_bits) {
  BinLayout L;
  if (use_binned(n_a, n_b, v, key_bits, &L)) return binned_tables_ws_bytes(n_b, L, key_bits, n_a);
  return 1024;
}

int hg_intersect_tables(const uint32_t* offsets_a, const void* edges_a, uint64_t n_a, const uint32_t* offsets_b,
                        const void* edges_b, const uint32_t* positions_b, uint64_t n_b, int key_bits, int kind,
                        uint32_t seed, uint64_t v, void* trace, size_t trace_bytes, uint32_t* mult, uint64_t* agg,
                        void* workspace, size_t workspace_bytes, void* stream) {
  int rc = check_common(n_b, key_bits, kind, v);
  if (rc) return rc;
  if (n_b && positions_b == nullptr) return set_error(HG_ERR_CONFIG, "positions_b is required");
  HashParams hp = make_hash_params(kind, seed, v, key_bits);
  cudaStream_t s = (cudaStream_t)stream;
  BinLayout Lp, Lt;
  if (use_binned(n_a, n_b, v, key_bits, &Lp) && binned_tables_ws_bytes(n_b, Lp, key_bits, n_a) <= workspace_bytes) {
    // the trace is only usable when the query table was built binned with it
    const bool traced = trace != nullptr && use_binned(n_b, n_b, v, key_bits, &Lt) &&
                        binned_ws_bytes(n_b, Lt, key_bits, kWsTraced) <= trace_bytes;
    Workspace ws{(char*)workspace, workspace_bytes, 0};
    if (key_bits == 32)
      return binned_tables<uint32_t>(offsets_a, (const uint32_t*)edges_a, n_a, offsets_b, (const uint32_t*)edges_b,
                                     positions_b, n_b, hp, v, Lp, traced ? &Lt : nullptr, traced ? trace : nullptr,
                                     trace_bytes, mult, agg, ws, s);
    return binned_tables<uint64_t>(offsets_a, (const uint64_t*)edges_a, n_a, offsets_b, (const uint64_t*)edges_b,
                                   positions_b, n_b, hp, v, Lp, traced ? &Lt : nullptr, traced ? trace : nullptr,
                                   trace_bytes, mult, agg, ws, s);
  }
  if (key_bits == 32)
    return intersect_impl<uint32_t>(offsets_a, (const uint32_t*)edges_a, (const uint32_t*)edges_b, positions_b, n_b, hp,
                                    mult, agg, s);
  return intersect_impl<uint64_t>(offsets_a, (const uint64_t*)edges_a, (const uint64_t*)edges_b, positions_b, n_b, hp,
                                  mult, agg, s);
}

}  // extern "C"
