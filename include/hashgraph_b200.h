/*
 * hashgraph_b200.h -- C ABI of libhashgraph_b200.so, the sm_100a (B200) HashGraph.
 *
 * This is the drop-in boundary for the reference package's hot path
 * (`hashgraph` 0.1.0, /root/reference/pkg/src/hashgraph).  Every entry point
 * names the reference interface it replaces (file:line, relative to that
 * directory).  The Python package `paper_2104_00792_b200` binds these with
 * ctypes; INTEGRATION.md shows the binding a maintainer adds to the reference.
 *
 * Conventions
 *  - Plain pointers and sizes only.  Every `const void* keys` / `void* edges`
 *    is DEVICE memory holding uint32 (key_bits == 32) or uint64 (key_bits ==
 *    64) keys.  Offsets and positions are device uint32 (a table holds < 2^32
 *    keys per shard); aggregates are device uint64.
 *  - Enqueue-only: work is launched on `stream` (a cudaStream_t, NULL = legacy
 *    default stream) and the call returns without synchronising, except where
 *    a function is documented as "host-synchronous".
 *  - The library never allocates device memory on the hot path: callers pass
 *    a workspace of at least the size the matching *_workspace_size() call
 *    returns.  Workspace contents need no initialisation.
 *  - Return value: 0 on success; HG_ERR_CONFIG for invalid arguments (the
 *    Python layer raises ConfigError, like the reference's validation);
 *    HG_ERR_CUDA for a CUDA launch/runtime failure (RuntimeError).
 *    hg_last_error() returns a thread-local message for the last failure.
 *  - Hash family: kind 0 = murmur32 (fmix32(key ^ seed) mod V; fmix64 for
 *    64-bit keys), kind 1 = identity (key mod V)  -- hashing.py:31-59, 77-114.
 */
#ifndef HASHGRAPH_B200_H
#define HASHGRAPH_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define HG_API __attribute__((visibility("default")))
#else
#define HG_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define HG_OK 0
#define HG_ERR_CONFIG (-1)
#define HG_ERR_CUDA (-2)

#define HG_KIND_MURMUR32 0
#define HG_KIND_IDENTITY 1

/* Library identity / diagnostics ---------------------------------------- */
HG_API const char* hg_version(void);
HG_API const char* hg_last_error(void);
/* Number of kernels this library has launched in this process. */
HG_API uint64_t hg_launch_count(void);
/* Per-launch CUDA-event timing (off by default).  While enabled every kernel
 * launch is bracketed by events on its stream; hg_timing_collect()
 * synchronises those events and returns up to `cap` (name, milliseconds)
 * records, oldest first, then clears the list.  Returns the record count. */
HG_API void hg_timing_enable(int on);
HG_API int hg_timing_collect(const char** names, float* ms, int cap);

/* Hashing -- replaces hashing.hash_array (hashing.py:98-114).
 * out[i] = hash(keys[i]) mod v as uint32 (v <= 2^32) or uint64 (out_bits 64). */
HG_API int hg_hash(const void* keys, uint64_t n, int key_bits, int kind, uint32_t seed, uint64_t v,
            void* out, int out_bits, void* stream);

/* Single-shard build -- replaces core.build / core.build_traced
 * (core.py:164-209, arrays from _build_arrays core.py:148-155).
 * offsets: uint32[v+1]; edges: keys grouped by bucket (order inside a bucket
 * unspecified, core.py:12-14); positions (nullable): uint32[n], input index of
 * the key at each edge slot. */
HG_API size_t hg_build_workspace_size(uint64_t n, uint64_t v, int key_bits);
/* Workspace for hg_build with positions on the binned path (build_traced):
 * the workspace then also holds the build's TRACE (position maps of both
 * partition levels, the grouped keys and their input indices), which
 * hg_intersect_tables reuses to return counts to input order by streaming
 * instead of scattering.  A smaller workspace runs the direct Alg. 1 kernels. */
HG_API size_t hg_build_traced_workspace_size(uint64_t n, uint64_t v, int key_bits);
HG_API int hg_build(const void* keys, uint64_t n, int key_bits, int kind, uint32_t seed, uint64_t v,
             uint32_t* offsets, void* edges, uint32_t* positions, void* workspace,
             size_t workspace_bytes, void* stream);

/* Intersection of two tables with equal v and family -- replaces
 * query.intersect_tables (query.py:120-179).  mult[positions_b[j]] = number of
 * keys in bucket h of table A equal to edges_b[j].  agg (nullable, uint64[3],
 * accumulated, caller zeroes): matched positions, total matches, comparisons
 * (sum over buckets of deg_a * deg_b, query.py:153-155). */
HG_API int hg_intersect(const uint32_t* offsets_a, const void* edges_a, const uint32_t* offsets_b,
                 const void* edges_b, const uint32_t* positions_b, uint64_t n_b, int key_bits,
                 int kind, uint32_t seed, uint64_t v, uint32_t* mult, uint64_t* agg, void* stream);

/* intersect_tables on the binned path (query.py:120-179), with the same depth
 * classes, sorted-bucket search and hash-table path as hg_query.  With `trace`
 * (the workspace of the hg_build that produced table B with positions,
 * hg_build_traced_workspace_size bytes; nullable), the trace's grouped query
 * keys are probed (at table A's probe layout when the trace's fine bins nest in
 * it, else at the trace's own) and the counts return to query order through its
 * position maps; without a trace table B's fine-bin slices are probed and the
 * counts scatter through positions_b.  n_a = table A's key
 * count.  Small inputs run hg_intersect's kernels.  agg accumulated (caller
 * zeroes). */
HG_API size_t hg_intersect_tables_workspace_size(uint64_t n_b, uint64_t v, uint64_t n_a, int key_bits);
HG_API int hg_intersect_tables(const uint32_t* offsets_a, const void* edges_a, uint64_t n_a,
                        const uint32_t* offsets_b, const void* edges_b, const uint32_t* positions_b,
                        uint64_t n_b, int key_bits, int kind, uint32_t seed, uint64_t v, void* trace,
                        size_t trace_bytes, uint32_t* mult, uint64_t* agg, void* workspace,
                        size_t workspace_bytes, void* stream);

/* Whole query against a built table -- replaces query.intersect /
 * intersect_timed (query.py:182-202): builds the query-side table with the
 * table's v (build_query_table, query.py:84-95) and intersects.  mult is
 * uint32[q] in query order; agg (nullable, uint64[3]) is ACCUMULATED like
 * hg_intersect's (caller zeroes), whichever kernels the query runs, so several
 * shard queries can sum into one buffer.  The workspace depends on the table's
 * key count n_table (its keys per bucket set the bin size; fine bins too large
 * for shared memory -- high-duplicate or skewed tables -- are answered from a
 * key -> count hash table of up to 2 * n_table slots). */
HG_API size_t hg_query_workspace_size(uint64_t q, uint64_t v, uint64_t n_table, int key_bits);
HG_API int hg_query(const uint32_t* offsets_a, const void* edges_a, uint64_t n_a, const void* queries,
             uint64_t q, int key_bits, int kind, uint32_t seed, uint64_t v, uint32_t* mult,
             uint64_t* agg, void* workspace, size_t workspace_bytes, void* stream);
/* hg_query plus a split point for intersect_timed (query.py:193-202): split_event
 * (a cudaEvent_t created by the caller) is recorded on the stream once the
 * query-side table (the binned grouping of the queries, or the direct query
 * CSR) is complete, before the intersection kernels. */
HG_API int hg_query_timed(const uint32_t* offsets_a, const void* edges_a, uint64_t n_a, const void* queries,
                   uint64_t q, int key_bits, int kind, uint32_t seed, uint64_t v, uint32_t* mult,
                   uint64_t* agg, void* workspace, size_t workspace_bytes, void* split_event, void* stream);

/* Partitioned build, Phase 1 -- replaces the bin histogram of
 * multishard.build_sharded.worker (multishard.py:371-377) and
 * plan_partition (multishard.py:266-291).  bin_counts: uint64[bins_g],
 * ACCUMULATED (caller zeroes), so several shards can add into one array or an
 * all-reduce can follow. */
HG_API int hg_bin_histogram(const void* keys, uint64_t n, int key_bits, int kind, uint32_t seed,
                     uint64_t hash_range, uint64_t bins_g, uint64_t bin_size,
                     uint64_t* bin_counts, void* stream);

/* Split search -- replaces _splits_from_counts (multishard.py:249-263).
 * splits: int64[shards+1] (device). */
HG_API int hg_split_plan(const uint64_t* bin_counts, uint64_t bins_g, uint64_t total_keys,
                  uint32_t shards, int64_t* splits, void* stream);

/* Phase 2 -- replaces _reorganize_hashed / reorganize (multishard.py:294-318).
 * Stable per-destination CSR: row_offsets uint64[shards+1], grouped keys in
 * input order inside each row; order (nullable) uint32[n]: input index of each
 * grouped slot; search_steps (nullable, uint64, accumulated): sum(dest+1). */
HG_API size_t hg_reorganize_workspace_size(uint64_t n, uint32_t shards);
HG_API int hg_reorganize(const void* keys, uint64_t n, int key_bits, int kind, uint32_t seed,
                  uint64_t hash_range, uint64_t bin_size, const int64_t* splits, uint32_t shards,
                  uint64_t* row_offsets, void* grouped, uint32_t* order, uint64_t* search_steps,
                  void* workspace, size_t workspace_bytes, void* stream);
/* Values per reorganized key back to input order: out[i] = vals[slot of key i]
 * for the rows hg_reorganize produced from these very keys (same hash, plan and
 * splits), whose `workspace` still holds that call's tile bases -- the query
 * answers of query_sharded (multishard.py:510-535) returned with coalesced
 * stores instead of a scatter through `order`. */
HG_API int hg_reorganize_gather(const void* keys, uint64_t n, int key_bits, int kind, uint32_t seed,
                         uint64_t hash_range, uint64_t bin_size, const int64_t* splits, uint32_t shards,
                         const uint64_t* row_offsets, const uint32_t* vals, uint32_t* out, const void* workspace,
                         size_t workspace_bytes, void* stream);

/* Phase 2 + Phase 3 fused over peer memory (one process per GPU; the receive
 * buffers are symmetric allocations mapped into every rank over NVLink /
 * NVSwitch) -- replaces reorganize + exchange (multishard.py:294-333).
 * hg_reorganize_count: count pass + scan, row_offsets uint64[shards+1] (device;
 *   row sizes = send counts); per-tile bases stay in `workspace`.
 * hg_reorganize_place_peers: same keys/splits/workspace; key i of row d is
 *   stored at ((K*)dest_ptrs[d])[dest_base[d] + its stable rank in row d];
 *   dest_ptrs / dest_base: uint64[shards] device arrays; order (nullable) as in
 *   hg_reorganize (local grouped positions).
 * hg_return_peers: reverse direction for uint32 answers: vals[i], i in sender
 *   s's segment [recv_bounds[s], recv_bounds[s+1]) of this rank's receive
 *   order, goes to ((uint32_t*)back_ptrs[s])[back_base[s] + i - recv_bounds[s]]. */
HG_API int hg_reorganize_count(const void* keys, uint64_t n, int key_bits, int kind, uint32_t seed,
                        uint64_t hash_range, uint64_t bin_size, const int64_t* splits, uint32_t shards,
                        uint64_t* row_offsets, uint64_t* search_steps, void* workspace,
                        size_t workspace_bytes, void* stream);
HG_API int hg_reorganize_place_peers(const void* keys, uint64_t n, int key_bits, int kind, uint32_t seed,
                              uint64_t hash_range, uint64_t bin_size, const int64_t* splits,
                              uint32_t shards, const uint64_t* row_offsets, const uint64_t* dest_ptrs,
                              const uint64_t* dest_base, uint32_t* order, void* workspace,
                              size_t workspace_bytes, void* stream);
/* Routing in one pass, for the distributed build and query when the
 * per-destination counts are already known (segment sums of the Phase-1 bin
 * histogram): per tile one claim per destination on cursors[d] (uint64[P]
 * device scratch, zeroed by the call); key -> ((K*)dest_ptrs[d])[dest_base[d]
 * + claim] when dest_ptrs is given (peer memory), else grouped[row_offsets[d]
 * + claim]; order (nullable) [row_offsets[d] + claim] = input index.  Rows are
 * complete but not in input order (see hg_reorganize for the stable form). */
HG_API int hg_route(const void* keys, uint64_t n, int key_bits, int kind, uint32_t seed, uint64_t hash_range,
             uint64_t bin_size, const int64_t* splits, uint32_t shards, const uint64_t* row_offsets,
             const uint64_t* dest_ptrs, const uint64_t* dest_base, void* grouped, uint32_t* order,
             uint64_t* cursors, void* stream);
HG_API int hg_return_peers(const uint32_t* vals, uint64_t n, const uint64_t* recv_bounds,
                    const uint64_t* back_ptrs, const uint64_t* back_base, uint32_t shards, void* stream);

/* Positional merge of per-shard multiplicities -- replaces
 * `multiplicities[order[off_d:off_d+1]] = res.multiplicities`
 * (multishard.py:523): out[order[i]] = src[i]. */
HG_API int hg_scatter_u32(const uint32_t* src, const uint32_t* order, uint64_t n, uint32_t* out,
                   void* stream);

/* Workload -- replaces workload.splitmix64_at / generate (workload.py:63-85).
 * out[i] = SplitMix64(seed, start + i); key_bits 32 -> 1 + (z mod 2^k) as
 * uint32, key_bits 64 -> the full word. */
HG_API int hg_generate(uint64_t seed, uint64_t start, uint64_t count, int k, int key_bits, void* out,
                void* stream);

/* uint32 -> int64 widening for host export (offsets, multiplicities). */
HG_API int hg_widen_u32(const uint32_t* src, uint64_t n, int64_t* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HASHGRAPH_B200_H */
