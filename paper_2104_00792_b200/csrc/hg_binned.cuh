// hg_binned.cuh -- interface of the binned build/query path (hg_binned.cu).
#pragma once
#include "hg_common.cuh"

namespace hg {

struct BinLayout {
  int s;               // log2 buckets per fine bin
  uint32_t nfine;      // F
  bool two_level;
  uint32_t nb1;        // level-1 bins (F when one level)
  int bits1;           // ballot bits for level 1
  int shift1;          // level-1 bin = bucket >> shift1
  uint32_t group;      // fine bins per level-1 bin (1 or sub)
  uint32_t sub;        // level-2 fan-out: 128, or 256 above 32768 fine bins
  uint32_t grid;       // CTAs of A / P1 / R1 (one chunk each)
  uint64_t chunk;      // keys per chunk (multiple of the tile)
  uint32_t tile;
  uint64_t ntiles1;
  uint64_t max_tiles2;
};

bool binned_layout(uint64_t n_table, uint64_t n, uint64_t v, int key_bits, BinLayout* L);
enum { kWsBuild = 0, kWsQuery = 1, kWsTraced = 2 };  // == PartMode
size_t binned_ws_bytes(uint64_t n, const BinLayout& L, int key_bits, int mode, uint64_t n_table = 0);
size_t binned_tables_ws_bytes(uint64_t q, const BinLayout& Lp, int key_bits, uint64_t n_table);
template <typename K>
int binned_build(const K* keys, uint64_t n, const HashParams& hp, uint64_t v, const BinLayout& L, uint32_t* offsets,
                 K* edges, Workspace& ws, cudaStream_t st, uint32_t* positions = nullptr);
template <typename K>
int binned_tables(const uint32_t* t_off, const K* t_edges, uint64_t n_table, const uint32_t* q_off, const K* q_edges,
                  const uint32_t* positions, uint64_t q, const HashParams& hp, uint64_t v, const BinLayout& Lp,
                  const BinLayout* Lt, void* trace, size_t trace_bytes, uint32_t* mult, uint64_t* agg, Workspace& ws,
                  cudaStream_t st);
template <typename K>
int binned_query(const uint32_t* t_off, const K* t_edges, uint64_t n_table, const K* queries, uint64_t q,
                 const HashParams& hp, uint64_t v, const BinLayout& L, uint32_t* mult, uint64_t* agg, Workspace& ws,
                 cudaStream_t st, cudaEvent_t split = nullptr);

}  // namespace hg
