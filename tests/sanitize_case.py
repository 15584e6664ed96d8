"""One small run of every binned kernel, for compute-sanitizer (tests/test_sanitizer_gpu.py).

`python tests/sanitize_case.py` builds and queries: u32 single-level (2^17
keys), u32 two-level (2^17 keys over V = 2^24: 1024 fine bins, 8 level-1
bins), a high-duplicate table (oversized fine bins, deep-bucket probe map)
and u64 two-level, each checked against the oracle so a sanitizer run also
proves the answers.  Round 2 adds: sorted deep buckets (V = N / 64),
all-identical keys (the chunked oversized-bin build, the hash-table query
path, hot-bin probe items), identical queries against a uniform table, the
65536-fine-bin layout, and the two-step query (traced build, k_repart,
k_perm_bins; the scatter path for foreign positions)."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
import paper_2104_00792_b200 as hg  # noqa: E402


def case(keys, queries, hash_range=None, key_bits=32):
    table = hg.build(keys, hash_range=hash_range, key_bits=key_bits)
    res = hg.intersect(table, queries)
    off, placed, _ = O.build_csr(keys, table.hash_range)
    assert np.array_equal(table.offset, off)
    assert np.array_equal(O.canonical(table.offset, table.keys)[1], O.canonical(off, placed)[1])
    assert np.array_equal(res.multiplicities, O.count_occurrences(keys, queries))


def main():
    n = 1 << 17
    case(O.generate_keys(17, n, 1), O.generate_keys(17, n, 2))
    case(O.generate_keys(24, n, 3), O.generate_keys(24, n, 4), hash_range=1 << 24)
    case(O.generate_keys(6, n, 5), O.generate_keys(6, n // 2, 6), hash_range=1 << 16)
    k64 = O.generate_keys(64, n, 7, key_bits=64)
    case(k64, np.concatenate([k64[: n // 2], O.generate_keys(64, n // 2, 8, key_bits=64)]), hash_range=1 << 22,
         key_bits=64)
    case(O.generate_keys(17, n, 9), O.generate_keys(17, n, 10), hash_range=n // 64)  # sorted deep buckets
    same = np.full(n, 7, np.uint32)
    case(same, np.concatenate([same[: n // 2], O.generate_keys(17, n // 2, 11)]))  # chunked build, hash table
    case(O.generate_keys(17, n, 12), np.full(n, 99, np.uint32))  # hot bin: extra probe items
    k = O.generate_keys(32, n // 2, 13)
    table = hg.build(k, hash_range=1 << 30)  # 65536 fine bins
    assert np.array_equal(hg.intersect(table, k[::3]).multiplicities, O.count_occurrences(k, k[::3]))
    keys, queries = O.generate_keys(17, n, 14), O.generate_keys(17, n, 15)
    table = hg.build(keys)
    qt, pos = hg.build_query_table(table, queries)  # traced build
    want = O.count_occurrences(keys, queries)
    assert np.array_equal(hg.intersect_tables(table, qt, pos).multiplicities, want)  # through the trace
    assert np.array_equal(hg.intersect_tables(table, qt, pos.copy()).multiplicities, want)  # scatter
    print("sanitize_case ok")


if __name__ == "__main__":
    main()
