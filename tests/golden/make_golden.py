"""Generate golden fixtures by running the REFERENCE implementation itself.

Run in the dev container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the unmodified reference package from /root/reference/pkg/src and
records its outputs on seeded inputs into tests/golden/*.npz.  Those fixtures
pin the oracle (oracle/restatement.py) and are compared directly against the
CUDA product path by the GPU tests.  Nothing at test or bench time reads
/root/reference; only this generator does.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _ref():
    sys.path.insert(0, REF)
    import hashgraph  # noqa: E402  (the reference package)

    return hashgraph


def _save(name: str, cases: list[dict], **shared) -> None:
    flat = {"ncases": np.array(len(cases))}
    flat.update({k: np.asarray(v) for k, v in shared.items()})
    for i, case in enumerate(cases):
        for k, v in case.items():
            flat[f"c{i}.{k}"] = np.asarray(v)
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **flat)
    print(f"{name}: {len(cases)} cases -> {os.path.getsize(path)} bytes")


def _fam(hg, kind: int, seed: int):
    return hg.HashFamily(hg.HashKind(kind), seed)


def main() -> None:
    hg = _ref()
    rng = np.random.default_rng(20261017)

    # ---- hashing: fmix32 + hash_array over families and ranges (hashing.py:77-114)
    cases = []
    probe = np.concatenate([
        np.array([0, 1, 2, 7, 0x2A, 0xDEADBEEF, 0xFFFFFFFF, 0x9E3779B9, 0x80000000], dtype=np.uint32),
        rng.integers(0, 1 << 32, size=4096, dtype=np.uint32),
    ])
    fm = np.array([hg.fmix32(int(k)) for k in probe[:64]], dtype=np.uint32)
    cases.append(dict(kind=-1, seed=0, v=0, keys=probe[:64], out=fm))  # case 0: raw fmix32
    for kind, seed in [(0, 0), (0, 42), (0, 0x9E3779B9), (0, 0xFFFFFFFF), (1, 0)]:
        for v in [1, 2, 3, 17, 1000, 65536, 1 << 20, (1 << 31) + 11, (1 << 32) - 1, 1 << 32, (1 << 32) + 5]:
            out = hg.hash_array(_fam(hg, kind, seed), probe, v)
            assert out.max() < (1 << 32)
            cases.append(dict(kind=kind, seed=seed, v=np.uint64(v), out=out.astype(np.uint32)))
    _save("hashing", cases, probe=probe)

    # ---- build (core.py:164-209): offsets, stable placement, positions
    cases = []
    specs = [
        (np.array([0, 2, 2, 5], dtype=np.uint32), 1.0, 1, 0, None),
        (np.array([], dtype=np.uint32), 1.0, 0, 0, None),
        (np.array([42], dtype=np.uint32), 1.0, 1, 0, None),
        (np.array([1, 2, 3, 4], dtype=np.uint32), 1.0, 1, 0, 2),
        (np.full(5000, 123456, dtype=np.uint32), 1.0, 0, 0, None),
    ]
    for n in [1, 2, 31, 32, 33, 1000, 4096, 5000, 1 << 14, 40000]:
        for lf in [0.5, 1.0, 2.0]:
            kind = int(rng.integers(0, 2))
            seed = int(rng.integers(0, 1 << 32)) if kind == 0 else 0
            kbits = int(rng.integers(4, 33))
            keys = rng.integers(0, 1 << kbits, size=n, dtype=np.uint64).astype(np.uint32)
            specs.append((keys, lf, kind, seed, None))
    # high-duplicate: 2^16 keys drawn from 2^6 values, explicit small range
    specs.append((rng.integers(1, 65, size=1 << 16, dtype=np.uint32), 1.0, 0, 0, 1 << 10))
    specs.append((rng.integers(1, 1 << 12, size=1 << 15, dtype=np.uint32), 1.0, 0, 7, 1 << 9))
    for keys, lf, kind, seed, hr in specs:
        table, counters, positions = hg.build_traced(keys, lf, _fam(hg, kind, seed), 1, hr)
        cases.append(dict(keys=keys, load_factor=lf, kind=kind, seed=seed,
                          hash_range=np.uint64(table.hash_range),
                          offset=table.offset, placed=table.keys, positions=positions))
    _save("build", cases)

    # ---- query (query.py:84-202): positional multiplicities + aggregates
    cases = []
    qspecs = [
        (np.array([0, 2, 2, 5], dtype=np.uint32), np.array([2, 7, 0], dtype=np.uint32), 1.0, 1, 0, None),
        (np.array([1, 2, 3], dtype=np.uint32), np.array([], dtype=np.uint32), 1.0, 0, 0, None),
        (np.array([], dtype=np.uint32), np.array([1, 2, 3], dtype=np.uint32), 1.0, 0, 0, None),
        (np.array([7, 7, 7], dtype=np.uint32), np.array([7, 7], dtype=np.uint32), 1.0, 0, 0, None),
    ]
    for n, q, dom, lf in [(1 << 12, 1 << 12, 1 << 12, 1.0), (1 << 14, 1 << 13, 1 << 14, 0.5),
                          (5000, 7000, 600, 2.0), (1 << 16, 1 << 16, 1 << 16, 1.0),
                          (1 << 15, 1 << 15, 64, 1.0), (3000, 100, 1 << 31, 1.0)]:
        kind = int(rng.integers(0, 2))
        seed = int(rng.integers(0, 1 << 32)) if kind == 0 else 0
        keys = rng.integers(1, dom + 1, size=n, dtype=np.uint64).astype(np.uint32)
        queries = rng.integers(1, dom + 1, size=q, dtype=np.uint64).astype(np.uint32)
        qspecs.append((keys, queries, lf, kind, seed, None))
    # duplicate-rate sweep shape (test_query.py:149-164): explicit small hash range
    keys = rng.integers(1, (1 << 14) + 1, size=1 << 14, dtype=np.uint32)
    queries = rng.integers(1, (1 << 14) + 1, size=1 << 14, dtype=np.uint32)
    qspecs.append((keys, queries, 1.0, 0, 0, (1 << 14) // 32))
    for keys, queries, lf, kind, seed, hr in qspecs:
        table = hg.build(keys, lf, _fam(hg, kind, seed), 1, hr)
        res = hg.intersect(table, queries)
        cases.append(dict(keys=keys, queries=queries, load_factor=lf, kind=kind, seed=seed,
                          hash_range=np.uint64(table.hash_range),
                          multiplicities=res.multiplicities, matched=res.matched_positions,
                          total=res.total_matches, comparisons=res.comparisons,
                          hash_values=res.hash_values))
    _save("query", cases)

    # ---- sharded build + query (multishard.py:266-542)
    cases = []
    sspecs = [
        ([np.array([0, 1], np.uint32), np.array([2, 3], np.uint32)], 2, 1.0, 1, 0, 4, 4,
         np.array([3, 9], np.uint32)),
        ([np.array([], np.uint32), np.array([], np.uint32)], 2, 1.0, 0, 0, 0, 0, np.array([1, 2, 3], np.uint32)),
        ([np.full(5000, 77, np.uint32)[:2500], np.full(2500, 77, np.uint32)], 2, 1.0, 0, 0, 0, 70,
         np.array([77, 78], np.uint32)),
    ]
    for p, n, dom, lf in [(1, 5000, 1 << 14, 1.0), (2, 1 << 14, 1 << 16, 1.0), (3, 4017, 1 << 12, 0.5),
                          (4, 1 << 15, 1 << 15, 1.0), (8, 1 << 16, 1 << 18, 2.0), (8, 1 << 15, 256, 1.0),
                          (16, 1 << 16, 1 << 16, 1.0), (5, 37, 1 << 10, 1.0)]:
        kind = int(rng.integers(0, 2))
        seed = int(rng.integers(0, 1 << 32)) if kind == 0 else 0
        keys = rng.integers(1, dom + 1, size=n, dtype=np.uint64).astype(np.uint32)
        parts = list(np.array_split(keys, p))
        queries = np.concatenate([rng.choice(keys, size=n // 4) if n else np.empty(0, np.uint32),
                                  rng.integers(1, dom + 1, size=n // 4, dtype=np.uint64).astype(np.uint32)])
        sspecs.append((parts, p, lf, kind, seed, 0, 0, queries.astype(np.uint32)))
    for parts, p, lf, kind, seed, hr, bins, queries in sspecs:
        cfg = hg.ShardConfig(shards=p, load_factor=lf, bins_g=bins, family=_fam(hg, kind, seed), hash_range=hr)
        table, report = hg.build_sharded(parts, cfg)
        res = hg.query_sharded(table, queries)
        case = dict(p=p, load_factor=lf, kind=kind, seed=seed, hr_in=hr, bins_in=bins,
                    hash_range=report.hash_range, bins_g=report.bins_g, bin_size=table.plan.bin_size,
                    splits=table.plan.bin_splits, received=np.array(report.shard_received_counts),
                    search_steps=report.search_steps, bytes_exchanged=report.bytes_exchanged,
                    queries=queries, multiplicities=res.multiplicities, matched=res.matched_positions,
                    total=res.total_matches, comparisons=res.comparisons, hash_values=res.hash_values)
        for d, a in enumerate(parts):
            case[f"in{d}"] = a
            sb = hg.reorganize(a, table.plan, _fam(hg, kind, seed))
            case[f"send_off{d}"] = sb.offsets
            case[f"send_keys{d}"] = sb.keys
        for d, s in enumerate(table.shards):
            case[f"off{d}"] = s.offset
            case[f"keys{d}"] = s.keys
        cases.append(case)
    _save("sharded", cases)

    # ---- workload (workload.py:63-85)
    idx = np.array([0, 1, 2, 3, 1000, (1 << 31) + 5, (1 << 40) + 3], dtype=np.uint64)
    cases = []
    for seed in [0, 1, 1234567, 0x51, (1 << 64) - 1]:
        cases.append(dict(seed=np.uint64(seed), idx=idx, out=hg.splitmix64_at(seed, idx)))
    for k, count, seed in [(24, 4096, 0), (16, 1000, 0x51), (32, 3000, 7), (1, 100, 3), (30, 5000, 2)]:
        keys = hg.generate(hg.WorkloadSpec(hg.WorkloadKind.RANDOM_WITH_REPLACEMENT, k, count, seed))
        cases.append(dict(seed=np.uint64(seed), k=k, count=count, keys=keys))
    _save("workload", cases)


if __name__ == "__main__":
    main()
