"""build_sharded / query_sharded with shards placed on devices (GPU).

VERDICT r1 N1: the reference's own partitioned build (multishard.py:336-542)
must reach real GPUs through an import swap.  `build_sharded(..., devices=)`
(default: one shard per visible GPU when the counts match) drives every shard
from one host thread.  Checked against the oracle's four-phase restatement
(oracle/restatement.py build_sharded / query_sharded):

* plan, received counts, search steps and bytes exchanged exact;
* every shard's offsets exact and bucket multisets equal (`canonical`);
* query multiplicities and aggregates exact.

The single-GPU boxes run the device-placement path with repeated device ids
and the per-row exchange forced (the copy path used between GPUs); the
multi-GPU case runs when more than one GPU is visible and skips otherwise.
"""

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

hg = pytest.importorskip("paper_2104_00792_b200")
from paper_2104_00792_b200 import multishard  # noqa: E402


def check_against_oracle(parts, shards, table, report, queries, lf=1.0):
    ref = O.build_sharded(parts, shards, load_factor=lf)
    assert np.array_equal(table.plan.bin_splits, ref["splits"])
    assert report.shard_received_counts == ref["received"]
    assert report.search_steps == ref["search_steps"]
    n = sum(len(p) for p in parts)
    assert report.bytes_exchanged == 4 * n
    for sh, (off, keys) in zip(table.shards, ref["tables"]):
        assert np.array_equal(sh.offset, off)
        assert np.array_equal(O.canonical(sh.offset, sh.keys)[1], O.canonical(off, keys)[1])
    res = hg.query_sharded(table, queries)
    mult, matched, total, comp, hv = O.query_sharded(ref, queries)
    assert np.array_equal(res.multiplicities, mult)
    assert (res.matched_positions, res.total_matches, res.comparisons, res.hash_values) == (matched, total, comp, hv)


@pytest.mark.parametrize("shards", [2, 3, 8])
def test_device_placement_path_on_one_gpu(shards, monkeypatch):
    import torch

    monkeypatch.setattr(multishard, "_EXCHANGE_BY_ROWS", True)
    rng = np.random.default_rng(211 + shards)
    keys = O.generate_keys(20, 1 << 20, shards)
    parts = list(np.array_split(keys, shards))
    parts[1] = parts[1][:0]  # an empty shard input
    queries = rng.integers(0, 1 << 20, size=1 << 18, dtype=np.uint32)
    devs = [torch.cuda.current_device()] * shards
    table, report = hg.build_sharded(parts, hg.ShardConfig(shards=shards), devices=devs)
    assert [d.index for d in table.devices] == devs
    check_against_oracle(parts, shards, table, report, queries)
    res, times = hg.query_sharded_timed(table, queries)
    assert times.total_ns > 0


def test_device_list_validation():
    import torch

    with pytest.raises(hg.ConfigError):
        hg.build_sharded([[1], [2]], hg.ShardConfig(shards=2), devices=[0])
    with pytest.raises(hg.ConfigError):
        hg.build_sharded([[1], [2]], hg.ShardConfig(shards=2), devices=[0, torch.cuda.device_count()])


def test_table_on_another_current_device_context():
    """A table is queried on its own device whatever device is current."""
    import torch

    keys = O.generate_keys(16, 1 << 16, 5)
    with torch.cuda.device(0):
        table = hg.build(keys)
    queries = O.generate_keys(16, 1 << 14, 6)
    res = hg.intersect(table, queries)
    assert np.array_equal(res.multiplicities, O.count_occurrences(keys, queries))


@pytest.mark.skipif(not __import__("torch").cuda.is_available() or __import__("torch").cuda.device_count() < 2,
                    reason="needs two or more visible GPUs (the pool's boxes have one)")
def test_one_shard_per_gpu():
    import torch

    p = torch.cuda.device_count()
    keys = O.generate_keys(22, 1 << 22, 0)
    parts = list(np.array_split(keys, p))
    queries = O.generate_keys(22, 1 << 20, 0x51)
    table, report = hg.build_sharded(parts, hg.ShardConfig(shards=p))  # default: shard d on GPU d
    assert [d.index for d in table.devices] == list(range(p))
    check_against_oracle(parts, p, table, report, queries)
