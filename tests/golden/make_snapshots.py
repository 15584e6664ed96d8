"""Golden snapshot / key-file / CLI-counter fixtures made by the REFERENCE itself.

Run in the dev container (where /root/reference exists):

    python tests/golden/make_snapshots.py

Writes, using the unmodified reference package (/root/reference/pkg/src):
  ref_murmur.hgr    save_table of build(keys k=12, 3000 rand, seed 7, lf 1.5, murmur seed 5)   (core.py:212-225)
  ref_identity.hgr  save_table of build(same keys, identity family, hash_range 1000)
  ref_keys.key      save_keys(same keys, k=12)                                                 (workload.py:95-101)
  cli_counters.json deterministic counters of `cli build` runs (cli.py:162-185), timings dropped
Nothing at test or bench time reads /root/reference; only this generator does.
"""

from __future__ import annotations

import json
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
import hashgraph as hg  # noqa: E402
from hashgraph.cli import main as ref_cli  # noqa: E402

CLI_RUNS = {
    "rand_k18_4shards": ["--kind", "rand", "--k", "18", "--count", "40000", "--shards", "4", "--rng-seed", "5"],
    "seq_k16_1shard": ["--kind", "seq", "--k", "16", "--count", "65536", "--shards", "1"],
    "rand_k16_3shards_lf2": ["--kind", "rand", "--k", "16", "--count", "50000", "--shards", "3", "--load-factor",
                             "2.0", "--seed", "11"],
    "identity_2shards": ["--kind", "rand", "--k", "20", "--count", "30000", "--shards", "2", "--hash", "identity"],
}
COUNTER_KEYS = ["schema", "shards", "total_keys", "hash_range", "bins_g", "load_factor", "family", "seed", "passes",
                "search_steps", "bytes_exchanged", "shard_received_counts"]


def main() -> None:
    keys = hg.generate(hg.WorkloadSpec(hg.WorkloadKind.RANDOM_WITH_REPLACEMENT, 12, 3000, 7))
    t = hg.build(keys, 1.5, hg.HashFamily(hg.HashKind.MURMUR32, 5))
    hg.save_table(t, os.path.join(HERE, "ref_murmur.hgr"))
    t = hg.build(keys, 1.0, hg.HashFamily(hg.HashKind.IDENTITY, 0), hash_range=1000)
    hg.save_table(t, os.path.join(HERE, "ref_identity.hgr"))
    hg.save_keys(keys, 12, os.path.join(HERE, "ref_keys.key"))
    out = {}
    with tempfile.TemporaryDirectory() as d:
        for name, args in CLI_RUNS.items():
            path = os.path.join(d, "r.json")
            assert ref_cli(["build", *args, "--out", path]) == 0
            rep = json.load(open(path))
            phases = {p: {k: v for k, v in st.items() if k != "time_ns"} for p, st in rep["phases"].items()}
            out[name] = {"args": args, "report": {k: rep[k] for k in COUNTER_KEYS}, "phases": phases}
    json.dump(out, open(os.path.join(HERE, "cli_counters.json"), "w"), indent=1)
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
