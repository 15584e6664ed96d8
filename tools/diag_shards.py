"""c09 shape: build_sharded wall time, 1 shard x 2^20 vs 8 shards x 2^20 (one GPU), with phase split."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2104_00792_b200 as hg  # noqa: E402

n_d = 1 << 20
rng = np.random.default_rng(909)
one = rng.integers(1, 1 << 20, size=n_d, dtype=np.uint32)
eight = [rng.integers(1, 1 << 20, size=n_d, dtype=np.uint32) for _ in range(8)]
fam = hg.HashFamily(hg.HashKind.MURMUR32, 0)
for label, parts, p in (("one", [one], 1), ("eight", eight, 8)):
    ts = []
    for _ in range(7):
        _, rep = hg.build_sharded(parts, hg.ShardConfig(shards=p, family=fam))
        ts.append(rep.total_time_ns)
    ph = {k: v.time_ns for k, v in rep.phases.items()}
    print(label, "median total us", sorted(ts)[3] / 1e3, "phases us", {k: v / 1e3 for k, v in ph.items()}, flush=True)

# host-side profile of one 8-shard build
import cProfile, pstats  # noqa: E402
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    hg.build_sharded(eight, hg.ShardConfig(shards=8, family=fam))
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
