"""Virtual shards on one GPU at scale: build_sharded / query_sharded with 8 shards x 2^25
keys vs one shard of 2^28, wall time after the inputs are resident (PhaseReport.total_time_ns) and query time."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2104_00792_b200 as hg  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 25
P = 8
r = hg.WorkloadKind.RANDOM_WITH_REPLACEMENT
parts = [hg.generate_device(hg.WorkloadSpec(r, L + 3, 1 << L, d)) for d in range(P)]
qs = hg.generate_device(hg.WorkloadSpec(r, L + 3, P << L, 0x51))
fam = hg.HashFamily(hg.HashKind.MURMUR32, 0)
for label, ps, p in (("one shard", [torch.cat(parts)], 1), ("8 virtual shards", parts, P)):
    bt, qt = [], []
    for _ in range(4):
        table, rep = hg.build_sharded(ps, hg.ShardConfig(shards=p, family=fam))
        bt.append(rep.total_time_ns / 1e6)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = hg.query_sharded(table, qs)
        _ = res.matched_positions
        torch.cuda.synchronize()
        qt.append(1e3 * (time.perf_counter() - t0))
    n = P << L
    print(f"{label}: build {sorted(bt)[1]:.2f} ms ({n / sorted(bt)[1] / 1e6:.1f} G keys/s), "
          f"query {sorted(qt)[1]:.2f} ms ({n / sorted(qt)[1] / 1e6:.1f} G keys/s)", flush=True)
