import sys, time
sys.path.insert(0, ".")
import torch
import paper_2104_00792_b200 as hg
from paper_2104_00792_b200 import _lib
from collections import defaultdict
L, P = 25, 8
r = hg.WorkloadKind.RANDOM_WITH_REPLACEMENT
parts = [hg.generate_device(hg.WorkloadSpec(r, L + 3, 1 << L, d)) for d in range(P)]
qs = hg.generate_device(hg.WorkloadSpec(r, L + 3, P << L, 0x51))
fam = hg.HashFamily(hg.HashKind.MURMUR32, 0)
for _ in range(3):
    table, rep = hg.build_sharded(parts, hg.ShardConfig(shards=P, family=fam))
print("total", rep.total_time_ns / 1e6, {k: v.time_ns / 1e6 for k, v in rep.phases.items()})
_lib.timing_enable(True); _lib.timing_collect()
table, rep = hg.build_sharded(parts, hg.ShardConfig(shards=P, family=fam))
torch.cuda.synchronize()
acc = defaultdict(float); cnt = defaultdict(int)
for name, ms in _lib.timing_collect(1 << 14):
    acc[name] += ms; cnt[name] += 1
print("build kernels", " ".join(f"{k} {v:.3f}x{cnt[k]}" for k, v in sorted(acc.items(), key=lambda kv: -kv[1])))
res = hg.query_sharded(table, qs); _ = res.matched_positions; torch.cuda.synchronize()
_lib.timing_collect()
t0 = time.perf_counter(); res = hg.query_sharded(table, qs); _ = res.matched_positions; torch.cuda.synchronize(); t1 = time.perf_counter()
acc = defaultdict(float); cnt = defaultdict(int)
for name, ms in _lib.timing_collect(1 << 14):
    acc[name] += ms; cnt[name] += 1
print("query wall", (t1 - t0) * 1e3, "kernels", " ".join(f"{k} {v:.3f}x{cnt[k]}" for k, v in sorted(acc.items(), key=lambda kv: -kv[1])))
ts = []
for _ in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = hg.query_sharded(table, qs)
    _ = res.matched_positions
    torch.cuda.synchronize()
    ts.append(1e3 * (time.perf_counter() - t0))
print("query wall x5 (ms)", " ".join(f"{x:.2f}" for x in ts))
