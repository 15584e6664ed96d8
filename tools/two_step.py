"""Device time of the reference's two-step query (build_query_table +
intersect_tables, query.py:84-179) vs the fused intersect() at 2^L.
usage: python tools/two_step.py [log2]"""
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2104_00792_b200 as hg  # noqa: E402
from paper_2104_00792_b200 import _device as D, _lib  # noqa: E402
from paper_2104_00792_b200.core import build_device  # noqa: E402
from paper_2104_00792_b200.hashing import family_code  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 28
n = 1 << L
rand = hg.WorkloadKind.RANDOM_WITH_REPLACEMENT
keys = hg.generate_device(hg.WorkloadSpec(rand, L, n, 0))
qs = hg.generate_device(hg.WorkloadSpec(rand, L, n, 0x51))
table = hg.build(keys)


def timed(fn, reps=5):
    ts = []
    for _ in range(reps + 1):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        out = fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return sorted(ts[1:])[reps // 2], out


kind, seed = family_code(table.family)
v = table.hash_range
t_fused, r = timed(lambda: hg.intersect(table, qs))


def bqt():
    return build_device(qs, v, table.family, 32, True, True)


t_bqt, (qoff, qedges, qpos, trace) = timed(bqt)
mult = torch.zeros(n, dtype=torch.int32, device="cuda")
agg = torch.zeros(3, dtype=torch.int64, device="cuda")
ws = D.workspace(_lib.load().hg_intersect_tables_workspace_size(n, v, table.num_keys, 32))


def tables(tr):
    agg.zero_()
    _lib.call("hg_intersect_tables", D.ptr(table.offset_device), D.ptr(table.keys_device), table.num_keys, D.ptr(qoff),
              D.ptr(qedges), D.ptr(qpos), n, 32, kind, seed, v, D.ptr(tr) if tr is not None else None,
              tr.numel() if tr is not None else 0, D.ptr(mult), D.ptr(agg), D.ptr(ws), ws.numel(), D.stream_ptr())
    return agg


t_it, a = timed(lambda: tables(trace))
ok = torch.equal(mult, r.multiplicities_device) and [int(x) for x in a.cpu()] == [r.matched_positions, r.total_matches, r.comparisons]
t_sc, _ = timed(lambda: tables(None))
ok2 = torch.equal(mult, r.multiplicities_device)
print(json.dumps({"log2": L, "intersect_ms": round(t_fused, 3), "build_query_table_ms": round(t_bqt, 3),
                  "intersect_tables_traced_ms": round(t_it, 3), "intersect_tables_scatter_ms": round(t_sc, 3),
                  "two_step_over_fused": round((t_bqt + t_it) / t_fused, 2), "exact": bool(ok and ok2)}))

# per-kernel device times of one two-step run (library-recorded CUDA events)
_lib.timing_enable(True)
_lib.timing_collect()
bqt()
tables(trace)
torch.cuda.synchronize()
from collections import defaultdict  # noqa: E402
acc = defaultdict(float)
for name, ms in _lib.timing_collect(1 << 14):
    acc[name] += ms
_lib.timing_enable(False)
print(" ".join(f"{k} {v:.3f}" for k, v in sorted(acc.items(), key=lambda kv: -kv[1])))
