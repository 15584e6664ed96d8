"""Direct (Alg. 1, global atomics) vs binned build device time by size (HG_FORCE_DIRECT=1 for the direct path)."""
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2104_00792_b200 as hg  # noqa: E402

for L in range(16, 26):
    n = 1 << L
    keys = hg.generate_device(hg.WorkloadSpec(hg.WorkloadKind.RANDOM_WITH_REPLACEMENT, min(L, 32), n, 0))
    qs = hg.generate_device(hg.WorkloadSpec(hg.WorkloadKind.RANDOM_WITH_REPLACEMENT, min(L, 32), n, 0x51))
    ts, tq = [], []
    for _ in range(6):
        a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        torch.cuda.synchronize()
        a.record()
        t = hg.build(keys)
        b.record()
        hg.intersect(t, qs)
        c.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
        tq.append(b.elapsed_time(c))
    print(os.environ.get("HG_FORCE_DIRECT", "binned"), L, "build_us", round(sorted(ts[1:])[2] * 1e3, 1),
          "query_us", round(sorted(tq[1:])[2] * 1e3, 1), flush=True)
