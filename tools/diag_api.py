"""Phases of one reference-API step with numpy in/out (what a reference caller
does): hg.build(numpy keys), hg.intersect(table, numpy queries),
res.multiplicities (int64 numpy) + aggregates.  usage: python tools/diag_api.py [log2]"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2104_00792_b200 as hg  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 28
n = 1 << L
rand = hg.WorkloadKind.RANDOM_WITH_REPLACEMENT
keys = hg.generate_device(hg.WorkloadSpec(rand, L, n, 0)).cpu().numpy().view(np.uint32)
qs = hg.generate_device(hg.WorkloadSpec(rand, L, n, 0x51)).cpu().numpy().view(np.uint32)


def step():
    t = [time.perf_counter()]
    tab = hg.build(keys)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    r = hg.intersect(tab, qs)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    m = r.multiplicities
    t.append(time.perf_counter())
    a = (r.matched_positions, r.total_matches, r.comparisons)
    t.append(time.perf_counter())
    return [1e3 * (t[i + 1] - t[i]) for i in range(4)], int(m[-1]) + a[0]


for i in range(4):
    ph, _ = step()
    print(f"step {i}: build {ph[0]:.1f} ms, intersect {ph[1]:.1f} ms, multiplicities {ph[2]:.1f} ms, aggregates {ph[3]:.1f} ms, "
          f"total {sum(ph):.1f} ms", flush=True)
