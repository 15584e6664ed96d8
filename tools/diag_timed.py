import sys; sys.path.insert(0, ".")
import time, torch, paper_2104_00792_b200 as hg
n = 1 << 28
keys = hg.generate_device(hg.WorkloadSpec(hg.WorkloadKind.RANDOM_WITH_REPLACEMENT, 28, n, 0))
qs = hg.generate_device(hg.WorkloadSpec(hg.WorkloadKind.RANDOM_WITH_REPLACEMENT, 28, n, 0x51))
t = hg.build(keys)
for _ in range(2): r, tm = hg.intersect_timed(t, qs)
r2 = hg.intersect(t, qs)
print("timed split ms", tm.table_build_ns / 1e6, tm.intersect_ns / 1e6, "same result", torch.equal(r.multiplicities_device, r2.multiplicities_device), r.matched_positions == r2.matched_positions)
