"""One build + query of the bench workload (for ncu captures).
usage: python tools/one_step.py [log2_keys] [k] [load_factor] [key_bits] [reps]"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2104_00792_b200 as hg  # noqa: E402

a = sys.argv[1:]
n = 1 << int(a[0]) if a else 1 << 28
k = int(a[1]) if len(a) > 1 else 28
lf = float(a[2]) if len(a) > 2 else 1.0
kb = int(a[3]) if len(a) > 3 else 32
reps = int(a[4]) if len(a) > 4 else 1
keys = hg.generate_device(hg.WorkloadSpec(hg.WorkloadKind.RANDOM_WITH_REPLACEMENT, k, n, 0), key_bits=kb)
qs = hg.generate_device(hg.WorkloadSpec(hg.WorkloadKind.RANDOM_WITH_REPLACEMENT, k, n, 0x51), key_bits=kb)
for _ in range(reps):
    t = hg.build(keys, lf, key_bits=kb)
    r = hg.intersect(t, qs)
torch.cuda.synchronize()
print("matched", r.matched_positions)
