import sys; sys.path.insert(0, ".")
import numpy as np
import paper_2104_00792_b200 as hg
import oracle as O
rng = np.random.default_rng(1)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 70000
keys = rng.integers(1, 1 << 20, size=n, dtype=np.uint32)
qs = rng.integers(1, 1 << 20, size=n, dtype=np.uint32)
t = hg.build(keys)
r = hg.intersect(t, qs)
m = r.multiplicities
print("ok", np.array_equal(m, O.count_occurrences(keys, qs)))
