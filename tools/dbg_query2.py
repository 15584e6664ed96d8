import sys; sys.path.insert(0, ".")
import numpy as np
from paper_2104_00792_b200 import _lib
if len(sys.argv) > 2: _lib.load(sys.argv[2])
import paper_2104_00792_b200 as hg
import oracle as O
rng = np.random.default_rng(1)
n = int(sys.argv[1])
keys = rng.integers(1, 1 << 20, size=n, dtype=np.uint32)
qs = rng.integers(1, 1 << 20, size=n, dtype=np.uint32)
t = hg.build(keys)
off, placed, _ = O.build_csr(keys, t.hash_range)
print("build ok", np.array_equal(t.offset, off))
r = hg.intersect(t, qs)
print("query ok", np.array_equal(r.multiplicities, O.count_occurrences(keys, qs)))
