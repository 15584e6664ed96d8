"""Per-kernel device times of one Zipf(1.1) build + query at 2^L (library-recorded events)."""
import sys
from collections import defaultdict

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2104_00792_b200 as hg  # noqa: E402
from paper_2104_00792_b200 import _lib  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 26
n = 1 << L


def zipf(count, seed, a=1.1):
    u = np.random.default_rng(seed).random(count)
    x = np.floor(np.maximum(u, 1e-300) ** (-1.0 / (a - 1.0)))
    return torch.from_numpy(np.mod(x, 2.0 ** 32).astype(np.uint64).astype(np.uint32).view(np.int32)).cuda()


k, q = zipf(n, 1), zipf(n, 2)
for it in range(3):
    _lib.timing_enable(True)
    _lib.timing_collect()
    t = hg.build(k)
    r = hg.intersect(t, q)
    torch.cuda.synchronize()
    acc = defaultdict(float)
    for name, ms in _lib.timing_collect(1 << 14):
        acc[name] += ms
    _lib.timing_enable(False)
print(" ".join(f"{a} {b:.3f}" for a, b in sorted(acc.items(), key=lambda kv: -kv[1])[:10]))
