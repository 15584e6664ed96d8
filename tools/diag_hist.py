"""Per-kernel device times of one build at 2^L keys for power-of-two and other hash ranges (virtual-shard sizes).
usage: python tools/diag_hist.py [L]"""
import sys
from collections import defaultdict

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2104_00792_b200 as hg  # noqa: E402
from paper_2104_00792_b200 import _lib  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 25
keys = hg.generate_device(hg.WorkloadSpec(hg.WorkloadKind.RANDOM_WITH_REPLACEMENT, L + 3, 1 << L, 0))
for v in (1 << L, (1 << L) + 12345, (1 << L) - 7):
    for _ in range(3):
        hg.build(keys, hash_range=v)
    torch.cuda.synchronize()
    _lib.timing_enable(True)
    _lib.timing_collect()
    hg.build(keys, hash_range=v)
    torch.cuda.synchronize()
    acc = defaultdict(float)
    for name, ms in _lib.timing_collect(1 << 12):
        acc[name] += ms
    _lib.timing_enable(False)
    print(v, " ".join(f"{k} {x:.3f}" for k, x in sorted(acc.items(), key=lambda kv: -kv[1])), flush=True)
