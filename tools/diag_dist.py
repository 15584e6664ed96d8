"""Per-phase device time of the distributed path at N=1 (CUDA events around
each host-visible phase), to separate kernel time from sync/barrier cost.
usage (GPU box): python tools/diag_dist.py [p2p|nccl]"""
import os
import sys
import time

sys.path.insert(0, ".")
import torch
import torch.distributed as dist

import paper_2104_00792_b200 as hg
from paper_2104_00792_b200 import distributed as hd

tr = sys.argv[1] if len(sys.argv) > 1 else "p2p"
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29771")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
n = 1 << 28
keys = hg.generate_device(hg.WorkloadSpec(hg.WorkloadKind.RANDOM_WITH_REPLACEMENT, 28, n, 0))
qs = hg.generate_device(hg.WorkloadSpec(hg.WorkloadKind.RANDOM_WITH_REPLACEMENT, 28, n, 0x51))
cfg = hd.DistConfig(transport=tr)
for _ in range(3):
    t = hd.build_distributed(keys, cfg)
    r = hd.query_distributed(t, qs)
torch.cuda.synchronize()
for rep in range(3):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    w0 = time.perf_counter()
    e[0].record()
    t = hd.build_distributed(keys, cfg)
    e[1].record()
    r = hd.query_distributed(t, qs)
    e[2].record()
    torch.cuda.synchronize()
    w1 = time.perf_counter()
    print(f"{tr}: build {e[0].elapsed_time(e[1]):.3f} ms, query {e[1].elapsed_time(e[2]):.3f} ms, wall {1e3*(w1-w0):.3f} ms, "
          f"host phases {t.phase_ns}")
dist.destroy_process_group()
