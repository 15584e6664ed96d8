"""Diagnose per-step device time vs kernel time (host gaps, allocator)."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2104_00792_b200 as hg
from paper_2104_00792_b200 import _lib

n = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 28
keys = hg.generate_device(hg.WorkloadSpec(hg.WorkloadKind.RANDOM_WITH_REPLACEMENT, 28, n, 0))
qs = hg.generate_device(hg.WorkloadSpec(hg.WorkloadKind.RANDOM_WITH_REPLACEMENT, 28, n, 0x51))
for _ in range(3):
    t = hg.build(keys); r = hg.intersect(t, qs)
torch.cuda.synchronize()
st0 = torch.cuda.memory_stats()
for mode in ["build", "query", "both"]:
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    e[0].record()
    for _ in range(5):
        if mode in ("build", "both"):
            t = hg.build(keys)
        if mode in ("query", "both"):
            r = hg.intersect(t, qs)
    e[1].record()
    w1 = time.perf_counter()
    torch.cuda.synchronize()
    w2 = time.perf_counter()
    print(f"{mode}: device {e[0].elapsed_time(e[1])/5:.3f} ms/step, host enqueue {(w1-w0)/5*1e3:.3f} ms/step, wall {(w2-w0)/5*1e3:.3f}")
st1 = torch.cuda.memory_stats()
for k in ["num_device_alloc", "num_device_free", "num_alloc_retries", "num_sync_all_streams"]:
    print(k, st1.get(k, 0) - st0.get(k, 0))
_lib.timing_enable(True)
t = hg.build(keys); r = hg.intersect(t, qs)
torch.cuda.synchronize()
for name, ms in _lib.timing_collect():
    print(f"  {name:20s} {ms:.3f}")
