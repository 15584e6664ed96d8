"""PCIe copy overlap and the e2e loop, diagnosed (GPU box): H2D / D2H alone and
concurrently, then where a pipelined e2e step blocks."""
import sys
import time

sys.path.insert(0, ".")
import torch

import paper_2104_00792_b200 as hg

n = 1 << 28
hk = torch.empty(n, dtype=torch.int32, pin_memory=True)
hq = torch.empty(n, dtype=torch.int32, pin_memory=True)
ho = torch.empty(n, dtype=torch.int32, pin_memory=True)
dk = torch.empty(n, dtype=torch.int32, device="cuda")
dq = torch.empty(n, dtype=torch.int32, device="cuda")
do = torch.empty(n, dtype=torch.int32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(f, reps=3):
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


def h2d():
    dk.copy_(hk, non_blocking=True)
    dq.copy_(hq, non_blocking=True)


def d2h():
    ho.copy_(do, non_blocking=True)


def both():
    with torch.cuda.stream(s1):
        h2d()
    with torch.cuda.stream(s2):
        d2h()


print(f"H2D 2 GiB {timed(h2d):.1f} ms, D2H 1 GiB {timed(d2h):.1f} ms, both on two streams {timed(both):.1f} ms")
keys = hg.generate_device(hg.WorkloadSpec(hg.WorkloadKind.RANDOM_WITH_REPLACEMENT, 28, n, 0))
hk.copy_(keys.cpu())
hq.copy_(hg.generate_device(hg.WorkloadSpec(hg.WorkloadKind.RANDOM_WITH_REPLACEMENT, 28, n, 0x51)).cpu())
for i in range(4):
    st = [s1, s2][i % 2]
    t0 = time.perf_counter()
    with torch.cuda.stream(st):
        t = hg.build(hk)
        t1 = time.perf_counter()
        r = hg.intersect(t, hq)
        t2 = time.perf_counter()
        ho.copy_(r.multiplicities_device, non_blocking=True)
    t3 = time.perf_counter()
    print(f"step {i}: enqueue build {1e3*(t1-t0):.2f} ms, intersect {1e3*(t2-t1):.2f} ms, d2h {1e3*(t3-t2):.2f} ms")
torch.cuda.synchronize()

# the bench's pipelined loop, with host timestamps
outs = [torch.empty(n, dtype=torch.int32, pin_memory=True) for _ in range(2)]
done = [None, None]
torch.cuda.synchronize()
T0 = time.perf_counter()
for i in range(8):
    slot = i % 2
    tw = time.perf_counter()
    if done[slot] is not None:
        done[slot].synchronize()
    tw2 = time.perf_counter()
    with torch.cuda.stream([s1, s2][slot]):
        t = hg.build(hk)
        r = hg.intersect(t, hq)
        outs[slot].copy_(r.multiplicities_device, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        done[slot] = ev
    print(f"step {i}: t={1e3*(tw-T0):.1f} waited {1e3*(tw2-tw):.1f} ms, enqueued at {1e3*(time.perf_counter()-T0):.1f}")
torch.cuda.synchronize()
print(f"total {1e3*(time.perf_counter()-T0):.1f} ms for 8 steps")
