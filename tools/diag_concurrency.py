"""Do two independent pipelines gain from running concurrently?  Times two 2^27-key builds (and two
build+query steps) on one stream vs on two streams (device time, CUDA events)."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2104_00792_b200 as hg  # noqa: E402

n = 1 << 27
r = hg.WorkloadKind.RANDOM_WITH_REPLACEMENT
ka = hg.generate_device(hg.WorkloadSpec(r, 27, n, 0))
kb = hg.generate_device(hg.WorkloadSpec(r, 27, n, 1))
qa = hg.generate_device(hg.WorkloadSpec(r, 27, n, 2))
qb = hg.generate_device(hg.WorkloadSpec(r, 27, n, 3))
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def step(k, q):
    t = hg.build(k)
    hg.intersect(t, q)


def timed(fn, reps=5):
    ts = []
    for _ in range(reps + 1):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record(torch.cuda.current_stream())
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts[1:])[reps // 2]


def serial():
    step(ka, qa)
    step(kb, qb)


def concurrent():
    main = torch.cuda.current_stream()
    ev = torch.cuda.Event()
    ev.record(main)
    for s, k, q in ((s1, ka, qa), (s2, kb, qb)):
        s.wait_event(ev)
        with torch.cuda.stream(s):
            step(k, q)
    main.wait_stream(s1)
    main.wait_stream(s2)


serial(); concurrent()
print("two 2^27 build+query steps: serial %.3f ms, two streams %.3f ms" % (timed(serial), timed(concurrent)))
