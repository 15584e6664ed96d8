"""Skew and duplicate-rate timings of build + query on one GPU (device time, CUDA events).

Cases (2^L keys and 2^L queries, uint32, murmur32):
  uniform   keys/queries from {1..2^L}, V = N                      (the bench workload)
  dup-d     the same keys, V = N / d for d in 1..128 (acceptance c05's sweep, core.py:164-209)
  identical every key = 7, queries = 7                              (one bucket holds everything)
  zipf      Pareto-discretised Zipf(1.1) keys and queries over 32-bit values

usage: python tools/skew.py [log2] [case ...]
"""
import json
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2104_00792_b200 as hg  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 28
cases = sys.argv[2:] or ["uniform", "dup", "identical", "zipf"]
n = 1 << L
dev = torch.device("cuda", 0)


def zipf(count, seed, a=1.1):
    g = torch.Generator(device=dev).manual_seed(seed)
    u = torch.rand(count, generator=g, device=dev, dtype=torch.float64).clamp_min_(1e-300)
    x = torch.floor(u.pow(-1.0 / (a - 1.0)))
    return torch.remainder(x, 2.0 ** 32).to(torch.int64).to(torch.int32)


def timed(fn, reps=3):
    ts = []
    out = None
    for _ in range(reps + 1):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s.record()
        out = fn()
        e.record()
        torch.cuda.synchronize()
        ts.append((s.elapsed_time(e), time.perf_counter() - t0))
        if ts[-1][1] > 20:  # far too slow: one sample is enough
            break
    ms = sorted(t[0] for t in ts[1:] or ts)[len(ts[1:] or ts) // 2]
    return out, ms


def run(label, keys, queries, hash_range=None):
    t, bms = timed(lambda: hg.build(keys, 1.0, hash_range=hash_range))
    r, qms = timed(lambda: hg.intersect(t, queries))
    line = {"case": label, "log2": L, "hash_range": t.hash_range, "build_ms": round(bms, 3),
            "build_gkeys": round(n / bms / 1e6, 2), "query_ms": round(qms, 3), "query_gkeys": round(n / qms / 1e6, 2),
            "matched": r.matched_positions, "total": r.total_matches, "comparisons": r.comparisons}
    print(json.dumps(line), flush=True)
    return t, r


rand = hg.WorkloadKind.RANDOM_WITH_REPLACEMENT
keys = hg.generate_device(hg.WorkloadSpec(rand, L, n, 0))
qs = hg.generate_device(hg.WorkloadSpec(rand, L, n, 0x51))
if "uniform" in cases:
    run("uniform", keys, qs)
if "dup" in cases:
    for d in (1, 2, 4, 8, 16, 32, 64, 128, 1024, 1 << 16):
        run(f"dup-{d}", keys, qs, hash_range=n // d)
del keys, qs
if "identical" in cases:
    k7 = torch.full((n,), 7, dtype=torch.int32, device=dev)
    t, r = run("identical", k7, k7)
    assert r.matched_positions == n and r.total_matches == n * n, (r.matched_positions, r.total_matches)
    del k7, t, r
if "zipf" in cases:
    run("zipf1.1", zipf(n, 1), zipf(n, 2))
