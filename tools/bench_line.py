"""Condense bench.py JSON lines (stdin) to one line each: throughput, step, build/query
ms + fractions, and each kernel's device ms per step.  usage: python bench.py ... | python tools/bench_line.py LABEL"""
import json
import sys

label = sys.argv[1] if len(sys.argv) > 1 else ""
for line in sys.stdin:
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    r = d.get("roofline") or {}
    kern = d.get("kernels", [])
    steps = max(1, sum(k["launches"] for k in kern if k["kernel"] == "hg_hist") // 2)  # two per step
    ks = ", ".join(f"{k['kernel']} {k['avg_ms'] * k['launches'] / steps:.3f}" for k in kern)
    print(f"{label} {d['value'] / 1e9:.2f} G/s step {d['ms_per_step']:.3f} build {r.get('build_ms', 0):.3f} "
          f"({r.get('build_frac', 0):.3f}) query {r.get('query_ms', 0):.3f} ({r.get('query_frac', 0):.3f}) | {ks}",
          flush=True)
