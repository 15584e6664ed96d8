"""Summarise an ncu report's SASS page: top instructions by stall samples and
by executed count.  usage: python tools/ncu_hot.py REPORT KERNEL_REGEX [N]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout.splitlines()
start = [i for i, l in enumerate(out) if l.startswith('"Address"')][0]
rows = list(csv.reader(out[start:]))
h = rows[0]
ix = {k: h.index(k) for k in ["Source", "Warp Stall Sampling (All Samples)", "Instructions Executed"]}
data = []
for r in rows[1:]:
    if len(r) < len(h):
        continue
    try:
        data.append((int(r[ix["Warp Stall Sampling (All Samples)"]] or 0), int(r[ix["Instructions Executed"]] or 0),
                     r[ix["Source"]].strip()))
    except ValueError:
        pass
tot_s = sum(d[0] for d in data) or 1
tot_i = sum(d[1] for d in data) or 1
print(f"total stall samples {tot_s}, warp instructions {tot_i}")
for s, i, src in sorted(data, key=lambda d: -d[0])[:top]:
    print(f"{100*s/tot_s:5.1f}%  {i:>12}  {src}")
# opcode histogram by executed count
from collections import Counter
c = Counter()
for s, i, src in data:
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    c[op.split(".")[0]] += i
print("executed by opcode:", ", ".join(f"{k}:{100*v/tot_i:.1f}%" for k, v in c.most_common(15)))
