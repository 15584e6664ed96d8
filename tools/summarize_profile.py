"""Summarise a round's ncu evidence into profiles/:
  - the launch list (gpu__time_duration per launch) -> per-kernel share table
  - the --set full capture -> DRAM bytes, throughput, issue stats per kernel
  - profiles/traffic.json: dram read+write bytes per launch keyed by the
    library's launch label (read by bench.py for roofline.traffic)
usage: python tools/summarize_profile.py ROUND LAUNCH_CSV NCU_REP"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

rnd, launch_csv, rep = sys.argv[1], sys.argv[2], sys.argv[3]
LABEL = {  # kernel function -> launch label used by the library / bench
    "k_hist": "hg_hist", "k_colscan": "hg_colscan", "k_starts": "hg_starts", "k_local_build_big": "hg_local_build_big",
    "k_local_build": "hg_local_build", "k_local_build_p": "hg_local_build", "k_local_probe": "hg_local_probe", "k_unpart<2>": "hg_unpart2",
    "k_unpart<1>": "hg_unpart1", "k_count": "hg_count", "k_scan": "hg_scan", "k_place": "hg_place",
    "k_intersect": "hg_intersect", "k_generate32": "hg_generate", "k_probe_plan": "hg_probe_plan",
    "k_big_count": "hg_big_count", "k_big_place": "hg_big_place", "k_ht_prep": "hg_ht_prep",
    "k_ht_insert": "hg_ht_insert", "k_ht_lookup": "hg_ht_lookup", "k_qstart": "hg_qstart",
    "k_perm_bins": "hg_perm_bins", "k_scatter_pos": "hg_scatter_pos",
}


def label(fn: str) -> str:
    name = fn.split("(")[0].replace("void ", "").replace("hg::", "").strip()
    base = name.split("<")[0]
    if base in ("k_part1", "k_part2"):
        targs = [t.strip() for t in name[name.index(">") + 1:].strip(" ,>").split(",")] if ">" in name else []
        q = ", true" in name or (len(targs) >= 1 and targs[0] == "1")
        return f"hg_{base[2:]}" + ("_q" if q else "")
    if base in ("k_unpart", "k_repart"):
        return f"hg_{base[2:]}" + ("2" if "<2>" in name else "1")
    return LABEL.get(base, name)


# ---- launch list
rows = list(csv.reader(open(launch_csv)))
hdr_i = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hdr_i]
per = defaultdict(list)
for r in rows[hdr_i + 1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    unit = d.get("Metric Unit", "")
    val = float(d["Metric Value"].replace(",", ""))
    ms = val / 1e6 if unit in ("nsecond", "ns") else val / 1e3 if unit in ("usecond", "us") else val
    per[label(d["Kernel Name"])].append(ms)
tot = sum(sum(v) for v in per.values())
lines = [f"# Round {rnd} ncu evidence", "",
         "## Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`, bench.py --steps 2 --warmup 1)", "",
         "Cold-cache, serialised per-launch times: compare shares, not absolutes.", "",
         "| kernel (label) | launches | avg ms | share |", "|---|---|---|---|"]
for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
    lines.append(f"| {k} | {len(v)} | {sum(v)/len(v):.3f} | {100*sum(v)/tot:.1f}% |")

# ---- full capture
mets = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active"]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(mets)],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
hh, units = r[0], r[1]
traffic = {}
lines += ["", "## Full capture (`ncu --set full --clock-control none --import-source on`), one launch per kernel", "",
          "| kernel | ms | DRAM read GB | DRAM write GB | DRAM % | SM % | issue-active % | regs | warp instr |",
          "|---|---|---|---|---|---|---|---|---|"]
for row in r[2:]:
    d = dict(zip(hh, row))
    lab = label(d["Kernel Name"])
    rd = float(d["dram__bytes_read.sum"]); wr = float(d["dram__bytes_write.sum"])
    ur = dict(zip(hh, units))
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}
    rd_b = rd * scale.get(ur["dram__bytes_read.sum"], 1)
    wr_b = wr * scale.get(ur["dram__bytes_write.sum"], 1)
    traffic.setdefault(lab, rd_b + wr_b)
    lines.append(f"| {lab} | {float(d['gpu__time_duration.sum']):.3f} | {rd_b/1e9:.3f} | {wr_b/1e9:.3f} | "
                 f"{float(d['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed']):.1f} | "
                 f"{float(d['sm__throughput.avg.pct_of_peak_sustained_elapsed']):.1f} | "
                 f"{float(d['smsp__issue_active.avg.pct_of_peak_sustained_active']):.1f} | "
                 f"{d['launch__registers_per_thread']} | {float(d['smsp__inst_executed.sum']):.3g} |")
os.makedirs("profiles", exist_ok=True)
open(f"profiles/{rnd}_ncu_summary.md", "w").write("\n".join(lines) + "\n")
old = json.load(open("profiles/traffic.json")) if os.path.exists("profiles/traffic.json") else {}
old.update(traffic)  # merge: a capture of some kernels keeps the others' figures
json.dump(old, open("profiles/traffic.json", "w"), indent=1)
print("\n".join(lines))
