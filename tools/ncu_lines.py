"""Per-CUDA-source-line executed instructions and stall samples for one kernel
of an ncu report (cuda,sass correlated view).
usage: python tools/ncu_lines.py REPORT KERNEL_REGEX [N]"""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}", "--launch-count", "1",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout.splitlines()
data = []
fname = ""
hdr = None
for row in csv.reader(out):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or not row[0] or row[0] == "Function Name":
        continue
    try:
        ss = float(row[4] or 0); ie = float(row[7] or 0)
    except (ValueError, IndexError):
        continue
    data.append((ie, ss, f"{fname}:{row[0]}", row[1].strip()[:100]))
ti = sum(d[0] for d in data) or 1; ts = sum(d[1] for d in data) or 1
print(f"warp instructions {ti:.3g}, stall samples {ts:.3g}")
for ie, ss, ln, src in sorted(data, key=lambda d: -d[0])[:top]:
    print(f"{100*ie/ti:5.1f}% inst {100*ss/ts:5.1f}% stall  {ln:>18}  {src}")
