"""Summaries of one ncu capture: headline metrics (details page) and the top stalled SASS
instructions with their dominant stall reason (source page).
  python tools/ncu_stalls.py gpurun_out/x.ncu-rep [--top 30] [--around ADDR]"""
import argparse
import csv
import io
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--top", type=int, default=25)
ap.add_argument("--kernel", default=None)
a = ap.parse_args()
det = subprocess.check_output(["ncu", "-i", a.rep, "--page", "details", "--csv"], text=True)
rows = list(csv.reader(io.StringIO(det)))
h = rows[0]
keys = ["Duration", "DRAM Throughput", "Memory Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "No Eligible", "L2 Hit Rate", "Achieved Occupancy", "Registers Per Thread",
        "Warp Cycles Per Issued Instruction"]
for r in rows[1:]:
    d = dict(zip(h, r))
    if a.kernel and a.kernel not in d["Kernel Name"]:
        continue
    if d.get("Metric Name") in keys:
        print(d["Kernel Name"][:40], "|", d["Metric Name"], "|", d["Metric Unit"], "|", d["Metric Value"])
src = subprocess.check_output(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "sass"]
                              + (["-k", a.kernel] if a.kernel else []), text=True)
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h)]
si = h.index("Warp Stall Sampling (All Samples)")
ie = h.index("Instructions Executed")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
num = lambda x: int(x) if x.isdigit() else 0
tot = sum(num(r[si]) for r in data)
print("total stall samples", tot)
agg = {}
for r in data:
    d = dict(zip(h, r))
    for c in reasons:
        agg[c] = agg.get(c, 0) + num(d[c])
print("by reason:", sorted(((v, k) for k, v in agg.items()), reverse=True)[:8])
for r in sorted(data, key=lambda r: -num(r[si]))[:a.top]:
    d = dict(zip(h, r))
    rs = sorted(((num(d[c]), c) for c in reasons), reverse=True)[:1]
    print(r[0][-5:], str(num(r[si])).rjust(6), r[ie].rjust(9), r[1][:64], rs)
