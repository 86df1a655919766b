"""Summarise an ncu --set full capture: speed-of-light lines and the stall
reasons aggregated over the kernel's SASS (tuning aid)."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
keep = ("Duration", "DRAM Throughput", "Memory Throughput", "Issue Slots Busy", "Registers Per Thread",
        "Achieved Active Warps Per SM", "No Eligible", "Eligible Warps Per Scheduler", "L2 Hit Rate")
for d in csv.DictReader(io.StringIO(det)):
    if d.get("Metric Name") in keep:
        print(f"{d['Metric Name']:32s} {d['Metric Value']} {d['Metric Unit']}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]
f = lambda x: float(x) if x else 0.0
agg = collections.Counter()
for d in data:
    for k in h:
        if k.startswith("stall_") and "Not Issued" not in k:
            agg[k] += f(d[k])
tot = sum(agg.values())
print("stalls:", ", ".join(f"{k[6:]} {v / tot * 100:.1f}%" for k, v in agg.most_common(8)))
key = "Warp Stall Sampling (All Samples)"
for d in sorted(data, key=lambda d: -f(d[key]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    top = max((k for k in h if k.startswith("stall_") and "Not Issued" not in k), key=lambda k: f(d[k]))
    print(f"  {d['Address'][-5:]} {f(d[key]) / tot * 100:5.1f}% {top[6:]:16s} {d['Source'][:70]}")
