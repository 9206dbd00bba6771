"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv) to per-kernel totals
of the LAST solve in the capture (from its k_init).  Usage: launch_summary.py in.csv title"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
title = sys.argv[2] if len(sys.argv) > 2 else ""
hdr, data = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
names = [d["Kernel Name"] for d in data]
t = [float(d["Metric Value"]) for d in data]
last = max(i for i, n in enumerate(names) if "k_init" in n)
solve = list(zip(names[last:], t[last:]))
tot = sum(x for _, x in solve)
agg = collections.OrderedDict()
for n, x in solve:
    k = n.split("(")[0].replace("void ", "")
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += x
print(f"# {title}")
print("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: compare shares)")
print(f"# total {tot / 1e3:.1f} us over {len(solve)} launches")
print("kernel,launches,total_us,share")
for k, (c, x) in agg.items():
    print(f"{k},{c},{x / 1e3:.1f},{x / tot:.3f}")
