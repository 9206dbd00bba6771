"""Print an ncu --csv launch list as one line per launch. Usage: python tools/ncu_rows.py file.csv"""
import csv
import sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
H = rows[hdr]
ki, mi, vi = H.index("Kernel Name"), H.index("Metric Name"), H.index("Metric Value")
out = {}
for r in rows[hdr + 1:]:
    if len(r) > vi:
        out.setdefault((int(r[0]), r[ki].split("::")[-1][:28]), {})[r[mi]] = r[vi]
for (i, k), m in sorted(out.items()):
    print(i, k, " ".join(f"{a.split('__')[0][:6]}.{a.split('__')[1][:22]}={v}" for a, v in sorted(m.items())))
