"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel.

    python tools/launch_summary.py launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}
t, n = collections.Counter(), collections.Counter()
for r in rows[start + 1:]:
    if len(r) != len(hdr):
        continue
    name = r[ik].split("(")[0].replace("void ", "").split("::")[-1]
    t[name] += float(r[iv].replace(",", "")) * scale[r[iu]]
    n[name] += 1
tot = sum(t.values())
print(f"{sum(n.values())} launches, {tot / 1e3:.1f} ms total (cold-cache, serialised)")
print("| kernel | share | launches | avg us |\n|---|---|---|---|")
for k, v in t.most_common(14):
    print(f"| {k} | {100 * v / tot:.1f}% | {n[k]} | {v / n[k]:.1f} |")
