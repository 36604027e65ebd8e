"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per-kernel launch count, total device time and share.  Usage:
    python profiles/summarize_launches.py profiles/r1_launches.csv"""
import csv
import re
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = OrderedDict()
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r[ki]).replace("void ", "")
    name = re.sub(r"<.*", "", name).split("::")[-1]
    v = float(r[vi].replace(",", ""))
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
    c, t = agg.get(name, (0, 0.0))
    agg[name] = (c + 1, t + v * scale)
tot = sum(t for _, t in agg.values())
print(f"{'kernel':28s} {'launches':>8s} {'total_us':>10s} {'share':>7s}")
for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{n:28s} {c:8d} {t:10.1f} {t / tot * 100:6.1f}%")
print(f"{'total':28s} {sum(c for c, _ in agg.values()):8d} {tot:10.1f}")
