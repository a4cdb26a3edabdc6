"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
launches, total ms, share and ms/launch per kernel.  usage: python tools/launch_summary.py launches.csv"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
kn, mn, mv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
tot, cnt = defaultdict(float), defaultdict(int)
unit = h.index("Metric Unit") if "Metric Unit" in h else None
for r in rows[hi + 1:]:
    if len(r) <= mv or r[mn] != "gpu__time_duration.sum":
        continue
    name = r[kn].split("(")[0].replace("void ", "")
    if not name.startswith("dm::"):
        name = "torch/other: " + name.split("<")[0][:40]
    v = float(r[mv].replace(",", ""))
    u = r[unit] if unit is not None else "ns"
    ms = v * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(u, 1e-6)
    tot[name] += ms
    cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':34s} {'launches':>8s} {'total ms':>10s} {'share':>7s} {'ms/launch':>10s}")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k:34s} {cnt[k]:8d} {tot[k]:10.2f} {100 * tot[k] / T:6.1f}% {tot[k] / cnt[k]:10.3f}")
