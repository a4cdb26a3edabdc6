"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv).

usage: python tools/launch_summary.py LAUNCHES.csv "HEADER LINE" > SUMMARY.txt"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.defaultdict(list)
for r in rows[1:]:
    agg[r[ik].split("(")[0].replace("void ", "")].append(float(r[iv].replace(",", "")) * scale[r[iu]])
tot = sum(sum(v) for v in agg.values())
print("# " + (sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]))
print("# serialised, per-launch cold cache (ncu): shares, not absolute step times")
print("# %-30s %8s %10s %10s %7s" % ("kernel", "launches", "mean_us", "total_ms", "share"))
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print("%-32s %8d %10.1f %10.2f %6.1f%%" % (k[:32], len(v), sum(v) / len(v), sum(v) / 1e3, 100 * sum(v) / tot))
