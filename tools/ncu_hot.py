"""Summarise an ncu report's SASS source page: stall reasons, stall samples by
opcode and the hottest instructions.

usage: python tools/ncu_hot.py report.ncu-rep [N] [kernel-regex] [launch-skip]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
topn = int(sys.argv[2]) if len(sys.argv) > 2 else 25
cmd = ["ncu", "-i", rep]
if len(sys.argv) > 3:
    cmd += ["-k", "regex:" + sys.argv[3], "--launch-count", "1"]
if len(sys.argv) > 4:
    cmd += ["--launch-skip", sys.argv[4]]
out = subprocess.run(cmd + ["--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if len(r) > 3 and r[0] == "Address")
h = rows[hi]
idx = {k: i for i, k in enumerate(h)}
samp = idx["Warp Stall Sampling (All Samples)"]
execd = idx["Instructions Executed"]
src = idx["Source"]
stall_cols = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
tot = 0
by_op = defaultdict(int)
by_op_n = defaultdict(int)
by_stall = defaultdict(int)
agg = []
for r in rows[hi + 1:]:
    if len(r) <= samp:
        continue
    try:
        s = int(r[samp])
        n = int(r[execd])
    except ValueError:
        continue
    tot += s
    for k in stall_cols:
        try:
            by_stall[k] += int(r[idx[k]])
        except ValueError:
            pass
    op = r[src].split()[0] if r[src].split() else "?"
    if op.startswith("@"):
        op = r[src].split()[1]
    op = op.split(".")[0]
    by_op[op] += s
    by_op_n[op] += n
    agg.append((s, r[0], r[src][:110]))
print("total samples", tot, " total warp-instructions", sum(by_op_n.values()))
print("stall reasons:", ", ".join(f"{k[6:]} {100 * v / max(tot, 1):.1f}%"
                                  for k, v in sorted(by_stall.items(), key=lambda x: -x[1])[:8]))
for op, s in sorted(by_op.items(), key=lambda x: -x[1])[:15]:
    print(f"  {op:10s} {100*s/tot:5.1f}% samples   {by_op_n[op]:>12d} instr")
agg.sort(reverse=True)
for s, a, t in agg[:topn]:
    print(f"{s:7d} {100*s/max(tot,1):5.1f}%  {a[-5:]}  {t}")
