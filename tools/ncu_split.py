"""Per-kernel SASS hot spots from a multi-kernel ncu report.
usage: python tools/ncu_split.py report.ncu-rep kernel_regex [N]"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

rep, pat = sys.argv[1], sys.argv[2]
topn = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{pat}",
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if len(r) > 3 and r[0] == "Address")
h = rows[hi]
idx = {k: i for i, k in enumerate(h)}
samp, execd, src = idx["Warp Stall Sampling (All Samples)"], idx["Instructions Executed"], idx["Source"]
tot, ninstr = 0, 0
by_op, by_op_n = defaultdict(int), defaultdict(int)
agg = []
for r in rows[hi + 1:]:
    if len(r) <= samp or r[0] == "Address":
        if r and r[0] == "Address":
            break
        continue
    try:
        s, n = int(r[samp]), int(r[execd])
    except ValueError:
        continue
    tot += s
    ninstr += n
    toks = r[src].split()
    op = toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "?")
    op = op.split(".")[0]
    by_op[op] += s
    by_op_n[op] += n
    agg.append((s, n, r[0][-5:], r[src][:100]))
print(f"samples {tot}  warp-instr {ninstr}")
for op, s in sorted(by_op.items(), key=lambda x: -x[1])[:14]:
    print(f"  {op:10s} {100*s/max(tot,1):5.1f}% samples  {by_op_n[op]:>11d} instr")
agg.sort(reverse=True)
for s, n, a, t in agg[:topn]:
    print(f"{s:6d} {100*s/max(tot,1):5.1f}% {n:>9d} {a} {t}")
