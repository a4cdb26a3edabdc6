"""Per-CUDA-source-line instruction counts and stall samples of one kernel in an
ncu report (cuda,sass view).  usage: python tools/ncu_lines.py rep kernel-regex [N] [skip]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
topn = int(sys.argv[3]) if len(sys.argv) > 3 else 30
cmd = ["ncu", "-i", rep, "-k", "regex:" + kre, "--launch-count", "1"]
if len(sys.argv) > 4:
    cmd += ["--launch-skip", sys.argv[4]]
out = subprocess.run(cmd + ["--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = []
fname = ""
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 8 or r[0] in ("Line No", "") or not r[0].isdigit():
        continue
    try:
        samp, ins = int(r[4]), int(r[7])
    except ValueError:
        continue
    agg.append((ins, samp, f"{fname}:{r[0]}", r[1].strip()[:90]))
ti = sum(a[0] for a in agg)
ts = sum(a[1] for a in agg)
print(f"total warp-instr {ti}  samples {ts}")
for ins, samp, loc, src in sorted(agg, reverse=True)[:topn]:
    print(f"{100*ins/ti:5.1f}% inst {100*samp/max(ts,1):5.1f}% stall  {loc:22s} {src}")
