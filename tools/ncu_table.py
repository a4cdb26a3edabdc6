"""Per-launch table of an ncu report: duration, DRAM bytes, instructions,
occupancy, issue activity.  usage: python tools/ncu_table.py report.ncu-rep [particles]"""
import csv
import io
import subprocess
import sys

M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
     "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
     "launch__registers_per_thread", "lts__t_bytes.sum"]
rep = sys.argv[1]
npart = float(sys.argv[2]) if len(sys.argv) > 2 else 16777216.0
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base", "--metrics", ",".join(M)],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
print(f"{'kernel':28s} {'us':>8s} {'DRAM MB':>9s} {'B/part':>7s} {'GB/s':>7s} {'winst/p':>8s} {'occ%':>5s} {'issue%':>6s} {'regs':>4s} {'L2 B/p':>7s}")
for r in rows[2:]:
    d = dict(zip(h, r))
    f = lambda k: float(d[k].replace(",", "")) if d.get(k) not in (None, "", "n/a") else 0.0
    t = f(M[0]) * 1e-9
    b = f(M[1]) + f(M[2])
    name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("dm::", "")[:28]
    print(f"{name:28s} {t*1e6:8.1f} {b/1e6:9.1f} {b/npart:7.1f} {b/t/1e9 if t else 0:7.0f} {f(M[3])/npart:8.2f} "
          f"{f(M[4]):5.1f} {f(M[5]):6.1f} {int(f(M[6])):4d} {f(M[7])/npart:7.1f}")
