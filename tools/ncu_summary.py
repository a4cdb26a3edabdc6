"""Per-kernel summary of ncu --set full reports -> JSON (profiles/): duration,
DRAM bytes read+write per launch and per particle, instructions per particle,
occupancy, issue activity, registers.  usage:
  python tools/ncu_summary.py OUT.json PARTICLES_PER_LAUNCH rep1.ncu-rep [rep2 ...]"""
import csv
import io
import json
import subprocess
import sys

M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
     "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
     "launch__registers_per_thread", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
     "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"]
out, npart, reps = sys.argv[1], float(sys.argv[2]), sys.argv[3:]
res = {}
for rep in reps:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base", "--metrics", ",".join(M)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[0]
    for r in rows[2:]:
        d = dict(zip(h, r))
        f = lambda k: float(d[k].replace(",", "")) if d.get(k) not in (None, "", "n/a") else 0.0
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("dm::", "")
        cls = name.split("<")[0].replace("k_", "")
        t = f(M[0]) * 1e-9
        b = f(M[1]) + f(M[2])
        res.setdefault(cls, {
            "kernel": name, "report": rep.split("/")[-1], "duration_us": t * 1e6, "dram_bytes": b,
            "dram_read": f(M[1]), "dram_write": f(M[2]), "dram_bytes_per_particle": b / npart,
            "dram_gbs": b / t / 1e9 if t else 0.0, "warp_inst_per_particle": f(M[3]) / npart,
            "occupancy_pct": f(M[4]), "issue_active_pct": f(M[5]), "registers": int(f(M[6])),
            "sm_throughput_pct": f(M[7]), "mem_throughput_pct": f(M[8])})
json.dump({"particles_per_launch": npart, "kernels": res}, open(out, "w"), indent=1)
for k, v in res.items():
    print(f"{k:10s} {v['duration_us']:8.1f} us  {v['dram_bytes_per_particle']:6.1f} B/p  {v['dram_gbs']:6.0f} GB/s  "
          f"{v['warp_inst_per_particle']:6.2f} winst/p  occ {v['occupancy_pct']:5.1f}  issue {v['issue_active_pct']:5.1f}  regs {v['registers']}")
