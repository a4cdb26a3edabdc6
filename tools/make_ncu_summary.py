"""profiles/ncu_summary_cfg<N>.json (and the per-round copy) from the details/raw CSV
exports of tools/r2_prof2.sh: per kernel duration, DRAM bytes (total and per
particle), warp instructions per particle, occupancy, issue, registers.

usage: python tools/make_ncu_summary.py TAG PARTICLES OUT.json [SOURCE_NOTE]"""
import csv
import glob
import json
import os
import sys

tag, npart, out = sys.argv[1], float(sys.argv[2]), sys.argv[3]
note = sys.argv[4] if len(sys.argv) > 4 else tag
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
names = {"k_p2g": "p2g", "k_g2p": "g2p", "k_g2p_adj": "g2p_adj", "k_p2g_adj": "p2g_adj", "k_bin": "bin",
         "k_cellsort": "cellsort", "k_grid": "grid", "k_grid_adj": "grid_adj"}
res = {}
for f in sorted(glob.glob("gpurun_out/%s_k_*_details.csv" % tag)):
    k = os.path.basename(f)[len(tag) + 1:-len("_details.csv")]
    rows = list(csv.reader(open(f)))
    h = rows[0]
    d = {}
    for r in rows[1:]:
        d[(r[h.index("Section Name")], r[h.index("Metric Name")])] = (r[h.index("Metric Value")], r[h.index("Metric Unit")])
    def dv(sec, name):
        v = d.get((sec, name))
        return float(v[0].replace(",", "")) if v and v[0] else None
    raw = list(csv.reader(open(f.replace("_details", "_raw"))))
    rh, ru, rv = raw[0], raw[1], raw[2]
    def rm(name):
        i = rh.index(name)
        return float(rv[i].replace(",", "")) * SCALE.get(ru[i], 1)
    rd, wr = rm("dram__bytes_read.sum"), rm("dram__bytes_write.sum")
    dur = dv("GPU Speed Of Light Throughput", "Duration")
    dunit = d[("GPU Speed Of Light Throughput", "Duration")][1]
    dur_us = dur * {"us": 1, "ms": 1e3, "ns": 1e-3}[dunit]
    inst = dv("Instruction Statistics", "Executed Instructions")
    res[names.get(k, k)] = {
        "kernel": rows[1][h.index("Kernel Name")].split("(")[0].replace("void ", ""),
        "duration_us": dur_us, "dram_bytes": rd + wr, "dram_read": rd, "dram_write": wr,
        "dram_bytes_per_particle": (rd + wr) / npart, "dram_gbs": (rd + wr) / (dur_us * 1e3),
        "warp_inst_per_particle": inst / npart,
        "occupancy_pct": dv("Occupancy", "Achieved Occupancy"),
        "issue_active_pct": dv("Compute Workload Analysis", "Issue Slots Busy"),
        "registers": dv("Launch Statistics", "Registers Per Thread"),
        "sm_throughput_pct": dv("GPU Speed Of Light Throughput", "Compute (SM) Throughput"),
        "mem_throughput_pct": dv("GPU Speed Of Light Throughput", "Memory Throughput"),
    }
json.dump({"source": note, "particles_per_launch": npart, "kernels": res}, open(out, "w"), indent=1)
for k, v in res.items():
    print("%-9s %-24s %8.1f us  %6.1f B/p  %5.0f GB/s  %5.1f inst/p  occ %5.1f  issue %5.1f  regs %3d" % (
        k, v["kernel"][:24], v["duration_us"], v["dram_bytes_per_particle"], v["dram_gbs"],
        v["warp_inst_per_particle"], v["occupancy_pct"], v["issue_active_pct"], v["registers"]))
