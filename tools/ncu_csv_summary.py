"""Summarise ncu --page details/raw CSV exports (tools/r2_prof.sh) into one
table: duration, DRAM bytes and throughput, occupancy, issue, top stalls."""
import csv
import glob
import json
import os
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "p1"
out = {}
for f in sorted(glob.glob("gpurun_out/%s_k_*_details.csv" % tag)):
    k = os.path.basename(f)[len(tag) + 1:-len("_details.csv")]
    rows = list(csv.reader(open(f)))
    if not rows:
        continue
    h = rows[0]
    try:
        iname, iv, iu = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    except ValueError:
        continue
    d = {}
    for r in rows[1:]:
        if len(r) > iv:
            d[r[iname]] = (r[iv], r[iu])
    raw = list(csv.reader(open(f.replace("_details", "_raw"))))
    rh, rv = raw[0], raw[2] if len(raw) > 2 else raw[-1]
    def rm(name):
        return float(rv[rh.index(name)].replace(",", "")) if name in rh else None
    st = {m: rm(m) for m in rh if m.startswith("smsp__pcsamp_warps_issue_stalled") and not m.endswith("not_issued")}
    tot = sum(v for v in st.values() if v) or 1
    top = sorted(((k2.replace("smsp__pcsamp_warps_issue_stalled_", ""), v / tot) for k2, v in st.items() if v),
                 key=lambda x: -x[1])[:4]
    out[k] = {"kernel": rv[rh.index("Kernel Name")] if "Kernel Name" in rh else k,
              "duration_us": d.get("Duration", ("", ""))[0], "dram_bytes": (rm("dram__bytes_read.sum") or 0) + (rm("dram__bytes_write.sum") or 0),
              "dram_gbs": d.get("DRAM Throughput", ("", ""))[0], "regs": d.get("Registers Per Thread", ("", ""))[0],
              "occupancy": d.get("Achieved Occupancy", ("", ""))[0], "ipc": d.get("Executed Ipc Active", ("", ""))[0],
              "inst": d.get("Executed Instructions", ("", ""))[0], "top_stalls": [(n, round(v, 3)) for n, v in top]}
print(json.dumps(out, indent=1))
