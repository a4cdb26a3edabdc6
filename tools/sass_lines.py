"""Per-source-line totals of an ncu SASS source-page CSV (tools/r2_prof*.sh,
--print-source sass): stall samples and executed warp instructions mapped to
CUDA lines through nvdisasm -gi line info of the same build's cubin.

usage: python tools/sass_lines.py gpurun_out/q4_k_grid_sass.csv.gz MANGLED_SUBSTR [top]
(needs the profiled build's libdiffmpm.so in place)."""
import collections
import csv
import gzip
import os
import re
import subprocess
import sys
import tempfile

src, fsub = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
depth = int(sys.argv[4]) if len(sys.argv) > 4 else 0  # > 0: also aggregate at this inline depth (1 = kernel level)
so = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2412_12089_b200", "libdiffmpm.so")
tmp = tempfile.mkdtemp()
subprocess.check_call(["cuobjdump", "-xelf", "all", so], cwd=tmp, stdout=subprocess.DEVNULL)
cub = [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-c", "-gi", cub], capture_output=True, text=True).stdout.splitlines()
loc_re = re.compile(r'//## File ".*?([^/]+)", line (\d+)(?: inlined at ".*?([^/]+)", line (\d+))?')
ins_re = re.compile(r"/\*([0-9a-f]{4,})\*/\s+(.*?);")
inner, outer, text, chain = {}, {}, {}, {}
infn, cur = False, []
for ln in dis:
    if ln.startswith("//----") and ".text." in ln:
        infn = fsub in ln
        continue
    if not infn:
        continue
    m = loc_re.search(ln)
    if m:
        if not ln.lstrip().startswith("//## File") or "inlined at" in ln or not cur or True:
            cur.append((m.group(1), int(m.group(2))))
        continue
    m = ins_re.search(ln)
    if m:
        off = int(m.group(1), 16)
        if cur:
            inner[off] = cur[0]
            outer[off] = cur[-1]
            chain[off] = cur[::-1]  # outermost first
        text[off] = m.group(2).strip()
        cur = []
rows = list(csv.reader(gzip.open(src, "rt")))
h = rows[1]
ia, isamp, iex = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
base = int(rows[2][ia], 16)
agg_i, agg_o = collections.Counter(), collections.Counter()
ex_i = collections.Counter()
tot_s = tot_e = 0
last_i = last_o = ("?", 0)
for r in rows[2:]:
    off = int(r[ia], 16) - base
    s, e = float(r[isamp] or 0), float(r[iex] or 0)
    li, lo = inner.get(off, last_i), outer.get(off, last_o)
    last_i, last_o = li, lo
    agg_i[li] += s
    agg_o[lo] += s
    ex_i[li] += e
    tot_s += s
    tot_e += e
print("total samples %d, warp instructions %.3g" % (tot_s, tot_e))
print("-- innermost line: samples%, inst%")
for k, v in agg_i.most_common(top):
    print("%-22s %6.2f%% %6.2f%%" % ("%s:%d" % k, 100 * v / tot_s, 100 * ex_i[k] / max(tot_e, 1)))
if depth:
    agg_d, ex_d = collections.Counter(), collections.Counter()
    last = ("?", 0)
    for r in rows[2:]:
        off = int(r[ia], 16) - base
        ch = chain.get(off)
        k = ch[min(depth, len(ch)) - 1] if ch else last
        last = k
        agg_d[k] += float(r[isamp] or 0)
        ex_d[k] += float(r[iex] or 0)
    print("-- inline depth %d: samples%%, inst%%" % depth)
    for k, v in sorted(agg_d.items(), key=lambda x: -ex_d[x[0]])[:top]:
        print("%-22s %6.2f%% %6.2f%%" % ("%s:%d" % k, 100 * v / tot_s, 100 * ex_d[k] / max(tot_e, 1)))
print("-- kernel-level line: samples%")
for k, v in agg_o.most_common(20):
    print("%-22s %6.2f%%" % ("%s:%d" % k, 100 * v / tot_s))
