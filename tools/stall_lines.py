"""Warp-stall samples of an ncu --set full capture of k_sets, attributed to
source lines and stall reasons (the SASS source page joined with the line
table of the same build's cubin).  Run here, on the .ncu-rep brought back
from the box:
  python tools/stall_lines.py gpurun_out/ncu_k_sets_c5.ncu-rep paper_2107_01143_b200/build/obj/k_sets.o"""
import collections
import csv
import io
import re
import subprocess
import sys
import tempfile
from pathlib import Path

rep, obj = sys.argv[1], sys.argv[2]
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                      capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(sass)))
hdr = rows[1]
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_e = hdr.index("Instructions Executed")
stall = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
with tempfile.TemporaryDirectory() as td:
    subprocess.run(["cuobjdump", "-xelf", "all", str(Path(obj).resolve())], cwd=td, capture_output=True, check=True)
    cub = sorted(Path(td).glob("*.cubin"))[0]
    dis = subprocess.run(["nvdisasm", "-g", "-gi", "-c", str(cub)], capture_output=True, text=True).stdout
m_off = re.compile(r"/\*([0-9a-f]{4,})\*/")
loc = {}
grp, last = [], False
for ln in dis.splitlines():
    if "//##" in ln:
        if not last:
            grp = []
        grp.append(ln)
        last = True
        continue
    m = m_off.search(ln)
    if m:
        last = False
        if grp:
            locs = re.findall(r'(\w+\.cuh?)", line (\d+)', grp[0])
            outer = re.findall(r'(\w+\.cuh?)", line (\d+)', grp[-1])
            loc[int(m.group(1), 16)] = (locs[0] if locs else None, outer[-1] if outer else None)
base = int(rows[2][0], 16)
by_line, by_reason = collections.Counter(), collections.Counter()
reasons = collections.defaultdict(collections.Counter)
total = 0
for r in rows[2:]:
    try:
        s = int(r[i_s])
    except (ValueError, IndexError):
        continue
    inner, _ = loc.get(int(r[0], 16) - base, (None, None))
    key = f"{inner[0]}:{inner[1]}" if inner else "?"
    by_line[key] += s
    total += s
    for i in stall:
        try:
            v = int(r[i])
        except ValueError:
            continue
        by_reason[hdr[i]] += v
        reasons[key][hdr[i]] += v
tr = sum(by_reason.values())
print(f"{rep}: {total} warp-stall samples, {len(rows) - 2} SASS instructions")
print("stall reasons (share of samples):")
for k, v in by_reason.most_common(10):
    print(f"  {k:28s} {100 * v / tr:5.1f} %")
print("top source lines (innermost inlined location):")
for k, v in by_line.most_common(30):
    top = ", ".join(f"{a[6:]} {100 * b / max(1, v):.0f}%" for a, b in reasons[k].most_common(2))
    print(f"  {100 * v / total:5.1f} %  {k:22s} {top}")
