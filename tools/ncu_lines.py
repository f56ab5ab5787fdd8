"""Aggregate ncu source-page warp-stall samples per CUDA source line.
usage: ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > s.csv; python tools/ncu_lines.py s.csv [N]"""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
agg = defaultdict(float); inst = defaultdict(float); text = {}
cur_file = None; hdr = None
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur_file = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or r[0] in ("Function Name",): continue
    try:
        line = int(r[0]); s = float(r[4]); ie = float(r[7])
    except (ValueError, IndexError):
        continue
    key = (cur_file, line)
    agg[key] += s; inst[key] += ie; text[key] = r[1][:100]
tot = sum(agg.values()) or 1
print("total stall samples", tot)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print("%5.1f%% inst=%10.0f %s:%d  %s" % (100 * v / tot, inst[k], k[0], k[1], text[k]))
