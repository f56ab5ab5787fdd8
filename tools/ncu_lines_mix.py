"""Aggregate an ncu source page (--print-source cuda,sass --csv) per CUDA
source line: stall samples, executed instructions and local-memory
instructions.  usage: python tools/ncu_lines_mix.py report.ncu-rep [top]"""
import csv, subprocess, sys, collections, io

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["/usr/local/cuda/bin/ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname = None; hdr = None; cur = None
agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0, ""])
for r in csv.reader(io.StringIO(txt)):
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if r[0] == "Function Name" or hdr is None: continue
    if r[0]:
        cur = (fname, int(r[0])); agg[cur][3] = r[1][:90]; continue
    if cur is None: continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        agg[cur][0] += float(d.get("Warp Stall Sampling (All Samples)", 0) or 0)
        agg[cur][1] += float(d.get("Instructions Executed", 0) or 0)
    except ValueError:
        continue
    s = d.get("Source", "")
    if "LDL" in s or "STL" in s: agg[cur][2] += float(d.get("Instructions Executed", 0) or 0)
tot = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
tl = sum(v[2] for v in agg.values())
print(f"samples {tot:.0f} inst {ti:.3g} local inst {tl:.3g}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*v[0]/tot:6.2f}% stall {100*v[1]/ti:6.2f}% inst local {v[2]:10.0f}  {k[0]}:{k[1]}  {v[3]}")
