"""Per-unit cost profile of the interval-union engine on a bench workload (GPU).
usage: python tools/unit_profile.py [C2|C3|C4]"""
import sys, json
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np
import bench
from paper_2107_01143_b200 import _native

ctx = _native.context()
L = _native.lib()
wl = sys.argv[1] if len(sys.argv) > 1 else "C2"
sp, _, _ = bench.build_shard(wl, 0, 1)
cfgs = sp.config_array(ctx)
kept = [type("K", (), {"key": sp.key(i)})() for i in range(len(sp))]
L.gvo_debug_units(ctx.h, 1, None, 0, None)
for _ in range(2):
    out = ctx.eval_configs_host(cfgs, 5, 2, 0)
n_items = _native.C.c_int64()
L.gvo_debug_units(ctx.h, 1, None, 0, _native.C.byref(n_items))
raw = np.zeros(n_items.value * 10 + 10 + 4096 * 10, dtype=np.int64)
L.gvo_debug_units(ctx.h, 0, _native._ptr(raw), raw.size, None)
st = raw[: n_items.value * 10].reshape(-1, 10)
nrng = int(raw[n_items.value * 10])
rng_rows = raw[n_items.value * 10 + 10: n_items.value * 10 + 10 + nrng * 10].reshape(-1, 10)
F = out["F"]; S = out["S"]
per_cfg = F * (S + 1)
rows = []
n_cfg = n_items.value // per_cfg
for i in range(n_items.value):
    if i < n_cfg * F:
        c, f = divmod(i, F); j = S
    else:
        r = i - n_cfg * F; c = r // (F * S); f = (r // S) % F; j = r % S
    if st[i, 3] == 0: continue
    rows.append((int(st[i, 3]), kept[c].key, f, "wave" if j == S else f"blk{j}", int(st[i, 0]), int(st[i, 1]), int(st[i, 2]), int(st[i, 4]), [int(v) for v in st[i, 6:10]]))
rows.sort(reverse=True)
tot = sum(r[0] for r in rows)
print("units", len(rows), "total Mcycles", tot / 1e6, "max", rows[0][0] / 1e6)
for r in rows[:40]: print(r)
cyc = np.array([r[0] for r in rows]); N = np.array([r[5] for r in rows])
print("smem fraction", np.mean([r[6] for r in rows]), "N p50/p90/max", np.percentile(N, [50, 90, 100]))
wave = [r for r in rows if r[3] == "wave"]; blk = [r for r in rows if r[3] != "wave"]
print("wave units cycles", sum(r[0] for r in wave) / 1e6, "block units", sum(r[0] for r in blk) / 1e6)
for name, grp in (("wave", wave), ("block", blk)):
    ph = np.array([r[8] for r in grp], dtype=float)
    print(name, "phase Mcycles runs/emit/sort/sweep", (ph.sum(0) / 1e6).round(2), "mean", ph.mean(0).round(0))
json.dump(rows, open(ROOT / "gpurun_out" / "unit_profile.json", "w"))
print("ranges processed", nrng)
if nrng:
    bund = [r for r in rng_rows.tolist() if r[8] == 3]
    if bund:
        cyc = sorted(r[4] for r in bund)
        print("bundles", len(bund), "total Mcycles", sum(cyc) / 1e6, "p50", cyc[len(cyc)//2], "max", cyc[-1], "fallbacks", sum(r[2] for r in bund))
    rr = sorted([r for r in rng_rows.tolist() if r[8] != 3], key=lambda r: -r[4])
    print("range cycles total M", sum(r[4] for r in rr) / 1e6, "max", rr[0][4])
    for r in rr[:15]: print("desc", r[0], "a", r[1], "b", r[2], "N", r[3], "cyc", r[4], "nr", r[5], "sm", r[6], "cfg", kept[r[7]].key, "queued" if r[8] == 1 else "first")
