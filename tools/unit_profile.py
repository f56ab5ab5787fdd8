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
if len(sys.argv) > 2:  # key filter, e.g. "D3Q27/zyxf"
    sp = sp.subset(np.array([i for i in range(len(sp)) if sys.argv[2] in sp.key(i)]))
cfgs = sp.config_array(ctx)
kept = [type("K", (), {"key": sp.key(i)})() for i in range(len(sp))]
L.gvo_debug_units(ctx.h, 1, None, 0, None)
for _ in range(2):
    out = ctx.eval_configs_host(cfgs, 5, 2, 0)
n_items = _native.C.c_int64()
L.gvo_debug_units(ctx.h, 1, None, 0, _native.C.byref(n_items))
raw = np.zeros(n_items.value * 10 + 10 + 4096 * 10 + 1024 * 16, dtype=np.int64)
L.gvo_debug_units(ctx.h, 0, _native._ptr(raw), raw.size, None)
st = raw[: n_items.value * 10].reshape(-1, 10)
nrng = int(raw[n_items.value * 10])
rng_rows = raw[n_items.value * 10 + 10: n_items.value * 10 + 10 + min(nrng, 4096) * 10].reshape(-1, 10)
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
    su = [r for r in rng_rows.tolist() if r[8] == 4]
    if su:
        su.sort(key=lambda r: -r[3])
        print("split units", len(su), "sum N", sum(r[3] for r in su))
        for r in su[:25]:
            print("  split", kept[r[7]].key, "field", r[0], "kind", r[1], "N", r[3], "nr", r[5], "span", r[6])
    rr = sorted([r for r in rng_rows.tolist() if r[8] not in (3, 4)], key=lambda r: -r[4])
    print("range cycles total M", sum(r[4] for r in rr) / 1e6, "max", rr[0][4])
    for r in rr[:15]: print("desc", r[0], "a", r[1], "b", r[2], "N", r[3], "cyc", r[4], "nr", r[5], "sm", r[6], "cfg", kept[r[7]].key, "queued" if r[8] == 1 else "first")
# per-CTA phase accounting (k_sets debug counters)
base = n_items.value * 10 + 10 + 4096 * 10
ph = raw[base: base + 1024 * 16].reshape(1024, 16)
ph = ph[ph.sum(1) != 0]
names = ["fetch-wait", "warp-items", "micro", "unit-runs", "unit-sort/sweep", "range-count", "range-bitmap",
         "range-emit/sort/sweep"]
tot = ph[:, :8].sum(0) / 1e6
print("CTAs", len(ph), "phase Gcycles (sum over CTAs):", {n: round(v / 1e3, 3) for n, v in zip(names, tot)})
print("ranges", int(ph[:, 8].sum()), "bitmap", int(ph[:, 9].sum()), "sum N", int(ph[:, 10].sum()), "sum nr", int(ph[:, 11].sum()), "seg ok", int(ph[:, 12].sum()), "seg no", int(ph[:, 13].sum()), "runs: pre-lattice Gcyc", round(ph[:, 14].sum() / 1e9, 3), "lattice Gcyc", round(ph[:, 15].sum() / 1e9, 3))
fw = ph[:, 0] / 1e3
busy = ph[:, 1:8].sum(1) / 1e3
print("per-CTA fetch-wait kcycles p10/p50/p90/max", np.percentile(fw, [10, 50, 90, 100]).round(0),
      "busy kcycles p10/p50/p90/max", np.percentile(busy, [10, 50, 90, 100]).round(0))
