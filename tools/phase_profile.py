"""Per-CTA phase accounting of the set kernel over one batch of a C5 part
(GPU; needs the prof build: GVO_BUILD_VARIANT=prof python -m
paper_2107_01143_b200.build, then GVO_LIB_VARIANT=prof).
usage: python tools/phase_profile.py [stencil|lbm] [first_config] [n]"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2107_01143_b200 import _native, workloads as W  # noqa: E402
from paper_2107_01143_b200.gvo.machine import b200_preset  # noqa: E402

part = sys.argv[1] if len(sys.argv) > 1 else "lbm"
c0 = int(sys.argv[2]) if len(sys.argv) > 2 else 0
n = int(sys.argv[3]) if len(sys.argv) > 3 else 16384
m = b200_preset()
ms = W.l2_variants(m)
if part == "stencil":
    sp = W.space_c3(m, radii=(1, 2, 3, 4), alignments=tuple(range(0, 256, 8)), machines=ms, machines_idx=(0, 1, 2))
else:
    sp = W.space_c4(m, alignments=tuple(range(0, 128, 8)), machines=ms, machines_idx=(0, 1, 2))
sp = sp.subset(np.arange(c0, min(len(sp), c0 + n)))
ctx = _native.context()
L = _native.lib()
cfgs = sp.config_array(ctx)
L.gvo_debug_units(ctx.h, 1, None, 0, None)
for _ in range(2):
    out = ctx.eval_configs_host(cfgs, 5, 2, 0)
n_items = _native.C.c_int64()
L.gvo_debug_units(ctx.h, 1, None, 0, _native.C.byref(n_items))
raw = np.zeros(n_items.value * 10 + 10 + 4096 * 10 + 1024 * 16, dtype=np.int64)
L.gvo_debug_units(ctx.h, 0, _native._ptr(raw), raw.size, None)
base = n_items.value * 10 + 10 + 4096 * 10
ph = raw[base: base + 1024 * 16].reshape(1024, 16)
ph = ph[ph.sum(1) != 0]
names = ["fetch-wait", "warp-items", "micro", "unit-runs", "unit-sort/sweep", "range-count", "range-bitmap",
         "range-emit/sort/sweep"]
tot = ph[:, :8].sum(0) / 1e9
print(f"{part} configs {c0}..{c0 + len(sp)}: CTAs {len(ph)}; phase Gcycles (sum over CTAs):",
      {k: round(float(v), 3) for k, v in zip(names, tot)})
print("ranges", int(ph[:, 8].sum()), "bitmap", int(ph[:, 9].sum()), "sum N", int(ph[:, 10].sum()), "sum nr",
      int(ph[:, 11].sum()), "seg ok", int(ph[:, 12].sum()), "seg no", int(ph[:, 13].sum()))
print("slots 12..15 Gcycles (bmprof build: bitmap zero/elements/big runs/measures)",
      np.round(ph[:, 12:16].sum(0) / 1e9, 3).tolist())
busy = ph[:, 1:8].sum(1) / 1e3
print("per-CTA fetch-wait kcycles p50/max", np.percentile(ph[:, 0] / 1e3, [50, 100]).round(0),
      "busy kcycles p10/p50/p90/max", np.percentile(busy, [10, 50, 90, 100]).round(0))
# per-unit statistics of the batch: cycles by (template kind/layout/folding, unit kind)
st = raw[: n_items.value * 10].reshape(-1, 10)
F, S = out["F"], out["S"]
n_cfg = n_items.value // (F * (S + 1))
from collections import defaultdict  # noqa: E402
agg = defaultdict(lambda: [0, 0, 0])
agg_ph = {}
nr_blk, n_blk = [], []
for i in np.flatnonzero(st[:, 3] > 0).tolist():
    if i < n_cfg * F:
        f, c = divmod(i, n_cfg)  # wave units field-major
        kind = "wave"
    else:
        r = i - n_cfg * F
        c = r // (F * S); f = (r // S) % F
        kind = "blk"
    t = sp.templates[int(sp.tpl[c])]
    lab = t.label.split("/a")[0] + "/" + t.folding
    a = agg[(lab, kind, f)]
    a[0] += int(st[i, 3]); a[1] += 1; a[2] += int(st[i, 1])
    if kind == "blk":
        nr_blk.append(int(st[i, 0])); n_blk.append(int(st[i, 1]))
    ph4 = agg_ph.setdefault(kind, np.zeros(5))
    ph4[:4] += st[i, 6:10]
    ph4[4] += st[i, 2]  # in shared memory (not split)
tot = sum(v[0] for v in agg.values())
print("unit cycles total G", round(tot / 1e9, 3))
if n_blk:
    nb_ = np.array(n_blk); nr_ = np.array(nr_blk)
    print("CTA-path block units", len(nb_), "N p10/p50/p90", np.percentile(nb_, [10, 50, 90]).tolist(),
          "runs p10/p50/p90", np.percentile(nr_, [10, 50, 90]).tolist(), "N>512", int((nb_ > 512).sum()),
          "runs>64", int((nr_ > 64).sum()))
nrng_ = int(raw[n_items.value * 10])
rr = raw[n_items.value * 10 + 10: n_items.value * 10 + 10 + min(nrng_, 4096) * 10].reshape(-1, 10)
bund = rr[rr[:, 8] == 3]
print("bundles (sampled)", len(bund), "fallbacks in them", int(bund[:, 2].sum()) if len(bund) else 0)
for k, v in agg_ph.items():
    print(f"  {k}: runs/emit/sort/sweep Gcyc {np.round(v[:4] / 1e9, 3).tolist()} units in smem {int(v[4])}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:20]:
    print(f"  {k[0]:28s} {k[1]:4s} f{k[2]} units {v[1]:6d} Gcyc {v[0]/1e9:7.3f} ({100*v[0]/tot:4.1f}%) mean kcyc {v[0]/v[1]/1e3:7.1f} mean N {v[2]/v[1]:8.0f}")
