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
busy = ph[:, 1:8].sum(1) / 1e3
print("per-CTA fetch-wait kcycles p50/max", np.percentile(ph[:, 0] / 1e3, [50, 100]).round(0),
      "busy kcycles p10/p50/p90/max", np.percentile(busy, [10, 50, 90, 100]).round(0))
