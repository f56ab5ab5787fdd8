"""C5's two halves (stencil C3-like part, LBM C4-like part) evaluated
separately: device ms per pipeline stage and sharing figures (GPU).
usage: python tools/c5_probe.py"""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2107_01143_b200 import _native, workloads as W  # noqa: E402
from paper_2107_01143_b200.gvo.machine import b200_preset  # noqa: E402

m = b200_preset()
ms = W.l2_variants(m)
parts = {
    "C5-stencil": W.space_c3(m, radii=(1, 2, 3, 4), alignments=tuple(range(0, 256, 8)), machines=ms, machines_idx=(0, 1, 2)),
    "C5-lbm": W.space_c4(m, alignments=tuple(range(0, 128, 8)), machines=ms, machines_idx=(0, 1, 2)),
}
ctx = _native.context()
L = _native.lib()
C = _native.C
L.gvo_set_timing(ctx.h, 1)
for name, sp in parts.items():
    cfgs = sp.config_array(ctx)
    ctx.sync_registries()
    for rep in range(2):
        L.gvo_dedup_stats(ctx.h, 1, None, None)
        L.gvo_kernel_times(ctx.h, None, None, 1)
        t0 = time.perf_counter()
        out = ctx.eval_configs_host(cfgs, 5, 2, 0)
        dt = time.perf_counter() - t0
        kms = (C.c_double * 8)()
        kcnt = (C.c_int64 * 8)()
        L.gvo_kernel_times(ctx.h, kms, kcnt, 1)
        u, f = C.c_int64(), C.c_int64()
        L.gvo_dedup_stats(ctx.h, 0, C.byref(u), C.byref(f))
        print(f"{name} n={len(sp)} wall={dt:.3f}s kernels(ms) setup={kms[0]:.1f} warp={kms[1]:.1f} sets={kms[2]:.1f}"
              f" finish={kms[3]:.1f} launches={list(kcnt)[:4]} shareable={u.value} copied={f.value}", flush=True)
