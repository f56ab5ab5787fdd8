"""Evaluate a workload space on the device; per-template status and time.
usage: python tools/wl_probe.py C4 [--per-template]"""
import sys
import time
from collections import Counter
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2107_01143_b200 import _native, workloads as W  # noqa: E402

name = sys.argv[1]
sp = W.space(name)
ctx = _native.context()
L = _native.lib()
cfgs = sp.config_array(ctx)
ctx.sync_registries()
C = _native.C
L.gvo_set_timing(ctx.h, 1)
for rep in range(2):
    L.gvo_kernel_times(ctx.h, None, None, 1)
    t0 = time.perf_counter()
    out = ctx.eval_configs_host(cfgs, 5, 2, 0)
    dt = time.perf_counter() - t0
    kms = (C.c_double * 8)()
    kcnt = (C.c_int64 * 8)()
    L.gvo_kernel_times(ctx.h, kms, kcnt, 1)
    st = out["counts"][:, _native.C_STATUS]
    print(f"{name} n={len(sp)} wall={dt:.3f}s cfg/s={len(sp)/dt:.0f} kernels(ms)={[round(kms[i],2) for i in range(5)]}"
          f" status={dict(Counter(st.tolist()))}", flush=True)
bad = Counter(sp.templates[int(t)].label for t in sp.tpl[st != 0])
print("failing templates", bad.most_common(10))
if "--per-template" in sys.argv:
    for t in range(len(sp.templates)):
        sub = sp.subset(np.flatnonzero(sp.tpl == t))
        c2 = sub.config_array(ctx)
        L.gvo_kernel_times(ctx.h, None, None, 1)
        t0 = time.perf_counter()
        o = ctx.eval_configs_host(c2, 5, 2, 0)
        dt = time.perf_counter() - t0
        L.gvo_kernel_times(ctx.h, kms, kcnt, 1)
        print(f"{sp.templates[t].label:40s} n={len(sub):4d} {dt*1e3:8.1f} ms  sets={kms[2]:8.1f} setup={kms[0]:6.1f}"
              f" bad={(o['counts'][:, _native.C_STATUS] != 0).sum()}", flush=True)
