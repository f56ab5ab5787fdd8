"""Evaluate a key-filtered subset of a workload space (for ncu captures).
usage: python tools/run_subset.py C4 D3Q27/zyxf/a0/none [reps]"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2107_01143_b200 import _native, workloads as W  # noqa: E402

sp = W.space(sys.argv[1])
if len(sys.argv) > 2:
    sp = sp.subset(np.array([i for i in range(len(sp)) if sys.argv[2] in sp.key(i)]))
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
ctx = _native.context()
cfgs = sp.config_array(ctx)
ctx.sync_registries()
for _ in range(reps):
    out = ctx.eval_configs_host(cfgs, 5, 2, 0)
print("n", len(sp), "status", np.unique(out["counts"][:, _native.C_STATUS], return_counts=True))
