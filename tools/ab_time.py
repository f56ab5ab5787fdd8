"""A/B timing of library builds (run on the GPU box):

  python tools/ab_time.py [variant ...]      ('' = the product library)

For each build (GVO_LIB_VARIANT=<name> -> libgvo_b200_<name>.so, built by
`GVO_BUILD_VARIANT=<name> GVO_BUILD_DEFS=... python -m paper_2107_01143_b200.build`)
a fresh process evaluates C2, C4 and a seeded 49,152-configuration sample of
C5 (3 batches) and reports device ms per workload (CUDA events around each
kernel, best of 3 after a warm-up) plus a result checksum (every variant must
agree)."""

from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def child():
    sys.path.insert(0, str(ROOT))
    import numpy as np
    import torch

    from paper_2107_01143_b200 import _native, workloads as W

    ctx = _native.context()
    L = _native.lib()
    C = _native.C
    out = {"variant": os.environ.get("GVO_LIB_VARIANT", ""), "build_id": _native.build_id(),
           "env": {k: v for k, v in os.environ.items() if k.startswith("GVO_") and k != "GVO_AB_CHILD"}}
    sp5 = W.space("C5")
    pick = np.sort(np.random.default_rng(7).choice(len(sp5), size=49152, replace=False))
    spaces = {"C2": W.space("C2"), "C4": W.space("C4"), "C5s": sp5.subset(pick)}
    for name, sp in spaces.items():
        cfg = sp.config_array(ctx)
        ctx.sync_registries()
        F = ctx.max_fields
        S, Wn = _native.effective_sampling(5, 2)
        stride = _native.counts_stride(F, S, Wn)
        n = len(cfg)
        dev = torch.device("cuda", 0)
        d_cfg = torch.from_numpy(cfg.view(np.uint8).copy()).to(dev)
        d_cnt = torch.zeros((n, stride), dtype=torch.int64, device=dev)
        d_rec = torch.zeros((n, _native.RECORD_LEN), dtype=torch.float64, device=dev)
        smp = _native.Sampling(5, 2, 0, 7, 0)
        st = torch.cuda.current_stream().cuda_stream
        best = None
        for rep in range(4):
            L.gvo_set_timing(ctx.h, 1)
            L.gvo_kernel_times(ctx.h, None, None, 1)
            ctx.check(L.gvo_eval_configs(ctx.h, C.c_void_p(d_cfg.data_ptr()), n, C.byref(smp), F,
                                         C.c_void_p(d_cnt.data_ptr()), None, C.c_void_p(d_rec.data_ptr()),
                                         None, None, 0, C.c_void_p(st)))
            torch.cuda.synchronize()
            kms = (C.c_double * 8)()
            L.gvo_kernel_times(ctx.h, kms, None, 1)
            L.gvo_set_timing(ctx.h, 0)
            if rep and (best is None or kms[2] < best[2]):
                best = [kms[i] for i in range(5)]
        status = d_cnt[:, 0].cpu().numpy()
        chk = float(d_rec[:, -1].double().sum().item())
        out[name] = {"n": n, "setup_ms": best[0], "sets_ms": best[2], "finish_ms": best[3],
                     "cfg_per_s": n / (sum(best) * 1e-3), "bad_status": int((status != 0).sum()), "glups_sum": chk}
    print("AB " + json.dumps(out), flush=True)


def main():
    if os.environ.get("GVO_AB_CHILD"):
        child()
        return
    variants = sys.argv[1:] or [""]
    for v in variants:
        # "name@KEY=VAL,KEY2=VAL2": a build plus runtime environment knobs
        name, _, kv = v.partition("@")
        env = dict(os.environ, GVO_AB_CHILD="1", GVO_LIB_VARIANT=name)
        env.update(dict(x.split("=", 1) for x in kv.split(",") if x))
        r = subprocess.run([sys.executable, __file__], env=env, capture_output=True, text=True, timeout=1800)
        line = [ln for ln in r.stdout.splitlines() if ln.startswith("AB ")]
        print(line[0][3:] if line else json.dumps({"variant": v, "error": r.stderr[-2000:]}), flush=True)


if __name__ == "__main__":
    main()
