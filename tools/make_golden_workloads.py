"""Golden vectors for the BASELINE.json configuration spaces (C1-C5), made by
running the UNMODIFIED reference estimator on descriptors of
paper_2107_01143_b200/workloads.py (handed over as kernel-spec dicts, the
reference's own interchange format, kernels.py:441-512).

Run in the build container (the reference is not on the GPU box):
    python tools/make_golden_workloads.py
writes tests/golden/workloads.json:
  * "records": full-size evaluations (42-column ranking record as float.hex,
    per-field down volumes, L1 per-access) of C1 and seeded-random samples of
    C3, C4 and C5;
  * "rankings": every configuration of C2 (246) and C4 (1,812) with its
    predicted GLup/s (hex) and limiter, and the reference ranking order
    (perf.py:131 key: -glups, block_dim, folding string, then input order).
"""

from __future__ import annotations

import json
import multiprocessing as mp
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
REF = next(c for c in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")) if (c / "gvo").exists())

from paper_2107_01143_b200 import workloads as W  # noqa: E402
from paper_2107_01143_b200.gvo.kernels import kernel_to_dict  # noqa: E402
from paper_2107_01143_b200.gvo.machine import b200_preset, machine_to_dict  # noqa: E402

OUT = ROOT / "tests" / "golden" / "workloads.json"
FOLD = {0: "2y", 1: "2z", 2: "none"}


def hx(v):
    if v is None:
        return None
    if isinstance(v, (bool, np.bool_)):
        return bool(v)
    if isinstance(v, (int, np.integer)):
        return int(v)
    return float(v).hex()


def _ref():
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import gvo

    return gvo


def ref_record(job):
    spec, mdict, full = job
    gvo = _ref()
    from gvo.machine import machine_from_dict
    from gvo.report import ranking_row_dict

    k = gvo.kernel_from_dict(spec)
    m = machine_from_dict(mdict)
    try:
        p = gvo.evaluate_kernel(k, m)
    except Exception as exc:  # noqa: BLE001
        return {"error": [type(exc).__name__, str(exc)]}
    if not full:
        return {"glups": hx(p.glups), "limiter": p.limiter}
    row = ranking_row_dict(gvo.SweepRow(gvo.SweepConfig(k.launch.block_dim), p))
    return {"record": {c: (hx(v) if not isinstance(v, str) else v) for c, v in row.items()},
            "per_access": [hx(v) for v in p.l1_cycles.per_access],
            "per_field_down": {lvl: {f: hx(v) for f, v in getattr(p.volumes, lvl).per_field_down.items()}
                               for lvl in ("l2l1_load", "l2l1_store", "dram_load", "dram_store")}}


def jobs_of(sp, idx, full):
    return [(kernel_to_dict(sp.kernel(int(i))), machine_to_dict(sp.machine(int(i))), full) for i in idx]


def entry(sp, i):
    t = sp.templates[int(sp.tpl[i])]
    return {"template": {"kind": t.kind, "grid": list(t.grid), "folding": t.folding, "layout": t.layout,
                         "components": t.components, "alignment": t.alignment, "radius": t.radius,
                         "stencil": t.stencil},
            "machine": int(sp.mach[i]), "block": [int(v) for v in sp.block[i]]}


def ranking_order(sp, glups):
    """perf.py:131 sort key over the space, stable in input order."""
    keys = []
    for i in range(len(sp)):
        b = tuple(int(v) for v in sp.block[i])
        keys.append((-float.fromhex(glups[i]), b, FOLD[int(sp.fold_rank[i])], i))
    return [k[-1] for k in sorted(keys)]


def main():
    m = b200_preset()
    rng = np.random.default_rng(20240811)
    spaces = {n: W.space(n, m) for n in ("C1", "C2", "C3", "C4", "C5")}
    out = {"machine_base": machine_to_dict(m), "machines": {n: [machine_to_dict(x) for x in s.machines]
                                                            for n, s in spaces.items()},
           "records": {}, "rankings": {}}
    with mp.get_context("spawn").Pool(os.cpu_count()) as pool:
        for name, n in (("C1", 1), ("C3", 48), ("C4", 32), ("C5", 48)):
            sp = spaces[name]
            idx = np.sort(rng.choice(len(sp), size=min(n, len(sp)), replace=False))
            res = pool.map(ref_record, jobs_of(sp, idx, True), chunksize=1)
            out["records"][name] = [dict(entry(sp, i), **r) for i, r in zip(idx, res)]
            print(name, "records", len(res), flush=True)
        for name in ("C2", "C4"):
            sp = spaces[name]
            res = pool.map(ref_record, jobs_of(sp, range(len(sp)), False), chunksize=4)
            glups = [r["glups"] for r in res]
            ents = [entry(sp, i) for i in range(len(sp))]
            tpls, tix = [], {}
            for e in ents:
                tix.setdefault(json.dumps(e["template"], sort_keys=True), len(tix))
                if len(tix) > len(tpls):
                    tpls.append(e["template"])
            cfg = [[tix[json.dumps(e["template"], sort_keys=True)], e["machine"], *e["block"]] for e in ents]
            out["rankings"][name] = {"templates": tpls, "cfg": cfg, "glups": glups,
                                     "limiter": [r["limiter"] for r in res], "order": ranking_order(sp, glups)}
            print(name, "ranking", len(res), flush=True)
    OUT.write_text(json.dumps(out, separators=(",", ":")))
    print("written", OUT, OUT.stat().st_size)


if __name__ == "__main__":
    main()
