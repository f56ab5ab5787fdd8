"""Calibration closed loop at scale (reference fit.py:94-243,
acceptance pattern test_acceptance.py:214-281) — test infrastructure shared
by tools/make_golden_calib.py (runs the unmodified reference's
derive_observations + calibrate_all on a device sweep) and
tests/test_calibration_scale.py (runs this package's on the same sweep).

The sweep is C3 (93,184 configurations, workloads.space_c3) on B200
parameters, evaluated on the device and written as the reference's ranking
CSV.  Measurements are synthesised from every row with known per-role
ratio curves (a Gompertz a*exp(-b*exp(-c*x)) per role), so the fit must
recover them: the closed loop the reference's acceptance test runs on a few
rows, here on ~10^5."""

from __future__ import annotations

import csv
import io
import math

# ground-truth (a, b, c) per role of the synthetic measurements
TRUE = {"l1": (0.85, 3.0, 2.5), "l2_load": (0.7, 6.0, 1.5), "l2_store": (0.6, 2.0, 4.0)}


def gompertz(p, x: float) -> float:
    a, b, c = p
    inner = -c * x
    if inner > 700.0:
        return 0.0
    return min(1.0, max(0.0, a * math.exp(-b * math.exp(inner))))


def space_c3():
    from paper_2107_01143_b200 import workloads as W
    from paper_2107_01143_b200.gvo.machine import b200_preset

    return W.space("C3", b200_preset())


def prefixes(sp) -> list[str]:
    """configKey,blockX,blockY,blockZ,folding of every configuration."""
    fold = [t.folding for t in sp.templates]
    return [f"{sp.key(i)},{int(sp.block[i][0])},{int(sp.block[i][1])},{int(sp.block[i][2])},{fold[int(sp.tpl[i])]}"
            for i in range(len(sp))]


def measurement_csv(sweep_csv: str) -> str:
    """Three measured per-LUP volumes per sweep row (fit.py MEASUREMENT_HEADER):
    L2->L1 loads on the l1 curve, DRAM loads on the l2_load curve (the overmiss
    share as estimated), DRAM stores on the l2_store curve."""
    out = io.StringIO()
    out.write("configKey,level,kind,measuredBytesPerLup\n")
    for row in csv.DictReader(io.StringIO(sweep_csv)):
        f = {k: (float(v) if v not in ("", None) else None) for k, v in row.items()
             if k not in ("configKey", "folding", "limiter")}
        key = row["configKey"]
        m1 = f["l2l1LoadComp"] + gompertz(TRUE["l1"], f["l2l1LoadOversub"]) * f["l2l1LoadRed"]
        base = f["dramLoadUnique"] - f["dramLoadOverlap"]
        m2 = base + f["dramLoadOvermiss"] + gompertz(TRUE["l2_load"], f["dramLoadOversub"]) * f["dramLoadRedL2"]
        m3 = f["dramStoreUnique"] + gompertz(TRUE["l2_store"], f["dramLoadOversub"]) * (
            f["dramStoreUp"] - f["dramStoreUnique"])
        out.write(f"{key},L2toL1,load,{m1!r}\n{key},DRAMtoL2,load,{m2!r}\n{key},DRAMtoL2,store,{m3!r}\n")
    return out.getvalue()
