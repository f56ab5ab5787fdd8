"""Golden bytes for the serialization / API / bindings layer (SURVEY.md §8f
N2-N4), produced by the UNMODIFIED reference (its gvo package and its
gvo_bindings, in process — byte-identical to its CLI per the reference's
own bindings/tests/test_parity.py).

Run in the build container:  python tools/make_golden_report.py
writes tests/golden/report.json.
"""

from __future__ import annotations

import json
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
REF = next(c for c in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")) if (c / "gvo").exists())
sys.path.insert(0, str(REF))
sys.path.insert(0, "/root/reference/pkg/bindings/src")

import gvo  # noqa: E402  (reference)
import gvo_bindings as gb  # noqa: E402  (reference)
from gvo import api  # noqa: E402
from gvo.report import render_estimate_csv, render_footprint_csv, render_table  # noqa: E402

OUT = ROOT / "tests" / "golden" / "report.json"
LIGHT = {"wave_samples": 1, "block_samples": 2, "blocks_per_wave": 40}
EST = [
    ("builtin:stencil", (16, 2, 32), "none", None),
    ("builtin:stencil", (32, 2, 16), "2z", None),
    ("builtin:stencil", (512, 2, 1), "2y", (512, 1024, 128)),
    ("builtin:stencil", (32, 1, 32), "2z", (512, 512, 128)),
    ("builtin:lbm", (32, 2, 2), "none", (256, 128, 128)),
    ("builtin:lbm", (2, 16, 16), "none", (128, 64, 64)),
]
SWEEPS = [
    ("builtin:stencil", "v100", 64, {"grid": (64, 64, 64), "stencil_range": 1, "wave_samples": 1, "block_samples": 1}),
    ("builtin:stencil", "v100", 1024, dict(folding_variants=True, **LIGHT)),
    ("builtin:lbm", "v100", 256, {"grid": (128, 128, 64), "wave_samples": 1, "block_samples": 2, "skip_invalid": True}),
    ("builtin:stencil", "v100", 256, {"grid": (256, 256, 64), "wave_samples": 1, "block_samples": 2}),
]


def main():
    out = {"estimates": [], "sweeps": [], "calibration": None, "footprints": []}
    for kernel, block, folding, grid in EST:
        kw = dict(folding=folding, grid=grid, **LIGHT)
        rep = gb.estimate(kernel, "v100", block, **kw)
        out["estimates"].append({"args": [kernel, list(block)], "kw": {k: (list(v) if isinstance(v, tuple) else v)
                                                                       for k, v in kw.items()},
                                 "json": gb.estimate_json(kernel, "v100", block, **kw),
                                 "csv": render_estimate_csv(rep), "table": render_table(rep)})
    for kernel, machine, threads, kw in SWEEPS:
        text = gb.sweep_csv(kernel, machine, threads, **kw)
        out["sweeps"].append({"args": [kernel, machine, threads],
                              "kw": {k: (list(v) if isinstance(v, tuple) else v) for k, v in kw.items()},
                              "csv": text})
    # calibration through files, as bindings/tests/test_parity.py:110-131
    sweep_text = out["sweeps"][3]["csv"]
    rows = sweep_text.strip().splitlines()
    idx = {n: i for i, n in enumerate(rows[0].split(","))}
    lines = ["configKey,level,kind,measuredBytesPerLup"]
    for r in rows[1:]:
        c = r.split(",")
        lines.append(f"{c[idx['configKey']]},L2toL1,load,{float(c[idx['l2l1LoadDown']]) * 1.05}")
        lines.append(f"{c[idx['configKey']]},DRAMtoL2,load,{c[idx['dramLoadDown']]}")
        lines.append(f"{c[idx['configKey']]},DRAMtoL2,store,{c[idx['dramStoreDown']]}")
    meas = "\n".join(lines) + "\n"
    with tempfile.TemporaryDirectory() as d:
        (Path(d) / "s.csv").write_text(sweep_text)
        (Path(d) / "m.csv").write_text(meas)
        cal = gb.calibrate(str(Path(d) / "m.csv"), str(Path(d) / "s.csv"))
    out["calibration"] = {"measurements": meas, "sweep": 3, "result": json.loads(json.dumps(cal))}
    for kernel, block, level, gran in (("builtin:stencil", (16, 4, 4), "block", None),
                                       ("builtin:lbm", (32, 2, 2), "wave", None),
                                       ("builtin:stencil", (32, 2, 2), "wave", 128)):
        res = api.run_footprint(kernel, "v100", block, level=level, granularity=gran,
                                grid=(128, 128, 64) if kernel == "builtin:stencil" else (128, 64, 64))
        out["footprints"].append({"args": [kernel, list(block), level, gran], "csv": render_footprint_csv(res)})
    OUT.write_text(json.dumps(out))
    print("written", OUT, OUT.stat().st_size)


if __name__ == "__main__":
    main()
