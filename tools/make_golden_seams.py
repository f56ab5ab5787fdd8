"""Golden vectors for the public seams beside the batched path, made by the
UNMODIFIED reference (run in the build container; the reference is not on
the GPU box):

    python tools/make_golden_seams.py   ->  tests/golden/seams.json

* "bulk": 1000 random address trees on the generator of the reference's own
  test (test_expr.py:136-168: +, -, constant *, floor // and % by positive
  constants over the six coordinates and BX/BY/BZ), rendered to text, with
  random coordinate arrays and the reference evaluate_bulk output
  (expr.py:281-304).
* "injected": estimate_volumes with injected BlockStats / WaveStats
  (volumes.py:421-445, the seam of test_volumes.py:194-199 and
  test_acceptance.py:293-300): seeded random statistics for stencil / LBM
  kernels at several L2 capacities, and the reference's four
  LevelKindVolumes (float.hex) plus predict() (perf.py:45-67).
* "file_sweeps": rank_sweep over KernelFamily("file", ...) (kernels.py:
  422-433: spec re-tiled per block, folding refused) for three spec files,
  with skip_invalid, the reference's ranked (block, folding, glups hex,
  limiter) rows.
"""

from __future__ import annotations

import dataclasses
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
REF = next(c for c in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")) if (c / "gvo").exists())
sys.path.insert(0, str(REF))

import gvo  # noqa: E402  (reference)
from gvo.expr import COORD_NAMES, BlockDimRef, CoordRef, IntConstant, fold, render  # noqa: E402
from gvo.volumes import BlockStats, WaveStats  # noqa: E402

OUT = ROOT / "tests" / "golden" / "seams.json"
BLOCK = (32, 4, 2)


def _random_tree(rng, depth=0):
    roll = rng.integers(0, 10)
    if depth >= 4 or roll < 3:
        choice = rng.integers(0, 3)
        if choice == 0:
            return IntConstant(int(rng.integers(-1000, 1000)))
        if choice == 1:
            return CoordRef(COORD_NAMES[rng.integers(0, 6)])
        return BlockDimRef(("BX", "BY", "BZ")[rng.integers(0, 3)])
    op = ("+", "-", "*", "//", "%")[rng.integers(0, 5)]
    left = _random_tree(rng, depth + 1)
    if op in ("//", "%"):
        return fold(op, left, IntConstant(int(rng.integers(1, 64))))
    if op == "*":
        return fold(op, left, IntConstant(int(rng.integers(-32, 33))))
    return fold(op, left, _random_tree(rng, depth + 1))


def bulk_cases(rng):
    out = []
    for _ in range(1000):
        tree = _random_tree(rng)
        n = int(rng.integers(1, 24))
        env = {name: rng.integers(-64, 64, size=n).astype(np.int64) for name in COORD_NAMES}
        val = gvo.evaluate_bulk(tree, env, BLOCK, {})
        out.append({"expr": render(tree), "env": {k: v.tolist() for k, v in env.items()},
                    "out": [int(x) for x in np.asarray(val).ravel()]})
    return out


def _hx(d):
    return {k: float(v).hex() for k, v in d.items()}


def _lkv(v):
    d = dataclasses.asdict(v)
    out = {}
    for k, x in d.items():
        if isinstance(x, dict):
            out[k] = _hx(x)
        elif x is None or isinstance(x, bool):
            out[k] = x
        else:
            out[k] = float(x).hex()
    return out


def _b200():
    """The B200 machine of this repo's workloads, as a reference descriptor."""
    sys.path.insert(1, str(ROOT))
    from paper_2107_01143_b200.gvo.machine import b200_preset, machine_to_dict
    from gvo.machine import machine_from_dict

    return machine_from_dict(machine_to_dict(b200_preset()))


def injected_cases(rng):
    kernels = [gvo.generate_star_stencil(4, (512, 512, 128), (32, 2, 16), folding="2z"),
               gvo.generate_star_stencil(2, (256, 256, 64), (64, 4, 1)),
               gvo.generate_lbm_d3q15((256, 128, 128), (32, 2, 2))]
    out = []
    for ki, k in enumerate(kernels):
        names = [f.name for f in k.fields]
        for rep in range(12):
            m = gvo.v100_preset() if rep % 2 == 0 else _b200()
            m = m.with_l2_capacity(int(m.l2_capacity_bytes // (1 << (rep % 3))))
            r = lambda lo, hi: float(rng.uniform(lo, hi))  # noqa: E731
            bs = BlockStats({n: r(0, 40) for n in names}, {n: r(0, 120) for n in names}, {n: r(0, 60) for n in names},
                            {n: r(0, 20) for n in names}, {n: r(0, 40) for n in names})
            has_pred = rep % 4 != 3
            lu = {n: r(0, 4e6) for n in names}
            ws = WaveStats(lu, {n: (r(0, 1) * lu[n] if has_pred else 0.0) for n in names},
                           r(0, 8e6) if has_pred else 0.0, {n: r(0, 2e6) for n in names}, r(1e5, 2e7),
                           float(int(rng.integers(1, 1 << 20))), 2 if has_pred else 0, has_pred)
            if rep == 5:  # zero previous footprint: coverage disabled
                ws = dataclasses.replace(ws, prev_unique_total=0.0)
            vols = gvo.estimate_volumes(k, m, block_stats=bs, wave_stats=ws)
            l1 = gvo.l1_register_cycles(k, m)
            p = gvo.predict(k, m, vols, l1)
            out.append({"kernel": ki, "machine": gvo.machine.machine_to_dict(m),
                        "block_stats": {f.name: _hx(getattr(bs, f.name)) for f in dataclasses.fields(bs)},
                        "wave_stats": {f.name: (_hx(getattr(ws, f.name)) if isinstance(getattr(ws, f.name), dict)
                                                else getattr(ws, f.name) if isinstance(getattr(ws, f.name), (bool, int))
                                                else float(getattr(ws, f.name)).hex())
                                       for f in dataclasses.fields(ws)},
                        "volumes": {lvl: _lkv(getattr(vols, lvl))
                                    for lvl in ("l2l1_load", "l2l1_store", "dram_load", "dram_store")},
                        "glups": float(p.glups).hex(), "limiter": p.limiter,
                        "times": _hx(p.times)})
    return [gvo.kernel_to_dict(k) for k in kernels], out


def file_sweeps():
    specs = [gvo.kernel_to_dict(gvo.generate_four_point_2d((256, 256), (32, 4, 1))),
             gvo.kernel_to_dict(gvo.generate_star_stencil(1, (64, 64, 64), (8, 8, 1))),
             gvo.kernel_to_dict(gvo.generate_lbm_d3q15((64, 32, 32), (32, 2, 2)))]
    out = []
    m = gvo.v100_preset()
    for si, spec in enumerate(specs):
        grid = tuple(int(v) for v in ((256, 256, 1) if si == 0 else (64, 64, 64) if si == 1 else (64, 32, 32)))
        fam = gvo.KernelFamily("file", grid, spec=spec)
        cfgs = list(gvo.enumerate_sweep(64)) + list(gvo.enumerate_sweep(256))
        cfgs += [gvo.SweepConfig((32, 2, 1), "2z")]  # folding refused -> skipped
        rows = gvo.rank_sweep(fam, cfgs, m, block_samples=2, wave_samples=1, skip_invalid=True)
        out.append({"spec": spec, "grid": list(grid),
                    "configs": [[list(c.block_dim), c.folding] for c in cfgs],
                    "rows": [[list(r.config.block_dim), r.config.folding, float(r.prediction.glups).hex(),
                              r.prediction.limiter] for r in rows]})
    return out


def main():
    rng = np.random.default_rng(20240811)
    kspecs, inj = injected_cases(rng)
    out = {"block": list(BLOCK), "bulk": bulk_cases(rng), "injected_kernels": kspecs, "injected": inj,
           "file_sweeps": file_sweeps()}
    OUT.write_text(json.dumps(out, separators=(",", ":")))
    print("written", OUT, OUT.stat().st_size)


if __name__ == "__main__":
    main()
