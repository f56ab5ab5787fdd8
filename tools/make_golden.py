"""Generate golden vectors by running the UNMODIFIED reference estimator.

Run in the build container (the reference is not available on the GPU box):
    python tools/make_golden.py
It imports `gvo` from baseline/_ref (pip-installed copy of /root/reference/pkg)
or /root/reference/pkg/src, and writes tests/golden/*.json.  Floats are stored
as float.hex() strings so comparisons are bit-exact.
"""

from __future__ import annotations

import dataclasses
import json
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
for cand in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
    if (cand / "gvo").exists():
        sys.path.insert(0, str(cand))
        break
import gvo  # noqa: E402  (the reference)
from gvo.expr import BaseRef, BinOp, CoordRef, IntConstant, fold  # noqa: E402
from gvo.footprint import CollaborativeGroup, wave_footprint  # noqa: E402
from gvo.kernels import kernel_to_dict  # noqa: E402
from gvo.machine import machine_to_dict  # noqa: E402
from gvo.report import ranking_row_dict  # noqa: E402

OUT = ROOT / "tests" / "golden"
COORDS = ("tidx", "tidy", "tidz", "bidx", "bidy", "bidz")


def hx(v):
    if v is None:
        return None
    if isinstance(v, (bool, np.bool_)):
        return bool(v)
    if isinstance(v, (int, np.integer)):
        return int(v)
    return float(v).hex()


def b200():
    return dataclasses.replace(
        gvo.v100_preset(), name="b200", sm_count=148, clock_ghz=1.965, l1_capacity_bytes=256 * 1024,
        l2_capacity_bytes=126 * 1024 * 1024, mem_bandwidth_gbps=6531.3, l2_bandwidth_gbps=20000.0)


# ------------------------------------------------------------- footprints
def random_kernel(rng, allow_divmod: bool, n_fields_max=3):
    block = [(1, 1, 1), (4, 1, 1), (8, 2, 1), (16, 2, 2), (32, 2, 1), (7, 3, 2), (64, 1, 1), (5, 3, 2)][rng.integers(0, 8)]
    grid = [(1, 1, 1), (2, 1, 1), (2, 2, 1), (3, 2, 2)][rng.integers(0, 4)]
    names = [f"f{i}" for i in range(int(rng.integers(1, n_fields_max + 1)))]
    align = {n: int(rng.choice([0, 0, 8, -1, 24, 100])) for n in names}
    fields = tuple(gvo.Field(n, 8, (1 << 20,), alignment=align[n]) for n in names)
    accesses = []
    for _ in range(int(rng.integers(1, 6))):
        name = names[rng.integers(0, len(names))]
        node = BaseRef(name)
        for _ in range(int(rng.integers(0, 5))):
            node = fold("+", node, fold("*", CoordRef(COORDS[rng.integers(0, 6)]), IntConstant(int(rng.integers(-64, 65)))))
        node = fold("+", node, IntConstant(int(rng.integers(-256, 257))))
        if allow_divmod and rng.integers(0, 2):
            op = ["//", "%"][rng.integers(0, 2)]
            node = BinOp(op, node, IntConstant(int(rng.choice([2, 4, 32, 100]))))
            node = fold("+", BaseRef(name), fold("*", node, IntConstant(1)))
            node = BinOp("-", node, BaseRef(name))
        accesses.append(gvo.Access(name, ["load", "store"][rng.integers(0, 2)], node, int(rng.integers(1, 4))))
    launch = gvo.LaunchConfig(block, grid)
    return gvo.KernelDescriptor(fields=fields, accesses=tuple(accesses), launch=launch)


def footprint_case(kernel, blocks, g):
    grp = CollaborativeGroup(kernel.launch, np.asarray(blocks, dtype=np.int64), "L2")
    r = gvo.grid_iteration(kernel, grp, g)
    return {"spec": kernel_to_dict(kernel), "blocks": [int(b) for b in blocks], "granularity": g,
            "per_field": [[f, k, c.unique_count, c.total_count] for (f, k), c in r.per_field.items()]}


def footprints():
    cases = []
    k = gvo.generate_four_point_2d((100, 100), (2, 2))
    cases.append(footprint_case(k, [0], 8))
    from gvo import parse

    names = ["a"]
    fa = (gvo.Field("a", 8, (4096, 64, 64), alignment=-1),)
    acc = (gvo.Access("a", "load", parse("a + (tidx + tidy * 100) * 8", fields=names)),
           gvo.Access("a", "store", parse("a + tidx * 8", fields=names)))
    kn = gvo.KernelDescriptor(fields=fa, accesses=acc, launch=gvo.LaunchConfig((8, 4, 1), (4, 2, 2)))
    for g in (8, 32, 128):
        cases.append(footprint_case(kn, [0], g))
    rng = np.random.default_rng(20240811)
    for i in range(400):
        kk = random_kernel(rng, allow_divmod=(i % 3 == 0))
        nb = kk.launch.total_blocks
        cnt = int(rng.integers(1, min(3, nb) + 1))
        start = int(rng.integers(0, nb - cnt + 1))
        g = int(rng.choice([8, 32, 128, 24]))
        try:
            cases.append(footprint_case(kk, list(range(start, start + cnt)), g))
        except gvo.AddressOverflowError:
            pass
    # a stencil block and a wave
    ks = gvo.generate_star_stencil(4, (128, 64, 32), (16, 4, 2))
    cases.append(footprint_case(ks, [37], 32))
    cases.append(footprint_case(ks, list(range(40, 200)), 32))
    return cases


# ------------------------------------------------------------- full evaluation
def evaluation(kernel, machine, fit_params=None, block_samples=5, wave_samples=2, override=None, ints=True):
    fits = machine.fit_params if fit_params is None else fit_params
    pred = gvo.evaluate_kernel(kernel, machine, fit_params, block_samples=block_samples,
                               wave_samples=wave_samples, override_blocks_per_wave=override)
    bs = gvo.sample_block_stats(kernel, machine, block_samples)
    ws = gvo.sample_wave_stats(kernel, machine, wave_samples, override)
    row = ranking_row_dict(gvo.SweepRow(gvo.SweepConfig(kernel.launch.block_dim), pred))
    rec = {k: hx(v) if not isinstance(v, str) else v for k, v in row.items()}
    out = {
        "spec": kernel_to_dict(kernel),
        "machine": machine_to_dict(dataclasses.replace(machine, fit_params=fits)),
        "sampling": [block_samples, wave_samples, override],
        "record": rec,
        "per_access": [hx(v) for v in pred.l1_cycles.per_access],
        "block_stats": {k: {f: hx(v) for f, v in getattr(bs, k).items()}
                        for k in ("load_comp", "load_up", "load_alloc", "store_unique", "store_up")},
        "wave_stats": {"load_unique": {f: hx(v) for f, v in ws.load_unique.items()},
                       "load_overlap": {f: hx(v) for f, v in ws.load_overlap.items()},
                       "store_unique": {f: hx(v) for f, v in ws.store_unique.items()},
                       "prev_unique_total": hx(ws.prev_unique_total), "alloc_total": hx(ws.alloc_total),
                       "wave_lups": hx(ws.wave_lups), "pairs_sampled": ws.pairs_sampled,
                       "has_predecessor": ws.has_predecessor},
        "per_field_down": {lvl: {f: hx(v) for f, v in getattr(pred.volumes, lvl).per_field_down.items()}
                           for lvl in ("l2l1_load", "l2l1_store", "dram_load", "dram_store")},
    }
    if ints:
        groups = gvo.representative_blocks(kernel, block_samples)
        out["block_ints"] = []
        for gr in groups:
            r32 = gvo.grid_iteration(kernel, gr, machine.sector_bytes)
            r128 = gvo.grid_iteration(kernel, gr, machine.l1_line_bytes, kinds=("load",))
            out["block_ints"].append({
                "block": int(gr.block_linear[0]),
                "sector": [[f, k, c.unique_count, c.total_count] for (f, k), c in r32.per_field.items()],
                "line": [[f, k, c.unique_count, c.total_count] for (f, k), c in r128.per_field.items()],
            })
        pairs = gvo.representative_wave_pairs(kernel, machine, wave_samples, override)
        out["wave_ints"] = []
        seen = {}
        for prev, curr in pairs:
            for w in (curr, prev):
                if w is not None and w.index not in seen:
                    fp = wave_footprint(kernel, w, machine.sector_bytes)
                    seen[w.index] = fp
                    out["wave_ints"].append({"index": w.index, "start": w.start, "count": w.count,
                                             "load": {f: s.count for f, s in fp.load_sets.items()},
                                             "store": dict(fp.store_counts), "alloc": fp.alloc_count})
        out["overlaps"] = []
        for prev, curr in pairs:
            if prev is not None:
                c, p = seen[curr.index], seen[prev.index]
                out["overlaps"].append({"curr": curr.index, "prev": prev.index,
                                        "per_field": {f: c.load_sets[f].intersection_count(p.load_sets[f])
                                                      for f in c.load_sets}})
    return out


def stencil2d5pt():
    from gvo import parse

    names = ["dst", "src"]
    fields = (gvo.Field("dst", 8, (256, 256)), gvo.Field("src", 8, (256, 256)))
    acc = []
    for dx, dy in ((0, 0), (1, 0), (-1, 0), (0, 1), (0, -1)):
        acc.append(gvo.Access("src", "load", parse(
            f"src + ((tidx + bidx*BX) + {dx} + ((tidy + bidy*BY) + {dy}) * 256) * 8", fields=names)))
    acc.append(gvo.Access("dst", "store", parse("dst + ((tidx + bidx*BX) + (tidy + bidy*BY) * 256) * 8", fields=names)))
    return gvo.KernelDescriptor(fields=fields, accesses=tuple(acc),
                                launch=gvo.LaunchConfig((32, 4, 1), (8, 64, 1)), flops_per_lup=5, name="2d5pt")


def evaluations():
    v100, m200 = gvo.v100_preset(), b200()
    cases = []
    k = stencil2d5pt()
    cases.append(evaluation(k, v100))
    cases.append(evaluation(k, m200))
    cases.append(evaluation(gvo.generate_star_stencil(4, (640, 512, 512), (16, 2, 32)), v100))
    cases.append(evaluation(gvo.generate_lbm_d3q15((256, 128, 128), (32, 2, 2)), v100))
    cases.append(evaluation(gvo.generate_lbm_d3q15((256, 128, 128), (32, 2, 2)), v100, gvo.zero_fit_params()))
    for shape, fold_ in (((16, 2, 32), "2z"), ((32, 32, 1), "2y"), ((1, 32, 32), "none"), ((128, 8, 1), "none"),
                         ((4, 4, 64), "none"), ((64, 4, 4), "2z")):
        cases.append(evaluation(gvo.generate_star_stencil(4, (640, 640, 640), shape, fold_), m200, ints=False))
    for shape in ((1, 128, 4), (8, 8, 8), (128, 2, 2)):
        cases.append(evaluation(gvo.generate_lbm_d3q15((256, 256, 256), shape), m200, ints=False))
    # sampling / override variants and a single-wave grid
    ks = gvo.generate_star_stencil(2, (128, 128, 64), (16, 4, 4))
    cases.append(evaluation(ks, v100, block_samples=2, wave_samples=1, override=40))
    cases.append(evaluation(ks, v100, block_samples=7, wave_samples=3))
    cases.append(evaluation(gvo.generate_star_stencil(1, (128, 128, 10), (32, 32, 1)), v100))
    return cases


def sweeps():
    out = []
    for kind, grid, threads, folds, radius in (("stencil", (128, 128, 64), 256, ("none", "2y", "2z"), 2),
                                               ("lbm", (64, 64, 32), 128, ("none",), 4)):
        fam = gvo.KernelFamily(kind, grid, radius=radius)
        cfgs = gvo.enumerate_sweep(threads, foldings=folds)
        rows = gvo.rank_sweep(fam, cfgs, gvo.v100_preset(), wave_samples=1, block_samples=2, skip_invalid=True)
        out.append({"kind": kind, "grid": list(grid), "threads": threads, "foldings": list(folds), "radius": radius,
                    "order": [r.config.key for r in rows],
                    "glups": [hx(r.prediction.glups) for r in rows]})
    return out


def errors():
    """Failing evaluations: exception class and message of the reference."""
    from gvo import parse

    out = []
    v100 = gvo.v100_preset()

    def case(fields, accs, block, grid, machine=v100, **kw):
        names = [f.name for f in fields]
        k = gvo.KernelDescriptor(fields=fields, accesses=tuple(gvo.Access(fn, kd, parse(t, fields=names))
                                                                for fn, kd, t in accs),
                                 launch=gvo.LaunchConfig(block, grid))
        try:
            gvo.evaluate_kernel(k, machine, **kw)
            res = None
        except Exception as exc:  # noqa: BLE001
            res = [type(exc).__name__, str(exc)]
        out.append({"spec": kernel_to_dict(k), "machine": machine_to_dict(machine), "kw": kw, "error": res})

    fa = (gvo.Field("a", 8, (1 << 20,)),)
    # phase 0: interior block bidx=2 overflows
    case(fa, [("a", "load", "a + tidx * 8 + bidx * 4611686018427387904")], (4, 1, 1), (4, 1, 1))
    # phase 1 only: interior blocks fine, the wave reaches bidx = 2
    case(fa, [("a", "load", "a + tidx * 8 + bidx * 4611686018427387904")], (4, 1, 1), (3, 1, 1))
    # a store overflowing after loads are fine (loads-before-stores order)
    case(fa, [("a", "load", "a + tidx * 8"), ("a", "store", "a + bidy * 4611686018427387904 + tidx")], (4, 1, 1), (3, 3, 1))
    # intermediate-node overflow that cancels at the root
    case(fa, [("a", "load", "a + (tidx * 4611686018427387904 + bidx * 4611686018427387904) - bidx * 4611686018427387904")],
         (4, 1, 1), (4, 1, 1))
    # block larger than the machine limit -> FootprintError in the wave phase
    case(fa, [("a", "load", "a + tidx * 8")], (1024, 2, 1), (1, 1, 1))
    # samples < 1
    case(fa, [("a", "load", "a + tidx * 8")], (32, 1, 1), (4, 4, 4), block_samples=0)
    case(fa, [("a", "load", "a + tidx * 8")], (32, 1, 1), (4, 4, 4), wave_samples=0)
    # override of 0 means computed; negative override is an error
    case(fa, [("a", "load", "a + tidx * 8")], (32, 1, 1), (4, 4, 4), override_blocks_per_wave=-3)
    # per-SM capacity
    import dataclasses
    small = dataclasses.replace(v100, max_threads_per_sm=512, max_threads_per_block=1024)
    case(fa, [("a", "load", "a + tidx * 8")], (1024, 1, 1), (4, 1, 1), machine=small)
    return out


if __name__ == "__main__":
    OUT.mkdir(parents=True, exist_ok=True)
    what = sys.argv[1:] or ["footprints", "evaluations", "sweeps", "errors"]
    if "errors" in what:
        (OUT / "errors.json").write_text(json.dumps(errors()))
    if "footprints" in what:
        (OUT / "footprints.json").write_text(json.dumps(footprints()))
    if "evaluations" in what:
        (OUT / "evaluations.json").write_text(json.dumps(evaluations()))
    if "sweeps" in what:
        (OUT / "sweeps.json").write_text(json.dumps(sweeps()))
    print("written", sorted(p.name for p in OUT.glob("*.json")))
