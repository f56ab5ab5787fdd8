"""Serialization of estimates and rankings (drop-in for reference
``gvo.report``, report.py:1-255): the estimate report dict / JSON, the
estimate and footprint CSVs, the plain table, and the 42-column ranking
record and CSV.

Byte-identical output is the contract (the reference's bindings and CLI
compare bytes, bindings/tests/test_parity.py:47-108).  Ranking CSVs of a
device sweep (``SweepRows`` from ``rank_sweep``) are formatted by the
native multi-threaded formatter (``gvo_format_ranking_csv``, csrc/h_report.cu)
straight from the f64 records in ranked order — 10^6 rows without building
one Python row object per configuration; any other row sequence goes
through ``ranking_row_dict`` and the same ``.10g`` rule in Python.
"""

from __future__ import annotations

import io
import json

from .. import _native
from .perf import PerfPrediction, SweepRow, SweepRows
from .volumes import LEVEL_DRAM, LEVEL_L2L1, LevelKindVolumes

REPORT_SCHEMA_VERSION = 1

ESTIMATE_CSV_HEADER = ("level,kind,vComp,vRed,vCap,vUp,vDown,vAlloc,oversubscription,"
                       "waveUnique,vOverlap,overmissBytes,coverage,vRedL2")
FOOTPRINT_CSV_HEADER = "field,kind,granularity,uniqueBytes,totalAccessBytes"
RANKING_CSV_COLUMNS = ("configKey", "blockX", "blockY", "blockZ", "folding") + _native.RECORD_COLUMNS


def _fmt(value) -> str:
    """Numeric cell: Python's '.10g' (report.py:19-22); None -> empty."""
    return "" if value is None else format(float(value), ".10g")


def _level_kind_dict(v: LevelKindVolumes, dram: bool) -> dict:
    d = {"vUp": v.v_up, "vComp": v.v_comp, "vRed": v.v_red, "vCap": v.v_cap, "vDown": v.v_down,
         "vAlloc": v.v_alloc, "oversubscription": v.oversubscription,
         "perFieldDown": dict(sorted(v.per_field_down.items()))}
    if dram:
        d["waveUnique"] = v.wave_unique
        d["vOverlap"] = v.v_overlap
        d["overmissBytes"] = v.overmiss_bytes
        d["coverage"] = v.coverage
        d["vRedL2"] = v.v_red_l2
    return d


def build_estimate_report(prediction: PerfPrediction, config_meta: dict) -> dict:
    """Estimate report document (report.py:48-81 schema)."""
    v = prediction.volumes
    return {
        "schemaVersion": REPORT_SCHEMA_VERSION,
        "config": config_meta,
        "kernel": {"flopsPerLup": prediction.flops_per_lup, "accessCount": config_meta.get("accessCount"),
                   "workPerThread": config_meta.get("workPerThread")},
        "l1Cycles": {"cyclesPerLup": prediction.l1_cycles.cycles_per_lup,
                     "perAccess": list(prediction.l1_cycles.per_access)},
        "volumes": {
            LEVEL_L2L1: {"load": _level_kind_dict(v.l2l1_load, False), "store": _level_kind_dict(v.l2l1_store, False)},
            LEVEL_DRAM: {"load": _level_kind_dict(v.dram_load, True), "store": _level_kind_dict(v.dram_store, True)},
        },
        "performance": {"times": dict(sorted(prediction.times.items())), "limiter": prediction.limiter,
                        "predictedGLups": prediction.glups},
    }


def render_json(report: dict) -> str:
    return json.dumps(report, indent=2, sort_keys=True)


def render_estimate_csv(report: dict) -> str:
    lines = [ESTIMATE_CSV_HEADER]
    for level in (LEVEL_L2L1, LEVEL_DRAM):
        for kind in ("load", "store"):
            v = report["volumes"][level][kind]
            cells = [level, kind] + [_fmt(v[k]) for k in ("vComp", "vRed", "vCap", "vUp", "vDown", "vAlloc",
                                                          "oversubscription")]
            cells += [_fmt(v.get(k)) for k in ("waveUnique", "vOverlap", "overmissBytes", "coverage", "vRedL2")]
            lines.append(",".join(cells))
    return "\n".join(lines) + "\n"


def render_table(report: dict) -> str:
    cfg, perf = report["config"], report["performance"]
    b = io.StringIO()
    b.write(f"kernel      : {cfg.get('kernel')}\n")
    b.write(f"machine     : {cfg.get('machine')}\n")
    b.write(f"block       : {tuple(cfg.get('block', ()))}  folding: {cfg.get('folding')}\n")
    b.write(f"grid        : {tuple(cfg.get('grid', ()))}\n")
    b.write(f"blocks/wave : {cfg.get('blocksPerWave')}\n")
    b.write("\nvolumes per lattice update [bytes]\n")
    b.write(f"{'level':10} {'kind':6} {'comp':>10} {'red':>10} {'cap':>10} {'up':>10} {'down':>10}\n")
    for level in (LEVEL_L2L1, LEVEL_DRAM):
        for kind in ("load", "store"):
            v = report["volumes"][level][kind]
            b.write(f"{level:10} {kind:6} {v['vComp']:10.2f} {v['vRed']:10.2f} "
                    f"{v['vCap']:10.2f} {v['vUp']:10.2f} {v['vDown']:10.2f}\n")
    b.write("\ntimes per lattice update [s]\n")
    for name, t in perf["times"].items():
        b.write(f"  {name:5}: {t:.4e}{' <- limiter' if name == perf['limiter'] else ''}\n")
    b.write(f"\npredicted throughput: {perf['predictedGLups']:.3f} GLup/s\n")
    b.write(f"L1 cycles per LUP   : {report['l1Cycles']['cyclesPerLup']:.4f}\n")
    return b.getvalue()


def render_footprint_csv(result) -> str:
    g = result.granularity
    lines = [FOOTPRINT_CSV_HEADER]
    lines += [f"{f},{k},{g},{c.unique_count * g},{c.total_count * g}" for (f, k), c in sorted(result.per_field.items())]
    return "\n".join(lines) + "\n"


def ranking_row_dict(row: SweepRow) -> dict:
    """The 42-column record of one ranked configuration (report.py:208-239)."""
    p, v = row.prediction, row.prediction.volumes
    bx, by, bz = row.config.block_dim
    d = {"configKey": row.config.key, "blockX": bx, "blockY": by, "blockZ": bz, "folding": row.config.folding,
         "l1CyclesPerLup": p.l1_cycles.cycles_per_lup}
    for prefix, lv, dram in (("l2l1Load", v.l2l1_load, False), ("l2l1Store", v.l2l1_store, False),
                             ("dramLoad", v.dram_load, True), ("dramStore", v.dram_store, True)):
        d[prefix + "Comp"] = lv.v_comp
        d[prefix + "Red"] = lv.v_red
        d[prefix + "Cap"] = lv.v_cap
        d[prefix + "Up"] = lv.v_up
        d[prefix + "Down"] = lv.v_down
        if prefix.endswith("Load"):
            d[prefix + "Alloc"] = lv.v_alloc
            d[prefix + "Oversub"] = lv.oversubscription
        if prefix == "dramLoad":
            d["dramLoadUnique"] = lv.wave_unique
            d["dramLoadOverlap"] = lv.v_overlap
            d["dramLoadOvermiss"] = lv.overmiss_bytes
            d["dramLoadCoverage"] = lv.coverage
            d["dramLoadRedL2"] = lv.v_red_l2
        if prefix == "dramStore":
            d["dramStoreUnique"] = lv.wave_unique
    d.update({"tDram": p.times["dram"], "tL2": p.times["l2"], "tL1": p.times["l1"], "tFp": p.times["fp"],
              "limiter": p.limiter, "predictedGLups": p.glups})
    return {c: d[c] for c in RANKING_CSV_COLUMNS}


def _cell(value) -> str:
    if isinstance(value, str):
        return value
    if isinstance(value, int):
        return str(value)
    return _fmt(value)


def render_ranking_csv(rows) -> str:
    """Ranking CSV (report.py:242-255).  Device sweeps take the native path."""
    head = ",".join(RANKING_CSV_COLUMNS) + "\n"
    if isinstance(rows, SweepRows):
        cfgs = rows.configs
        prefixes = [f"{c.key},{c.block_dim[0]},{c.block_dim[1]},{c.block_dim[2]},{c.folding}" for c in cfgs]
        return head + _native.format_ranking_csv(rows.records, prefixes, rows.order)
    body = "".join(",".join(_cell(v) for v in ranking_row_dict(r).values()) + "\n" for r in rows)
    return head + body
