"""Glue between the drop-in API objects and the device pipeline.

A batch is a list of (template, launch, flops, machine) rows encoded as
``gvo_config`` records; ``run`` launches the whole pipeline for the batch
(setup -> warp statistics -> interval-union engine -> assembly) through the
C ABI and returns the integer numerators, float statistics, f64 records and
per-field volumes.  Errors are re-raised with the reference's exception
classes and messages (the device reports which group/access failed; the
message text is rebuilt from that group's coordinate bounds).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .. import _native
from .expr import AddressOverflowError, value_bounds

FOLD_RANK = {"2y": 0, "2z": 1, "none": 2}  # string order of perf.py:131


@dataclass
class Result:
    F: int
    S: int
    W: int
    counts: np.ndarray
    stats: np.ndarray
    records: np.ndarray
    field_down: np.ndarray | None
    l1_access: np.ndarray | None


class Batch:
    def __init__(self):
        self.ctx = _native.context()
        self.rows: list[tuple] = []
        self.meta: list = []

    def add(self, fields, accesses, launch, flops, machine, fit_params=None, fold_rank=2, meta=None) -> int:
        tid = self.ctx.template_id(fields, accesses)
        mid = self.ctx.machine_id(machine, fit_params)
        self.rows.append((tid, mid, tuple(launch.block_dim), fold_rank, tuple(launch.grid_dim),
                          launch.work_per_thread, flops))
        self.meta.append(meta)
        return len(self.rows) - 1

    def config_array(self) -> np.ndarray:
        a = np.zeros(len(self.rows), dtype=_native.CONFIG_DTYPE)
        if self.rows:
            tid, mid, blk, fr, grd, wpt, fl = zip(*self.rows)
            a["template_id"] = tid
            a["machine_id"] = mid
            a["block"] = np.array(blk, dtype=np.int32)
            a["fold_rank"] = fr
            a["grid"] = np.array(grd, dtype=np.int64)
            a["work_per_thread"] = wpt
            a["flops_per_lup"] = fl
        return a

    def run(self, block_samples=5, wave_samples=2, override=None, phases=7, want_l1=False) -> Result:
        out = self.ctx.eval_configs_host(self.config_array(), block_samples, wave_samples, override or 0,
                                         want_l1_access=want_l1, phases=phases)
        return Result(out["F"], out["S"], out["W"], out["counts"], out["stats"], out["records"],
                      out["field_down"], out["l1_access"])


# ---------------------------------------------------------------------------
# decoding


def block_counts(res: Result, i: int) -> np.ndarray:
    """[n_samples][F][5] integer numerators of config i."""
    n = int(res.counts[i, _native.C_NSAMPLES])
    blk = res.counts[i, _native.C_HDR:_native.C_HDR + res.S * res.F * 5].reshape(res.S, res.F, 5)
    return blk[:n]


def wave_counts(res: Result, i: int) -> tuple[np.ndarray, np.ndarray]:
    """([U][F][4] set counts, [U] wave lups)."""
    U = int(res.counts[i, _native.C_NUWAVES])
    off = _native.C_HDR + res.S * res.F * 5
    wv = res.counts[i, off:off + (res.W + 1) * res.F * 4].reshape(res.W + 1, res.F, 4)
    wl = res.counts[i, off + (res.W + 1) * res.F * 4: off + (res.W + 1) * res.F * 4 + res.W + 1]
    return wv[:U], wl[:U]


def stats_view(res: Result, i: int):
    F = res.F
    s = res.stats[i]
    return {
        "load_comp": s[0:F], "load_up": s[F:2 * F], "load_alloc": s[2 * F:3 * F],
        "store_unique": s[3 * F:4 * F], "store_up": s[4 * F:5 * F],
        "w_load_unique": s[5 * F:6 * F], "w_load_overlap": s[6 * F:7 * F], "w_store_unique": s[7 * F:8 * F],
        "prev_total": s[8 * F], "alloc_total": s[8 * F + 1], "wave_lups": s[8 * F + 2],
        "has_pred": bool(s[8 * F + 3]), "cycles_per_lup": s[8 * F + 4],
    }


_FOOTPRINT_MESSAGES = {
    0: "sample count must be >= 1",
    1: "block of {t} threads exceeds machine limit {m}",
    2: "block of {t} threads exceeds per-SM thread capacity",
    3: "blocks per wave must be >= 1",
}


def raise_for_status(res: Result, i: int, kernel, machine, block_samples, wave_samples, override):
    """Raise the reference's exception for a failed config."""
    from .footprint import FootprintError, build_waves, representative_blocks, representative_wave_pairs

    row = res.counts[i]
    status = int(row[_native.C_STATUS])
    if status == 0:
        return
    phase = int(row[_native.C_ERR_PHASE])
    group = int(row[_native.C_ERR_GROUP])
    acc = int(row[_native.C_ERR_ACCESS])
    if status == 4:  # FootprintError
        msg = _FOOTPRINT_MESSAGES.get(acc, "footprint error").format(
            t=kernel.launch.threads_per_block, m=machine.max_threads_per_block)
        raise FootprintError(msg)
    if status == 2:  # AddressOverflowError: rebuild the message on that group
        if phase == 0:
            grp = representative_blocks(kernel, block_samples)[group]
        elif phase == 1:
            waves = build_waves(kernel.launch, machine, override)
            first = int(row[_native.C_FIRSTWAVE])
            from .footprint import wave_group

            grp = wave_group(kernel.launch, waves[first + group])
        else:
            groups = representative_blocks(kernel, 5)
            grp = groups[len(groups) // 2]
        bounds = group_bounds(kernel, grp)
        value_bounds(kernel.accesses[acc].expr, bounds, kernel.launch.block_dim, kernel.base_substitution)
        raise AddressOverflowError("subexpression bound outside 64-bit signed range")
    raise _native.EngineError(status, f"config {i}: engine status {status}")


def group_bounds(kernel, group) -> dict:
    bx, by, bz = kernel.launch.block_dim
    xs, ys, zs = group.block_coords()
    return {"tidx": (0, bx - 1), "tidy": (0, by - 1), "tidz": (0, bz - 1),
            "bidx": (int(xs.min()), int(xs.max())), "bidy": (int(ys.min()), int(ys.max())),
            "bidz": (int(zs.min()), int(zs.max()))}


def check_group_bounds(kernel, group, accesses):
    """The reference evaluates value_bounds per access before enumerating a
    group (footprint.py:331, 343); same order, same exception."""
    if not accesses:
        return
    b = group_bounds(kernel, group)
    for a in accesses:
        value_bounds(a.expr, b, kernel.launch.block_dim, kernel.base_substitution)


def runs_of(block_linear: np.ndarray) -> list[tuple[int, int]]:
    """Consecutive runs of a block list (order kept)."""
    lin = [int(v) for v in np.asarray(block_linear).ravel()]
    runs: list[list[int]] = []
    for v in lin:
        if runs and runs[-1][0] + runs[-1][1] == v:
            runs[-1][1] += 1
        else:
            runs.append([v, 1])
    return [(a, b) for a, b in runs]
