"""Four-limiter performance model and configuration ranking (drop-in for
reference ``gvo.perf``, perf.py:1-132).

``rank_sweep`` is the batching point: instead of building one descriptor per
configuration and looping (perf.py:115-130), it builds one device template
per distinct access structure, validates each configuration with the
family's tiling rule, evaluates the whole batch in one pipeline launch and
ranks it with the device radix sort (key of perf.py:131).
"""

from __future__ import annotations

from dataclasses import dataclass
from collections.abc import Sequence
from typing import Iterable, Mapping

from itertools import repeat
from operator import attrgetter

import numpy as np

from .. import _native
from . import _engine
from .fit import GompertzParams
from .kernels import KernelDescriptor, KernelFamily, SweepConfig
from .machine import MachineDescriptor
from .volumes import L1CycleEstimate, VolumeBreakdown, _levels_from

LIMITER_ORDER = ("dram", "l2", "l1", "fp")


class PerfError(ValueError):
    pass


@dataclass(frozen=True)
class PerfPrediction:
    times: dict[str, float]
    limiter: str
    glups: float
    volumes: VolumeBreakdown
    l1_cycles: L1CycleEstimate
    flops_per_lup: int


def binding_limiter(times: Mapping[str, float]) -> str:
    """Largest time; ties resolved in the order (dram, l2, l1, fp) (perf.py:38-42)."""
    order = [n for n in LIMITER_ORDER if n in times] + [n for n in times if n not in LIMITER_ORDER]
    best = order[0]
    for n in order[1:]:
        if times[n] > times[best]:
            best = n
    return best


def predict(kernel: KernelDescriptor, machine: MachineDescriptor, volumes: VolumeBreakdown,
            l1_cycles: L1CycleEstimate) -> PerfPrediction:
    if machine.mem_bandwidth_bps <= 0 or machine.l2_bandwidth_bps <= 0:
        raise PerfError("bandwidths must be positive")
    ctx = _native.context()
    mid = ctx.machine_id(machine)
    out = _native.predict(np.array([mid]), np.array([volumes.dram_load.v_down + volumes.dram_store.v_down]),
                          np.array([volumes.l2l1_load.v_down + volumes.l2l1_store.v_down]),
                          np.array([l1_cycles.cycles_per_lup]), np.array([kernel.flops_per_lup]))[0]
    times = {"dram": float(out[0]), "l2": float(out[1]), "l1": float(out[2]), "fp": float(out[3])}
    return PerfPrediction(times, LIMITER_ORDER[int(out[4])], float(out[5]), volumes, l1_cycles,
                          kernel.flops_per_lup)


def _prediction(res, i, names, flops, per_access) -> PerfPrediction:
    rec = res.records[i]
    c = dict(zip(_native.RECORD_COLUMNS, rec))
    times = {"dram": float(c["tDram"]), "l2": float(c["tL2"]), "l1": float(c["tL1"]), "fp": float(c["tFp"])}
    vols = _levels_from(rec, res.field_down[i], names)
    l1 = L1CycleEstimate(float(c["l1CyclesPerLup"]), per_access)
    return PerfPrediction(times, LIMITER_ORDER[int(c["limiter"])], float(c["predictedGLups"]), vols, l1, flops)


def _per_access(res, i, n_acc) -> tuple[float, ...]:
    l1 = res.l1_access[i, :n_acc]
    return tuple((float(r[1]) / 2.0) / float(r[2]) for r in l1)


def evaluate_kernel(kernel: KernelDescriptor, machine: MachineDescriptor,
                    fit_params: Mapping[str, GompertzParams] | None = None, *, block_samples: int = 5,
                    wave_samples: int = 2, override_blocks_per_wave: int | None = None) -> PerfPrediction:
    """Footprints, volumes, cycles and prediction in one device pipeline."""
    b = _engine.Batch()
    b.add(kernel.fields, kernel.accesses, kernel.launch, kernel.flops_per_lup, machine, fit_params)
    res = b.run(block_samples, wave_samples, override_blocks_per_wave, phases=7, want_l1=True)
    _engine.raise_for_status(res, 0, kernel, machine, block_samples, wave_samples, override_blocks_per_wave)
    return _prediction(res, 0, [f.name for f in kernel.fields], kernel.flops_per_lup,
                       _per_access(res, 0, len(kernel.accesses)))


@dataclass(frozen=True)
class SweepRow:
    config: SweepConfig
    prediction: PerfPrediction


_FOLD_FACTORS = {"none": (1, 1, 1), "2y": (1, 2, 1), "2z": (1, 1, 2)}
_BLOCK_DIM = attrgetter("block_dim")
_FOLDING = attrgetter("folding")


# (family, template key) -> (template descriptor, context, template id):
# generator families build the same descriptor for every sweep, so repeated
# sweeps skip rebuilding and re-hashing the access trees (descriptors are
# immutable; file families are not cached: their spec does not enter the
# family's hash)
_TPL_CACHE: dict = {}


class SweepPlan:
    """A validated sweep in columnar form: the kept configurations (input
    order), one device template per distinct access structure and the
    gvo_config array, built without one descriptor per configuration.

    Validation follows the reference loop (perf.py:115-121): build errors
    (ValueError from family.build) skip the configuration with
    ``skip_invalid`` and otherwise stop the sweep at the first invalid
    configuration.  Stencil / LBM families validate the whole batch with
    array arithmetic; any configuration the vector check does not accept
    goes through family.launch_of, which raises exactly what build raises.
    """

    def __init__(self, family: KernelFamily, configs, machine, fit_params=None, *, skip_invalid=False):
        self.family = family
        configs = list(configs)
        if not configs:
            raise PerfError("empty sweep")
        ctx = _native.context()
        self.machine_id = ctx.machine_id(machine, fit_params)
        n = len(configs)
        block = np.zeros((n, 3), dtype=np.int64)
        grid = np.zeros((n, 3), dtype=np.int64)
        wpt = np.ones(n, dtype=np.int64)
        flops = np.zeros(n, dtype=np.int64)
        # template key of each configuration as an id into key_list (keys are
        # large tuples: hashed once per distinct folding, not per config)
        key_list: list = []
        key_ix: dict = {}

        def key_id(k) -> int:
            j = key_ix.get(k)
            if j is None:
                j = key_ix[k] = len(key_list)
                key_list.append(k)
            return j

        tk = np.full(n, -1, dtype=np.int64)
        fast = np.zeros(n, dtype=bool)
        # rejected by the vector check with every block extent >= 1 and a
        # string folding: launch_of raises KernelError (a ValueError) for
        # these, so a skip_invalid sweep skips them without the call
        sure_bad = np.zeros(n, dtype=bool)
        folds = None
        if family.kind in ("stencil", "lbm") and len(tuple(family.grid)) == 3:
            try:
                b = np.array(list(map(_BLOCK_DIM, configs)), dtype=np.int64)
                ok_shape = b.shape == (n, 3)
            except (TypeError, ValueError):
                ok_shape = False
            if ok_shape:
                # foldings as codes into their distinct values (a handful per sweep)
                folds = list(map(_FOLDING, configs))
                try:
                    ufolds = [f for f in dict.fromkeys(folds) if isinstance(f, str)]
                    ucode = {f: i for i, f in enumerate(ufolds)}
                    fcode = np.array(list(map(ucode.get, folds, repeat(-1))), dtype=np.int64)
                except TypeError:  # unhashable foldings: none of them is valid
                    ufolds = []
                    fcode = np.full(n, -1, dtype=np.int64)
                uff = np.array([_FOLD_FACTORS.get(f, (0, 0, 0)) for f in ufolds] + [(0, 0, 0)], dtype=np.int64)
                ff = uff[fcode]
                g = np.array([int(v) for v in family.grid], dtype=np.int64)
                eff = b * ff
                ok = (ff > 0).all(axis=1) & (b >= 1).all(axis=1) & (g >= 1).all()
                ok &= ((g[None, :] % np.where(eff > 0, eff, 1)) == 0).all(axis=1)
                if family.kind == "stencil":
                    ok &= family.radius >= 1
                    fl = 6 * family.radius + 1
                else:
                    ok &= ff.prod(axis=1) == 1  # lbm: folding "none" only
                    fl = 250 if family.flops_per_lup is None else family.flops_per_lup
                fast = ok
                sure_bad = ~ok & (b >= 1).all(axis=1) & (fcode >= 0) & (g >= 1).all()
                block[ok] = b[ok]
                grid[ok] = g[None, :] // np.where(eff[ok] > 0, eff[ok], 1)
                wpt[ok] = ff[ok].prod(axis=1)
                flops[ok] = fl
                # stencil / lbm template keys depend on the folding only: one
                # key per distinct folding, from its first valid configuration
                for u in np.unique(fcode[ok]).tolist():
                    rows = ok & (fcode == u)
                    tk[rows] = key_id(family.template_key(configs[int(np.argmax(rows))]))
        self.build_error = None  # (index, exception) of the first invalid config (skip_invalid=False)
        keep = np.ones(n, dtype=bool)
        todo = ~fast
        if skip_invalid:
            keep[sure_bad] = False
            todo &= ~sure_bad
        for i in np.flatnonzero(todo):
            cfg = configs[i]
            try:
                launch, fl = family.launch_of(cfg)
                tk[i] = key_id(family.template_key(cfg))
            except ValueError as exc:
                keep[i] = False
                if skip_invalid:
                    continue
                self.build_error = (int(i), exc)
                keep[i:] = False  # the reference loop stops here
                break
            block[i], grid[i], wpt[i], flops[i] = launch.block_dim, launch.grid_dim, launch.work_per_thread, fl
        idx = np.flatnonzero(keep)
        self.configs = configs if len(idx) == n else list(map(configs.__getitem__, idx.tolist()))
        self.block, self.grid, self.wpt, self.flops = block[idx], grid[idx], wpt[idx], flops[idx]
        # one template per key (built from its first configuration), ids registered once
        self.templates: list = []
        ukid, first, kid = np.unique(tk[idx], return_index=True, return_inverse=True)
        cacheable = family.kind in ("stencil", "lbm")
        for u, j in zip(ukid.tolist(), first.tolist()):
            key, i = key_list[u], int(idx[j])
            hit = _TPL_CACHE.get((family, key)) if cacheable else None
            if hit is not None and hit[1] is ctx:
                self.templates.append((hit[0], hit[2]))
            else:
                k = family.build(configs[i])
                tid = ctx.template_id(k.fields, k.accesses)
                self.templates.append((k, tid))
                if cacheable:
                    if len(_TPL_CACHE) >= 4096:
                        _TPL_CACHE.clear()
                    _TPL_CACHE[(family, key)] = (k, ctx, tid)
        self.tpl = kid.astype(np.int32).reshape(-1)
        fr = _engine.FOLD_RANK
        if folds is not None and all(isinstance(f, str) for f in ufolds):
            ufr = np.array([fr.get(f, -1) for f in ufolds] + [-1], dtype=np.int32)
            self.fold_rank = ufr[fcode[idx]]
            if (self.fold_rank < 0).any():  # a folding the rank table lacks: the reference's KeyError
                self.fold_rank = np.array([fr[c.folding] for c in self.configs], dtype=np.int32)
        else:
            self.fold_rank = np.array([fr[c.folding] for c in self.configs], dtype=np.int32)

    def __len__(self) -> int:
        return len(self.configs)

    def config_array(self) -> np.ndarray:
        a = np.zeros(len(self), dtype=_native.CONFIG_DTYPE)
        tid = np.array([t[1] for t in self.templates], dtype=np.int32)
        a["template_id"] = tid[self.tpl] if len(self) else 0
        a["machine_id"] = self.machine_id
        a["block"] = self.block
        a["fold_rank"] = self.fold_rank
        a["grid"] = self.grid
        a["work_per_thread"] = self.wpt
        a["flops_per_lup"] = self.flops
        return a

    def kernel_row(self, i: int):
        """(template descriptor, LaunchConfig, flops) of kept config i."""
        from .kernels import LaunchConfig

        k = self.templates[int(self.tpl[i])][0]
        launch = LaunchConfig(tuple(int(v) for v in self.block[i]), tuple(int(v) for v in self.grid[i]),
                              int(self.wpt[i]))
        return k, launch, int(self.flops[i])

    def raise_first_error(self, res, machine, block_samples, wave_samples, override):
        """Reference order: the first configuration that fails (to evaluate,
        or to build) raises; evaluation errors of earlier configs first."""
        bad = np.flatnonzero(res.counts[:, _native.C_STATUS]) if res is not None else []
        if len(bad):
            i = int(bad[0])
            k, launch, _ = self.kernel_row(i)
            _engine.raise_for_status(res, i, k.with_launch(launch), machine, block_samples, wave_samples, override)
        if self.build_error is not None:
            raise self.build_error[1]


class _KernelRows(Sequence):
    """(descriptor, launch, flops) per kept configuration, built on access."""

    def __init__(self, plan: SweepPlan):
        self._plan = plan

    def __len__(self) -> int:
        return len(self._plan)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self._plan.kernel_row(j) for j in range(*i.indices(len(self)))]
        return self._plan.kernel_row(i)


def evaluate_sweep(family: KernelFamily, configs: Iterable[SweepConfig], machine: MachineDescriptor,
                   fit_params=None, *, block_samples=5, wave_samples=2, override_blocks_per_wave=None,
                   skip_invalid=False):
    """Batched evaluation: (kept configs, per-config (descriptor, launch,
    flops) rows, device result, ranking order).  One columnar batch, one
    evaluate + rank call (gvo_sweep_host_ex); validation and error order
    follow perf.py:115-130."""
    plan = SweepPlan(family, configs, machine, fit_params, skip_invalid=skip_invalid)
    if not len(plan):
        plan.raise_first_error(None, machine, block_samples, wave_samples, override_blocks_per_wave)
        raise PerfError("empty sweep")
    ctx = _native.context()
    out = ctx.sweep_host(plan.config_array(), block_samples, wave_samples, override_blocks_per_wave or 0)
    res = _engine.Result(out["F"], out["S"], out["W"], out["counts"], out["stats"], out["records"],
                         out["field_down"], out["l1_access"])
    plan.raise_first_error(res, machine, block_samples, wave_samples, override_blocks_per_wave)
    return plan.configs, _KernelRows(plan), res, out["order"]


class SweepRows(Sequence):
    """Ranked sweep rows (reference: list[SweepRow], perf.py:132).  Rows are
    materialised on access from the device records; ``records`` / ``order``
    / ``configs`` expose the batch for bulk consumers (the native ranking
    CSV formatter, report.render_ranking_csv)."""

    def __init__(self, kept, kernels, res, order):
        self.configs = list(kept)
        self._kernels = kernels
        self._res = res
        self.records = res.records
        self.order = np.asarray(order, dtype=np.int64)

    def __len__(self) -> int:
        return len(self.order)

    def _row(self, r: int) -> SweepRow:
        i = int(self.order[r])
        k, launch, flops = self._kernels[i]
        return SweepRow(self.configs[i], _prediction(self._res, i, [f.name for f in k.fields], flops,
                                                     _per_access(self._res, i, len(k.accesses))))

    def __getitem__(self, idx):
        if isinstance(idx, slice):
            return [self._row(r) for r in range(*idx.indices(len(self)))]
        r = int(idx)
        if r < 0:
            r += len(self)
        if not 0 <= r < len(self):
            raise IndexError("sweep row index out of range")
        return self._row(r)

    def __eq__(self, other):
        return list(self) == list(other)


def rank_sweep(family: KernelFamily, configs: Iterable[SweepConfig], machine: MachineDescriptor,
               fit_params: Mapping[str, GompertzParams] | None = None, *, block_samples: int = 5,
               wave_samples: int = 2, override_blocks_per_wave: int | None = None,
               skip_invalid: bool = False) -> SweepRows:
    """Evaluate every configuration and order by descending predicted
    throughput, ties by (block_dim, folding) then input order (perf.py:98-132)."""
    kept, kernels, res, order = evaluate_sweep(
        family, configs, machine, fit_params, block_samples=block_samples, wave_samples=wave_samples,
        override_blocks_per_wave=override_blocks_per_wave, skip_invalid=skip_invalid)
    return SweepRows(kept, kernels, res, order)
