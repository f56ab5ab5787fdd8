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


def evaluate_sweep(family: KernelFamily, configs: Iterable[SweepConfig], machine: MachineDescriptor,
                   fit_params=None, *, block_samples=5, wave_samples=2, override_blocks_per_wave=None,
                   skip_invalid=False):
    """Batched evaluation: (kept configs, per-config descriptors' field names,
    device result, ranking order).  Validation errors follow perf.py:115-121."""
    configs = list(configs)
    if not configs:
        raise PerfError("empty sweep")
    batch = _engine.Batch()
    templates: dict = {}
    kept, kernels = [], []
    for cfg in configs:
        try:
            launch, flops = family.launch_of(cfg)
            key = family.template_key(cfg)
            if key not in templates:
                templates[key] = family.build(cfg)
        except ValueError:
            if skip_invalid:
                continue
            raise
        k = templates[key]
        batch.add(k.fields, k.accesses, launch, flops, machine, fit_params, _engine.FOLD_RANK[cfg.folding])
        kept.append(cfg)
        kernels.append((k, launch, flops))
    res = batch.run(block_samples, wave_samples, override_blocks_per_wave, phases=7, want_l1=True)
    for i, (k, launch, flops) in enumerate(kernels):
        if res.counts[i, _native.C_STATUS]:
            _engine.raise_for_status(res, i, k.with_launch(launch), machine, block_samples, wave_samples,
                                     override_blocks_per_wave)
    order = _native.rank_host(batch.config_array(), res.records)
    return kept, kernels, res, order


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
