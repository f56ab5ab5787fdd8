"""Per-level volumes and L1 bank-conflict cycles (drop-in for reference
``gvo.volumes``, volumes.py:1-445).

All numbers come from the device: the integer numerators from the
enumeration engine, the float statistics, clamped assembly and Gompertz
ratios from csrc/k_assemble.cu (bit-identical to the Python reference).
Injected ``block_stats`` / ``wave_stats`` are shipped to the device
assembly kernel as they are.
"""

from __future__ import annotations

from dataclasses import dataclass, field as dc_field
from typing import Mapping

import numpy as np

from .. import _native
from . import _engine
from .fit import GompertzParams
from .footprint import CollaborativeGroup, representative_blocks
from .kernels import KernelDescriptor
from .machine import MachineDescriptor

LEVEL_L2L1 = "L2toL1"
LEVEL_DRAM = "DRAMtoL2"


@dataclass(frozen=True)
class L1CycleEstimate:
    cycles_per_lup: float
    per_access: tuple[float, ...]


@dataclass(frozen=True)
class BlockStats:
    load_comp: dict[str, float]
    load_up: dict[str, float]
    load_alloc: dict[str, float]
    store_unique: dict[str, float]
    store_up: dict[str, float]


@dataclass(frozen=True)
class WaveStats:
    load_unique: dict[str, float]
    load_overlap: dict[str, float]
    prev_unique_total: float
    store_unique: dict[str, float]
    alloc_total: float
    wave_lups: float
    pairs_sampled: int
    has_predecessor: bool


@dataclass(frozen=True)
class LevelKindVolumes:
    v_up: float
    v_comp: float
    v_red: float
    v_cap: float
    v_down: float
    v_alloc: float
    oversubscription: float
    per_field_down: dict[str, float] = dc_field(default_factory=dict)
    wave_unique: float | None = None
    v_overlap: float | None = None
    overmiss_bytes: float | None = None
    coverage: float | None = None
    v_red_l2: float | None = None


@dataclass(frozen=True)
class VolumeBreakdown:
    l2l1_load: LevelKindVolumes
    l2l1_store: LevelKindVolumes
    dram_load: LevelKindVolumes
    dram_store: LevelKindVolumes

    def level_kind(self, level: str, kind: str) -> LevelKindVolumes:
        return {
            (LEVEL_L2L1, "load"): self.l2l1_load, (LEVEL_L2L1, "store"): self.l2l1_store,
            (LEVEL_DRAM, "load"): self.dram_load, (LEVEL_DRAM, "store"): self.dram_store,
        }[(level, kind)]


# ---------------------------------------------------------------------------
# engine helpers


def _run_one(kernel, machine, fit_params, phases, block_samples=5, wave_samples=2, override=None,
             want_l1=False):
    b = _engine.Batch()
    b.add(kernel.fields, kernel.accesses, kernel.launch, kernel.flops_per_lup, machine, fit_params)
    res = b.run(block_samples, wave_samples, override, phases=phases, want_l1=want_l1)
    _engine.raise_for_status(res, 0, kernel, machine, block_samples, wave_samples, override)
    return res


def _block_stats_from(res, i, names) -> BlockStats:
    v = _engine.stats_view(res, i)
    pick = lambda arr: {n: float(arr[k]) for k, n in enumerate(names)}
    return BlockStats(pick(v["load_comp"]), pick(v["load_up"]), pick(v["load_alloc"]),
                      pick(v["store_unique"]), pick(v["store_up"]))


def _wave_stats_from(res, i, names) -> WaveStats:
    v = _engine.stats_view(res, i)
    pick = lambda arr: {n: float(arr[k]) for k, n in enumerate(names)}
    return WaveStats(pick(v["w_load_unique"]), pick(v["w_load_overlap"]), float(v["prev_total"]),
                     pick(v["w_store_unique"]), float(v["alloc_total"]), float(v["wave_lups"]),
                     int(res.counts[i, _native.C_NPAIRS]), v["has_pred"])


def l1_register_cycles(kernel: KernelDescriptor, machine: MachineDescriptor,
                       group: CollaborativeGroup | None = None) -> L1CycleEstimate:
    """Bank-conflict wavefronts of a representative block (volumes.py:111-134)."""
    if group is None:
        groups = representative_blocks(kernel, samples=5)
        group = groups[len(groups) // 2]
    _engine.check_group_bounds(kernel, group, list(kernel.accesses))
    blocks = [int(b) for b in group.block_linear]
    if len(blocks) > 1 and kernel.launch.threads_per_block % 32:
        raise NotImplementedError("multi-block L1 groups need whole warps per block")
    acc = np.zeros((len(kernel.accesses), 3), dtype=np.int64)
    for blk in blocks:
        acc += _native.l1_cycles(kernel, blk, machine.bank_width_bytes, machine.l1_banks)
    total = 0.0
    for a, row in zip(kernel.accesses, acc):
        total += a.multiplicity * float(row[0])
    per_access = tuple((float(r[1]) / 2.0) / float(r[2]) for r in acc)
    return L1CycleEstimate(cycles_per_lup=total / kernel.launch.lups_per_block, per_access=per_access)


def sample_block_stats(kernel: KernelDescriptor, machine: MachineDescriptor, samples: int = 5) -> BlockStats:
    res = _run_one(kernel, machine, None, phases=1, block_samples=samples)
    return _block_stats_from(res, 0, [f.name for f in kernel.fields])


def sample_wave_stats(kernel: KernelDescriptor, machine: MachineDescriptor, samples: int = 2,
                      override_blocks_per_wave: int | None = None) -> WaveStats:
    res = _run_one(kernel, machine, None, phases=2, wave_samples=samples, override=override_blocks_per_wave)
    return _wave_stats_from(res, 0, [f.name for f in kernel.fields])


# ---------------------------------------------------------------------------
# assembly


def _stats_row(F, names, lups_per_block, block_stats=None, wave_stats=None, cycles=0.0, l2l1=None):
    s = np.zeros(_native.stats_len(F), dtype=np.float64)
    if block_stats is not None:
        for k, d in enumerate((block_stats.load_comp, block_stats.load_up, block_stats.load_alloc,
                               block_stats.store_unique, block_stats.store_up)):
            for fi, n in enumerate(names):
                s[k * F + fi] = d.get(n, 0.0)
    if wave_stats is not None:
        for k, d in enumerate((wave_stats.load_unique, wave_stats.load_overlap, wave_stats.store_unique)):
            for fi, n in enumerate(names):
                s[(5 + k) * F + fi] = d.get(n, 0.0)
        s[8 * F + 0] = wave_stats.prev_unique_total
        s[8 * F + 1] = wave_stats.alloc_total
        s[8 * F + 2] = wave_stats.wave_lups
        s[8 * F + 3] = 1.0 if wave_stats.has_predecessor else 0.0
    s[8 * F + 4] = cycles
    s[8 * F + 5] = float(lups_per_block)
    if l2l1 is not None:
        ld, st = l2l1
        for fi, n in enumerate(names):
            s[8 * F + 6 + fi] = ld.per_field_down.get(n, 0.0)
            s[9 * F + 6 + fi] = st.per_field_down.get(n, 0.0)
        s[10 * F + 6] = 1.0
    return s


def _levels_from(rec: np.ndarray, fd: np.ndarray, names) -> VolumeBreakdown:
    c = {k: float(rec[i]) for i, k in enumerate(_native.RECORD_COLUMNS)}
    pf = lambda l: {n: float(fd[l, i]) for i, n in enumerate(names)}
    cov = c["dramLoadCoverage"]
    l2l1_load = LevelKindVolumes(c["l2l1LoadUp"], c["l2l1LoadComp"], c["l2l1LoadRed"], c["l2l1LoadCap"],
                                 c["l2l1LoadDown"], c["l2l1LoadAlloc"], c["l2l1LoadOversub"], pf(0))
    l2l1_store = LevelKindVolumes(c["l2l1StoreUp"], c["l2l1StoreComp"], c["l2l1StoreRed"], c["l2l1StoreCap"],
                                  c["l2l1StoreDown"], c["l2l1LoadAlloc"], c["l2l1LoadOversub"], pf(1))
    dram_load = LevelKindVolumes(c["dramLoadUp"], c["dramLoadComp"], c["dramLoadRed"], c["dramLoadCap"],
                                 c["dramLoadDown"], c["dramLoadAlloc"], c["dramLoadOversub"], pf(2),
                                 wave_unique=c["dramLoadUnique"], v_overlap=c["dramLoadOverlap"],
                                 overmiss_bytes=c["dramLoadOvermiss"],
                                 coverage=None if np.isnan(cov) else cov, v_red_l2=c["dramLoadRedL2"])
    dram_store = LevelKindVolumes(c["dramStoreUp"], c["dramStoreComp"], c["dramStoreRed"], c["dramStoreCap"],
                                  c["dramStoreDown"], c["dramLoadAlloc"], c["dramLoadOversub"], pf(3),
                                  wave_unique=c["dramStoreUnique"])
    return VolumeBreakdown(l2l1_load, l2l1_store, dram_load, dram_store)


def _assemble(kernel, machine, fit_params, block_stats, wave_stats, l2l1=None):
    names = [f.name for f in kernel.fields]
    F = len(names)
    ctx = _native.context()
    mid = ctx.machine_id(machine, fit_params)
    s = _stats_row(F, names, kernel.launch.lups_per_block, block_stats, wave_stats, 0.0, l2l1)
    rec, fd = _native.assemble(s[None, :], F, np.array([mid]), np.array([kernel.flops_per_lup]))
    return _levels_from(rec[0], fd[0], names)


def l2_to_l1_volume(kernel: KernelDescriptor, machine: MachineDescriptor,
                    fit_params: Mapping[str, GompertzParams] | None = None,
                    block_stats: BlockStats | None = None, samples: int = 5):
    stats = block_stats or sample_block_stats(kernel, machine, samples)
    v = _assemble(kernel, machine, fit_params, stats, None)
    return v.l2l1_load, v.l2l1_store


def dram_to_l2_volume(kernel: KernelDescriptor, machine: MachineDescriptor, l2l1_load: LevelKindVolumes,
                      l2l1_store: LevelKindVolumes, fit_params: Mapping[str, GompertzParams] | None = None,
                      wave_stats: WaveStats | None = None, samples: int = 2,
                      override_blocks_per_wave: int | None = None):
    stats = wave_stats or sample_wave_stats(kernel, machine, samples, override_blocks_per_wave)
    v = _assemble(kernel, machine, fit_params, None, stats, (l2l1_load, l2l1_store))
    return v.dram_load, v.dram_store


def estimate_volumes(kernel: KernelDescriptor, machine: MachineDescriptor,
                     fit_params: Mapping[str, GompertzParams] | None = None, *, block_samples: int = 5,
                     wave_samples: int = 2, override_blocks_per_wave: int | None = None,
                     block_stats: BlockStats | None = None, wave_stats: WaveStats | None = None
                     ) -> VolumeBreakdown:
    phases = (0 if block_stats else 1) | (0 if wave_stats else 2)
    names = [f.name for f in kernel.fields]
    if phases:
        res = _run_one(kernel, machine, fit_params, phases, block_samples, wave_samples,
                       override_blocks_per_wave)
        block_stats = block_stats or _block_stats_from(res, 0, names)
        wave_stats = wave_stats or _wave_stats_from(res, 0, names)
    return _assemble(kernel, machine, fit_params, block_stats, wave_stats)
