"""Collaborative groups and unique-footprint enumeration (drop-in for
reference ``gvo.footprint``, footprint.py:1-637).

Group geometry (waves, representative blocks) is integer bookkeeping kept on
the host for the single-call API; the batched path computes it on the
device (csrc/k_setup.cu).  Every footprint count — unique granules per
(field, kind), per-warp coalesced requests, wave unions and overlaps — is
computed by the sm_100a engine through the C ABI.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable, Iterator

import numpy as np

from .. import _native
from . import _engine
from .expr import ThreadCoord
from .kernels import KernelDescriptor, LaunchConfig
from .machine import MachineDescriptor, WARP_SIZE


class FootprintError(ValueError):
    pass


@dataclass(frozen=True)
class Wave:
    index: int
    start: int
    count: int

    @property
    def block_linear(self) -> np.ndarray:
        return np.arange(self.start, self.start + self.count, dtype=np.int64)


def blocks_per_wave(launch: LaunchConfig, machine: MachineDescriptor) -> int:
    """Co-resident blocks of one wave (reference footprint.py:48-57)."""
    t = launch.threads_per_block
    if t > machine.max_threads_per_block:
        raise FootprintError(f"block of {t} threads exceeds machine limit {machine.max_threads_per_block}")
    per_sm = min(machine.max_blocks_per_sm, machine.max_threads_per_sm // t)
    if per_sm < 1:
        raise FootprintError(f"block of {t} threads exceeds per-SM thread capacity")
    return machine.sm_count * per_sm


def build_waves(launch: LaunchConfig, machine: MachineDescriptor,
                override_blocks_per_wave: int | None = None) -> list[Wave]:
    per = override_blocks_per_wave or blocks_per_wave(launch, machine)
    if per < 1:
        raise FootprintError("blocks per wave must be >= 1")
    total = launch.total_blocks
    return [Wave(i, s, min(per, total - s)) for i, s in enumerate(range(0, total, per))]


@dataclass(frozen=True)
class CollaborativeGroup:
    launch: LaunchConfig
    block_linear: np.ndarray
    level: str

    def __post_init__(self):
        if self.block_linear.size == 0:
            raise FootprintError("collaborative group needs at least one block")
        if self.level == "L1" and self.block_linear.size != 1:
            raise FootprintError("an L1 group is exactly one thread block")

    @property
    def block_count(self) -> int:
        return int(self.block_linear.size)

    @property
    def thread_count(self) -> int:
        return self.block_count * self.launch.threads_per_block

    @property
    def lups(self) -> int:
        return self.block_count * self.launch.lups_per_block

    def block_coords(self):
        gx, gy, _ = self.launch.grid_dim
        lin = self.block_linear
        return lin % gx, (lin // gx) % gy, lin // (gx * gy)

    def thread_coords(self) -> Iterator[ThreadCoord]:
        bx, by, bz = self.launch.block_dim
        xs, ys, zs = self.block_coords()
        for b in zip(xs.tolist(), ys.tolist(), zs.tolist()):
            for t in range(bx * by * bz):
                yield ThreadCoord(t % bx, (t // bx) % by, t // (bx * by), *b)


def block_group(launch: LaunchConfig, linear_index: int) -> CollaborativeGroup:
    if not 0 <= linear_index < launch.total_blocks:
        raise FootprintError(f"block index {linear_index} outside grid")
    return CollaborativeGroup(launch, np.array([linear_index], dtype=np.int64), "L1")


def wave_group(launch: LaunchConfig, wave: Wave) -> CollaborativeGroup:
    return CollaborativeGroup(launch, wave.block_linear, "L2")


# ---------------------------------------------------------------------------
# results


@dataclass(frozen=True)
class KindCounts:
    unique_count: int
    total_count: int


@dataclass(frozen=True)
class FootprintResult:
    granularity: int
    per_field: dict

    def _pick(self, field, kind):
        return [c for (f, k), c in self.per_field.items()
                if (field is None or f == field) and (kind is None or k == kind)]

    def unique_bytes(self, field=None, kind=None) -> int:
        return sum(c.unique_count for c in self._pick(field, kind)) * self.granularity

    def total_bytes(self, field=None, kind=None) -> int:
        return sum(c.total_count for c in self._pick(field, kind)) * self.granularity

    def unique_count(self, field=None, kind=None) -> int:
        return sum(c.unique_count for c in self._pick(field, kind))

    def total_count(self, field=None, kind=None) -> int:
        return sum(c.total_count for c in self._pick(field, kind))


def _check_kinds(granularity: int, kinds) -> tuple[str, ...]:
    if granularity < 1:
        raise FootprintError(f"granularity must be positive, got {granularity}")
    kinds = ("load", "store") if kinds is None else tuple(kinds)
    bad = set(kinds) - {"load", "store"}
    if bad:
        raise FootprintError(f"unknown access kinds: {sorted(bad)}")
    return kinds


def grid_iteration(kernel: KernelDescriptor, group: CollaborativeGroup, granularity: int,
                   kinds: Iterable[str] | None = None) -> FootprintResult:
    """Unique and per-warp-request granule counts per (field, kind)
    (reference footprint.py:441-471), computed by the device engine."""
    kinds = _check_kinds(granularity, kinds)
    for f in kernel.fields:
        for kind in kinds:
            _engine.check_group_bounds(kernel, group, [a for a in kernel.accesses
                                                       if a.field == f.name and a.kind == kind])
    out = _native.group_footprint(kernel, _engine.runs_of(group.block_linear), granularity)
    per_field = {}
    for fi, f in enumerate(kernel.fields):
        for kind in kinds:
            if any(a.field == f.name and a.kind == kind for a in kernel.accesses):
                k = 0 if kind == "load" else 1
                per_field[(f.name, kind)] = KindCounts(int(out[fi, k, 0]), int(out[fi, k, 1]))
    return FootprintResult(granularity, per_field)


def naive_footprint_oracle(kernel: KernelDescriptor, group: CollaborativeGroup, granularity: int,
                           kinds: Iterable[str] | None = None) -> FootprintResult:
    """Brute-force twin of grid_iteration (reference footprint.py:474-507):
    every thread's address evaluated by the device bytecode interpreter
    (gvo_eval_addresses), granules deduplicated per field/kind and per
    (block, warp) on the device.  Independent of the interval engine, so the
    two cross-check each other exactly as in the reference's tests."""
    import torch

    kinds = _check_kinds(granularity, kinds)
    bx, by, bz = kernel.launch.block_dim
    s = bx * by * bz
    xs, ys, zs = group.block_coords()
    t = np.arange(s, dtype=np.int64)
    nb = len(xs)
    coords = np.empty((nb * s, 6), dtype=np.int64)
    coords[:, 0] = np.tile(t % bx, nb)
    coords[:, 1] = np.tile((t // bx) % by, nb)
    coords[:, 2] = np.tile(t // (bx * by), nb)
    coords[:, 3] = np.repeat(np.asarray(xs, dtype=np.int64), s)
    coords[:, 4] = np.repeat(np.asarray(ys, dtype=np.int64), s)
    coords[:, 5] = np.repeat(np.asarray(zs, dtype=np.int64), s)
    dev = torch.device("cuda", _native.context().device)
    idx = torch.arange(nb * s, dtype=torch.int64, device=dev)
    warp_key = (idx // s) * ((s + 31) // 32) + (idx % s) // 32
    bases = kernel.base_substitution
    per_field = {}
    for f in kernel.fields:
        for kind in kinds:
            accesses = [a for a in kernel.accesses if a.field == f.name and a.kind == kind]
            if not accesses:
                continue
            allg, total = [], 0
            for a in accesses:
                addr = torch.from_numpy(_native.eval_addresses(a.expr, bases, kernel.launch.block_dim, coords)).to(dev)
                gran = torch.div(addr, granularity, rounding_mode="floor")
                allg.append(gran)
                pairs = torch.stack([warp_key, gran], dim=1)
                total += a.multiplicity * int(torch.unique(pairs, dim=0).shape[0])
            per_field[(f.name, kind)] = KindCounts(int(torch.unique(torch.cat(allg)).numel()), total)
    return FootprintResult(granularity, per_field)


# ---------------------------------------------------------------------------
# waves


class WaveSet:
    """Unique-granule set of one field's loads in one wave.  Holds its count;
    intersections with another wave's set are computed on the device."""

    __slots__ = ("kernel", "wave", "field", "granularity", "count")

    def __init__(self, kernel, wave, field, granularity, count):
        self.kernel, self.wave, self.field, self.granularity, self.count = kernel, wave, field, granularity, count

    def intersection_count(self, other: "WaveSet") -> int:
        if self.count == 0 or other.count == 0:
            return 0
        out = _native.group_sets(self.kernel, [(other.wave.start, other.wave.count),
                                               (self.wave.start, self.wave.count)], self.granularity)
        fi = [f.name for f in self.kernel.fields].index(self.field)
        return int(out[1, fi, 3])

    def union_count(self, other: "WaveSet") -> int:
        return self.count + other.count - self.intersection_count(other)


@dataclass(frozen=True)
class WaveFootprint:
    load_sets: dict
    store_counts: dict
    alloc_count: int
    lups: int
    granularity: int

    def load_unique_bytes(self, field: str | None = None) -> int:
        if field is not None:
            return self.load_sets[field].count * self.granularity
        return sum(s.count for s in self.load_sets.values()) * self.granularity

    def store_unique_bytes(self, field: str | None = None) -> int:
        if field is not None:
            return self.store_counts[field] * self.granularity
        return sum(self.store_counts.values()) * self.granularity


def _wave_guard(kernel, wave):
    grp = wave_group(kernel.launch, wave)
    for f in kernel.fields:
        for kind in ("load", "store"):
            _engine.check_group_bounds(kernel, grp, [a for a in kernel.accesses
                                                     if a.field == f.name and a.kind == kind])


def wave_footprint(kernel: KernelDescriptor, wave: Wave, granularity: int) -> WaveFootprint:
    """Per-field unique loads/stores and Σ|L∪S| of one wave (footprint.py:535-555)."""
    if granularity < 1:
        raise FootprintError(f"granularity must be positive, got {granularity}")
    _wave_guard(kernel, wave)
    out = _native.group_sets(kernel, [(wave.start, wave.count)], granularity)[0]
    load_sets, store_counts, alloc = {}, {}, 0
    for fi, f in enumerate(kernel.fields):
        load_sets[f.name] = WaveSet(kernel, wave, f.name, granularity, int(out[fi, 0]))
        store_counts[f.name] = int(out[fi, 1])
        alloc += int(out[fi, 2])
    return WaveFootprint(load_sets, store_counts, alloc, wave.count * kernel.launch.lups_per_block, granularity)


def wave_overlap(kernel: KernelDescriptor, wave_curr: Wave, wave_prev: Wave, granularity: int) -> int:
    """Σ_f |L_curr ∩ L_prev| in bytes (footprint.py:567-577)."""
    if granularity < 1:
        raise FootprintError(f"granularity must be positive, got {granularity}")
    _wave_guard(kernel, wave_curr)
    _wave_guard(kernel, wave_prev)
    out = _native.group_sets(kernel, [(wave_prev.start, wave_prev.count),
                                      (wave_curr.start, wave_curr.count)], granularity)
    return int(out[1, :, 3].sum()) * granularity


def overlap_bytes(curr: WaveFootprint, prev: WaveFootprint) -> int:
    return sum(s.intersection_count(prev.load_sets[n]) for n, s in curr.load_sets.items()) * curr.granularity


# ---------------------------------------------------------------------------
# representative groups (closed forms of footprint.py:591-637)


def _interior(extent: int) -> tuple[int, int]:
    return (1, extent - 2) if extent > 2 else (0, extent)


def spread_indices(n: int, samples: int) -> list[int]:
    """np.unique(np.round(np.linspace(0, n-1, samples))) without the meshgrid."""
    if n <= samples:
        return list(range(n))
    if samples == 1:
        return [0]
    step = (n - 1) / (samples - 1)
    picks = [int(np.rint(i * step)) for i in range(samples - 1)] + [n - 1]
    return sorted(set(picks))


def representative_blocks(kernel: KernelDescriptor, samples: int = 5) -> list[CollaborativeGroup]:
    if samples < 1:
        raise FootprintError("sample count must be >= 1")
    launch = kernel.launch
    gx, gy, gz = launch.grid_dim
    (ox, nx), (oy, ny), (oz, nz) = _interior(gx), _interior(gy), _interior(gz)
    out = []
    for k in spread_indices(nx * ny * nz, samples):
        x, y, z = k % nx, (k // nx) % ny, k // (nx * ny)
        out.append(block_group(launch, (x + ox) + gx * ((y + oy) + gy * (z + oz))))
    return out


def representative_wave_pairs(kernel: KernelDescriptor, machine: MachineDescriptor, samples: int = 2,
                              override_blocks_per_wave: int | None = None):
    if samples < 1:
        raise FootprintError("sample count must be >= 1")
    waves = build_waves(kernel.launch, machine, override_blocks_per_wave)
    if len(waves) == 1:
        return [(None, waves[0])]
    hi = len(waves) - 2 if len(waves) >= 3 else len(waves) - 1
    lo = 1
    count = min(samples, hi - lo + 1)
    start = min(max(lo, (lo + hi) // 2 - (count - 1) // 2), hi - count + 1)
    return [(waves[i - 1], waves[i]) for i in range(start, start + count)]
