"""Configuration spaces of BASELINE.json and the
generators they need beyond the reference's own.

The reference ships the star stencil and D3Q15 generators
(reference kernels.py:193-244, 296-341).  The BASELINE workloads also name
multi-component field layouts (fzyx / zyxf), a D3Q27 hydrodynamics kernel and
folded LBM kernels; none is a reference concept, so they are written here on
the reference's own recipe (``global_coord`` / ``folded_coord`` /
``linear_address``, kernels.py:151-173) and reach the estimator as ordinary
descriptors — exactly what the reference evaluates for any raw kernel spec
(``kernel_to_dict`` round-trips them; tools/make_golden.py pins them against
the unmodified reference).

Layouts, for a field with ``F`` components on a (w, h, d) grid:
  * ``fzyx`` — component slowest: extents (w, h, d*F), component c at z + c*d
    (the reference's own pdf layout, kernels.py:316-330);
  * ``zyxf`` — component fastest: extents (w, h, d), strides (8F, 8Fw, 8Fwh),
    component c at +8c bytes.
With F == 1 both layouts give the same field and the same trees.

A ``Space`` holds a configuration space as arrays (template index, machine
index, block, grid, work per thread, flops, fold rank) so 10^6-config spaces
are built without one Python descriptor per configuration; templates are
shared by every launch shape of one access pattern (the trees use BX/BY/BZ).
"""

from __future__ import annotations

import dataclasses
from dataclasses import dataclass, field as dc_field
from typing import Sequence

import numpy as np

from .gvo.expr import IntConstant, fold
from .gvo.kernels import (
    Access,
    D3Q15_DIRECTIONS,
    FOLDINGS,
    PHI_STENCIL,
    Field,
    KernelDescriptor,
    KernelError,
    LaunchConfig,
    check_tiling,
    fold_factors,
    folded_coord,
    global_coord,
    linear_address,
    star_offsets,
)

LAYOUTS = ("fzyx", "zyxf")

# D3Q27: rest, 6 faces, 12 edges, 8 corners
D3Q27_DIRECTIONS = (
    ((0, 0, 0),)
    + ((1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1))
    + ((1, 1, 0), (-1, -1, 0), (1, -1, 0), (-1, 1, 0),
       (1, 0, 1), (-1, 0, -1), (1, 0, -1), (-1, 0, 1),
       (0, 1, 1), (0, -1, -1), (0, 1, -1), (0, -1, 1))
    + ((1, 1, 1), (-1, -1, -1), (1, 1, -1), (-1, -1, 1), (1, -1, 1), (-1, 1, -1), (-1, 1, 1), (1, -1, -1))
)
LBM_STENCILS = {"D3Q15": D3Q15_DIRECTIONS, "D3Q27": D3Q27_DIRECTIONS}
LBM_FLOPS = {"D3Q15": 250, "D3Q27": 450}
FOLD_RANK = {"2y": 0, "2z": 1, "none": 2}  # string order of perf.py:131


# ---------------------------------------------------------------------------
# fields with components


def component_field(name: str, grid: Sequence[int], components: int, layout: str, alignment: int = 0,
                    element_size: int = 8) -> Field:
    if layout not in LAYOUTS:
        raise KernelError(f"layout must be one of {LAYOUTS}, got {layout!r}")
    if components < 1:
        raise KernelError("components must be >= 1")
    w, h, d = (int(g) for g in grid)
    if layout == "fzyx" or components == 1:
        return Field(name, element_size, (w, h, d * components), alignment)
    e = element_size * components
    return Field(name, element_size, (w, h, d), alignment, (e, e * w, e * w * h))


def component_address(field: Field, coords, offsets: Sequence[int], comp: int, grid: Sequence[int],
                      layout: str):
    """Address of component ``comp`` at ``coords + offsets``."""
    ox, oy, oz = offsets
    if layout == "fzyx" or len(field.extents) == 3 and field.strides[0] == field.element_size:
        return linear_address(field, coords, (ox, oy, oz + comp * int(grid[2])))
    node = linear_address(field, coords, (ox, oy, oz))
    return fold("+", node, IntConstant(comp * field.element_size)) if comp else node


def _folded_coords(fy: int, fz: int, iy: int, iz: int):
    return (global_coord(0), folded_coord(1, fy, iy), folded_coord(2, fz, iz))


# ---------------------------------------------------------------------------
# generators


def generate_jacobi_2d5pt(grid: Sequence[int] = (256, 256), block_dim: Sequence[int] = (32, 4, 1), *,
                          element_size: int = 8) -> KernelDescriptor:
    """C1: 2D five-point Jacobi sweep (PR1 oracle config)."""
    w, h = (int(g) for g in grid)
    block_dim = tuple(int(b) for b in block_dim)
    grid_dim = check_tiling((w, h, 1), block_dim)
    src = Field("src", element_size, (w, h))
    dst = Field("dst", element_size, (w, h))
    coords = (global_coord(0), global_coord(1))
    acc = [Access("src", "load", linear_address(src, coords, o))
           for o in ((0, 0), (1, 0), (-1, 0), (0, 1), (0, -1))]
    acc.append(Access("dst", "store", linear_address(dst, coords, (0, 0))))
    return KernelDescriptor(fields=(src, dst), accesses=tuple(acc), launch=LaunchConfig(block_dim, grid_dim),
                            flops_per_lup=5, name="2d5pt")


def generate_star_stencil_fields(radius: int, grid: Sequence[int], block_dim: Sequence[int],
                                 folding: str = "none", *, layout: str = "fzyx", components: int = 1,
                                 alignment: int = 0) -> KernelDescriptor:
    """3D star stencil on ``components``-component fields (C3): per folded
    iteration every component reads the 6r+1 star and writes the centre.
    With components == 1 and alignment 0 this is the reference's
    generate_star_stencil (kernels.py:193-244) access for access."""
    if radius < 1:
        raise KernelError("stencil range must be >= 1")
    grid = tuple(int(g) for g in grid)
    block_dim = tuple(int(b) for b in block_dim)
    if len(grid) != 3 or len(block_dim) != 3:
        raise KernelError("grid and block must be 3D")
    fx, fy, fz = fold_factors(folding)
    grid_dim = check_tiling(grid, (block_dim[0] * fx, block_dim[1] * fy, block_dim[2] * fz))
    src = component_field("src", grid, components, layout, alignment)
    dst = component_field("dst", grid, components, layout, alignment)
    offs = star_offsets(radius)
    acc = []
    for iy in range(fy):
        for iz in range(fz):
            coords = _folded_coords(fy, fz, iy, iz)
            for c in range(components):
                acc.extend(Access("src", "load", component_address(src, coords, o, c, grid, layout)) for o in offs)
                acc.append(Access("dst", "store", component_address(dst, coords, (0, 0, 0), c, grid, layout)))
    name = f"star{radius}" if components == 1 else f"star{radius}_{layout}_c{components}"
    return KernelDescriptor(fields=(src, dst), accesses=tuple(acc),
                            launch=LaunchConfig(block_dim, grid_dim, work_per_thread=fx * fy * fz),
                            flops_per_lup=(6 * radius + 1) * components, name=name)


def generate_lbm(stencil: str, grid: Sequence[int], block_dim: Sequence[int], folding: str = "none", *,
                 layout: str = "fzyx", alignment: int = 0, flops_per_lup: int | None = None) -> KernelDescriptor:
    """Two-phase LBM kernels (C4): pull streaming of a DdQq pdf field
    (q loads from the upstream neighbours, q aligned stores) plus the
    7-point phase-field read, per folded iteration.  D3Q15/fzyx/none/0 is the
    reference's generate_lbm_d3q15 (kernels.py:296-341) access for access;
    D3Q27 is the hydrodynamics kernel on the same recipe."""
    if stencil not in LBM_STENCILS:
        raise KernelError(f"stencil must be one of {tuple(LBM_STENCILS)}, got {stencil!r}")
    dirs = LBM_STENCILS[stencil]
    grid = tuple(int(g) for g in grid)
    block_dim = tuple(int(b) for b in block_dim)
    if len(grid) != 3 or len(block_dim) != 3:
        raise KernelError("grid and block must be 3D")
    fx, fy, fz = fold_factors(folding)
    grid_dim = check_tiling(grid, (block_dim[0] * fx, block_dim[1] * fy, block_dim[2] * fz))
    q = len(dirs)
    pdf_src = component_field("pdf_src", grid, q, layout, alignment)
    pdf_dst = component_field("pdf_dst", grid, q, layout, alignment)
    phi = component_field("phi", grid, 1, layout, alignment)
    acc = []
    for iy in range(fy):
        for iz in range(fz):
            coords = _folded_coords(fy, fz, iy, iz)
            acc += [Access("pdf_src", "load", component_address(pdf_src, coords, (-cx, -cy, -cz), i, grid, layout))
                    for i, (cx, cy, cz) in enumerate(dirs)]
            acc += [Access("pdf_dst", "store", component_address(pdf_dst, coords, (0, 0, 0), i, grid, layout))
                    for i in range(q)]
            acc += [Access("phi", "load", component_address(phi, coords, o, 0, grid, layout)) for o in PHI_STENCIL]
    flops = LBM_FLOPS[stencil] if flops_per_lup is None else flops_per_lup
    name = f"lbm_{stencil.lower()}" + ("" if (layout, folding) == ("fzyx", "none") else f"_{layout}_{folding}")
    return KernelDescriptor(fields=(pdf_src, pdf_dst, phi), accesses=tuple(acc),
                            launch=LaunchConfig(block_dim, grid_dim, work_per_thread=fx * fy * fz),
                            flops_per_lup=flops, name=name)


# ---------------------------------------------------------------------------
# configuration spaces


@dataclass(frozen=True)
class TemplateSpec:
    """One access pattern (shared by every launch shape)."""

    kind: str  # "star" | "lbm" | "jacobi2d"
    grid: tuple[int, int, int]
    folding: str = "none"
    layout: str = "fzyx"
    components: int = 1
    alignment: int = 0
    radius: int = 4
    stencil: str = ""

    def build(self, block_dim) -> KernelDescriptor:
        if self.kind == "star":
            return generate_star_stencil_fields(self.radius, self.grid, block_dim, self.folding, layout=self.layout,
                                                components=self.components, alignment=self.alignment)
        if self.kind == "lbm":
            return generate_lbm(self.stencil, self.grid, block_dim, self.folding, layout=self.layout,
                                alignment=self.alignment)
        if self.kind == "jacobi2d":
            return generate_jacobi_2d5pt(self.grid[:2], block_dim)
        raise KernelError(f"unknown template kind {self.kind!r}")

    def n_accesses(self) -> int:
        """Accesses of the generated kernel, without building its trees."""
        _, fy, fz = fold_factors(self.folding)
        if self.kind == "star":
            return fy * fz * self.components * (6 * self.radius + 2)
        if self.kind == "lbm":
            return fy * fz * (2 * len(LBM_STENCILS[self.stencil]) + len(PHI_STENCIL))
        if self.kind == "jacobi2d":
            return 6
        raise KernelError(f"unknown template kind {self.kind!r}")

    @property
    def label(self) -> str:
        if self.kind == "star":
            return f"star{self.radius}/{self.layout}/c{self.components}/a{self.alignment}/{self.folding}"
        if self.kind == "lbm":
            return f"{self.stencil}/{self.layout}/a{self.alignment}/{self.folding}"
        return self.kind


@dataclass
class Space:
    """A configuration space as arrays; ``templates[i]`` / ``machines[j]``
    are referenced by ``tpl`` / ``mach``."""

    name: str
    templates: list[TemplateSpec]
    machines: list
    tpl: np.ndarray
    mach: np.ndarray
    block: np.ndarray  # [n][3] int32
    grid_dim: np.ndarray  # [n][3] int64
    wpt: np.ndarray
    flops: np.ndarray
    fold_rank: np.ndarray
    _kernels: dict = dc_field(default_factory=dict, repr=False)

    def __len__(self) -> int:
        return int(len(self.tpl))

    def template_kernel(self, t: int) -> KernelDescriptor:
        """Descriptor of template t (at its first valid launch shape)."""
        if t not in self._kernels:
            i = int(np.flatnonzero(self.tpl == t)[0])
            self._kernels[t] = self.templates[t].build(tuple(int(v) for v in self.block[i]))
        return self._kernels[t]

    def kernel(self, i: int) -> KernelDescriptor:
        """Full descriptor of configuration i (for the reference / oracle)."""
        return self.templates[int(self.tpl[i])].build(tuple(int(v) for v in self.block[i]))

    def machine(self, i: int):
        return self.machines[int(self.mach[i])]

    def key(self, i: int) -> str:
        b = self.block[i]
        return f"{self.templates[int(self.tpl[i])].label}/{b[0]}x{b[1]}x{b[2]}/m{int(self.mach[i])}"

    def subset(self, idx) -> "Space":
        idx = np.asarray(idx, dtype=np.int64)
        return Space(self.name, self.templates, self.machines, self.tpl[idx], self.mach[idx], self.block[idx],
                     self.grid_dim[idx], self.wpt[idx], self.flops[idx], self.fold_rank[idx], self._kernels)

    def config_array(self, ctx) -> np.ndarray:
        """gvo_config records; registers templates and machines with ctx."""
        from . import _native

        tid = np.zeros(len(self.templates), dtype=np.int32)
        for t in np.unique(self.tpl):
            k = self.template_kernel(int(t))
            tid[t] = ctx.template_id(k.fields, k.accesses)
        mid = np.array([ctx.machine_id(m) for m in self.machines], dtype=np.int32)
        a = np.zeros(len(self), dtype=_native.CONFIG_DTYPE)
        a["template_id"] = tid[self.tpl]
        a["machine_id"] = mid[self.mach]
        a["block"] = self.block
        a["fold_rank"] = self.fold_rank
        a["grid"] = self.grid_dim
        a["work_per_thread"] = self.wpt
        a["flops_per_lup"] = self.flops
        return a

    def n_accesses(self) -> np.ndarray:
        per_t = np.array([t.n_accesses() for t in self.templates], dtype=np.int64)
        return per_t[self.tpl]

    def kind_weight(self) -> np.ndarray:
        """Per-configuration device cost weight of its template kind (shard.KIND_WEIGHT)."""
        from .shard import KIND_WEIGHT

        per_t = np.array([KIND_WEIGHT.get(t.kind, 1.0) for t in self.templates])
        return per_t[self.tpl]

    def sharing_groups(self, sector_bytes: int = 32) -> np.ndarray:
        """Group id per configuration: equal ids share their wave sets on the
        device (csrc/k_dedup.cu: same accesses up to the field base, base
        residue modulo the sector, launch and machine integer parameters)."""
        tkey = {}
        tcls = np.zeros(len(self.templates), dtype=np.int64)
        for t, spec in enumerate(self.templates):
            k = dataclasses.replace(spec, alignment=spec.alignment % sector_bytes)
            tcls[t] = tkey.setdefault(k, len(tkey))
        mkey = {}
        mcls = np.zeros(len(self.machines), dtype=np.int64)
        for j, m in enumerate(self.machines):
            k = (m.sm_count, m.l1_line_bytes, m.sector_bytes, m.l1_banks, m.bank_width_bytes,
                 m.max_threads_per_sm, m.max_blocks_per_sm, m.max_threads_per_block)
            mcls[j] = mkey.setdefault(k, len(mkey))
        b = self.block.astype(np.int64)
        if len(tkey) < (1 << 20) and len(mkey) < (1 << 10) and (b < (1 << 11)).all() and (b >= 0).all():
            key = ((tcls[self.tpl] << 10 | mcls[self.mach]) << 33) | (b[:, 0] << 22) | (b[:, 1] << 11) | b[:, 2]
            _, gid = np.unique(key, return_inverse=True)
        else:
            key = np.stack([tcls[self.tpl], mcls[self.mach], b[:, 0], b[:, 1], b[:, 2]], axis=1)
            _, gid = np.unique(key, axis=0, return_inverse=True)
        return gid.reshape(-1)


def pow2_shapes(threads: Sequence[int], x_max=512, y_max=512, z_max=64) -> np.ndarray:
    """Power-of-two (X, Y, Z), X*Y*Z in ``threads`` (reference kernels.py:367-395 order per count)."""
    out = []
    for t in threads:
        x = 1
        while x <= x_max:
            y = 1
            while y <= y_max:
                if t % (x * y) == 0 and t // (x * y) <= z_max:
                    out.append((x, y, t // (x * y)))
                y <<= 1
            x <<= 1
    return np.array(sorted(set(out), key=lambda s: (s[0] * s[1] * s[2], s)), dtype=np.int32).reshape(-1, 3)


def _tile(grid, shapes: np.ndarray, folding: str):
    fx, fy, fz = fold_factors(folding)
    eff = shapes.astype(np.int64) * np.array([fx, fy, fz], dtype=np.int64)
    g = np.array(grid, dtype=np.int64)
    ok = (g[None, :] % eff == 0).all(axis=1)
    return ok, g[None, :] // eff, fx * fy * fz


class _Builder:
    def __init__(self, name, machines):
        self.name = name
        self.machines = list(machines)
        self.templates: list[TemplateSpec] = []
        self.cols = {k: [] for k in ("tpl", "mach", "block", "grid", "wpt", "flops", "fold")}

    def add(self, spec: TemplateSpec, shapes: np.ndarray, flops: int, machines: Sequence[int] = (0,)):
        ok, gd, wpt = _tile(spec.grid, shapes, spec.folding)
        if not ok.any():
            return
        t = len(self.templates)
        self.templates.append(spec)
        n = int(ok.sum())
        for m in machines:
            c = self.cols
            c["tpl"].append(np.full(n, t, np.int32))
            c["mach"].append(np.full(n, m, np.int32))
            c["block"].append(shapes[ok])
            c["grid"].append(gd[ok])
            c["wpt"].append(np.full(n, wpt, np.int32))
            c["flops"].append(np.full(n, flops, np.int64))
            c["fold"].append(np.full(n, FOLD_RANK[spec.folding], np.int32))

    def done(self) -> Space:
        c = self.cols
        cat = lambda k, dt, shp=(-1,): (np.concatenate(c[k]).astype(dt).reshape(shp) if c[k]
                                         else np.zeros((0,) + shp[1:], dt))
        return Space(self.name, self.templates, self.machines, cat("tpl", np.int32), cat("mach", np.int32),
                     cat("block", np.int32, (-1, 3)), cat("grid", np.int64, (-1, 3)), cat("wpt", np.int32),
                     cat("flops", np.int64), cat("fold", np.int32))


def l2_variants(machine, fractions=(1, 2, 4)):
    """{full, 1/2, 1/4} L2 capacity (the knob of reference test_acceptance.py:284-306)."""
    return [machine if f == 1 else dataclasses.replace(machine, name=f"{machine.name}-l2/{f}",
                                                       l2_capacity_bytes=machine.l2_capacity_bytes // f)
            for f in fractions]


STENCIL_THREADS = tuple(1 << i for i in range(11))  # 1..1024
LBM_THREADS = (64, 128, 256, 512)


def space_c1(machine) -> Space:
    b = _Builder("C1", [machine])
    b.add(TemplateSpec("jacobi2d", (256, 256, 1)), np.array([[32, 4, 1]], np.int32), 5)
    return b.done()


def space_c2(machine, grid=(640, 640, 640), radius=4, alignment=0) -> Space:
    b = _Builder("C2", [machine])
    b.add(TemplateSpec("star", tuple(grid), "none", radius=radius, alignment=alignment),
          pow2_shapes(STENCIL_THREADS), 6 * radius + 1)
    return b.done()


def space_c3(machine, grid=(640, 640, 640), radii=(2, 4), components=(2, 4), alignments=tuple(range(0, 128, 8)),
             layouts=LAYOUTS, foldings=FOLDINGS, name="C3", machines_idx=(0,), machines=None) -> Space:
    b = _Builder(name, machines or [machine])
    shapes = pow2_shapes(STENCIL_THREADS)
    for r in radii:
        for fc in components:
            for lay in layouts:
                for al in alignments:
                    for fo in foldings:
                        b.add(TemplateSpec("star", tuple(grid), fo, lay, fc, al, r), shapes, (6 * r + 1) * fc,
                              machines_idx)
    return b.done()


def space_c4(machine, grid=(256, 256, 256), stencils=("D3Q15", "D3Q27"), layouts=LAYOUTS, foldings=FOLDINGS,
             alignments=(0,), name="C4", machines_idx=(0,), machines=None) -> Space:
    b = _Builder(name, machines or [machine])
    shapes = pow2_shapes(LBM_THREADS)
    for st in stencils:
        for lay in layouts:
            for al in alignments:
                for fo in foldings:
                    b.add(TemplateSpec("lbm", tuple(grid), fo, lay, 1, al, stencil=st), shapes, LBM_FLOPS[st],
                          machines_idx)
    return b.done()


def space_c5(machine) -> Space:
    """C3 (radius 1-4, alignments 0..248) and C4 (alignments 0..120), each
    at {full, 1/2, 1/4} L2 capacity: ~1.2e6 configurations."""
    ms = l2_variants(machine)
    s3 = space_c3(machine, radii=(1, 2, 3, 4), alignments=tuple(range(0, 256, 8)), machines=ms,
                  machines_idx=(0, 1, 2))
    s4 = space_c4(machine, alignments=tuple(range(0, 128, 8)), machines=ms, machines_idx=(0, 1, 2))
    return concat("C5", [s3, s4])


def concat(name: str, spaces: Sequence[Space]) -> Space:
    """Concatenate spaces that share one machine list."""
    templates, cols = [], {k: [] for k in ("tpl", "mach", "block", "grid_dim", "wpt", "flops", "fold_rank")}
    for s in spaces:
        off = len(templates)
        templates += s.templates
        cols["tpl"].append(s.tpl + off)
        for k in ("mach", "block", "grid_dim", "wpt", "flops", "fold_rank"):
            cols[k].append(getattr(s, k))
    c = {k: np.concatenate(v) for k, v in cols.items()}
    return Space(name, templates, spaces[0].machines, c["tpl"].astype(np.int32), c["mach"], c["block"],
                 c["grid_dim"], c["wpt"], c["flops"], c["fold_rank"])


def space(name: str, machine=None) -> Space:
    from .gvo.machine import b200_preset

    m = machine or b200_preset()
    return {"C1": space_c1, "C2": space_c2, "C3": space_c3, "C4": space_c4, "C5": space_c5}[name](m)


# ---------------------------------------------------------------------------
# batched evaluation of a space (device pipeline; no CPU path)


def evaluate_space(sp: Space, *, block_samples: int = 5, wave_samples: int = 2, override: int | None = None,
                   want_l1: bool = False):
    """Evaluate every configuration of ``sp`` on the device and rank them
    (perf.py:131 key).  Returns (engine Result, ranking order).  The first
    failing configuration raises the reference's exception."""
    from . import _native
    from .gvo import _engine

    ctx = _native.context()
    cfgs = sp.config_array(ctx)
    out = ctx.eval_configs_host(cfgs, block_samples, wave_samples, override or 0, want_l1_access=want_l1)
    res = _engine.Result(out["F"], out["S"], out["W"], out["counts"], out["stats"], out["records"],
                         out["field_down"], out["l1_access"])
    bad = np.flatnonzero(res.counts[:, _native.C_STATUS])
    if len(bad):
        i = int(bad[0])
        _engine.raise_for_status(res, i, sp.kernel(i), sp.machine(i), block_samples, wave_samples, override)
    return res, _native.rank_host(cfgs, res.records)


def prediction(sp: Space, res, i: int):
    """PerfPrediction of configuration i from an evaluate_space result."""
    from .gvo import perf

    k = sp.template_kernel(int(sp.tpl[i]))
    per = perf._per_access(res, i, len(k.accesses)) if res.l1_access is not None else ()
    return perf._prediction(res, i, [f.name for f in k.fields], int(sp.flops[i]), per)


def space_from_entries(entries, machines) -> Space:
    """Space of explicit (template, machine index, block) entries (golden files)."""
    b = _Builder("entries", machines)
    idx = {}
    for e in entries:
        t = e["template"]
        spec = TemplateSpec(t["kind"], tuple(t["grid"]), t["folding"], t["layout"], t["components"], t["alignment"],
                            t["radius"], t["stencil"])
        if spec not in idx:
            idx[spec] = len(b.templates)
            b.templates.append(spec)
        ti = idx[spec]
        shape = np.array([e["block"]], np.int32)
        ok, gd, wpt = _tile(spec.grid, shape, spec.folding)
        if not ok[0]:
            raise KernelError(f"entry {e} does not tile its grid")
        k = spec.build(tuple(e["block"]))
        c = b.cols
        c["tpl"].append(np.array([ti], np.int32))
        c["mach"].append(np.array([e["machine"]], np.int32))
        c["block"].append(shape)
        c["grid"].append(gd)
        c["wpt"].append(np.array([wpt], np.int32))
        c["flops"].append(np.array([k.flops_per_lup], np.int64))
        c["fold"].append(np.array([FOLD_RANK[spec.folding]], np.int32))
    return b.done()
