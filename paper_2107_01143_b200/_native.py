"""ctypes binding of libgvo_b200.so (the C ABI in include/gvo_b200.h).

The library is the only compute path: there is no CPU fallback.  If the
shared object is missing or no CUDA device is visible, every entry point
raises ``NativeUnavailable``.
"""

from __future__ import annotations

import atexit
import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
# GVO_LIB_VARIANT=<name> loads a variant build (libgvo_b200_<name>.so: the
# phase-counter build "prof" or an A/B experiment); default: the product
_VARIANT = os.environ.get("GVO_LIB_VARIANT", "")
LIB_PATH = _HERE / (f"libgvo_b200_{_VARIANT}.so" if _VARIANT else "libgvo_b200.so")

ABI_VERSION = 4  # include/gvo_b200.h GVO_ABI_VERSION
GVO_MAX_FIELDS = 16
GVO_MAX_ACCESSES = 1024
GVO_MAX_BLOCK_SAMPLES = 32
GVO_MAX_UNIQUE_WAVES = 16
C_HDR = 16
C_STATUS, C_ERR_PHASE, C_ERR_GROUP, C_ERR_ACCESS = 0, 1, 2, 3
C_NSAMPLES, C_NUWAVES, C_NPAIRS, C_HASPRED = 4, 5, 6, 7
C_PERWAVE, C_NWAVES, C_L1BLOCK, C_L1CYCLES, C_FIRSTWAVE, C_FIRSTBLOCK = 8, 9, 10, 11, 12, 13

STATUS_CAPACITY = 7
STATUS = {0: "OK", 1: "EXPR", 2: "ADDRESS_OVERFLOW", 3: "KERNEL", 4: "FOOTPRINT", 5: "MACHINE",
          6: "PERF", 7: "CAPACITY", 8: "UNSUPPORTED", 15: "INVALID", 16: "CUDA", 17: "NCCL"}

RECORD_COLUMNS = (
    "l1CyclesPerLup",
    "l2l1LoadComp", "l2l1LoadRed", "l2l1LoadCap", "l2l1LoadUp", "l2l1LoadDown", "l2l1LoadAlloc",
    "l2l1LoadOversub",
    "l2l1StoreComp", "l2l1StoreRed", "l2l1StoreCap", "l2l1StoreUp", "l2l1StoreDown",
    "dramLoadComp", "dramLoadRed", "dramLoadCap", "dramLoadUp", "dramLoadDown", "dramLoadAlloc",
    "dramLoadOversub", "dramLoadUnique", "dramLoadOverlap", "dramLoadOvermiss", "dramLoadCoverage",
    "dramLoadRedL2",
    "dramStoreComp", "dramStoreRed", "dramStoreCap", "dramStoreUp", "dramStoreDown", "dramStoreUnique",
    "tDram", "tL2", "tL1", "tFp", "limiter", "predictedGLups",
)
RECORD_LEN = len(RECORD_COLUMNS)
LIMITERS = ("dram", "l2", "l1", "fp")


def stats_len(F: int) -> int:
    return 10 * F + 7


def counts_stride(F: int, S: int, W: int) -> int:
    return C_HDR + S * F * 5 + (W + 1) * F * 4 + (W + 1)


def effective_sampling(block_samples: int, wave_samples: int) -> tuple[int, int]:
    S = min(max(int(block_samples), 1), GVO_MAX_BLOCK_SAMPLES)
    W = min(max(int(wave_samples), 1), GVO_MAX_UNIQUE_WAVES - 1)
    return S, W


class NativeUnavailable(RuntimeError):
    pass


class EngineError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"gvo_b200 status {STATUS.get(status, status)}: {message}")
        self.status = status


class Machine(C.Structure):
    _fields_ = [
        ("sm_count", C.c_int64), ("clock_ghz", C.c_double), ("l1_capacity_bytes", C.c_int64),
        ("l2_capacity_bytes", C.c_int64), ("l1_line_bytes", C.c_int64), ("sector_bytes", C.c_int64),
        ("l1_banks", C.c_int64), ("bank_width_bytes", C.c_int64), ("mem_bandwidth_gbps", C.c_double),
        ("l2_bandwidth_gbps", C.c_double), ("max_threads_per_sm", C.c_int64),
        ("max_blocks_per_sm", C.c_int64), ("max_threads_per_block", C.c_int64),
        ("flop_per_byte_balance", C.c_double), ("fit", (C.c_double * 3) * 4),
    ]


class Insn(C.Structure):
    _fields_ = [("op", C.c_int32), ("pad", C.c_int32), ("arg", C.c_int64)]


class Template(C.Structure):
    _fields_ = [
        ("n_fields", C.c_int32), ("n_accesses", C.c_int32),
        ("field_base", C.POINTER(C.c_int64)), ("access_field", C.POINTER(C.c_int32)),
        ("access_kind", C.POINTER(C.c_int32)), ("access_mult", C.POINTER(C.c_int64)),
        ("access_code_off", C.POINTER(C.c_int32)), ("access_code_len", C.POINTER(C.c_int32)),
        ("code", C.POINTER(Insn)), ("n_code", C.c_int32), ("pad", C.c_int32),
    ]


class Config(C.Structure):
    _fields_ = [
        ("template_id", C.c_int32), ("machine_id", C.c_int32), ("block", C.c_int32 * 3),
        ("fold_rank", C.c_int32), ("grid", C.c_int64 * 3), ("work_per_thread", C.c_int64),
        ("flops_per_lup", C.c_int64),
    ]


class Sampling(C.Structure):
    _fields_ = [("block_samples", C.c_int32), ("wave_samples", C.c_int32),
                ("blocks_per_wave_override", C.c_int64), ("phases", C.c_int32), ("pad", C.c_int32)]


# numpy mirror of gvo_config for vectorised batch construction
CONFIG_DTYPE = np.dtype([
    ("template_id", "<i4"), ("machine_id", "<i4"), ("block", "<i4", (3,)), ("fold_rank", "<i4"),
    ("grid", "<i8", (3,)), ("work_per_thread", "<i8"), ("flops_per_lup", "<i8"),
])
assert CONFIG_DTYPE.itemsize == C.sizeof(Config)

_lib = None
_lib_lock = threading.Lock()


def lib():
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise NativeUnavailable(
                f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(str(LIB_PATH))
        P = C.c_void_p
        i32, i64 = C.c_int32, C.c_int64
        p64 = C.POINTER(C.c_int64)
        sig = {
            "gvo_abi_version": (C.c_int, []),
            "gvo_open": (C.c_int, [C.c_int, C.POINTER(P)]),
            "gvo_close": (None, [P]),
            "gvo_last_error": (C.c_char_p, [P]),
            "gvo_set_templates": (C.c_int, [P, C.POINTER(Template), i32]),
            "gvo_set_machines": (C.c_int, [P, C.POINTER(Machine), i32]),
            "gvo_counts_stride_eff": (i64, [i32, C.POINTER(Sampling)]),
            "gvo_eval_configs": (C.c_int, [P, P, i64, C.POINTER(Sampling), i32, P, P, P, P, P, i32, P]),
            "gvo_eval_configs_host": (C.c_int, [P, P, i64, C.POINTER(Sampling), i32, P, P, P, P, P, i32]),
            "gvo_rank": (C.c_int, [P, P, P, i64, P, P]),
            "gvo_sweep_host": (C.c_int, [P, P, i64, C.POINTER(Sampling), i32, P, P, P, P]),
            "gvo_rank_gathered": (C.c_int, [P, P, P, i64, P, i64, P, P, P]),
            "gvo_sweep_host_ex": (C.c_int, [P, P, i64, C.POINTER(Sampling), i32, P, P, P, P, P, i32, P]),
            "gvo_build_id": (C.c_char_p, []),
            "gvo_group_footprint": (C.c_int, [P, i32, C.POINTER(C.c_int32), p64, p64, p64, i32, i64, p64]),
            "gvo_group_sets": (C.c_int, [P, i32, C.POINTER(C.c_int32), p64, p64, p64, i32, i64, p64]),
            "gvo_l1_cycles": (C.c_int, [P, i32, C.POINTER(C.c_int32), p64, i64, i64, i64, p64]),
            "gvo_eval_addresses": (C.c_int, [P, i32, i32, C.POINTER(C.c_int32), p64, i64, p64]),
            "gvo_assemble_host": (C.c_int, [P, P, i32, P, P, i64, P, P]),
            "gvo_predict_host": (C.c_int, [P, P, P, P, P, P, i64, P]),
            "gvo_set_timing": (C.c_int, [P, C.c_int]),
            "gvo_kernel_times": (C.c_int, [P, P, P, C.c_int]),
            "gvo_int_peak": (C.c_int, [P, C.POINTER(C.c_double)]),
            "gvo_debug_units": (C.c_int, [P, C.c_int, P, i64, C.POINTER(C.c_int64)]),
            "gvo_dedup_stats": (C.c_int, [P, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
            "gvo_set_dedup": (C.c_int, [P, C.c_int]),
            "gvo_set_batch": (C.c_int, [P, C.c_int64]),
            "gvo_format_ranking_csv": (C.c_int, [P, i64, P, C.c_char_p, P, i32, P, i64, C.POINTER(C.c_int64)]),
        }
        L.gvo_abi_version.restype = C.c_int
        L.gvo_abi_version.argtypes = []
        if L.gvo_abi_version() != ABI_VERSION:
            raise NativeUnavailable(f"{LIB_PATH.name} ABI version {L.gvo_abi_version()} != {ABI_VERSION}; rebuild it")
        for name, (res, args) in sig.items():
            try:
                fn = getattr(L, name)
            except AttributeError as exc:
                raise NativeUnavailable(f"{LIB_PATH.name} does not export {name}; rebuild it") from exc
            fn.restype = res
            fn.argtypes = args
        _lib = L
        return L


EXPORTED_SYMBOLS = (
    "gvo_abi_version", "gvo_open", "gvo_close", "gvo_last_error", "gvo_set_templates",
    "gvo_set_machines", "gvo_counts_stride_eff", "gvo_eval_configs", "gvo_eval_configs_host",
    "gvo_rank", "gvo_sweep_host", "gvo_rank_gathered", "gvo_build_id", "gvo_sweep_host_ex", "gvo_group_footprint", "gvo_group_sets", "gvo_l1_cycles", "gvo_eval_addresses",
    "gvo_assemble_host", "gvo_predict_host", "gvo_set_timing", "gvo_kernel_times", "gvo_int_peak",
    "gvo_debug_units", "gvo_format_ranking_csv", "gvo_dedup_stats", "gvo_set_dedup",
    "gvo_set_batch",
)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _p64(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int64))


# ---------------------------------------------------------------------------
# encoding of host descriptors


def encode_machine(machine, fit_params=None) -> Machine:
    from .gvo.fit import ROLES

    fits = machine.fit_params if fit_params is None else fit_params
    m = Machine()
    for name, _ in Machine._fields_:
        if name != "fit":
            setattr(m, name, getattr(machine, name))
    for i, role in enumerate(ROLES):
        p = fits[role]
        m.fit[i][0], m.fit[i][1], m.fit[i][2] = float(p.a), float(p.b), float(p.c)
    return m


def machine_key(machine, fit_params=None):
    from .gvo.fit import ROLES

    fits = machine.fit_params if fit_params is None else fit_params
    return tuple(getattr(machine, n) for n, _ in Machine._fields_ if n != "fit") + tuple(
        (float(fits[r].a), float(fits[r].b), float(fits[r].c)) for r in ROLES)


class EncodedTemplate:
    """Arrays backing one gvo_template (kept alive while registered)."""

    def __init__(self, fields, accesses):
        from .gvo.expr import compile_postfix

        index = {f.name: i for i, f in enumerate(fields)}
        self.n_fields = len(fields)
        self.field_names = [f.name for f in fields]
        self.field_base = np.array([f.alignment for f in fields], dtype=np.int64)
        code, off, ln = [], [], []
        for a in accesses:
            prog = compile_postfix(a.expr, index)
            off.append(len(code))
            ln.append(len(prog))
            code.extend(prog)
        self.access_field = np.array([index[a.field] for a in accesses], dtype=np.int32)
        self.access_kind = np.array([0 if a.kind == "load" else 1 for a in accesses], dtype=np.int32)
        self.access_mult = np.array([a.multiplicity for a in accesses], dtype=np.int64)
        self.code_off = np.array(off, dtype=np.int32)
        self.code_len = np.array(ln, dtype=np.int32)
        self.code = (Insn * max(len(code), 1))()
        for i, (op, arg) in enumerate(code):
            self.code[i].op = op
            self.code[i].arg = arg
        self.n_code = len(code)
        self.n_accesses = len(accesses)

    def struct(self) -> Template:
        t = Template()
        t.n_fields = self.n_fields
        t.n_accesses = self.n_accesses
        t.field_base = self.field_base.ctypes.data_as(C.POINTER(C.c_int64))
        t.access_field = self.access_field.ctypes.data_as(C.POINTER(C.c_int32))
        t.access_kind = self.access_kind.ctypes.data_as(C.POINTER(C.c_int32))
        t.access_mult = self.access_mult.ctypes.data_as(C.POINTER(C.c_int64))
        t.access_code_off = self.code_off.ctypes.data_as(C.POINTER(C.c_int32))
        t.access_code_len = self.code_len.ctypes.data_as(C.POINTER(C.c_int32))
        t.code = C.cast(self.code, C.POINTER(Insn))
        t.n_code = self.n_code
        return t


def template_key(fields, accesses):
    return (tuple((f.name, f.alignment) for f in fields),
            tuple((a.field, a.kind, a.multiplicity, a.expr) for a in accesses))


# ---------------------------------------------------------------------------
# context


class Context:
    """One library context per (process, device); registries of uploaded
    templates and machines.  Not thread-safe (reference SPEC.md:484-485)."""

    def __init__(self, device: int = 0):
        L = lib()
        try:
            import torch

            if not torch.cuda.is_available():
                raise NativeUnavailable("no CUDA device visible: the B200 path has no CPU fallback")
        except ImportError:
            pass
        h = C.c_void_p()
        rc = L.gvo_open(device, C.byref(h))
        if rc != 0:
            raise NativeUnavailable(f"gvo_open(device={device}) failed with status {STATUS.get(rc, rc)}")
        self.h = h
        self.device = device
        self.templates: list[EncodedTemplate] = []
        self.tkeys: dict = {}
        self.machines: list[Machine] = []
        self.mkeys: dict = {}
        self._tdirty = False
        self._mdirty = False

    def close(self):
        if self.h:
            lib().gvo_close(self.h)
            self.h = None

    def check(self, rc: int):
        if rc != 0:
            msg = lib().gvo_last_error(self.h)
            raise EngineError(rc, msg.decode() if msg else "")

    def template_id(self, fields, accesses) -> int:
        key = template_key(fields, accesses)
        tid = self.tkeys.get(key)
        if tid is None:
            tid = len(self.templates)
            self.templates.append(EncodedTemplate(fields, accesses))
            self.tkeys[key] = tid
            self._tdirty = True
        return tid

    def machine_id(self, machine, fit_params=None) -> int:
        key = machine_key(machine, fit_params)
        mid = self.mkeys.get(key)
        if mid is None:
            mid = len(self.machines)
            self.machines.append(encode_machine(machine, fit_params))
            self.mkeys[key] = mid
            self._mdirty = True
        return mid

    def sync_registries(self):
        L = lib()
        if self._tdirty:
            arr = (Template * len(self.templates))(*[t.struct() for t in self.templates])
            self.check(L.gvo_set_templates(self.h, arr, len(self.templates)))
            self._tdirty = False
        if self._mdirty:
            arr = (Machine * len(self.machines))(*self.machines)
            self.check(L.gvo_set_machines(self.h, arr, len(self.machines)))
            self._mdirty = False
        if not self.machines:
            self.machine_id_default()

    def machine_id_default(self):
        from .gvo.machine import v100_preset

        self.machine_id(v100_preset())
        self.sync_registries()

    @property
    def max_fields(self) -> int:
        return max((t.n_fields for t in self.templates), default=1)

    @property
    def max_accesses(self) -> int:
        return max((t.n_accesses for t in self.templates), default=1)

    # -- batched evaluation, host buffers
    def eval_configs_host(self, cfgs: np.ndarray, block_samples: int, wave_samples: int,
                          bpw_override: int, want_l1_access: bool = False, want_field_down: bool = True,
                          phases: int = 7):
        self.sync_registries()
        F = self.max_fields
        S, W = effective_sampling(block_samples, wave_samples)
        smp = Sampling(int(block_samples), int(wave_samples), int(bpw_override or 0), int(phases), 0)
        n = len(cfgs)
        cfgs = np.ascontiguousarray(cfgs, dtype=CONFIG_DTYPE)
        stride = counts_stride(F, S, W)
        counts = np.zeros((n, stride), dtype=np.int64)
        stats = np.zeros((n, stats_len(F)), dtype=np.float64)
        records = np.zeros((n, RECORD_LEN), dtype=np.float64)
        fd = np.zeros((n, 4, F), dtype=np.float64) if want_field_down else None
        A = self.max_accesses
        l1 = np.zeros((n, A, 3), dtype=np.int64) if want_l1_access else None
        self.check(lib().gvo_eval_configs_host(
            self.h, _ptr(cfgs), n, C.byref(smp), F, _ptr(counts), _ptr(stats), _ptr(records),
            _ptr(fd) if fd is not None else None, _ptr(l1) if l1 is not None else None, A))
        return {"F": F, "S": S, "W": W, "counts": counts, "stats": stats, "records": records,
                "field_down": fd, "l1_access": l1}


    def sweep_host(self, cfgs: np.ndarray, block_samples: int, wave_samples: int, bpw_override: int,
                   want_l1_access: bool = True, want_field_down: bool = True):
        """Evaluate + rank host configurations in one call (gvo_sweep_host_ex)."""
        self.sync_registries()
        F = self.max_fields
        S, W = effective_sampling(block_samples, wave_samples)
        smp = Sampling(int(block_samples), int(wave_samples), int(bpw_override or 0), 7, 0)
        n = len(cfgs)
        cfgs = np.ascontiguousarray(cfgs, dtype=CONFIG_DTYPE)
        counts = np.empty((n, counts_stride(F, S, W)), dtype=np.int64)
        stats = np.empty((n, stats_len(F)), dtype=np.float64)
        records = np.empty((n, RECORD_LEN), dtype=np.float64)
        fd = np.zeros((n, 4, F), dtype=np.float64) if want_field_down else None
        A = self.max_accesses
        l1 = np.zeros((n, A, 3), dtype=np.int64) if want_l1_access else None
        order = np.empty(n, dtype=np.int64)
        self.check(lib().gvo_sweep_host_ex(
            self.h, _ptr(cfgs), n, C.byref(smp), F, _ptr(counts), _ptr(stats), _ptr(records),
            _ptr(fd) if fd is not None else None, _ptr(l1) if l1 is not None else None, A, _ptr(order)))
        return {"F": F, "S": S, "W": W, "counts": counts, "stats": stats, "records": records,
                "field_down": fd, "l1_access": l1, "order": order}


_ctx: Context | None = None


def context() -> Context:
    global _ctx
    if _ctx is None:
        dev = 0
        try:
            import torch

            if torch.cuda.is_available():
                dev = torch.cuda.current_device()
        except ImportError:
            pass
        _ctx = Context(dev)
        atexit.register(_close_context)
    return _ctx


def _close_context():
    """Release the process-wide context (device buffers) at exit."""
    global _ctx
    if _ctx is not None:
        _ctx.close()
        _ctx = None


# ---------------------------------------------------------------------------
# fine-grained entry points


def _launch_of(kernel):
    block = (C.c_int32 * 3)(*kernel.launch.block_dim)
    grid = np.array(kernel.launch.grid_dim, dtype=np.int64)
    return block, grid


def group_footprint(kernel, runs: list[tuple[int, int]], granularity: int) -> np.ndarray:
    """[F][kind][unique, total] for the union of block runs."""
    ctx = context()
    tid = ctx.template_id(kernel.fields, kernel.accesses)
    ctx.sync_registries()
    block, grid = _launch_of(kernel)
    rs = np.array([r[0] for r in runs], dtype=np.int64)
    rc = np.array([r[1] for r in runs], dtype=np.int64)
    F = len(kernel.fields)
    out = np.zeros((F, 2, 2), dtype=np.int64)
    ctx.check(lib().gvo_group_footprint(ctx.h, tid, block, _p64(grid), _p64(rs), _p64(rc), len(runs),
                                        int(granularity), _p64(out)))
    return out


def group_sets(kernel, runs: list[tuple[int, int]], granularity: int) -> np.ndarray:
    """[G][F][|L|, |S|, |L u S|, |L n L_prev|] for consecutive groups."""
    ctx = context()
    tid = ctx.template_id(kernel.fields, kernel.accesses)
    ctx.sync_registries()
    block, grid = _launch_of(kernel)
    rs = np.array([r[0] for r in runs], dtype=np.int64)
    rc = np.array([r[1] for r in runs], dtype=np.int64)
    F = len(kernel.fields)
    out = np.zeros((len(runs), F, 4), dtype=np.int64)
    ctx.check(lib().gvo_group_sets(ctx.h, tid, block, _p64(grid), _p64(rs), _p64(rc), len(runs),
                                   int(granularity), _p64(out)))
    return out


def l1_cycles(kernel, block_linear: int, bank_width: int, n_banks: int) -> np.ndarray:
    """[A][cycles, 2*sum metric, warps]."""
    ctx = context()
    tid = ctx.template_id(kernel.fields, kernel.accesses)
    ctx.sync_registries()
    block, grid = _launch_of(kernel)
    out = np.zeros((len(kernel.accesses), 3), dtype=np.int64)
    ctx.check(lib().gvo_l1_cycles(ctx.h, tid, block, _p64(grid), int(block_linear), int(bank_width),
                                  int(n_banks), _p64(out)))
    return out


def eval_addresses(expr, bases, block_dim, coords: np.ndarray) -> np.ndarray:
    """Device evaluation of one expression at explicit coordinates."""
    from .gvo.expr import base_refs
    from .gvo.kernels import Access, Field

    ctx = context()
    refs = base_refs(expr)
    names = list(dict.fromkeys(refs)) or ["__nofield"]
    fields = tuple(Field(n, 8, (1,), alignment=int(bases.get(n, 0))) for n in names)
    acc = (_RawAccess(names[0], expr),)
    tid = ctx.template_id(fields, acc)
    ctx.sync_registries()
    block = (C.c_int32 * 3)(*block_dim)
    coords = np.ascontiguousarray(coords, dtype=np.int64)
    out = np.zeros(len(coords), dtype=np.int64)
    ctx.check(lib().gvo_eval_addresses(ctx.h, tid, 0, block, _p64(coords), len(coords), _p64(out)))
    return out


class _RawAccess:
    """Minimal access record for evaluate_bulk templates (no base-ref check)."""

    def __init__(self, field, expr):
        self.field = field
        self.kind = "load"
        self.expr = expr
        self.multiplicity = 1


def assemble(stats: np.ndarray, F: int, machine_ids: np.ndarray, flops: np.ndarray):
    ctx = context()
    ctx.sync_registries()
    n = len(stats)
    stats = np.ascontiguousarray(stats, dtype=np.float64)
    mids = np.ascontiguousarray(machine_ids, dtype=np.int32)
    fl = np.ascontiguousarray(flops, dtype=np.int64)
    rec = np.zeros((n, RECORD_LEN), dtype=np.float64)
    fd = np.zeros((n, 4, F), dtype=np.float64)
    ctx.check(lib().gvo_assemble_host(ctx.h, _ptr(stats), F, _ptr(mids), _ptr(fl), n, _ptr(rec), _ptr(fd)))
    return rec, fd


def predict(machine_ids: np.ndarray, dram_down: np.ndarray, l2_down: np.ndarray, cycles: np.ndarray,
            flops: np.ndarray) -> np.ndarray:
    """Device four-limiter prediction; returns [n][6] = t_dram, t_l2, t_l1, t_fp, limiter, glups."""
    ctx = context()
    ctx.sync_registries()
    n = len(machine_ids)
    mids = np.ascontiguousarray(machine_ids, dtype=np.int32)
    a = np.ascontiguousarray(dram_down, dtype=np.float64)
    b = np.ascontiguousarray(l2_down, dtype=np.float64)
    c = np.ascontiguousarray(cycles, dtype=np.float64)
    f = np.ascontiguousarray(flops, dtype=np.int64)
    out = np.zeros((n, 6), dtype=np.float64)
    ctx.check(lib().gvo_predict_host(ctx.h, _ptr(mids), _ptr(a), _ptr(b), _ptr(c), _ptr(f), n, _ptr(out)))
    return out


def rank_device(d_records, d_cfgs, n: int, d_order, stream: int = 0):
    """Device ranking on caller-owned device buffers (torch tensors' data_ptr)."""
    ctx = context()
    ctx.check(lib().gvo_rank(ctx.h, C.c_void_p(d_records), C.c_void_p(d_cfgs), int(n), C.c_void_p(d_order),
                             C.c_void_p(stream)))


def rank_gathered(d_rows, d_gidx, n_rows: int, d_cfgs, n_global: int, d_records_global, d_order,
                  stream: int = 0):
    """Device ranking of all-gathered shard rows carrying their global index
    (-1: padding) over the whole space in global order (gvo_rank_gathered)."""
    ctx = context()
    ctx.check(lib().gvo_rank_gathered(ctx.h, C.c_void_p(d_rows), C.c_void_p(d_gidx), int(n_rows),
                                      C.c_void_p(d_cfgs), int(n_global),
                                      C.c_void_p(d_records_global) if d_records_global else None,
                                      C.c_void_p(d_order), C.c_void_p(stream)))


def build_id() -> str:
    """gvo_build_id() of the loaded library (hash of sources + flags)."""
    return lib().gvo_build_id().decode()


def rank_host(cfgs: np.ndarray, records: np.ndarray) -> np.ndarray:
    """Ranking order of host arrays, computed by the device sort (k_rank.cu)."""
    import torch

    n = len(cfgs)
    if n == 0:
        return np.zeros(0, dtype=np.int64)
    dev = torch.device("cuda", context().device)
    rec = torch.from_numpy(np.ascontiguousarray(records, dtype=np.float64)).to(dev)
    raw = np.ascontiguousarray(cfgs, dtype=CONFIG_DTYPE).view(np.uint8)
    cf = torch.from_numpy(raw.copy()).to(dev)
    order = torch.empty(n, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)
    rank_device(rec.data_ptr(), cf.data_ptr(), n, order.data_ptr(), stream.cuda_stream)
    return order.cpu().numpy()


def format_ranking_csv(records: np.ndarray, prefixes: list[str], order=None, n_threads: int = 0) -> str:
    """Ranking CSV body rows (no header) via the native formatter; byte-identical
    to the reference's render_ranking_csv rows (report.py:242-255)."""
    rec = np.ascontiguousarray(records, dtype=np.float64).reshape(-1, RECORD_LEN)
    n = len(rec)
    if len(prefixes) != n:
        raise ValueError("one prefix per record")
    enc = [p.encode() for p in prefixes]
    off = np.zeros(n + 1, dtype=np.int64)
    if n:
        np.cumsum([len(e) for e in enc], out=off[1:])
    blob = b"".join(enc)
    ordr = None if order is None else np.ascontiguousarray(order, dtype=np.int64)
    L = lib()
    need = C.c_int64(0)
    args = (_ptr(rec) if n else None, n, _ptr(ordr) if ordr is not None else None, blob, _ptr(off), int(n_threads))
    rc = L.gvo_format_ranking_csv(*args, None, 0, C.byref(need))
    if rc not in (0, STATUS_CAPACITY):
        raise EngineError(rc, "gvo_format_ranking_csv: invalid arguments")
    buf = C.create_string_buffer(max(1, need.value))
    rc = L.gvo_format_ranking_csv(*args, buf, need.value, C.byref(need))
    if rc != 0:
        raise EngineError(rc, "gvo_format_ranking_csv failed")
    return buf.raw[: need.value].decode()
