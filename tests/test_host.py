"""CPU-side tests: descriptor layer, host geometry, bytecode, C-ABI surface."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from golden_util import load
from oracle import gvo_oracle as ora
from paper_2107_01143_b200 import _native, gvo
from paper_2107_01143_b200.gvo import expr as E

ROOT = Path(__file__).resolve().parents[1]


def test_parse_render_round_trip():
    for text in ("A + (tidx + bidx*BX)*8", "src + ((tidx + 4) + (tidy - 3) * 640 + tidz * 327680) * 8",
                 "a % 7 + b // 32 - -5", "(tidx + tidy) * (bidx + 1)", "-(tidx) * 3"):
        t = gvo.parse(text)
        assert gvo.parse(gvo.render(t)) == t


def test_parse_errors_and_positions():
    with pytest.raises(gvo.ExprSyntaxError) as e:
        gvo.parse("tidx + + 3")
    assert e.value.position == 7
    for bad in ("tidx + (tidy * 2", "", "tidx // 0", "tidx % -3", "B + tidx"):
        with pytest.raises(gvo.ExprError):
            gvo.parse(bad, fields=["A"] if bad.startswith("B") else None)


def test_overflow_guard_and_affine_parts():
    big = E.BinOp("*", E.CoordRef("tidx"), E.IntConstant(2 ** 60))
    with pytest.raises(gvo.AddressOverflowError):
        gvo.evaluate(big, [E.ThreadCoord(tidx=9)], (32, 4, 2), {})
    assert E.affine_parts(gvo.parse("3 * (tidx + 2) * 4"), (32, 4, 2), {}) == (24, {"tidx": 12})
    assert E.affine_parts(gvo.parse("tidx // 4"), (1, 1, 1), {}) is None
    assert E.affine_parts(gvo.parse("tidx * tidy"), (1, 1, 1), {}) is None


def test_generators_match_reference_specs():
    """Our generators build the same trees as the reference (spec equality)."""
    for case in load("evaluations"):
        spec = case["spec"]
        k = gvo.kernel_from_dict(spec)
        if spec["name"].startswith("star"):
            matches = 0
            for fold in ("none", "2y", "2z"):
                f = gvo.kernels.fold_factors(fold)
                grid = [k.launch.grid_dim[i] * k.launch.block_dim[i] * f[i] for i in range(3)]
                try:
                    mine = gvo.generate_star_stencil(int(spec["name"][4:]), grid, k.launch.block_dim, fold)
                except gvo.KernelError:
                    continue
                matches += gvo.kernel_to_dict(mine) == spec
            assert matches == 1, spec["name"]
        elif spec["name"] == "lbm_d3q15":
            grid = [k.launch.grid_dim[i] * k.launch.block_dim[i] for i in range(3)]
            assert gvo.kernel_to_dict(gvo.generate_lbm_d3q15(grid, k.launch.block_dim)) == spec


def test_enumerate_sweep_cardinalities():
    assert len(gvo.enumerate_sweep(1024)) == 54
    assert len(gvo.enumerate_sweep(1024, foldings=("none", "2y", "2z"))) == 162
    assert len(gvo.enumerate_sweep(512)) == 49


def test_representative_blocks_closed_form_vs_meshgrid():
    rng = np.random.default_rng(3)
    for _ in range(300):
        grid = tuple(int(v) for v in rng.integers(1, 40, size=3))
        k = gvo.generate_star_stencil(1, grid, (1, 1, 1))
        s = int(rng.integers(1, 12))
        mine = [int(g.block_linear[0]) for g in gvo.representative_blocks(k, s)]
        assert mine == ora.representative_blocks(k, s)


def test_wave_pairs_closed_form():
    m = gvo.v100_preset()
    k = gvo.generate_star_stencil(4, (256, 256, 128), (32, 4, 8))
    pairs = gvo.representative_wave_pairs(k, m, 2)
    w, op = ora.wave_pairs(k.launch, m, 2)
    assert [(p.index, c.index) for p, c in pairs] == op


def test_bytecode_postfix_shape():
    t = gvo.parse("a + (tidx + bidx*BX) * 8 // 3", fields=["a"])
    prog = E.compile_postfix(t, {"a": 0})
    depth = 0
    for op, _ in prog:
        depth += 1 if op <= E.OP_BASE else -1
        assert depth >= 1
    assert depth == 1


def test_library_exports_every_header_symbol():
    header = (ROOT / "include" / "gvo_b200.h").read_text()
    declared = set(re.findall(r"^\s*(?:int|void|const char\*|int64_t)\s+(gvo_\w+)\s*\(", header, re.M))
    assert declared, "no declarations parsed"
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    for name in declared:
        assert hasattr(lib, name), name
    assert declared <= set(_native.EXPORTED_SYMBOLS) | {"gvo_counts_stride"}
    assert lib.gvo_abi_version() == _native.ABI_VERSION == 4


def test_struct_layouts_match_header():
    assert ctypes.sizeof(_native.Config) == 64
    assert ctypes.sizeof(_native.Machine) == 14 * 8 + 12 * 8
    assert ctypes.sizeof(_native.Insn) == 16
    assert ctypes.sizeof(_native.Sampling) == 24
    assert _native.counts_stride(2, 5, 2) == 16 + 5 * 2 * 5 + 3 * 2 * 4 + 3


def test_no_gpu_means_loud_failure(monkeypatch):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_native.NativeUnavailable):
        _native.Context(0)
