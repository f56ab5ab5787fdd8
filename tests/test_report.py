"""Serialization / API / bindings layer (SURVEY.md §8b callers, §8f N2-N4)
against bytes produced by the unmodified reference (tests/golden/report.json,
tools/make_golden_report.py): estimate JSON/CSV/table, ranking CSVs of
whole sweeps (native formatter), footprint CSV, calibration."""

import json
import math

import numpy as np
import pytest

from golden_util import load
from paper_2107_01143_b200 import _native
from paper_2107_01143_b200 import gvo_bindings as gb
from paper_2107_01143_b200.gvo import api, report


def _kw(d):
    return {k: (tuple(v) if isinstance(v, list) else v) for k, v in d.items()}


# ------------------------------------------------------------------ CPU
def test_native_g10_formatter_matches_python_format():
    rng = np.random.default_rng(5)
    n = 20000
    rec = np.empty((n, _native.RECORD_LEN))
    mant = rng.standard_normal((n, _native.RECORD_LEN))
    expo = rng.integers(-30, 30, (n, _native.RECORD_LEN)).astype(float)
    rec[:] = mant * 10.0 ** expo
    rec[::7, 3] = np.round(rec[::7, 3])  # integral values
    rec[::11, 4] = 0.0
    rec[::13, 5] = -0.0
    rec[::17, 6] = 5e-324
    rec[::19, 7] = 1.7976931348623157e308
    rec[::23, 8] = 0.1 + 0.2
    rec[::3, 23] = np.nan  # coverage None
    rec[:, 35] = rng.integers(0, 4, n)
    prefixes = [f"k{i},1,2,3,none" for i in range(n)]
    order = rng.permutation(n)
    got = _native.format_ranking_csv(rec, prefixes, order, n_threads=4)
    lim = ("dram", "l2", "l1", "fp")
    want = "".join(prefixes[i] + "," + ",".join(
        lim[int(v)] if c == 35 else ("" if math.isnan(v) else format(float(v), ".10g"))
        for c, v in enumerate(rec[i])) + "\n" for i in order)
    assert got == want


def test_estimate_csv_and_table_from_reference_reports():
    for e in load("report")["estimates"]:
        rep = json.loads(e["json"])
        assert report.render_estimate_csv(rep) == e["csv"]
        assert report.render_table(rep) == e["table"]
        assert report.render_json(rep) == e["json"]


def test_calibration_from_reference_sweep_csv(tmp_path):
    g = load("report")
    cal = g["calibration"]
    (tmp_path / "s.csv").write_text(g["sweeps"][cal["sweep"]]["csv"])
    (tmp_path / "m.csv").write_text(cal["measurements"])
    got = json.loads(json.dumps(gb.calibrate(str(tmp_path / "m.csv"), str(tmp_path / "s.csv"))))
    assert got == cal["result"]


def test_spec_builder_validates():
    b = (gb.KernelSpecBuilder("copy").field("a", 8, (1024,)).load("a", "a + tidx * 8")
         .launch((32, 1, 1), (32, 1, 1)).flops(1))
    spec = b.build()
    assert spec["launch"]["blockDim"] == [32, 1, 1]
    b._data["accesses"][0]["expr"] = "a + tidx // 0"
    with pytest.raises(ValueError):
        b.build()


def test_resolve_machine_and_fits(tmp_path):
    assert api.resolve_machine(None).name == "v100"
    assert api.resolve_machine("b200").sm_count == 148
    with pytest.raises(FileNotFoundError):
        api.resolve_machine("nope", machine_dir=str(tmp_path))
    m = api.resolve_machine("v100")
    z = api.resolve_fit_params("zero", m)
    assert all(p.a == 0.0 for p in z.values())


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
def test_estimate_json_byte_identical():
    for e in load("report")["estimates"]:
        kernel, block = e["args"]
        assert gb.estimate_json(kernel, "v100", tuple(block), **_kw(e["kw"])) == e["json"], e["args"]


@pytest.mark.gpu
def test_sweep_csv_byte_identical():
    for s in load("report")["sweeps"]:
        kernel, machine, threads = s["args"]
        assert gb.sweep_csv(kernel, machine, threads, **_kw(s["kw"])) == s["csv"], s["args"]


@pytest.mark.gpu
def test_sweep_rows_python_path_equals_native_path():
    s = load("report")["sweeps"][0]
    kernel, machine, threads = s["args"]
    rows = api.run_sweep(kernel, machine, threads, **_kw(s["kw"]))
    assert report.render_ranking_csv(list(rows)) == report.render_ranking_csv(rows) == s["csv"]
    d = gb.sweep(kernel, machine, threads, **_kw(s["kw"]))
    assert [r["configKey"] for r in d] == [ln.split(",")[0] for ln in s["csv"].splitlines()[1:]]


@pytest.mark.gpu
def test_footprint_csv_byte_identical():
    for f in load("report")["footprints"]:
        kernel, block, level, gran = f["args"]
        res = api.run_footprint(kernel, "v100", tuple(block), level=level, granularity=gran,
                                grid=(128, 128, 64) if kernel == "builtin:stencil" else (128, 64, 64))
        assert report.render_footprint_csv(res) == f["csv"], f["args"]
