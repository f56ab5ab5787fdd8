"""Calibration closed loop at scale: the C3 sweep
(93,184 configurations) evaluated on the device, written as the reference's
ranking CSV by the native formatter, measurements synthesised from known
per-role curves (tests/calib_util.py), then derive_observations +
calibrate_all.  The golden (tests/golden/calib_c3.json,
tools/make_golden_calib.py) is the unmodified reference's fit of the same
sweep and measurements: the device sweep must hash to the rows the
reference fitted, and this package's fit must equal the reference's to the
bit (reference fit.py:94-243, api.py:280-287)."""

from __future__ import annotations

import hashlib
import json

import pytest

import calib_util
from golden_util import load

pytestmark = pytest.mark.gpu


def test_calibration_closed_loop_on_device_c3_sweep(tmp_path):
    from paper_2107_01143_b200 import _native, workloads as W
    from paper_2107_01143_b200.gvo import api, report

    gold = load("calib_c3")
    sp = calib_util.space_c3()
    res, order = W.evaluate_space(sp)
    sweep = ",".join(report.RANKING_CSV_COLUMNS) + "\n" + _native.format_ranking_csv(
        res.records, calib_util.prefixes(sp), order)
    assert sweep.count("\n") - 1 == gold["rows"] == 93184
    assert hashlib.sha256(sweep.encode()).hexdigest() == gold["sweep_sha256"]
    meas = calib_util.measurement_csv(sweep)
    assert hashlib.sha256(meas.encode()).hexdigest() == gold["measurements_sha256"]
    (tmp_path / "s.csv").write_text(sweep)
    (tmp_path / "m.csv").write_text(meas)
    got = api.run_calibrate(str(tmp_path / "m.csv"), str(tmp_path / "s.csv"))
    assert json.loads(json.dumps(got["fitParams"])) == gold["fitParams"]
    assert json.loads(json.dumps(got["residuals"])) == gold["residuals"]
    assert got["observationCounts"] == gold["observationCounts"]
    assert len(got["skipped"]) == gold["skipped"]
    obs = json.dumps(got["observations"], sort_keys=True).encode()
    assert hashlib.sha256(obs).hexdigest() == gold["observations_sha256"]
    # the closed loop: the generating curves are recovered
    for role, (a, b, c) in calib_util.TRUE.items():
        p = got["fitParams"][role]
        assert abs(p["a"] - a) < 1e-9 and abs(p["b"] - b) < 1e-9 and abs(p["c"] - c) < 1e-9, (role, p)
