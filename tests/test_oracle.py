"""Pin the CPU oracle (test infrastructure) against the reference itself:
golden vectors produced by the unmodified reference (tools/make_golden.py)
and the reference test-suite's known answers."""

import math

import numpy as np
import pytest

from golden_util import load, unhex
from oracle import gvo_oracle as ora
from paper_2107_01143_b200 import gvo
from paper_2107_01143_b200.gvo.machine import machine_from_dict


def test_paper_figure_known_answer():
    # reference test_footprint.py:30-38 / PAPER Fig. footprint: 16 accesses, 10 unique
    k = gvo.generate_four_point_2d((100, 100), (2, 2))
    r = ora.footprint(k, [0], 8, kinds=("load",))
    assert r[("src", "load")] == (10, 16)


def test_contiguous_sector_known_answer():
    # reference test_footprint.py:41-47: 8 sectors, 8 warp requests
    f = (gvo.Field("a", 8, (4096, 64, 64)),)
    acc = (gvo.Access("a", "load", gvo.parse("a + tidx * 8", fields=["a"])),)
    k = gvo.KernelDescriptor(fields=f, accesses=acc, launch=gvo.LaunchConfig((32, 1, 1), (4, 2, 2)))
    assert ora.footprint(k, [0], 32)[("a", "load")] == (8, 8)


def test_bank_triptych_known_answer():
    # reference test_volumes.py:41-52: per_access == (1.0, 2.0, 32.0)
    names = ["a", "b", "d"]
    fields = tuple(gvo.Field(n, 8, (65536,)) for n in names)
    acc = tuple(gvo.Access(n, "load", gvo.parse(f"{n} + tidx * {s}", fields=names))
                for n, s in zip(names, (8, 16, 256)))
    k = gvo.KernelDescriptor(fields=fields, accesses=acc, launch=gvo.LaunchConfig((32, 1, 1), (4, 2, 2)))
    _, per = ora.l1_cycles(k, gvo.v100_preset(), 0)
    assert per == (1.0, 2.0, 32.0)


@pytest.mark.parametrize("chunk", range(4))
def test_oracle_footprints_match_reference_golden(chunk):
    cases = load("footprints")
    for case in cases[chunk::4]:
        k = gvo.kernel_from_dict(case["spec"])
        got = ora.footprint(k, case["blocks"], case["granularity"])
        want = {(f, kd): (u, t) for f, kd, u, t in case["per_field"]}
        assert got == want, case["spec"]["accesses"]


def _check_eval(case, strict_float=True):
    k = gvo.kernel_from_dict(case["spec"])
    m = machine_from_dict(case["machine"])
    bsz, wsz, ovr = case["sampling"]
    ev = ora.evaluate_kernel(k, m, None, bsz, wsz, ovr)
    rec = ora.record(ev)
    for col, v in case["record"].items():
        if col in ("configKey", "blockX", "blockY", "blockZ", "folding"):
            continue
        want = unhex(v)
        assert rec[col] == want, (col, rec[col], want)
    assert [float(x).hex() for x in ev["per_access"]] == case["per_access"]


def test_oracle_evaluations_match_reference_golden_v100():
    cases = [c for c in load("evaluations") if c["machine"]["name"] == "v100"]
    assert len(cases) >= 6
    for case in cases:
        _check_eval(case)


def test_oracle_evaluation_b200_sample():
    cases = [c for c in load("evaluations") if c["machine"]["name"] == "b200"]
    _check_eval(cases[0])


def test_oracle_rank_matches_reference_sweep_golden():
    for sw in load("sweeps"):
        fam = gvo.KernelFamily(sw["kind"], tuple(sw["grid"]), radius=sw["radius"])
        m = gvo.v100_preset()
        rows = []
        for cfg in gvo.enumerate_sweep(sw["threads"], foldings=sw["foldings"]):
            try:
                k = fam.build(cfg)
            except ValueError:
                continue
            if sw["kind"] == "stencil" and cfg.key not in sw["order"]:
                continue
            ev = ora.evaluate_kernel(k, m, None, 2, 1)
            rows.append((ev["glups"], cfg.block_dim, cfg.folding, cfg.key))
        order = ora.rank([(g, b, f) for g, b, f, _ in rows])
        assert [rows[i][3] for i in order] == sw["order"]
        assert [float(rows[i][0]).hex() for i in order] == sw["glups"]
