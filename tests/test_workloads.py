"""BASELINE.json configuration spaces (C1-C5): generators, cardinalities,
and device parity against the unmodified reference run on the same
descriptors (tests/golden/workloads.json, tools/make_golden_workloads.py).

GPU tests: every integer-derived volume, time, limiter and GLup/s value of
the sampled full-size C1/C3/C4/C5 configurations is bit-identical to the
reference (tolerance 0, stricter than north_star's 1e-6 relative), and the
complete C2 (246) and C4 two-phase LBM (1,812) sweeps rank in exactly the
reference's order with bit-identical GLup/s."""

import numpy as np
import pytest

from golden_util import load, unhex
from oracle import gvo_oracle as ora
from paper_2107_01143_b200 import gvo, workloads as W
from paper_2107_01143_b200.gvo.machine import machine_from_dict

SKIP_COLS = ("configKey", "blockX", "blockY", "blockZ", "folding")


def _machines(name):
    return [machine_from_dict(d) for d in load("workloads")["machines"][name]]


# ------------------------------------------------------------------ CPU
def test_space_cardinalities():
    m = gvo.b200_preset()
    assert len(W.pow2_shapes(W.STENCIL_THREADS)) == 264
    assert len(W.pow2_shapes(W.LBM_THREADS)) == 154
    assert len(W.space("C1", m)) == 1
    assert len(W.space("C2", m)) == 246
    assert len(W.space("C3", m)) == 93184
    assert len(W.space("C4", m)) == 1812
    assert len(W.space("C5", m)) == 1205184


def test_generators_reduce_to_reference_generators():
    d = gvo.kernel_to_dict
    assert d(W.generate_lbm("D3Q15", (256, 128, 128), (32, 2, 2))) == d(
        gvo.generate_lbm_d3q15((256, 128, 128), (32, 2, 2)))
    for fo in ("none", "2y", "2z"):
        assert d(W.generate_star_stencil_fields(4, (640, 640, 640), (16, 2, 16), fo)) == d(
            gvo.generate_star_stencil(4, (640, 640, 640), (16, 2, 16), fo))
    # one component: both layouts are the same field and trees
    a = W.generate_star_stencil_fields(2, (64, 64, 64), (8, 8, 2), "2z", layout="zyxf", components=1)
    b = W.generate_star_stencil_fields(2, (64, 64, 64), (8, 8, 2), "2z", layout="fzyx", components=1)
    assert d(a) == d(b)


def test_layout_addresses():
    """zyxf: component c of point (x,y,z) at ((z*h+y)*w+x)*F*8 + 8c."""
    k = W.generate_star_stencil_fields(1, (16, 8, 4), (4, 2, 2), layout="zyxf", components=4, alignment=0)
    f = k.fields[0]
    assert f.strides == (32, 32 * 16, 32 * 16 * 8)
    tc = gvo.ThreadCoord(tidx=1, tidy=1, tidz=1, bidx=2, bidy=1, bidz=0)
    x, y, z = 1 + 2 * 4, 1 + 1 * 2, 1
    per_c = 7 + 1
    for c in range(4):
        centre = k.accesses[c * per_c]
        assert gvo.evaluate(centre.expr, [tc], (4, 2, 2), {"src": 0}) == [((z * 8 + y) * 16 + x) * 32 + 8 * c]
    kf = W.generate_lbm("D3Q27", (16, 8, 4), (4, 2, 2), layout="fzyx")
    assert len(kf.accesses) == 27 + 27 + 7 and kf.fields[0].extents == (16, 8, 4 * 27)
    kz = W.generate_lbm("D3Q27", (16, 8, 4), (4, 2, 1), "2z", layout="zyxf")
    assert len(kz.accesses) == 2 * 61 and kz.launch.work_per_thread == 2


def test_oracle_matches_reference_on_workload_records():
    """The CPU oracle reproduces the reference records of the C1 config and
    a small C4 two-phase LBM sample (pins the oracle on the new generators)."""
    g = load("workloads")
    for name, n in (("C1", 1), ("C4", 2)):
        ents = g["records"][name][:n]
        sp = W.space_from_entries(ents, _machines(name))
        for i, e in enumerate(ents):
            if "error" in e:
                continue
            ev = ora.evaluate_kernel(sp.kernel(i), sp.machine(i))
            assert float(ev["glups"]).hex() == e["record"]["predictedGLups"], (name, e["template"], e["block"])
            assert ev["limiter"] == e["record"]["limiter"]


# ------------------------------------------------------------------ GPU
def _pred_cols(p):
    v = p.volumes
    return {
        "l1CyclesPerLup": p.l1_cycles.cycles_per_lup,
        "l2l1LoadComp": v.l2l1_load.v_comp, "l2l1LoadRed": v.l2l1_load.v_red, "l2l1LoadCap": v.l2l1_load.v_cap,
        "l2l1LoadUp": v.l2l1_load.v_up, "l2l1LoadDown": v.l2l1_load.v_down, "l2l1LoadAlloc": v.l2l1_load.v_alloc,
        "l2l1LoadOversub": v.l2l1_load.oversubscription,
        "l2l1StoreComp": v.l2l1_store.v_comp, "l2l1StoreRed": v.l2l1_store.v_red,
        "l2l1StoreCap": v.l2l1_store.v_cap, "l2l1StoreUp": v.l2l1_store.v_up, "l2l1StoreDown": v.l2l1_store.v_down,
        "dramLoadComp": v.dram_load.v_comp, "dramLoadRed": v.dram_load.v_red, "dramLoadCap": v.dram_load.v_cap,
        "dramLoadUp": v.dram_load.v_up, "dramLoadDown": v.dram_load.v_down, "dramLoadAlloc": v.dram_load.v_alloc,
        "dramLoadOversub": v.dram_load.oversubscription, "dramLoadUnique": v.dram_load.wave_unique,
        "dramLoadOverlap": v.dram_load.v_overlap, "dramLoadOvermiss": v.dram_load.overmiss_bytes,
        "dramLoadCoverage": v.dram_load.coverage, "dramLoadRedL2": v.dram_load.v_red_l2,
        "dramStoreComp": v.dram_store.v_comp, "dramStoreRed": v.dram_store.v_red, "dramStoreCap": v.dram_store.v_cap,
        "dramStoreUp": v.dram_store.v_up, "dramStoreDown": v.dram_store.v_down,
        "dramStoreUnique": v.dram_store.wave_unique,
        "tDram": p.times["dram"], "tL2": p.times["l2"], "tL1": p.times["l1"], "tFp": p.times["fp"],
        "limiter": p.limiter, "predictedGLups": p.glups,
    }


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["C1", "C3", "C4", "C5"])
def test_workload_records_bit_exact_vs_reference(name):
    ents = [e for e in load("workloads")["records"][name] if "error" not in e]
    sp = W.space_from_entries(ents, _machines(name))
    res, _ = W.evaluate_space(sp, want_l1=True)
    bad = []
    for i, e in enumerate(ents):
        p = W.prediction(sp, res, i)
        got = _pred_cols(p)
        for col, want in e["record"].items():
            if col not in SKIP_COLS and got[col] != unhex(want):
                bad.append((sp.key(i), col, got[col], unhex(want)))
        if [float(x).hex() for x in p.l1_cycles.per_access] != e["per_access"]:
            bad.append((sp.key(i), "per_access"))
        for lvl, d in e["per_field_down"].items():
            gv = getattr(p.volumes, lvl).per_field_down
            bad += [(sp.key(i), lvl, f) for f, w in d.items() if gv[f] != unhex(w)]
    assert not bad, bad[:5]


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["C2", "C4"])
def test_full_sweep_ranking_identical_to_reference(name):
    g = load("workloads")["rankings"][name]
    ents = [{"template": g["templates"][t], "machine": m, "block": [bx, by, bz]} for t, m, bx, by, bz in g["cfg"]]
    sp = W.space_from_entries(ents, _machines(name))
    res, order = W.evaluate_space(sp)
    glups = [float(r).hex() for r in res.records[:, -1]]
    assert glups == g["glups"]
    lim = [gvo.perf.LIMITER_ORDER[int(x)] for x in res.records[:, -2]]
    assert lim == g["limiter"]
    assert list(map(int, order)) == g["order"]


@pytest.mark.gpu
@pytest.mark.parametrize("name,pad", [("C3", False), ("C5", False), ("C3", True), ("C5", True)])
def test_seeded_subset_records_and_ranking_vs_reference(name, pad):
    """512 seeded configurations of each large space: every
    record column bit-identical to the reference's and the subset ranked in
    the reference's order (tests/golden/subsets.json)."""
    g = load("subsets")
    s = g["spaces"][name]
    cols = g["columns"]
    ents = [{"template": s["templates"][t], "machine": mm, "block": [bx, by, bz]} for t, mm, bx, by, bz in s["cfg"]]
    assert all(isinstance(r, list) for r in s["records"])
    sp = W.space_from_entries(ents, _machines(name))
    if pad:
        # the same configurations inside one call of >= 1024 (the set
        # kernel's large-batch paths: micro handoffs, residency picked per
        # batch); the padding repeats them, so every copy must match too
        sp = sp.subset(np.concatenate([np.arange(len(sp))] * 3))
    res, order = W.evaluate_space(sp)
    if pad:
        n0 = len(s["records"])
        for k in (1, 2):
            assert np.array_equal(res.records[k * n0:(k + 1) * n0].view(np.int64), res.records[:n0].view(np.int64))
        res = type(res)(res.F, res.S, res.W, res.counts[:n0], None if res.stats is None else res.stats[:n0],
                        res.records[:n0], None, None)
        order = [o for o in order if o < n0]
    lim_col = cols.index("limiter")
    bad = []
    for i, want in enumerate(s["records"]):
        for c, (col, w) in enumerate(zip(cols, want)):
            got = res.records[i, c]
            if c == lim_col:
                ok = gvo.perf.LIMITER_ORDER[int(got)] == w
            elif w is None:
                ok = np.isnan(got)
            else:
                ok = float(got).hex() == w
            if not ok:
                bad.append((sp.key(i), col, float(got).hex(), w))
    assert not bad, bad[:5]
    assert list(map(int, order)) == s["order"]
