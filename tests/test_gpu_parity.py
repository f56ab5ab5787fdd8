"""Device parity: the sm_100a engine vs the reference golden vectors and the
CPU oracle.  Integer volumes bit-exact, floats bit-exact (tolerance 0 —
stricter than north_star's 1e-6 relative), rankings identical."""

import math

import numpy as np
import pytest

from golden_util import load, unhex
from oracle import gvo_oracle as ora
from paper_2107_01143_b200 import gvo
from paper_2107_01143_b200.gvo.footprint import CollaborativeGroup, wave_footprint
from paper_2107_01143_b200.gvo.machine import machine_from_dict

pytestmark = pytest.mark.gpu


def test_native_library_loaded():
    from paper_2107_01143_b200 import _native

    ctx = _native.context()
    assert ctx.h


def test_footprints_match_reference_golden():
    bad = []
    for case in load("footprints"):
        k = gvo.kernel_from_dict(case["spec"])
        grp = CollaborativeGroup(k.launch, np.asarray(case["blocks"], dtype=np.int64), "L2")
        r = gvo.grid_iteration(k, grp, case["granularity"])
        got = {(f, kd): (c.unique_count, c.total_count) for (f, kd), c in r.per_field.items()}
        want = {(f, kd): (u, t) for f, kd, u, t in case["per_field"]}
        if got != want:
            bad.append((case["spec"]["accesses"], case["blocks"], case["granularity"], got, want))
    assert not bad, bad[:3]


def _compare_eval(case):
    k = gvo.kernel_from_dict(case["spec"])
    m = machine_from_dict(case["machine"])
    bsz, wsz, ovr = case["sampling"]
    p = gvo.evaluate_kernel(k, m, block_samples=bsz, wave_samples=wsz, override_blocks_per_wave=ovr)
    v = p.volumes
    got = {
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
    diffs = []
    for col, want in case["record"].items():
        if col in ("configKey", "blockX", "blockY", "blockZ", "folding"):
            continue
        w = unhex(want)
        if got[col] != w:
            diffs.append((col, got[col], w))
    per = [float(x).hex() for x in p.l1_cycles.per_access]
    if per != case["per_access"]:
        diffs.append(("per_access", per[:4], case["per_access"][:4]))
    for lvl, d in case["per_field_down"].items():
        gv = getattr(v, lvl).per_field_down
        for f, w in d.items():
            if gv[f] != unhex(w):
                diffs.append((lvl, f, gv[f], unhex(w)))
    return diffs


@pytest.mark.parametrize("idx", range(len(load("evaluations"))))
def test_evaluate_kernel_bit_exact_vs_reference(idx):
    case = load("evaluations")[idx]
    diffs = _compare_eval(case)
    assert not diffs, diffs


def test_block_and_wave_integers_vs_reference():
    for case in load("evaluations"):
        if "block_ints" not in case:
            continue
        k = gvo.kernel_from_dict(case["spec"])
        m = machine_from_dict(case["machine"])
        for bi in case["block_ints"]:
            grp = gvo.block_group(k.launch, bi["block"])
            r32 = gvo.grid_iteration(k, grp, m.sector_bytes)
            assert [[f, kd, c.unique_count, c.total_count] for (f, kd), c in r32.per_field.items()] == bi["sector"]
            r128 = gvo.grid_iteration(k, grp, m.l1_line_bytes, kinds=("load",))
            assert [[f, kd, c.unique_count, c.total_count] for (f, kd), c in r128.per_field.items()] == bi["line"]
        waves = {}
        for wi in case["wave_ints"]:
            w = gvo.Wave(wi["index"], wi["start"], wi["count"])
            fp = wave_footprint(k, w, m.sector_bytes)
            waves[w.index] = (w, fp)
            assert {f: s.count for f, s in fp.load_sets.items()} == wi["load"]
            assert fp.store_counts == wi["store"]
            assert fp.alloc_count == wi["alloc"]
        for ov in case["overlaps"]:
            (wc, fc), (wp, fpv) = waves[ov["curr"]], waves[ov["prev"]]
            got = {f: fc.load_sets[f].intersection_count(fpv.load_sets[f]) for f in fc.load_sets}
            assert got == ov["per_field"]


def test_block_and_wave_stats_bit_exact():
    for case in load("evaluations")[:6]:
        k = gvo.kernel_from_dict(case["spec"])
        m = machine_from_dict(case["machine"])
        bsz, wsz, ovr = case["sampling"]
        bs = gvo.sample_block_stats(k, m, bsz)
        for key, d in case["block_stats"].items():
            assert {f: float(v).hex() for f, v in getattr(bs, key).items()} == d, key
        ws = gvo.sample_wave_stats(k, m, wsz, ovr)
        for key in ("load_unique", "load_overlap", "store_unique"):
            assert {f: float(v).hex() for f, v in getattr(ws, key).items()} == case["wave_stats"][key]
        for key in ("prev_unique_total", "alloc_total", "wave_lups"):
            assert float(getattr(ws, key)).hex() == case["wave_stats"][key]
        assert ws.has_predecessor == case["wave_stats"]["has_predecessor"]


def test_rank_sweep_order_identical_to_reference():
    for sw in load("sweeps"):
        fam = gvo.KernelFamily(sw["kind"], tuple(sw["grid"]), radius=sw["radius"])
        cfgs = gvo.enumerate_sweep(sw["threads"], foldings=sw["foldings"])
        rows = gvo.rank_sweep(fam, cfgs, gvo.v100_preset(), wave_samples=1, block_samples=2, skip_invalid=True)
        assert [r.config.key for r in rows] == sw["order"]
        assert [float(r.prediction.glups).hex() for r in rows] == sw["glups"]


def _rand_kernel(rng, divmod_ok):
    coords = ("tidx", "tidy", "tidz", "bidx", "bidy", "bidz")
    block = [(1, 1, 1), (4, 1, 1), (8, 2, 1), (16, 2, 2), (32, 2, 1), (7, 3, 2), (33, 1, 2), (64, 2, 1)][rng.integers(0, 8)]
    grid = [(1, 1, 1), (2, 1, 1), (2, 2, 1), (3, 2, 2), (5, 3, 2)][rng.integers(0, 5)]
    names = [f"f{i}" for i in range(int(rng.integers(1, 4)))]
    fields = tuple(gvo.Field(n, 8, (1 << 20,), alignment=int(rng.choice([0, -1, 8, 100]))) for n in names)
    acc = []
    for _ in range(int(rng.integers(1, 7))):
        n = names[rng.integers(0, len(names))]
        terms = " + ".join(f"{coords[rng.integers(0, 6)]} * {int(rng.integers(-64, 65))}"
                           for _ in range(int(rng.integers(0, 5)))) or "0"
        text = f"{n} + ({terms}) + {int(rng.integers(-256, 257))}"
        if divmod_ok and rng.integers(0, 2):
            text = f"{n} + (({terms}) {['//', '%'][rng.integers(0, 2)]} {int(rng.choice([2, 4, 32, 100]))})"
        acc.append(gvo.Access(n, ["load", "store"][rng.integers(0, 2)], gvo.parse(text, fields=names),
                              int(rng.integers(1, 4))))
    return gvo.KernelDescriptor(fields=fields, accesses=tuple(acc), launch=gvo.LaunchConfig(block, grid))


def test_random_kernels_vs_oracle():
    rng = np.random.default_rng(7)
    for i in range(300):
        k = _rand_kernel(rng, divmod_ok=i % 2 == 0)
        nb = k.launch.total_blocks
        cnt = int(rng.integers(1, nb + 1))
        start = int(rng.integers(0, nb - cnt + 1))
        g = int(rng.choice([1, 8, 24, 32, 128]))
        grp = CollaborativeGroup(k.launch, np.arange(start, start + cnt, dtype=np.int64), "L2")
        r = gvo.grid_iteration(k, grp, g)
        got = {(f, kd): (c.unique_count, c.total_count) for (f, kd), c in r.per_field.items()}
        assert got == ora.footprint(k, grp.block_linear, g), (i, [gvo.render(a.expr) for a in k.accesses])


def test_random_kernels_l1_cycles_vs_oracle():
    rng = np.random.default_rng(11)
    m = gvo.v100_preset()
    for i in range(120):
        k = _rand_kernel(rng, divmod_ok=i % 3 == 0)
        b = int(rng.integers(0, k.launch.total_blocks))
        est = gvo.volumes.l1_register_cycles(k, m, gvo.block_group(k.launch, b))
        cyc, per = ora.l1_cycles(k, m, b)
        assert est.cycles_per_lup == cyc and est.per_access == per, i


def test_lbm_and_layout_variants_vs_oracle():
    m = gvo.b200_preset()
    cases = [gvo.generate_lbm_d3q15((64, 32, 32), (16, 2, 2)), gvo.generate_lbm_d3q15((64, 32, 32), (1, 8, 4)),
             gvo.generate_star_stencil(3, (64, 64, 64), (8, 8, 2), "2z")]
    for k in cases:
        p = gvo.evaluate_kernel(k, m)
        ev = ora.evaluate_kernel(k, m)
        assert p.glups == ev["glups"] and p.limiter == ev["limiter"]
        assert p.volumes.dram_load.v_down == ev["volumes"]["dram_load"]["down"]


def test_errors_match_reference_class_and_message():
    for case in load("errors"):
        k = gvo.kernel_from_dict(case["spec"])
        m = machine_from_dict(case["machine"])
        try:
            gvo.evaluate_kernel(k, m, **case["kw"])
            got = None
        except Exception as exc:  # noqa: BLE001
            got = [type(exc).__name__, str(exc)]
        assert got == case["error"], (case["spec"]["accesses"], case["kw"], got)


def test_split_ranges_forced_small_capacity():
    """Run the parity checks in a subprocess whose engine may keep only 96
    intervals in shared memory: every unit then splits into many key ranges
    (queued to other CTAs, clipped, re-split) — results must not change."""
    import os
    import subprocess
    import sys

    env = dict(os.environ, GVO_SMEM_ELEMS="96")
    tests = ["tests/test_gpu_parity.py::test_footprints_match_reference_golden",
             "tests/test_gpu_parity.py::test_block_and_wave_integers_vs_reference",
             "tests/test_gpu_parity.py::test_rank_sweep_order_identical_to_reference",
             "tests/test_gpu_parity.py::test_random_kernels_vs_oracle"]
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", *tests], env=env,
                       capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def _interleaved_kernel(rng, W=16, H=8, D=6):
    """A field with Q interleaved 8-byte components per cell (zyxf layout), read
    by pull loads q <- cell + c_q (c_q random neighbour offsets) and written in
    place: the translate classes whose residues tile a cell, which the set
    engine covers by segment boxes (k_sets.cu cover_segments)."""
    Q = int(rng.choice([3, 5, 9, 15, 27]))
    block = [(4, 2, 1), (8, 1, 2), (2, 4, 2), (16, 2, 1), (1, 4, 2), (4, 4, 2)][rng.integers(0, 6)]
    grid = (W // block[0], H // block[1], D // block[2])
    fields = (gvo.Field("src", 8, (W * H * D * Q,), alignment=int(rng.choice([0, 8, 24]))),
              gvo.Field("dst", 8, (W * H * D * Q,), alignment=0))
    full = rng.integers(0, 3) > 0  # every component read (residues tile the cell)
    comps = range(Q) if full else sorted(set(int(v) for v in rng.integers(0, Q, size=max(1, Q // 2))))
    x = f"(tidx + bidx * {block[0]})"
    y = f"(tidy + bidy * {block[1]})"
    z = f"(tidz + bidz * {block[2]})"
    acc = []
    for q in comps:
        dx, dy, dz = (int(v) for v in rng.integers(-1, 2, size=3))
        text = f"src + ((({x} + {-dx}) * {Q} + {q}) + (({y} + {-dy}) * {W} + ({z} + {-dz}) * {W * H}) * {Q}) * 8"
        acc.append(gvo.Access("src", "load", gvo.parse(text, fields=["src", "dst"]), 1))
        text = f"dst + (({x} * {Q} + {q}) + ({y} * {W} + {z} * {W * H}) * {Q}) * 8"
        acc.append(gvo.Access("dst", "store", gvo.parse(text, fields=["src", "dst"]), 1))
    return gvo.KernelDescriptor(fields=fields, accesses=tuple(acc), launch=gvo.LaunchConfig(block, grid))


def test_interleaved_translates_vs_oracle():
    rng = np.random.default_rng(2107)
    for i in range(60):
        k = _interleaved_kernel(rng)
        nb = k.launch.total_blocks
        cnt = int(rng.integers(1, nb + 1))
        start = int(rng.integers(0, nb - cnt + 1))
        g = int(rng.choice([8, 24, 32, 128]))
        grp = CollaborativeGroup(k.launch, np.arange(start, start + cnt, dtype=np.int64), "L2")
        r = gvo.grid_iteration(k, grp, g)
        got = {(f, kd): (c.unique_count, c.total_count) for (f, kd), c in r.per_field.items()}
        assert got == ora.footprint(k, grp.block_linear, g), (i, k.launch, len(k.accesses) // 2)


def test_interleaved_evaluations_vs_oracle():
    rng = np.random.default_rng(143)
    m = gvo.b200_preset()
    for i in range(8):
        k = _interleaved_kernel(rng)
        ov = int(rng.choice([0, 3, 7]))
        p = gvo.evaluate_kernel(k, m, override_blocks_per_wave=ov or None)
        ev = ora.evaluate_kernel(k, m, override=ov or None)
        assert p.glups == ev["glups"] and p.limiter == ev["limiter"], i
        assert p.volumes.dram_load.v_down == ev["volumes"]["dram_load"]["down"], i


def test_interleaved_long_rows_vs_oracle():
    """Rows of 64 cells: boundary layers with partial component sets become
    pattern runs (k_sets.cu emit_pattern / bm_pattern)."""
    rng = np.random.default_rng(1143)
    for i in range(40):
        k = _interleaved_kernel(rng, W=64, H=4, D=4)
        nb = k.launch.total_blocks
        cnt = int(rng.integers(max(1, nb // 4), nb + 1))
        start = int(rng.integers(0, nb - cnt + 1))
        g = int(rng.choice([8, 24, 32, 128]))
        grp = CollaborativeGroup(k.launch, np.arange(start, start + cnt, dtype=np.int64), "L2")
        r = gvo.grid_iteration(k, grp, g)
        got = {(f, kd): (c.unique_count, c.total_count) for (f, kd), c in r.per_field.items()}
        assert got == ora.footprint(k, grp.block_linear, g), (i, k.launch, len(k.accesses) // 2, g)


def test_rank_sweep_sharded_matches_rank_sweep():
    """The multi-GPU sweep API (one all-gather + device ranking) on one rank
    with a real NCCL process group, and without one: same order and records
    as rank_sweep."""
    import os
    import socket

    import torch.distributed as dist

    m = gvo.b200_preset()
    fam = gvo.KernelFamily("stencil", (64, 64, 64), radius=3)
    cfgs = list(gvo.enumerate_sweep(128, foldings=("none", "2y", "2z"))) + list(gvo.enumerate_sweep(256))
    ref = gvo.rank_sweep(fam, cfgs, m, skip_invalid=True)
    kept, order, rec = gvo.rank_sweep_sharded(fam, cfgs, m, skip_invalid=True)
    assert [kept[i].key for i in order] == [r.config.key for r in ref]
    np.testing.assert_array_equal(rec[order], np.asarray(ref.records)[ref.order])
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        kept2, order2, rec2 = gvo.rank_sweep_sharded(fam, cfgs, m, skip_invalid=True)
    finally:
        dist.destroy_process_group()
    assert [k.key for k in kept2] == [k.key for k in kept]
    np.testing.assert_array_equal(order2, order)
    np.testing.assert_array_equal(rec2, rec)


def test_sweep_host_matches_eval_and_rank():
    """gvo_sweep_host (evaluate + rank in one call) == gvo_eval_configs_host
    followed by the device ranking."""
    from paper_2107_01143_b200 import _native

    m = gvo.b200_preset()
    fam = gvo.KernelFamily("stencil", (64, 64, 64), radius=2)
    cfgs = list(gvo.enumerate_sweep(64, foldings=("none", "2z"))) + list(gvo.enumerate_sweep(512))
    kept, kernels, res, order = gvo.perf.evaluate_sweep(fam, cfgs, m, skip_invalid=True)
    batch = gvo._engine.Batch()
    for cfg, (k, launch, flops) in zip(kept, kernels):
        batch.add(k.fields, k.accesses, launch, flops, m, None, gvo._engine.FOLD_RANK[cfg.folding])
    ca = batch.config_array()
    ctx = _native.context()
    n, F = len(ca), ctx.max_fields
    S, W = _native.effective_sampling(5, 2)
    stride = _native.counts_stride(F, S, W)
    counts = np.zeros((n, stride), dtype=np.int64)
    rec = np.zeros((n, _native.RECORD_LEN))
    o = np.zeros(n, dtype=np.int64)
    ctx.check(_native.lib().gvo_sweep_host(ctx.h, _native._ptr(ca), n, _native.C.byref(_native.Sampling(5, 2, 0, 7, 0)),
                                           F, _native._ptr(counts), None, _native._ptr(rec), _native._ptr(o)))
    np.testing.assert_array_equal(o, order)
    np.testing.assert_array_equal(rec, res.records)
