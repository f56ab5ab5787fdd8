"""Public seams beside the batched path against goldens made by the
unmodified reference (tests/golden/seams.json, tools/make_golden_seams.py):

* evaluate_bulk on 1000 random trees (reference test_expr.py:136-168;
  expr.py:281-304) — device bytecode interpreter, exact int64;
* estimate_volumes with injected BlockStats / WaveStats (volumes.py:421-445)
  and predict (perf.py:45-67) — device assembly (gvo_assemble_host /
  gvo_predict_host), bit-exact floats;
* rank_sweep over KernelFamily("file") (kernels.py:422-433) — spec files
  re-tiled per block on the batched path, identical ranked rows;
* naive_footprint_oracle == grid_iteration (footprint.py:474-507 contract).
"""

import dataclasses

import numpy as np
import pytest

from golden_util import load, unhex
from paper_2107_01143_b200 import gvo
from paper_2107_01143_b200.gvo.machine import machine_from_dict
from paper_2107_01143_b200.gvo.volumes import BlockStats, WaveStats

pytestmark = pytest.mark.gpu


def test_evaluate_bulk_matches_reference_on_random_trees():
    g = load("seams")
    block = tuple(g["block"])
    bad = []
    for case in g["bulk"]:
        tree = gvo.parse(case["expr"])
        env = {k: np.array(v, dtype=np.int64) for k, v in case["env"].items()}
        got = gvo.evaluate_bulk(tree, env, block, {})
        if got.tolist() != case["out"]:
            bad.append((case["expr"], got.tolist()[:4], case["out"][:4]))
    assert not bad, bad[:3]


def _stats(d, cls):
    kw = {}
    for f in dataclasses.fields(cls):
        v = d[f.name]
        kw[f.name] = {k: unhex(x) for k, x in v.items()} if isinstance(v, dict) else unhex(v)
    return cls(**kw)


def test_estimate_volumes_with_injected_stats_bit_exact():
    g = load("seams")
    kernels = [gvo.kernel_from_dict(s) for s in g["injected_kernels"]]
    bad = []
    for case in g["injected"]:
        k = kernels[case["kernel"]]
        m = machine_from_dict(case["machine"])
        bs = _stats(case["block_stats"], BlockStats)
        ws = _stats(case["wave_stats"], WaveStats)
        vols = gvo.estimate_volumes(k, m, block_stats=bs, wave_stats=ws)
        for lvl, want in case["volumes"].items():
            got = dataclasses.asdict(getattr(vols, lvl))
            for key, w in want.items():
                gv = got[key]
                if isinstance(w, dict):
                    if {a: float(b).hex() for a, b in gv.items()} != w:
                        bad.append((lvl, key))
                elif w is None or isinstance(w, bool):
                    if gv != w:
                        bad.append((lvl, key, gv, w))
                elif float(gv).hex() != w:
                    bad.append((lvl, key, float(gv).hex(), w))
        p = gvo.predict(k, m, vols, gvo.l1_register_cycles(k, m))
        if float(p.glups).hex() != case["glups"] or p.limiter != case["limiter"]:
            bad.append(("predict", float(p.glups).hex(), case["glups"]))
        if {a: float(b).hex() for a, b in p.times.items()} != case["times"]:
            bad.append(("times",))
    assert not bad, bad[:5]


def test_file_family_sweep_ranked_identically():
    m = gvo.v100_preset()
    for case in load("seams")["file_sweeps"]:
        fam = gvo.KernelFamily("file", tuple(case["grid"]), spec=case["spec"])
        cfgs = [gvo.SweepConfig(tuple(b), f) for b, f in case["configs"]]
        rows = gvo.rank_sweep(fam, cfgs, m, block_samples=2, wave_samples=1, skip_invalid=True)
        got = [[list(r.config.block_dim), r.config.folding, float(r.prediction.glups).hex(), r.prediction.limiter]
               for r in rows]
        assert got == case["rows"]


def test_file_family_refuses_folding_without_skip():
    spec = load("seams")["file_sweeps"][1]["spec"]
    fam = gvo.KernelFamily("file", (64, 64, 64), spec=spec)
    with pytest.raises(gvo.KernelError, match="thread folding is not available"):
        gvo.rank_sweep(fam, [gvo.SweepConfig((8, 8, 1)), gvo.SweepConfig((8, 8, 1), "2z")], gvo.v100_preset())


@pytest.mark.parametrize("level", ["block", "wave"])
def test_naive_footprint_oracle_equals_grid_iteration(level):
    k = gvo.generate_star_stencil(2, (64, 32, 32), (16, 2, 4), "2z")
    m = gvo.v100_preset()
    if level == "block":
        grp = gvo.representative_blocks(k, 3)[1]
    else:
        grp = gvo.wave_group(k.launch, gvo.build_waves(k.launch, m, 12)[1])
    for g in (8, 32, 128):
        a = gvo.grid_iteration(k, grp, g)
        b = gvo.naive_footprint_oracle(k, grp, g)
        assert a.per_field == b.per_field
