"""Host-side columnar sweep plan (gvo.perf.SweepPlan) against the per-
configuration path it replaces: family.launch_of / template_key for every
configuration, in the reference loop's order (perf.py:115-121), with a
stand-in registry instead of the device context (no GPU needed)."""
import random

import numpy as np
import pytest

from paper_2107_01143_b200 import _native, gvo
from paper_2107_01143_b200.gvo import _engine, perf
from paper_2107_01143_b200.gvo.kernels import SweepConfig


class _Registry:
    def __init__(self):
        self.t, self.m = {}, {}

    def machine_id(self, machine, fit_params=None):
        return self.m.setdefault(_native.machine_key(machine, fit_params), len(self.m))

    def template_id(self, fields, accesses):
        return self.t.setdefault(_native.template_key(fields, accesses), len(self.t))


@pytest.fixture()
def registry(monkeypatch):
    reg = _Registry()
    monkeypatch.setattr(_native, "context", lambda: reg)
    perf._TPL_CACHE.clear()
    yield reg
    perf._TPL_CACHE.clear()


def _expected(fam, cfgs, skip):
    kept, err = [], None
    for i, c in enumerate(cfgs):
        try:
            launch, fl = fam.launch_of(c)
        except ValueError as exc:
            if skip:
                continue
            err = (i, type(exc), str(exc))
            break
        kept.append((c, launch, fl))
    return kept, err


@pytest.mark.parametrize("seed", range(6))
def test_sweep_plan_matches_per_config_launches(registry, seed):
    rng = random.Random(seed)
    m = gvo.b200_preset()
    fams = [gvo.KernelFamily("stencil", (64, 32, 16), radius=2), gvo.KernelFamily("lbm", (32, 32, 32)),
            gvo.KernelFamily("stencil", (640, 640, 640), radius=4)]
    folds = ["none", "2y", "2z", "3x", None, "none"]
    for _ in range(40):
        fam = rng.choice(fams)
        cfgs = [SweepConfig(tuple(rng.choice([1, 2, 4, 8, 16, 32, 3]) for _ in range(3)), rng.choice(folds))
                for _ in range(rng.randint(1, 40))]
        for skip in (True, False):
            kept, err = _expected(fam, cfgs, skip)
            if not kept:
                continue
            p = perf.SweepPlan(fam, cfgs, m, skip_invalid=skip)
            assert len(p) == len(kept)
            assert p.block.tolist() == [list(k[1].block_dim) for k in kept]
            assert p.grid.tolist() == [list(k[1].grid_dim) for k in kept]
            assert p.wpt.tolist() == [k[1].work_per_thread for k in kept]
            assert p.flops.tolist() == [k[2] for k in kept]
            assert p.fold_rank.tolist() == [_engine.FOLD_RANK[k[0].folding] for k in kept]
            tids = [p.templates[t][1] for t in p.tpl.tolist()]
            for (c, _, _), tid in zip(kept, tids):
                k = fam.build(c)
                assert tid == registry.template_id(k.fields, k.accesses)
            if err is None:
                assert p.build_error is None
            else:
                assert p.build_error[0] == err[0] and isinstance(p.build_error[1], err[1])
                assert str(p.build_error[1]) == err[2]
            a = p.config_array()
            assert np.array_equal(a["block"], p.block) and np.array_equal(a["fold_rank"], p.fold_rank)
