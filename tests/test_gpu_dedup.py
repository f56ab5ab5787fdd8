"""Cross-configuration sharing of identical set problems (csrc/k_dedup.cu)
must not change a single number: every count, statistic, record and
per-access L1 figure with sharing on equals the run with sharing off, on a
structured slice of C5 where sharing is dense (every alignment and every L2
variant of each template at a few launch shapes, stencil and LBM, two
batches so that later batches copy from earlier ones)."""

from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from paper_2107_01143_b200 import _native, workloads as W

pytestmark = pytest.mark.gpu

SHAPES = {(16, 2, 32), (32, 4, 2), (64, 1, 4), (1, 1, 64), (32, 2, 2), (8, 8, 4), (128, 1, 1)}


def _slice():
    sp = W.space("C5")
    keep = np.array([tuple(int(v) for v in b) in SHAPES for b in sp.block])
    return sp.subset(np.flatnonzero(keep))


def _run(ctx, cfgs, on: bool):
    L = _native.lib()
    ctx.check(L.gvo_set_dedup(ctx.h, 1 if on else 0))
    L.gvo_dedup_stats(ctx.h, 1, None, None)
    out = ctx.eval_configs_host(cfgs, 5, 2, 0, want_l1_access=True)
    units, follow = C.c_int64(), C.c_int64()
    L.gvo_dedup_stats(ctx.h, 0, C.byref(units), C.byref(follow))
    return out, units.value, follow.value


@pytest.fixture()
def small_batches():
    """Batches of 16,384 configurations for the test (the slice then spans
    three batches: later batches copy from earlier ones), default after."""
    ctx = _native.context()
    ctx.check(_native.lib().gvo_set_batch(ctx.h, 16384))
    yield ctx
    ctx.check(_native.lib().gvo_set_batch(ctx.h, 65536))


def test_sharing_changes_nothing_on_structured_c5_slice(small_batches):
    sp = _slice()
    assert len(sp) > 16384  # at least two batches: cross-batch sharing
    ctx = small_batches
    cfgs = sp.config_array(ctx)
    try:
        off, _, f_off = _run(ctx, cfgs, False)
        on, units, follow = _run(ctx, cfgs, True)
    finally:
        _native.lib().gvo_set_dedup(ctx.h, 1)
    assert f_off == 0
    assert follow > units // 2, (units, follow)  # the slice is mostly shared
    assert (on["counts"][:, _native.C_STATUS] == 0).all()
    for k in ("counts", "l1_access"):
        assert np.array_equal(on[k], off[k]), k
    for k in ("stats", "records", "field_down"):
        assert np.array_equal(on[k].view(np.int64), off[k].view(np.int64)), k


def test_sharing_respects_machine_integer_parameters():
    """Machines that differ in an integer parameter (sector size / SM count)
    never share; machines that differ only in capacities do."""
    import dataclasses

    from paper_2107_01143_b200.gvo.machine import b200_preset

    m = b200_preset()
    ms = [m, dataclasses.replace(m, name="l2-half", l2_capacity_bytes=m.l2_capacity_bytes // 2),
          dataclasses.replace(m, name="sm-100", sm_count=100)]
    sp = W.space_c3(m, radii=(2,), components=(2,), alignments=(0, 32, 8), machines=ms, machines_idx=(0, 1, 2))
    ctx = _native.context()
    cfgs = sp.config_array(ctx)
    try:
        off, _, _ = _run(ctx, cfgs, False)
        on, units, follow = _run(ctx, cfgs, True)
    finally:
        _native.lib().gvo_set_dedup(ctx.h, 1)
    assert follow > 0
    for k in ("counts", "l1_access"):
        assert np.array_equal(on[k], off[k]), k
    assert np.array_equal(on["records"].view(np.int64), off["records"].view(np.int64))


def test_plan_sharing_with_failing_leaders():
    """Plan sharing (k_setup.cu): configurations equal up to field-base
    translation and machine capacities take their leader's plan; a leader
    whose plan is not shareable (here: a FootprintError, 1024-thread blocks
    on a machine limited to 512 threads per block) leaves every follower to
    compute its own — statuses and records equal the unshared run's."""
    import dataclasses

    from paper_2107_01143_b200.gvo.machine import b200_preset

    m = b200_preset()
    ms = [m, dataclasses.replace(m, name="l2-quarter", l2_capacity_bytes=m.l2_capacity_bytes // 4),
          dataclasses.replace(m, name="tpb-512", max_threads_per_block=512)]
    sp = W.space_c3(m, radii=(1,), components=(2,), alignments=(0, 8, 16, 136), machines=ms, machines_idx=(0, 1, 2))
    ctx = _native.context()
    cfgs = sp.config_array(ctx)
    try:
        off, _, _ = _run(ctx, cfgs, False)
        on, _, follow = _run(ctx, cfgs, True)
    finally:
        _native.lib().gvo_set_dedup(ctx.h, 1)
    st = on["counts"][:, _native.C_STATUS]
    assert (st != 0).sum() > 0 and (st == 0).sum() > 0
    assert follow > 0
    for k in ("counts", "l1_access"):
        assert np.array_equal(on[k], off[k]), k
    for k in ("stats", "records"):
        assert np.array_equal(on[k].view(np.int64), off[k].view(np.int64)), k


def test_pinned_sweep_host_pipelines_copies_identically(small_batches):
    """gvo_sweep_host_ex with page-locked outputs copies every batch to the
    host behind the next batches' kernels (a second stream); every output
    equals the pageable path's (one copy after the last batch)."""
    import torch

    sp = _slice()
    ctx = small_batches
    cfgs = np.ascontiguousarray(sp.config_array(ctx))
    assert len(cfgs) > 16384
    ref = ctx.sweep_host(cfgs, 5, 2, 0)
    F, S, Wn = ref["F"], ref["S"], ref["W"]
    n, A = len(cfgs), ctx.max_accesses
    pin = lambda shape, dt: torch.zeros(shape, dtype=dt, pin_memory=True).numpy()  # noqa: E731
    counts = pin((n, _native.counts_stride(F, S, Wn)), torch.int64)
    stats = pin((n, _native.stats_len(F)), torch.float64)
    rec = pin((n, _native.RECORD_LEN), torch.float64)
    fd = pin((n, 4, F), torch.float64)
    l1 = pin((n, A, 3), torch.int64)
    order = pin((n,), torch.int64)
    smp = _native.Sampling(5, 2, 0, 7, 0)
    ctx.check(_native.lib().gvo_sweep_host_ex(ctx.h, _native._ptr(cfgs), n, C.byref(smp), F, _native._ptr(counts),
                                              _native._ptr(stats), _native._ptr(rec), _native._ptr(fd),
                                              _native._ptr(l1), A, _native._ptr(order)))
    assert np.array_equal(counts, ref["counts"])
    assert np.array_equal(l1, ref["l1_access"])
    assert np.array_equal(order, ref["order"])
    for got, want in ((stats, ref["stats"]), (rec, ref["records"]), (fd, ref["field_down"])):
        assert np.array_equal(got.view(np.int64), want.view(np.int64))
