"""Multi-GPU sweep: one process per GPU under
torch.distributed (NCCL over NVLink/NVSwitch on a B200 box).

Every rank validates the whole sweep on the host exactly as rank_sweep does
(perf.py:115-121), deals the configurations by estimated cost
(paper_2107_01143_b200.shard), evaluates its shard on its own GPU, and one
all-gather of fixed-size rows — the 37-double ranking record
(include/gvo_b200.h GVO_R_*), the configuration's global index (-1 for the
padding that equalises shard lengths) and its error header — precedes the
device ranking of the whole space in global order (gvo_rank_gathered), so
ties break by input order as the reference's stable sort does
(perf.py:131).  Every rank returns the same global order and records,
bit-identical to a single-GPU rank_sweep of the same configurations, and
every rank raises the reference's exception for the first failing
configuration (no rank is left waiting in the collective).
"""

from __future__ import annotations

from typing import Iterable, Mapping

import numpy as np

from .. import _native, shard
from . import _engine
from .kernels import KernelFamily, SweepConfig
from .machine import MachineDescriptor
from .perf import PerfError, SweepPlan

# error header columns gathered with every row (what raise_for_status reads)
_HDR = (_native.C_STATUS, _native.C_ERR_PHASE, _native.C_ERR_GROUP, _native.C_ERR_ACCESS, _native.C_FIRSTWAVE)


def rank_sweep_sharded(family: KernelFamily, configs: Iterable[SweepConfig], machine: MachineDescriptor,
                       fit_params: Mapping | None = None, *, block_samples: int = 5, wave_samples: int = 2,
                       override_blocks_per_wave: int | None = None, skip_invalid: bool = False,
                       group=None):
    """(kept configs, order, records): the sweep's valid configurations in
    input order, their global ranking (indices into kept) and their ranking
    records [len(kept)][RECORD_LEN], identical on every rank of ``group``."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    plan = SweepPlan(family, configs, machine, fit_params, skip_invalid=skip_invalid)
    n = len(plan)
    if n == 0:
        plan.raise_first_error(None, machine, block_samples, wave_samples, override_blocks_per_wave)
        raise PerfError("empty sweep")
    n_acc = np.array([len(t[0].accesses) for t in plan.templates], dtype=np.int64)[plan.tpl]
    mine = shard.shard_indices(shard.config_cost(plan.block, n_acc), world, rank)
    m = shard.pad_to(n, world)
    ctx = _native.context()
    dev = torch.device("cuda", ctx.device)
    R, H = _native.RECORD_LEN, len(_HDR)
    local = np.zeros((m, R + 1 + H), dtype=np.float64)
    local[:, R] = -1.0  # global index column (-1: padding)
    cfg_all = plan.config_array()
    if len(mine):
        out = ctx.eval_configs_host(cfg_all[mine], block_samples, wave_samples, override_blocks_per_wave or 0,
                                    want_field_down=False)
        local[: len(mine), :R] = out["records"]
        local[: len(mine), R] = mine
        local[: len(mine), R + 1:] = out["counts"][:, list(_HDR)]
    # gloo gathers host tensors, NCCL device tensors
    backend = dist.get_backend(group) if dist.is_initialized() else "none"
    t_local = torch.from_numpy(local)
    if backend == "nccl":
        t_local = t_local.to(dev)
    gathered = shard.gather_records(t_local, world, group) if world > 1 else t_local
    g = gathered.cpu().numpy()
    gidx = g[:, R].astype(np.int64)
    # the reference raises at the first failing configuration: every rank
    # sees every row's status, so every rank raises the same exception
    status = np.zeros(n, dtype=np.int64)
    valid = gidx >= 0
    status[gidx[valid]] = g[valid, R + 1].astype(np.int64)
    if status.any() or plan.build_error is not None:
        i = int(np.flatnonzero(status)[0]) if status.any() else None
        if i is not None:
            row = g[np.flatnonzero(gidx == i)[0]]
            counts = np.zeros((1, _native.C_HDR), dtype=np.int64)
            counts[0, list(_HDR)] = row[R + 1:].astype(np.int64)
            res = _engine.Result(0, 0, 0, counts, None, None, None, None)
            k, launch, _ = plan.kernel_row(i)
            _engine.raise_for_status(res, 0, k.with_launch(launch), machine, block_samples, wave_samples,
                                     override_blocks_per_wave)
        raise plan.build_error[1]
    # device ranking of the whole space in global order
    d_rows = torch.from_numpy(np.ascontiguousarray(g[:, :R])).to(dev)
    d_gidx = torch.from_numpy(gidx.copy()).to(dev)
    d_cfg = torch.from_numpy(cfg_all.view(np.uint8).copy()).to(dev)
    records = torch.empty((n, R), dtype=torch.float64, device=dev)
    order = torch.empty(n, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    _native.rank_gathered(d_rows.data_ptr(), d_gidx.data_ptr(), len(gidx), d_cfg.data_ptr(), n,
                          records.data_ptr(), order.data_ptr(), stream)
    return plan.configs, order.cpu().numpy(), records.cpu().numpy()
