"""Multi-GPU sweep: one process per GPU under
torch.distributed (NCCL over NVLink/NVSwitch on a B200 box).

Every rank validates the whole sweep on the host exactly as rank_sweep does
(perf.py:115-121), deals the configurations by estimated cost
(paper_2107_01143_b200.shard), evaluates its shard on its own GPU, and one
all-gather of the fixed-size per-config records (the 37-double ranking
record, include/gvo_b200.h GVO_R_*) precedes the device ranking of the
gathered records with the reference's key (perf.py:131).  Every rank returns
the same global order and records, bit-identical to a single-GPU rank_sweep
of the same configurations.
"""

from __future__ import annotations

from typing import Iterable, Mapping

import numpy as np

from .. import _native, shard
from . import _engine
from .kernels import KernelFamily, SweepConfig
from .machine import MachineDescriptor
from .perf import PerfError, evaluate_sweep


def rank_sweep_sharded(family: KernelFamily, configs: Iterable[SweepConfig], machine: MachineDescriptor,
                       fit_params: Mapping | None = None, *, block_samples: int = 5, wave_samples: int = 2,
                       override_blocks_per_wave: int | None = None, skip_invalid: bool = False,
                       group=None):
    """(kept configs, order, records): the sweep's valid configurations in
    input order, their global ranking (indices into kept) and their ranking
    records [len(kept)][RECORD_LEN], identical on every rank."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    configs = list(configs)
    if not configs:
        raise PerfError("empty sweep")
    kept, blocks, n_acc = [], [], []
    templates: dict = {}
    for cfg in configs:  # the same validation on every rank: identical kept lists
        try:
            launch, _ = family.launch_of(cfg)
            key = family.template_key(cfg)
            if key not in templates:
                templates[key] = family.build(cfg)
        except ValueError:
            if skip_invalid:
                continue
            raise
        kept.append(cfg)
        blocks.append(launch.block_dim)
        n_acc.append(len(templates[key].accesses))
    n = len(kept)
    mine = shard.shard_indices(shard.config_cost(np.asarray(blocks), np.asarray(n_acc)), world, rank)
    m = shard.pad_to(n, world)
    dev = torch.device("cuda", _native.context().device)
    local = torch.zeros((m, _native.RECORD_LEN + 1), dtype=torch.float64, device=dev)
    local[:, -1] = -1.0  # global index column (-1: padding)
    if len(mine):
        _, _, res, _ = evaluate_sweep(family, [kept[i] for i in mine], machine, fit_params,
                                      block_samples=block_samples, wave_samples=wave_samples,
                                      override_blocks_per_wave=override_blocks_per_wave)
        local[: len(mine), :-1] = torch.from_numpy(np.ascontiguousarray(res.records)).to(dev)
        local[: len(mine), -1] = torch.from_numpy(mine.astype(np.float64)).to(dev)
    gathered = shard.gather_records(local, world) if world > 1 else local
    idx = gathered[:, -1].to(torch.int64)
    keep = idx >= 0
    records = torch.empty((n, _native.RECORD_LEN), dtype=torch.float64, device=dev)
    records[idx[keep]] = gathered[keep, :-1]
    # device ranking of all records (tie-break on block dims / folding as perf.py:131)
    batch = _engine.Batch()
    for cfg, b in zip(kept, blocks):
        launch, flops = family.launch_of(cfg)
        k = templates[family.template_key(cfg)]
        batch.add(k.fields, k.accesses, launch, flops, machine, fit_params, _engine.FOLD_RANK[cfg.folding])
    cf = torch.from_numpy(np.ascontiguousarray(batch.config_array()).view(np.uint8).copy()).to(dev)
    order = torch.empty(n, dtype=torch.int64, device=dev)
    _native.rank_device(records.data_ptr(), cf.data_ptr(), n, order.data_ptr(),
                        torch.cuda.current_stream(dev).cuda_stream)
    return kept, order.cpu().numpy(), records.cpu().numpy()
