"""Strong-scaling proxy on one GPU: C5 dealt to N ranks (bench.py's
sharing-group shards, and the plain cost round robin for comparison); each
shard evaluated alone on this GPU, device time per shard.  The N-GPU step
is bounded below by the slowest shard (plus one all-gather of the records
and the global ranking).  usage: python tools/shard_probe.py [N ...]"""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2107_01143_b200 import _native, shard, workloads as W  # noqa: E402
from paper_2107_01143_b200.gvo.machine import b200_preset  # noqa: E402

Ns = [int(a) for a in sys.argv[1:]] or [1, 2, 4, 8]
sp = W.space("C5", b200_preset())
ctx = _native.context()
L = _native.lib()
C = _native.C
cfg_all = sp.config_array(ctx)
ctx.sync_registries()
F = ctx.max_fields
S, Wn = _native.effective_sampling(5, 2)
stride = _native.counts_stride(F, S, Wn)
smp = _native.Sampling(5, 2, 0, 7, 0)
dev = torch.device("cuda", 0)
st = torch.cuda.current_stream().cuda_stream
cost = shard.config_cost(sp.block, sp.n_accesses()) * sp.kind_weight()
groups = sp.sharing_groups()


def run(idx):
    cfg = np.ascontiguousarray(cfg_all[idx])
    n = len(cfg)
    d_cfg = torch.from_numpy(cfg.view(np.uint8).copy()).to(dev)
    d_cnt = torch.zeros((n, stride), dtype=torch.int64, device=dev)
    d_rec = torch.zeros((n, _native.RECORD_LEN), dtype=torch.float64, device=dev)
    best = None
    for rep in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.check(L.gvo_eval_configs(ctx.h, C.c_void_p(d_cfg.data_ptr()), n, C.byref(smp), F,
                                     C.c_void_p(d_cnt.data_ptr()), None, C.c_void_p(d_rec.data_ptr()), None, None, 0,
                                     C.c_void_p(st)))
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if rep and (best is None or ms < best):
            best = ms
    return best


out = {}
for N in Ns:
    for how in ("groups", "round-robin"):
        if N == 1 and how == "round-robin":
            continue
        if how == "groups":
            parts = shard.group_shards(cost, groups, N) if N > 1 else [np.arange(len(sp))]
        else:
            parts = [shard.shard_indices(cost, N, r) for r in range(N)]
        ms = [run(p) for p in parts]
        out[f"{how}/{N}"] = {"max_ms": max(ms), "ms": [round(x, 1) for x in ms],
                             "configs_per_s_at_max": len(sp) / (max(ms) * 1e-3)}
        print(json.dumps({f"{how}/{N}": out[f"{how}/{N}"]}), flush=True)
