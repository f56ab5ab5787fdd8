"""End-to-end C5 through gvo_sweep_host: pinned vs pageable host outputs vs
the device-resident call (GPU).  usage: python tools/e2e_probe.py"""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2107_01143_b200 import _native, workloads as W  # noqa: E402
from paper_2107_01143_b200.gvo.machine import b200_preset  # noqa: E402

sp = W.space("C5", b200_preset())
ctx = _native.context()
L, C = _native.lib(), _native.C
cfg = np.ascontiguousarray(sp.config_array(ctx))
ctx.sync_registries()
n, F = len(cfg), ctx.max_fields
S, Wn = _native.effective_sampling(5, 2)
stride = _native.counts_stride(F, S, Wn)
R = _native.RECORD_LEN
smp = _native.Sampling(5, 2, 0, 7, 0)
dev = torch.device("cuda", 0)
st = torch.cuda.current_stream().cuda_stream
d_cfg = torch.from_numpy(cfg.view(np.uint8).copy()).to(dev)
d_cnt = torch.zeros((n, stride), dtype=torch.int64, device=dev)
d_st = torch.zeros((n, _native.stats_len(F)), dtype=torch.float64, device=dev)
d_rec = torch.zeros((n, R), dtype=torch.float64, device=dev)
d_ord = torch.zeros(n, dtype=torch.int64, device=dev)


def device():
    ctx.check(L.gvo_eval_configs(ctx.h, C.c_void_p(d_cfg.data_ptr()), n, C.byref(smp), F, C.c_void_p(d_cnt.data_ptr()),
                                 C.c_void_p(d_st.data_ptr()), C.c_void_p(d_rec.data_ptr()), None, None, 0,
                                 C.c_void_p(st)))
    ctx.check(L.gvo_rank(ctx.h, C.c_void_p(d_rec.data_ptr()), C.c_void_p(d_cfg.data_ptr()), n,
                         C.c_void_p(d_ord.data_ptr()), C.c_void_p(st)))
    torch.cuda.synchronize()


def host(pin):
    mk = (lambda s, dt: torch.zeros(s, dtype=dt, pin_memory=True).numpy()) if pin else \
        (lambda s, dt: np.zeros(s, dtype={torch.int64: np.int64, torch.float64: np.float64}[dt]))
    cfg_h = cfg
    if pin:
        buf = torch.empty(cfg.nbytes, dtype=torch.uint8, pin_memory=True).numpy()
        buf[:] = cfg.view(np.uint8).reshape(-1)
        cfg_h = buf.view(cfg.dtype)
    cnt, sts, rec, order = mk((n, stride), torch.int64), mk((n, _native.stats_len(F)), torch.float64), \
        mk((n, R), torch.float64), mk((n,), torch.int64)

    def go():
        ctx.check(L.gvo_sweep_host(ctx.h, _native._ptr(cfg_h), n, C.byref(smp), F, _native._ptr(cnt), _native._ptr(sts),
                                   _native._ptr(rec), _native._ptr(order)))
    return go


for name, fn in (("device", device), ("pinned", host(True)), ("pageable", host(False))):
    fn()
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    print(f"{name:9s} best {min(ts)*1e3:8.1f} ms  -> {n/min(ts)/1e6:.3f} M configs/s", flush=True)
