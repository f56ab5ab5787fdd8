"""Benchmark: kernel configurations evaluated per second (BASELINE.json metric).

Workload (BASELINE.json configs[1]): the range-four 3D25pt
star stencil on a 640^3 grid, full block-size sweep — every power-of-two
block (X, Y <= 512, Z <= 64) with X*Y*Z <= 1024 threads, 264 shapes of which
246 tile the grid (skip_invalid) — evaluated with the B200 machine
parameters, default fits, block_samples=5, wave_samples=2, then ranked.
A step = evaluate + rank the whole sweep.  With N GPUs each rank evaluates
its own 246-config shard (the same sweep with field alignment 8*rank bytes,
so every rank's configs are distinct), records are all-gathered over NCCL
and the global ranking runs on the device (weak scaling).

--workload C1|C3|C4|C5 runs the other BASELINE.json configuration spaces
(paper_2107_01143_b200/workloads.py): the space is dealt to ranks by
estimated cost (shard.py), one NCCL all-gather of the records, device rank
of the whole space (strong scaling: total work fixed).

--impl reference times the reference's own CPU estimator (pip-installed
unmodified under baseline/_ref; the CPU oracle port if that is missing) on a
bounded sample of the same workload with all host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

GRID = (640, 640, 640)
RADIUS = 4
# kernels per step (one batch): k_setup, k_sets (warp statistics fused),
# k_finish, k_rank_small (n <= 2048)
LAUNCHES_PER_STEP = 4


def b200_machine():
    from paper_2107_01143_b200 import gvo

    return gvo.b200_preset()


# ---------------------------------------------------------------- device arm
WORKLOADS = {
    "C1": "C1: 2D5pt Jacobi 256^2, block 32x4x1 (PR1 oracle config)",
    "C2": "C2: 3D25pt r4 640^3 full power-of-two block sweep (246 valid configs/rank), "
          "B200 machine params, samples 5/2, evaluate+rank",
    "C3": "C3: 3D25pt/13pt (r4/r2) 640^3 x folding x layout fzyx/zyxf x 2/4 components x 16 alignments "
          "(93,184 configs), B200 params, samples 5/2, evaluate+rank",
    "C4": "C4: two-phase LBM 256^3 (D3Q27 hydro + D3Q15 phase field) x 154 blocks x folding x layout "
          "(1,812 configs), B200 params, samples 5/2, evaluate+rank",
    "C5": "C5: C3 (r1-4, 32 alignments) + C4 (16 alignments) x L2 capacity {1, 1/2, 1/4} "
          "(1,205,184 configs), B200 params, samples 5/2, evaluate+rank",
}


def build_shard(workload: str, rank: int, world: int):
    """(Space of this rank's shard, padded shard length m, real configs of
    the whole job).  C2: every rank evaluates its own 246-config sweep
    (alignment 8*rank; weak scaling).  Others: the space is dealt by cost
    and padded to equal length for the all-gather (strong scaling)."""
    from paper_2107_01143_b200 import shard, workloads as W

    m = b200_machine()
    if workload == "C2":
        sp = W.space_c2(m, GRID, RADIUS, alignment=8 * rank)
        return sp, len(sp), len(sp) * world
    sp = W.space(workload, m)
    idx = shard.shard_indices(shard.config_cost(sp.block, sp.n_accesses()), world, rank)
    mlen = shard.pad_to(len(sp), world)
    if len(idx) < mlen:  # pad with this shard's own configs (evaluated, not counted)
        idx = np.concatenate([idx, idx[: mlen - len(idx)]])
    return sp.subset(idx), mlen, len(sp)


def n_addr(sp, m) -> int:
    """Brute-force address-granule evaluations the reference performs for the
    configs of a space: blocks n_b*T*A (+ lines), L1 T*A,
    waves U*B_w*T*A."""
    t = sp.block.astype(np.int64).prod(axis=1)
    per_sm = np.minimum(m.max_blocks_per_sm, m.max_threads_per_sm // t)
    bw = m.sm_count * per_sm
    total = sp.grid_dim.prod(axis=1)
    nw = -(-total // bw)
    u = np.where(nw == 1, 1, 3)
    n_b = np.minimum(5, np.maximum(1, np.clip(sp.grid_dim - 2, 1, None).prod(axis=1)))
    a = sp.n_accesses()
    return int((n_b * t * a + t * a + u * np.minimum(bw, total) * t * a).sum())


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                vals = [v.strip() for v in out.stdout.strip().split(",")]
                if len(vals) == 6:
                    self.samples.append(vals)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(s[0]) for s in self.samples)
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({n for s in self.samples for n, v in zip(names, s[2:]) if v.lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(self.samples[0][1]), "reasons": reasons,
                "samples": len(self.samples)}


def cpu_jobs(sp, n, rng):
    """n seeded-random (kind, spec dict, machine dict) jobs of a space."""
    from paper_2107_01143_b200.gvo.kernels import kernel_to_dict
    from paper_2107_01143_b200.gvo.machine import machine_to_dict

    kind = _ref_kind()
    pick = rng.choice(len(sp), size=min(n, len(sp)), replace=False)
    return [(kind, kernel_to_dict(sp.kernel(int(i))), machine_to_dict(sp.machine(int(i)))) for i in pick]


def cpu_sample_rate(sp, workload):
    """Reference CPU estimator on a bounded sample (multiprocessing pool)."""
    import multiprocessing as mp

    cores = len(os.sched_getaffinity(0))
    jobs = cpu_jobs(sp, max(3 * cores, 24), np.random.default_rng(20240811))
    with mp.get_context("spawn").Pool(min(cores, len(jobs))) as pool:
        pool.map(_warm, range(min(cores, len(jobs))))  # imports outside the timed sample
        t0 = time.perf_counter()
        list(pool.imap_unordered(_cpu_eval, jobs, chunksize=1))
        dt = time.perf_counter() - t0
    return {"value": len(jobs) / dt, "unit": "configs/s", "cores": min(cores, len(jobs)), "kind": jobs[0][0],
            "sample": f"{len(jobs)} seeded-random configs of the {workload} space, "
                      f"reference evaluate_kernel (B200 params, samples 5/2), {dt:.1f} s"}


def _warm(_):
    if (ROOT / "baseline" / "_ref" / "gvo").exists():
        sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
        import gvo  # noqa: F401
    return 0


def _ref_kind():
    return "reference" if (ROOT / "baseline" / "_ref" / "gvo").exists() else "port"


def _cpu_eval(arg):
    """One configuration through the reference's public API (kernel spec +
    machine JSON, as its CLI/bindings take them), or the oracle port."""
    kind, spec, mdict = arg
    if kind == "reference":
        sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
        import gvo as ref
        from gvo.machine import machine_from_dict as ref_machine

        return ref.evaluate_kernel(ref.kernel_from_dict(spec), ref_machine(mdict)).glups
    from oracle import gvo_oracle as ora
    from paper_2107_01143_b200 import gvo
    from paper_2107_01143_b200.gvo.machine import machine_from_dict

    return ora.evaluate_kernel(gvo.kernel_from_dict(spec), machine_from_dict(mdict))["glups"]


def run_device(args, rank, world):
    import torch
    import torch.distributed as dist

    from paper_2107_01143_b200 import _native

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    ctx = _native.context()
    L = _native.lib()
    sp, n, n_real = build_shard(args.workload, rank, world)
    cfg_np = sp.config_array(ctx)
    ctx.sync_registries()
    F = ctx.max_fields
    S, W = _native.effective_sampling(5, 2)
    smp = _native.Sampling(5, 2, 0, 7, 0)
    stride = _native.counts_stride(F, S, W)
    d_cfgs = torch.from_numpy(cfg_np.view(np.uint8).copy()).to(dev)
    d_counts = torch.zeros((n, stride), dtype=torch.int64, device=dev)
    d_stats = torch.zeros((n, _native.stats_len(F)), dtype=torch.float64, device=dev)
    d_rec = torch.zeros((n, _native.RECORD_LEN), dtype=torch.float64, device=dev)
    d_order = torch.zeros(n * world, dtype=torch.int64, device=dev)
    if world > 1:
        g_rec = torch.zeros((n * world, _native.RECORD_LEN), dtype=torch.float64, device=dev)
        g_cfgs = torch.zeros(n * world * cfg_np.itemsize, dtype=torch.uint8, device=dev)
        dist.all_gather_into_tensor(g_cfgs, d_cfgs)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream
    C = _native.C

    def step():
        ctx.check(L.gvo_eval_configs(ctx.h, C.c_void_p(d_cfgs.data_ptr()), n, C.byref(smp), F,
                                     C.c_void_p(d_counts.data_ptr()), C.c_void_p(d_stats.data_ptr()),
                                     C.c_void_p(d_rec.data_ptr()), None, None, 0, C.c_void_p(sptr)))
        if world > 1:
            dist.all_gather_into_tensor(g_rec, d_rec)
            ctx.check(L.gvo_rank(ctx.h, C.c_void_p(g_rec.data_ptr()), C.c_void_p(g_cfgs.data_ptr()), n * world,
                                 C.c_void_p(d_order.data_ptr()), C.c_void_p(sptr)))
        else:
            ctx.check(L.gvo_rank(ctx.h, C.c_void_p(d_rec.data_ptr()), C.c_void_p(d_cfgs.data_ptr()), n,
                                 C.c_void_p(d_order.data_ptr()), C.c_void_p(sptr)))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    status = d_counts[:, _native.C_STATUS].cpu().numpy()
    assert (status == 0).all(), f"engine status {np.unique(status)}"
    L.gvo_set_timing(ctx.h, 1)
    L.gvo_kernel_times(ctx.h, None, None, 1)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clk:
        for i in range(args.steps):
            flush.fill_(i & 0xFF)  # > L2: evict between timed steps
            starts[i].record(stream)
            step()
            ends[i].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    kms = (C.c_double * 8)()
    kcnt = (C.c_int64 * 8)()
    L.gvo_kernel_times(ctx.h, kms, kcnt, 1)
    L.gvo_set_timing(ctx.h, 0)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_step = ms_max / args.steps
    value = n_real * args.steps / (ms_max * 1e-3)

    # ---- e2e through the C ABI with host buffers (copies inside the region)
    # host buffers in pinned memory (the inputs a user stages for the DMA engines)
    counts_h = torch.zeros((n, stride), dtype=torch.int64, pin_memory=True).numpy()
    stats_h = torch.zeros((n, _native.stats_len(F)), dtype=torch.float64, pin_memory=True).numpy()
    rec_h = torch.zeros((n, _native.RECORD_LEN), dtype=torch.float64, pin_memory=True).numpy()
    cfg_pin = torch.empty(cfg_np.nbytes, dtype=torch.uint8, pin_memory=True).numpy()
    cfg_pin[:] = cfg_np.view(np.uint8).reshape(-1)
    cfg_np = cfg_pin.view(cfg_np.dtype).reshape(cfg_np.shape)
    e2e_steps = max(3, args.steps // 2)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    order_pin = torch.zeros(n, dtype=torch.int64, pin_memory=True).numpy()
    for _ in range(e2e_steps):
        if world == 1:  # the one-call sweep entry: evaluate + rank, one synchronisation
            ctx.check(L.gvo_sweep_host(ctx.h, _native._ptr(cfg_np), n, C.byref(smp), F, _native._ptr(counts_h),
                                       _native._ptr(stats_h), _native._ptr(rec_h), _native._ptr(order_pin)))
            order_h = order_pin
            continue
        ctx.check(L.gvo_eval_configs_host(ctx.h, _native._ptr(cfg_np), n, C.byref(smp), F, _native._ptr(counts_h),
                                          _native._ptr(stats_h), _native._ptr(rec_h), None, None, 0))
        rec_d = torch.from_numpy(rec_h).to(dev, non_blocking=False)
        dist.all_gather_into_tensor(g_rec, rec_d)
        ctx.check(L.gvo_rank(ctx.h, C.c_void_p(g_rec.data_ptr()), C.c_void_p(g_cfgs.data_ptr()), n * world,
                             C.c_void_p(d_order.data_ptr()), C.c_void_p(sptr)))
        order_h = d_order.cpu().numpy()
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    te = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = n_real * e2e_steps / float(te.item())
    h2d = n * cfg_np.itemsize + (n * _native.RECORD_LEN * 8 if world > 1 else 0)
    d2h = n * stride * 8 + n * _native.stats_len(F) * 8 + n * _native.RECORD_LEN * 8 + n * world * 8
    del order_h

    if rank != 0:
        return
    # ---- roofline: dominant kernel (interval-union engine) vs measured INT32 issue rate
    names = ("setup", "warp", "sets", "finish", "rank")
    kernel_ms = {names[i]: kms[i] / max(1, args.steps) for i in range(5)}
    top = max(("setup", "warp", "sets", "finish"), key=lambda k: kernel_ms[k])
    peak = C.c_double()
    ctx.check(L.gvo_int_peak(ctx.h, C.byref(peak)))
    n_addr_total = n_addr(sp, b200_machine())
    k_int = 8
    sets_s = kernel_ms["sets"] * 1e-3
    achieved = k_int * n_addr_total / sets_s / 1e9
    algo_bytes = n * (cfg_np.itemsize + stride * 8 + _native.stats_len(F) * 8 + _native.RECORD_LEN * 8)
    cpu = cpu_sample_rate(sp, args.workload) if world == 1 and not args.no_cpu else None
    line = {
        "metric": "kernel configs evaluated/sec (1/2/4/8 B200) vs host-CPU reference; % int/HBM roofline",
        "value": value, "unit": "configs/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak" if args.workload == "C2" else "strong", "vs_baseline": None,
        "dtype": "int64", "data": "synthetic (deterministic config-space enumeration)",
        "config": {"workload": WORKLOADS[args.workload], "configs_total": n_real,
                   "configs_per_rank": n, "parallelism": f"dp{world} (config shards, NCCL all-gather + device rank)",
                   "l2": "flushed between timed steps (256 MiB write)"},
        "e2e": {"value": e2e_value, "unit": "configs/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": int(sum(kcnt[i] for i in range(5))),
        "kernel_ms_per_step": kernel_ms,
        "roofline": {"bound": "int", "kernel": "k_sets (interval-union engine)",
                     "achieved": achieved, "peak": peak.value / 1e9, "unit": "Gop/s (int32, address-equivalent)",
                     "frac": achieved / (peak.value / 1e9),
                     "note": "achieved = 8 int ops x brute-force address-granules the reference enumerates "
                             "(SURVEY §8d N_addr) / k_sets time; >1 means the lattice collapse does less work "
                             "than enumeration. peak = measured INT32 issue rate (gvo_int_peak).",
                     "hbm": {"achieved": algo_bytes / (ms_step * 1e-3) / 1e9, "peak": 6531.3, "unit": "GB/s",
                             "frac": algo_bytes / (ms_step * 1e-3) / 1e9 / 6531.3},
                     "traffic": _ncu_traffic(),
                     "hw": _ncu_hw()},
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def run_reference(args, rank, world):
    """The reference's own CPU estimator on bounded samples of the workload,
    all host cores (rank 0 only under torchrun)."""
    if rank != 0:
        return
    import multiprocessing as mp

    from paper_2107_01143_b200 import workloads as W

    cores = len(os.sched_getaffinity(0))
    sp = W.space_c2(b200_machine(), GRID, RADIUS) if args.workload == "C2" else W.space(args.workload)
    rng = np.random.default_rng(20240811)
    per_step = max(3 * cores, 24)
    times = []
    kind = _ref_kind()
    with mp.get_context("spawn").Pool(cores) as pool:
        pool.map(_warm, range(cores))
        for i in range(args.warmup + args.steps):
            jobs = cpu_jobs(sp, per_step, rng)
            t0 = time.perf_counter()
            list(pool.imap_unordered(_cpu_eval, jobs, chunksize=1))
            if i >= args.warmup:
                times.append((len(jobs), time.perf_counter() - t0))
    n_done = sum(a for a, _ in times)
    secs = sum(b for _, b in times)
    value = n_done / secs
    line = {
        "impl": "reference",
        "metric": "kernel configs evaluated/sec (1/2/4/8 B200) vs host-CPU reference; % int/HBM roofline",
        "value": value, "unit": "configs/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": secs / len(times) * 1e3, "higher_is_better": True,
        "scaling": "weak" if args.workload == "C2" else "strong", "vs_baseline": None,
        "dtype": "int64", "data": "synthetic (deterministic config-space enumeration)",
        "config": {"workload": WORKLOADS[args.workload], "per_step_sample": per_step},
        "cpu_baseline": {"value": value, "unit": "configs/s", "cores": cores, "kind": kind,
                         "sample": f"{per_step} seeded-random configs per step of the {args.workload} space, "
                                   "unmodified reference evaluate_kernel"},
        "e2e": {"value": value, "unit": "configs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _ncu_traffic():
    """dram read+write bytes per k_sets launch from the committed ncu capture
    (profiles/r01_ncu_k_sets.json), or None."""
    p = ROOT / "profiles" / "r01_ncu_k_sets.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text())
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        v, u = d[k]
        tot += float(v) * scale.get(u, 1)
    return tot


def _ncu_hw():
    """Hardware utilisation of the same k_sets launch from the committed ncu
    capture: issue slots, ALU pipe, shared-memory wavefronts (the counters the
    north star names), or None."""
    p = ROOT / "profiles" / "r01_ncu_k_sets.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text())
    pick = {"issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "alu_pipe_pct": "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
            "smem_wavefronts_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed",
            "dram_pct": "dram__throughput.avg.pct_of_peak_sustained_elapsed"}
    out = {k: float(d[v][0]) for k, v in pick.items() if v in d}
    out["source"] = "profiles/r01_ncu_k_sets.json (ncu --set full, C2 bench k_sets launch)"
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=("b200", "reference"))
    ap.add_argument("--no-cpu", action="store_true", help="skip the in-run CPU baseline")
    ap.add_argument("--workload", default="C2", choices=sorted(WORKLOADS))
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        dist.init_process_group("nccl")
    try:
        run_device(args, rank, world)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
