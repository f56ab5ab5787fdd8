"""Benchmark: kernel configurations evaluated per second (BASELINE.json metric).

Workload (default): BASELINE.json configs[4], C5 — the combined stencil + LBM
configuration space at B200 cache/HBM parameters, 1,205,184 configurations
(paper_2107_01143_b200/workloads.py space_c5: the 3D25pt/13pt/19pt/7pt star
stencils (r = 1..4) on 640^3 x every power-of-two block <= 1024 threads x
folding {none, 2y, 2z} x layout {fzyx, zyxf} x {2, 4} components x 32 field
alignments, and the two-phase LBM kernels (D3Q27 hydro + D3Q15 phase field)
on 256^3 x 154 blocks x folding x layout x 16 alignments, each at L2
capacity {full, 1/2, 1/4}), evaluated with block_samples=5, wave_samples=2
and default fits, then ranked (perf.py:131 key).  It is the largest
single-GPU space of BASELINE.json, so it is the headline.

A step = evaluate + rank the whole space.  With N GPUs (torchrun) the space
is dealt to ranks by estimated cost (shard.py; strong scaling: total work
fixed), every rank evaluates its shard, one all-gather of the fixed-size
records (+ their global index), and the device ranks the whole space in
global order (gvo_rank_gathered: ties break by input order, padding dropped).

--workload C1|C2|C3|C4 runs the other BASELINE.json spaces (parity cases).

--impl reference times the reference's own CPU estimator (pip-installed
unmodified under baseline/_ref; the CPU oracle port if that is missing) on
bounded seeded samples of the same workload with all host cores.
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

METRIC = "kernel configs evaluated/sec (1/2/4/8 B200) vs host-CPU reference; % int/HBM roofline"
SEED = 20240811  # BASELINE.md §3 / SURVEY §8d seeded subsets
CPU_SAMPLE = 512  # >= 500 configurations for the 1e5 / 1e6 spaces
CPU_SAMPLE_1P = 12  # single-process rate: a bounded prefix of the same sample
# ncu capture of the dominant kernel for the default workload (tools/ncu_capture.py)
CAPTURE = ROOT / "profiles" / "r02_ncu_capture_c5.json"
ISSUE_SLOTS_PER_SM = 4  # warp schedulers per SM (one warp-instruction issue per cycle each)


def b200_machine():
    from paper_2107_01143_b200 import gvo

    return gvo.b200_preset()


WORKLOADS = {
    "C1": "C1: 2D5pt Jacobi 256^2, block 32x4x1 (PR1 oracle config)",
    "C2": "C2: 3D25pt r4 640^3 full power-of-two block sweep (246 valid configs), "
          "B200 machine params, samples 5/2, evaluate+rank",
    "C3": "C3: 3D25pt/13pt (r4/r2) 640^3 x folding x layout fzyx/zyxf x 2/4 components x 16 alignments "
          "(93,184 configs), B200 params, samples 5/2, evaluate+rank",
    "C4": "C4: two-phase LBM 256^3 (D3Q27 hydro + D3Q15 phase field) x 154 blocks x folding x layout "
          "(1,812 configs), B200 params, samples 5/2, evaluate+rank",
    "C5": "C5: C3 (r1-4, 32 alignments) + C4 (16 alignments) x L2 capacity {1, 1/2, 1/4} "
          "(1,205,184 configs), B200 params, samples 5/2, evaluate+rank",
}


def build_shard(workload: str, rank: int, world: int):
    """(whole space, this rank's global indices, padded shard length m).
    The space is dealt in sharing groups (configurations whose set problems
    are exact translates stay on one rank) by estimated cost, longest first
    to the least-loaded rank (strong scaling)."""
    from paper_2107_01143_b200 import shard, workloads as W

    sp = W.space(workload, b200_machine())
    if world == 1:
        return sp, np.arange(len(sp)), len(sp)
    cost = shard.config_cost(sp.block, sp.n_accesses()) * sp.kind_weight()
    shards = shard.group_shards(cost, sp.sharing_groups(), world)
    return sp, shards[rank], max(len(x) for x in shards)


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


# ---------------------------------------------------------------- CPU legs
def _ref_kind():
    return "reference" if (ROOT / "baseline" / "_ref" / "gvo").exists() else "port"


def cpu_jobs(sp, pick):
    """(kind, spec dict, machine dict) jobs of the configurations `pick`."""
    from paper_2107_01143_b200.gvo.kernels import kernel_to_dict
    from paper_2107_01143_b200.gvo.machine import machine_to_dict

    kind = _ref_kind()
    return [(kind, kernel_to_dict(sp.kernel(int(i))), machine_to_dict(sp.machine(int(i)))) for i in pick]


def _warm(_):
    if (ROOT / "baseline" / "_ref" / "gvo").exists():
        sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
        import gvo  # noqa: F401
    return 0


def _cpu_eval(arg):
    """One configuration through the reference's public API (kernel spec +
    machine JSON, as its CLI/bindings take them), or the oracle port:
    (glups, limiter)."""
    kind, spec, mdict = arg
    if kind == "reference":
        sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
        import gvo as ref
        from gvo.machine import machine_from_dict as ref_machine

        p = ref.evaluate_kernel(ref.kernel_from_dict(spec), ref_machine(mdict))
        return p.glups, p.limiter
    from oracle import gvo_oracle as ora
    from paper_2107_01143_b200 import gvo
    from paper_2107_01143_b200.gvo.machine import machine_from_dict

    ev = ora.evaluate_kernel(gvo.kernel_from_dict(spec), machine_from_dict(mdict))
    return ev["glups"], ev["limiter"]


def cpu_baseline(sp, workload):
    """The reference CPU estimator on CPU_SAMPLE seeded-random configurations
    of the space with a process per host core, plus a single-process rate on
    a prefix of the same sample.  Returns (cpu_baseline dict, sample indices,
    reference (glups, limiter) per sampled config)."""
    import multiprocessing as mp

    cores = len(os.sched_getaffinity(0))
    pick = np.random.default_rng(SEED).choice(len(sp), size=min(CPU_SAMPLE, len(sp)), replace=False)
    jobs = cpu_jobs(sp, pick)
    with mp.get_context("spawn").Pool(cores) as pool:
        pool.map(_warm, range(cores))  # imports outside the timed sample
        t0 = time.perf_counter()
        ref = pool.map(_cpu_eval, jobs, chunksize=1)
        dt = time.perf_counter() - t0
    n1 = min(CPU_SAMPLE_1P, len(jobs))
    with mp.get_context("spawn").Pool(1) as pool:
        pool.map(_warm, [0])
        t1 = time.perf_counter()
        pool.map(_cpu_eval, jobs[:n1], chunksize=1)
        dt1 = time.perf_counter() - t1
    out = {"value": len(jobs) / dt, "unit": "configs/s", "cores": cores, "kind": jobs[0][0],
           "single_process": {"value": n1 / dt1, "unit": "configs/s", "cores": 1, "configs": n1,
                              "seconds": round(dt1, 2)},
           "sample": f"{len(jobs)} configurations of the {workload} space drawn with "
                     f"np.random.default_rng({SEED}) (BASELINE.md §3), unmodified reference evaluate_kernel "
                     f"(B200 params, samples 5/2), multiprocessing pool of {cores}: {dt:.1f} s; "
                     f"single process: the first {n1} of them, {dt1:.1f} s"}
    return out, pick, ref


# ---------------------------------------------------------------- device arm
def _capture_for(workload: str, bid: str):
    """The committed ncu capture of the dominant kernel for this workload,
    if it was taken with this very library build (same gvo_build_id)."""
    p = ROOT / "profiles" / f"r02_ncu_capture_{workload.lower()}.json"
    if not p.exists():
        return None, f"no capture {p.name}"
    d = json.loads(p.read_text())
    if d.get("build_id") != bid:
        return None, f"{p.name} was taken with build {d.get('build_id')}, this library is {bid}"
    return d, str(p.relative_to(ROOT))


def run_device(args, rank, world):
    import torch
    import torch.distributed as dist

    from paper_2107_01143_b200 import _native

    ndev = torch.cuda.device_count()
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)) % max(1, ndev))
    torch.cuda.set_device(dev)
    nccl = world > 1 and dist.get_backend() == "nccl"
    ctx = _native.context()
    L = _native.lib()
    C = _native.C
    sp, mine, m = build_shard(args.workload, rank, world)
    N = len(sp)
    cfg_all = sp.config_array(ctx)
    ctx.sync_registries()
    cfg_np = np.ascontiguousarray(cfg_all[mine])
    n = len(cfg_np)
    F = ctx.max_fields
    S, W = _native.effective_sampling(5, 2)
    smp = _native.Sampling(5, 2, 0, 7, 0)
    stride = _native.counts_stride(F, S, W)
    R = _native.RECORD_LEN
    d_cfgs = torch.from_numpy(cfg_np.view(np.uint8).copy()).to(dev)
    d_counts = torch.zeros((max(n, 1), stride), dtype=torch.int64, device=dev)
    d_stats = torch.zeros((max(n, 1), _native.stats_len(F)), dtype=torch.float64, device=dev)
    d_rec = torch.zeros((max(m, 1), R), dtype=torch.float64, device=dev)
    d_order = torch.zeros(N, dtype=torch.int64, device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream
    if world > 1:
        gidx = np.full(m, -1, dtype=np.int64)
        gidx[:n] = mine
        g_gidx = torch.from_numpy(np.concatenate(_gather_np(gidx, world))).to(dev)
        g_rec = torch.zeros((m * world, R), dtype=torch.float64, device=dev)
        d_cfg_all = torch.from_numpy(cfg_all.view(np.uint8).copy()).to(dev)

    def gather_rec(src):
        if nccl:
            dist.all_gather_into_tensor(g_rec, src)
        else:  # gloo (test mode: several ranks on one GPU): host round trip
            parts = [torch.empty((m, R), dtype=torch.float64) for _ in range(world)]
            dist.all_gather(parts, src.cpu())
            g_rec.copy_(torch.cat(parts))

    def rank_all():
        if world > 1:
            gather_rec(d_rec)
            ctx.check(L.gvo_rank_gathered(ctx.h, C.c_void_p(g_rec.data_ptr()), C.c_void_p(g_gidx.data_ptr()),
                                          m * world, C.c_void_p(d_cfg_all.data_ptr()), N, None,
                                          C.c_void_p(d_order.data_ptr()), C.c_void_p(sptr)))
        else:
            ctx.check(L.gvo_rank(ctx.h, C.c_void_p(d_rec.data_ptr()), C.c_void_p(d_cfgs.data_ptr()), n,
                                 C.c_void_p(d_order.data_ptr()), C.c_void_p(sptr)))

    def step():
        if n:
            ctx.check(L.gvo_eval_configs(ctx.h, C.c_void_p(d_cfgs.data_ptr()), n, C.byref(smp), F,
                                         C.c_void_p(d_counts.data_ptr()), C.c_void_p(d_stats.data_ptr()),
                                         C.c_void_p(d_rec.data_ptr()), None, None, 0, C.c_void_p(sptr)))
        rank_all()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    status = d_counts[:n, _native.C_STATUS].cpu().numpy()
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
    sharing = sharing_leg(ctx, step, stream, flush, n) if not args.no_e2e else None
    per_rank = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        allr = _gather_np(np.array([ms]), world)
        ms_all = [float(a[0]) for a in allr]
    else:
        ms_all = [ms]
    ms_max = max(ms_all)
    del per_rank
    ms_step = ms_max / args.steps
    value = N * args.steps / (ms_max * 1e-3)
    final_order = d_order.cpu().numpy()

    # ---- e2e through the C ABI with host buffers (copies inside the region)
    e2e = None
    if not args.no_e2e:
        counts_h = torch.zeros((max(n, 1), stride), dtype=torch.int64, pin_memory=True).numpy()
        stats_h = torch.zeros((max(n, 1), _native.stats_len(F)), dtype=torch.float64, pin_memory=True).numpy()
        rec_h = torch.zeros((max(m, 1), R), dtype=torch.float64, pin_memory=True).numpy()
        cfg_pin = torch.empty(max(cfg_np.nbytes, 1), dtype=torch.uint8, pin_memory=True).numpy()
        cfg_pin[: cfg_np.nbytes] = cfg_np.view(np.uint8).reshape(-1)
        cfg_h = cfg_pin[: cfg_np.nbytes].view(cfg_np.dtype)
        order_pin = torch.zeros(N, dtype=torch.int64, pin_memory=True).numpy()
        e2e_steps = max(2, args.steps // 4)

        def e2e_step():
            if world == 1:  # the one-call sweep entry: evaluate + rank, one synchronisation
                ctx.check(L.gvo_sweep_host(ctx.h, _native._ptr(cfg_h), n, C.byref(smp), F, _native._ptr(counts_h),
                                           _native._ptr(stats_h), _native._ptr(rec_h), _native._ptr(order_pin)))
                return
            if n:
                ctx.check(L.gvo_eval_configs_host(ctx.h, _native._ptr(cfg_h), n, C.byref(smp), F,
                                                  _native._ptr(counts_h), _native._ptr(stats_h), _native._ptr(rec_h),
                                                  None, None, 0))
            d_rec.copy_(torch.from_numpy(rec_h), non_blocking=False)
            rank_all()
            order_pin[:] = d_order.cpu().numpy()

        e2e_step()  # warm-up: staging buffers, copy stream
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        torch.cuda.synchronize()
        e2e_s = time.perf_counter() - t0
        e2e_all = _gather_np(np.array([e2e_s]), world) if world > 1 else [np.array([e2e_s])]
        e2e_value = N * e2e_steps / max(float(a[0]) for a in e2e_all)
        h2d = n * cfg_np.itemsize + (m * R * 8 if world > 1 else 0)
        d2h = n * stride * 8 + n * _native.stats_len(F) * 8 + n * R * 8 + N * 8
        e2e = {"value": e2e_value, "unit": "configs/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "steps": e2e_steps,
               "path": "gvo_sweep_host (pinned host configs in, counts/stats/records/order out)" if world == 1
               else "gvo_eval_configs_host per shard + all-gather + gvo_rank_gathered, order to host"}
        if world == 1 and not np.array_equal(order_pin, final_order):
            raise AssertionError("e2e ranking differs from the device-timed ranking")

    api = api_leg(ctx, smp) if world == 1 and not args.no_e2e else None

    if args.dump_order and rank == 0:
        np.save(args.dump_order, final_order)
    if rank != 0:
        return
    names = ("setup", "warp", "sets", "finish", "rank")
    kernel_ms = {names[i]: kms[i] / max(1, args.steps) for i in range(5)}
    launches = {names[i]: int(kcnt[i]) for i in range(5)}
    clocks = clk.summary()
    bid = _native.build_id()
    roof = roofline(args, kernel_ms, launches, clocks, n, cfg_np.itemsize, stride, F, ms_step, bid)
    cpu = None
    parity = None
    if world == 1 and not args.no_cpu:
        cpu, pick, ref = cpu_baseline(sp, args.workload)
        parity = same_run_parity(ctx, cfg_all, pick, ref, smp, F)
    line = {
        "metric": METRIC,
        "value": value, "unit": "configs/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "int64", "data": "synthetic (deterministic config-space enumeration)",
        "config": {"workload": WORKLOADS[args.workload], "configs_total": N,
                   "configs_per_rank_max": m, "parallelism": f"dp{world} (cost-dealt sharing-group shards, "
                   f"{'NCCL' if nccl or world == 1 else 'gloo'} all-gather + device rank)",
                   "l2": "flushed between timed steps (256 MiB write)", "batch": int(os.environ.get("GVO_BATCH", 65536))},
        "e2e": e2e,
        "gpu_launches": int(sum(kcnt[i] for i in range(5))),
        "launches_per_step": {k: v / max(1, args.steps) for k, v in launches.items()},
        "kernel_ms_per_step": kernel_ms,
        "e2e_api": api,
        "sharing": sharing,
        "rank_ms": ms_all if world > 1 else None,
        "roofline": roof,
        "cpu_baseline": cpu,
        "parity_same_run": parity,
        "clocks": clocks,
        "build_id": bid,
    }
    print(json.dumps(line), flush=True)


def sharing_leg(ctx, step, stream, flush, n):
    """Cross-configuration sharing of identical set problems (k_dedup.cu)
    is part of every timed step above.  Here: how much of the step it
    shared (one counted step), and the same step with sharing switched off
    (one step, CUDA events, same L2 flush) -- the rate of an engine that
    evaluates every configuration from scratch."""
    import ctypes as C

    import torch

    from paper_2107_01143_b200 import _native

    L = _native.lib()
    L.gvo_dedup_stats(ctx.h, 1, None, None)
    step()
    torch.cuda.synchronize()
    units, follow = C.c_int64(), C.c_int64()
    L.gvo_dedup_stats(ctx.h, 0, C.byref(units), C.byref(follow))
    ctx.check(L.gvo_set_dedup(ctx.h, 0))
    try:
        step()  # warm the unshared path
        flush.fill_(7)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        step()
        b.record(stream)
        torch.cuda.synchronize()
        ms_off = a.elapsed_time(b)
    finally:
        ctx.check(L.gvo_set_dedup(ctx.h, 1))
    return {"shareable_units": units.value, "units_copied": follow.value,
            "copied_fraction": follow.value / units.value if units.value else 0.0,
            "no_sharing": {"value": n / (ms_off * 1e-3), "unit": "configs/s", "ms_per_step": ms_off, "steps": 1},
            "note": "units = (config, field) wave sets, (config, field, sample) block sets, (config, sample) "
                    "warp/L1 items; a copied unit is an exact translate of one computed in the same call "
                    "(same accesses up to the field base, base residue, launch and machine integer parameters)"}


def api_leg(ctx, smp, reps: int = 5):
    """The drop-in Python API (gvo.rank_sweep, reference perf.py:98-132)
    against the one-call C ABI (gvo_sweep_host) on the same sweep: the
    reference's own KernelFamily("stencil", 640^3, r=4) over every
    power-of-two block <= 1024 threads (C2, skip_invalid).  Host-side
    validation, batch construction, evaluation, ranking and row access
    (len / first row) are inside the timed region."""
    from paper_2107_01143_b200 import _native, gvo

    m = gvo.b200_preset()
    fam = gvo.KernelFamily("stencil", (640, 640, 640), radius=4)
    cfgs = [c for t in (1 << i for i in range(11)) for c in gvo.enumerate_sweep(t)]
    rows = gvo.rank_sweep(fam, cfgs, m, skip_invalid=True)  # warm: templates registered
    t0 = time.perf_counter()
    for _ in range(reps):
        rows = gvo.rank_sweep(fam, cfgs, m, skip_invalid=True)
        _ = rows[0].prediction.glups
    api_s = (time.perf_counter() - t0) / reps
    n = len(rows)
    plan = gvo.perf.SweepPlan(fam, cfgs, m, skip_invalid=True)
    ca = plan.config_array()
    ctx.sync_registries()
    F = ctx.max_fields
    S, W = _native.effective_sampling(5, 2)
    counts = np.zeros((n, _native.counts_stride(F, S, W)), dtype=np.int64)
    rec = np.zeros((n, _native.RECORD_LEN))
    order = np.zeros(n, dtype=np.int64)
    C = _native.C
    t0 = time.perf_counter()
    for _ in range(reps):
        ctx.check(_native.lib().gvo_sweep_host(ctx.h, _native._ptr(ca), n, C.byref(smp), F, _native._ptr(counts),
                                               None, _native._ptr(rec), _native._ptr(order)))
    abi_s = (time.perf_counter() - t0) / reps
    assert np.array_equal(order, rows.order)
    return {"workload": f"C2 sweep through gvo.rank_sweep ({len(cfgs)} configs, {n} valid)",
            "value": n / api_s, "unit": "configs/s", "c_abi_value": n / abi_s, "fraction_of_c_abi": abi_s / api_s}


def _gather_np(a: np.ndarray, world: int):
    """All-gather a small host array over the default group (any backend)."""
    import torch
    import torch.distributed as dist

    t = torch.from_numpy(np.ascontiguousarray(a))
    if dist.get_backend() == "nccl":
        t = t.cuda()
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t)
    return [p.cpu().numpy() for p in parts]


def roofline(args, kernel_ms, launches, clocks, n, cfg_bytes, stride, F, ms_step, bid):
    """Dominant kernel (the interval-union engine k_sets) against the
    integer-issue roof: warp-instructions it issues per second vs
    148 SMs x 4 schedulers x SM clock.  The instruction count and DRAM bytes
    per launch come from an ncu capture of the same workload taken with this
    very library build (tools/ncu_capture.py; build id checked), the time
    from this run's CUDA events on the launching stream."""
    from paper_2107_01143_b200 import _native

    top = max(("setup", "sets", "finish", "rank"), key=lambda k: kernel_ms[k])
    cap, src = _capture_for(args.workload, bid)
    clk_mhz = clocks.get("sm_mhz") or clocks.get("sm_max_mhz") or 1965.0
    peak = 148 * ISSUE_SLOTS_PER_SM * clk_mhz * 1e6  # warp-instructions / s
    sets_s = kernel_ms["sets"] * 1e-3
    R = _native.RECORD_LEN
    algo_bytes = n * (cfg_bytes + stride * 8 + _native.stats_len(F) * 8 + R * 8)
    out = {"bound": "int", "kernel": "k_sets (interval-union engine)", "dominant": top,
           "kernel_share_of_step": kernel_ms["sets"] / ms_step if ms_step else None,
           "unit": "warp-inst/s", "peak": peak,
           "peak_note": f"148 SMs x {ISSUE_SLOTS_PER_SM} issue slots x {clk_mhz:.0f} MHz (median SM clock sampled "
                        "in the timed region): the integer/control-flow issue roof of a kernel with no "
                        "tensor-core or HBM-bound work",
           "achieved": None, "frac": None, "traffic": None, "capture": src,
           "hbm": {"algorithmic_bytes_per_step": algo_bytes, "achieved": algo_bytes / (ms_step * 1e-3) / 1e9,
                   "peak": 6537.0, "unit": "GB/s", "frac": algo_bytes / (ms_step * 1e-3) / 1e9 / 6537.0}}
    if cap is not None and sets_s > 0:
        inst = cap["k_sets"]["inst_executed_per_step"]
        out["achieved"] = inst / sets_s
        out["frac"] = out["achieved"] / peak
        out["inst_executed_per_step"] = inst
        out["traffic"] = cap["k_sets"]["dram_bytes_per_launch"]
        out["traffic_per_step"] = cap["k_sets"]["dram_bytes_per_step"]
        out["ncu"] = {k: cap["k_sets"].get(k) for k in ("issue_active_pct", "launches_per_step",
                                                          "share_of_step_ncu", "hw")}
    return out


def same_run_parity(ctx, cfg_all, pick, ref, smp, F):
    """GPU records of the CPU-baseline sample vs the reference's results of
    the same run: GLup/s bit-exact, limiter equal, subset ranking equal."""
    from paper_2107_01143_b200 import _native

    sub = np.ascontiguousarray(cfg_all[pick])
    out = ctx.sweep_host(sub, 5, 2, 0, want_l1_access=False, want_field_down=False)
    g = out["records"][:, -1]
    lim = out["records"][:, -2].astype(int)
    exact = sum(1 for i, (rg, rl) in enumerate(ref) if g[i] == rg and _native.LIMITERS[lim[i]] == rl)
    fold = {0: "2y", 1: "2z", 2: "none"}
    keys = sorted(range(len(ref)), key=lambda i: (-ref[i][0], tuple(int(v) for v in sub["block"][i]),
                                                 fold[int(sub["fold_rank"][i])], i))
    return {"configs": len(ref), "glups_bit_exact_and_limiter_equal": exact,
            "subset_ranking_identical": bool(list(map(int, out["order"])) == keys),
            "reference_kind": _ref_kind()}


def run_reference(args, rank, world):
    """The reference's own CPU estimator on bounded seeded samples of the
    workload, all host cores (rank 0 only under torchrun)."""
    if rank != 0:
        return
    import multiprocessing as mp

    from paper_2107_01143_b200 import workloads as W

    cores = len(os.sched_getaffinity(0))
    sp = W.space(args.workload, b200_machine())
    rng = np.random.default_rng(SEED)
    per_step = max(3 * cores, 24)
    times = []
    kind = _ref_kind()
    with mp.get_context("spawn").Pool(cores) as pool:
        pool.map(_warm, range(cores))
        for i in range(args.warmup + args.steps):
            pick = rng.choice(len(sp), size=min(per_step, len(sp)), replace=False)
            jobs = cpu_jobs(sp, pick)
            t0 = time.perf_counter()
            pool.map(_cpu_eval, jobs, chunksize=1)
            if i >= args.warmup:
                times.append((len(jobs), time.perf_counter() - t0))
    n_done = sum(a for a, _ in times)
    secs = sum(b for _, b in times)
    value = n_done / secs
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value, "unit": "configs/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": secs / len(times) * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None,
        "dtype": "int64", "data": "synthetic (deterministic config-space enumeration)",
        "config": {"workload": WORKLOADS[args.workload], "per_step_sample": per_step},
        "cpu_baseline": {"value": value, "unit": "configs/s", "cores": cores, "kind": kind,
                         "sample": f"{per_step} configurations per step of the {args.workload} space "
                                   f"(np.random.default_rng({SEED}) stream, {n_done} timed in total), "
                                   "unmodified reference evaluate_kernel, process per core"},
        "e2e": {"value": value, "unit": "configs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=("b200", "reference"))
    ap.add_argument("--no-cpu", action="store_true", help="skip the in-run CPU baseline")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer end-to-end leg")
    ap.add_argument("--workload", default="C5", choices=sorted(WORKLOADS))
    ap.add_argument("--dump-order", default="", help="save the final global ranking (rank 0, .npy)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        # GVO_BENCH_BACKEND=gloo: several ranks sharing one GPU (tests); NCCL otherwise
        backend = os.environ.get("GVO_BENCH_BACKEND", "nccl")
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)) % max(1, torch.cuda.device_count()))
        dist.init_process_group(backend)
    try:
        run_device(args, rank, world)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
