"""Multi-process (gloo, world_size 2) tests of the sharding and the single
all-gather of the multi-GPU path; the device ranking itself is covered by
the GPU tests."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2107_01143_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(3)
    blocks = rng.integers(1, 64, size=(n, 3))
    cost = shard.config_cost(blocks, np.full(n, 26))
    mine = shard.shard_indices(cost, world, rank)
    m = shard.pad_to(n, world)
    # "records": global index and a value derived from it, padded
    rec = torch.full((m, 2), -1.0, dtype=torch.float64)
    rec[: len(mine), 0] = torch.from_numpy(mine.astype(np.float64))
    rec[: len(mine), 1] = torch.from_numpy((mine * 7 + 1).astype(np.float64))
    g = shard.gather_records(rec, world)
    shards = [shard.shard_indices(cost, world, r) for r in range(world)]
    gi = shard.global_index(shards, m)
    out_q.put((rank, g.numpy(), gi, cost))
    dist.destroy_process_group()


def test_shard_partition_is_exact_and_balanced():
    n = 1001
    cost = shard.config_cost(np.random.default_rng(1).integers(1, 64, size=(n, 3)), np.full(n, 26))
    parts = [shard.shard_indices(cost, 4, r) for r in range(4)]
    allidx = np.concatenate(parts)
    assert sorted(allidx.tolist()) == list(range(n))
    loads = [cost[p].sum() for p in parts]
    assert max(loads) / min(loads) < 1.1


def test_group_shards_keep_sharing_groups_whole_and_balance():
    """Sharing groups (bench.py's strong-scaled C5 sharding) never straddle
    ranks, every configuration lands on exactly one rank, and the dealt
    group costs stay balanced."""
    from paper_2107_01143_b200 import workloads as W
    from paper_2107_01143_b200.gvo.machine import b200_preset

    m = b200_preset()
    sp = W.space_c3(m, radii=(2,), components=(2,), alignments=tuple(range(0, 128, 8)), machines=W.l2_variants(m),
                    machines_idx=(0, 1, 2))
    g = sp.sharing_groups()
    cost = shard.config_cost(sp.block, sp.n_accesses()) * sp.kind_weight()
    for world in (2, 3, 8):
        parts = shard.group_shards(cost, g, world)
        allidx = np.concatenate(parts)
        assert sorted(allidx.tolist()) == list(range(len(sp)))
        owner = np.empty(len(sp), dtype=np.int64)
        for r, p_ in enumerate(parts):
            owner[p_] = r
        for gid in np.unique(g)[:500]:
            assert len(np.unique(owner[g == gid])) == 1
        gc = np.zeros(g.max() + 1)
        np.maximum.at(gc, g, cost)
        loads = [gc[np.unique(g[p_])].sum() for p_ in parts]
        assert max(loads) / min(loads) < 1.05
    # alignments equal modulo the sector share a group; other residues do not
    t0 = [i for i, t in enumerate(sp.templates) if t.alignment in (0, 32)]
    t1 = [i for i, t in enumerate(sp.templates) if t.alignment == 8]
    a = np.flatnonzero(np.isin(sp.tpl, t0))
    b = np.flatnonzero(np.isin(sp.tpl, t1))
    assert len(np.unique(g[a])) < len(a) and not set(g[a]) & set(g[b])


def test_gloo_world2_all_gather_reassembles_every_config():
    world, n = 2, 37
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda t: t[0])
    g0, gi = res[0][1], res[0][2]
    assert np.array_equal(g0, res[1][1])  # identical on both ranks
    valid = gi >= 0
    assert sorted(gi[valid].tolist()) == list(range(n))
    assert np.array_equal(g0[valid, 0], gi[valid].astype(float))
    assert np.array_equal(g0[valid, 1], gi[valid] * 7 + 1.0)


# ------------------------------------------------------------------ GPU: the real engine, two ranks
def _engine_worker(rank, world, port, out_q, case):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)  # every rank shares the one GPU of the test box
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2107_01143_b200 import gvo

    try:
        m = gvo.b200_preset()
        fam = gvo.KernelFamily("stencil", (64, 64, 64), radius=2)
        cfgs = list(gvo.enumerate_sweep(64, foldings=("none", "2y", "2z"))) + list(gvo.enumerate_sweep(512))
        group = None
        if case == "subgroup":
            group = dist.new_group([0, 2])
            if rank == 1:
                out_q.put((rank, None, None, None))
                return
        if case == "error":
            cfgs = cfgs[:40] + [gvo.SweepConfig((64, 32, 1))] + cfgs[40:]  # 2048 threads: FootprintError
        try:
            kept, order, rec = gvo.rank_sweep_sharded(fam, cfgs, m, skip_invalid=True, group=group)
            out_q.put((rank, [c.key for c in kept], order, rec))
        except Exception as exc:  # noqa: BLE001
            out_q.put((rank, "raised", type(exc).__name__, str(exc)))
    finally:
        dist.destroy_process_group()


def _run_world(world, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_engine_worker, args=(r, world, port, q, case)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["world2", "subgroup"])
def test_sharded_engine_equals_single_gpu_rank_sweep(case):
    """rank_sweep_sharded through the real engine on two ranks (gloo; both
    on the box's one GPU) gives rank_sweep's kept configs, order and
    records on every rank — including a subgroup of a three-rank world."""
    from paper_2107_01143_b200 import gvo

    res = _run_world(3 if case == "subgroup" else 2, case)
    m = gvo.b200_preset()
    fam = gvo.KernelFamily("stencil", (64, 64, 64), radius=2)
    cfgs = list(gvo.enumerate_sweep(64, foldings=("none", "2y", "2z"))) + list(gvo.enumerate_sweep(512))
    rows = gvo.rank_sweep(fam, cfgs, m, skip_invalid=True)
    want_keys = [c.key for c in rows.configs]
    members = [r for r in res if r[1] is not None]
    assert len(members) == 2
    for _, keys, order, rec in members:
        assert keys == want_keys
        np.testing.assert_array_equal(order, rows.order)
        np.testing.assert_array_equal(rec, rows.records)


@pytest.mark.gpu
def test_sharded_engine_every_rank_raises_the_reference_error():
    """An evaluation error on one rank's shard raises the reference's
    exception on every rank (no rank left waiting in the collective)."""
    res = _run_world(2, "error")
    for r in res:
        assert r[1] == "raised" and r[2] == "FootprintError", r
        assert "exceeds machine limit" in r[3]


@pytest.mark.gpu
def test_torchrun_bench_two_ranks_ranks_like_one(tmp_path):
    """bench.py under torchrun with two ranks (gloo on the one test GPU):
    cost-dealt shards, all-gather, gvo_rank_gathered — the global ranking
    equals the single-rank one."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ, GVO_BENCH_BACKEND="gloo")
    common = ["--workload", "C4", "--steps", "1", "--warmup", "1", "--no-cpu"]
    one = subprocess.run([sys.executable, str(root / "bench.py"), *common, "--dump-order", str(tmp_path / "o1.npy")],
                         capture_output=True, text=True, timeout=900, cwd=root, env=env)
    assert one.returncode == 0, one.stderr[-3000:]
    two = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(root / "bench.py"),
                          *common, "--gpus", "2", "--dump-order", str(tmp_path / "o2.npy")],
                         capture_output=True, text=True, timeout=900, cwd=root, env=env)
    assert two.returncode == 0, two.stderr[-3000:]
    line = json.loads([ln for ln in two.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong" and line["e2e"]["value"] > 0
    np.testing.assert_array_equal(np.load(tmp_path / "o1.npy"), np.load(tmp_path / "o2.npy"))
