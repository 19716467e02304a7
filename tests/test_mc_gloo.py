"""Multi-process Monte Carlo sharding + final gather (world_size 2, gloo, CPU)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2501_07942_b200.mc import gather_rmse, run_error_sums, shard


def test_shard_covers_all_runs():
    for total in (1, 7, 4096, 4097):
        for world in (1, 2, 3, 8):
            parts = [shard(total, world, r) for r in range(world)]
            allr = np.concatenate(parts)
            assert np.array_equal(allr, np.arange(total))
            assert max(len(p) for p in parts) - min(len(p) for p in parts) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, d, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    runs = shard(total, world, rank)
    rng = np.random.default_rng(100 + rank)
    B, S, kf = len(runs), 3, 4
    means = rng.normal(size=(B, S, d))
    states = rng.normal(size=(B, kf, d))
    ks = rng.integers(0, kf, size=(B, S))
    ok = rng.random((B, S)) > 0.3
    local = run_error_sums(means, states, ks, ok, d)
    rmse, allrows = gather_rmse(local)
    q.put((rank, rmse.tolist(), allrows.tolist(), local.tolist()))
    dist.barrier()
    dist.destroy_process_group()


def test_gather_rmse_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    total, d, world = 11, 3, 2
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, d, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    locals_ = [np.array(r[3]) for r in res]
    ref = np.concatenate(locals_)
    ref_rmse = np.sqrt(ref[:, :d].sum(0) / ref[:, d].sum())
    for r in res:
        assert np.allclose(np.array(r[2]), ref)
        assert np.allclose(r[1], ref_rmse)


def _bank_worker(rank, world, port, total, q):
    """One rank of the sharded Monte Carlo driver over the engine's host
    emulation (FilterBank.run), gloo all-gather of the error sums."""
    import sys
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    from hostsim import HostBackend
    from paper_2501_07942_b200.configs import SCENARIOS
    from paper_2501_07942_b200.mc import run_monte_carlo
    from scenario_util import bank_config
    sc = SCENARIOS["radar_deg"]
    rmse, allrows, recs, runs = run_monte_carlo(sc["spec"], bank_config(sc, ws_bytes=64 << 20), sc["x0_mean"],
                                                sc["x0_cov"], total, sc["steps"], 3, backend=HostBackend())
    q.put((rank, rmse.tolist(), allrows.tolist(), runs.tolist(), recs["status"].tolist()))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _run_ranks(world, total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bank_worker, args=(r, world, port, total, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


def test_filterbank_run_sharded_gloo_world2():
    """2 gloo ranks running FilterBank.run on their shards reproduce the
    1-rank run: same per-run error rows, same RMSE, bit for bit."""
    total = 5
    one = _run_ranks(1, total)[0]
    two = _run_ranks(2, total)
    assert two[0][3] + two[1][3] == list(range(total))
    for r in two:
        assert np.array_equal(np.array(r[2]), np.array(one[2]))
        assert r[1] == one[1]
    assert np.all(np.isfinite(one[1])) and np.array(one[2])[:, -1].sum() > 0
