"""Monte Carlo sharding across GPUs.

Independent filter runs are the only parallel axis: run ids are split into
contiguous per-rank blocks with no data-path collective; at the end one
``all_gather_into_tensor`` collects each run's squared-error sums and step
counts, from which every rank forms the RMSE exactly as the reference
harness does (bench.py:369-371: sqrt of the mean squared error per state
component over all runs and steps).
"""

from __future__ import annotations

import numpy as np


def shard(total_runs: int, world: int, rank: int) -> np.ndarray:
    """Contiguous block of run ids owned by ``rank`` (sizes differ by <= 1)."""
    base, extra = divmod(int(total_runs), int(world))
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return np.arange(lo, hi)


def run_error_sums(means, states, ks, ok, d):
    """Per-run squared-error sums and completed-step counts from step records.

    means: (B, S, >=d) filtering means; states: (B, kf, d) true states;
    ks: (B, S) trajectory index of each record; ok: (B, S) completed mask.
    Returns (B, d + 1): columns 0..d-1 squared-error sums, column d counts.
    """
    B, S = ok.shape
    out = np.zeros((B, d + 1))
    for i in range(B):
        for s in range(S):
            if ok[i, s]:
                e = means[i, s, :d] - states[i, ks[i, s]]
                out[i, :d] += e * e
                out[i, d] += 1
    return out


def gather_rmse(local, group=None, device=None):
    """All-gather per-run (d+1)-vectors from every rank and return the RMSE.

    ``local`` is this rank's (B_r, d+1) array; ranks may hold different B_r
    (padded to the max for the collective).  Works with NCCL (CUDA tensors)
    and gloo (CPU tensors).
    """
    import torch
    import torch.distributed as dist
    local = np.asarray(local, dtype=np.float64)
    d1 = local.shape[1]
    if not (dist.is_available() and dist.is_initialized()):
        allrows = local
    else:
        world = dist.get_world_size(group)
        dev = device if device is not None else torch.device("cpu")
        n = torch.tensor([local.shape[0]], dtype=torch.int64, device=dev)
        ns = [torch.zeros_like(n) for _ in range(world)]
        dist.all_gather(ns, n, group=group)
        bmax = int(max(int(v) for v in ns))
        pad = np.zeros((bmax, d1))
        pad[: local.shape[0]] = local
        t = torch.tensor(pad, dtype=torch.float64, device=dev)
        out = torch.empty((world * bmax, d1), dtype=torch.float64, device=dev)
        dist.all_gather_into_tensor(out, t, group=group)
        full = out.cpu().numpy()
        allrows = np.concatenate([full[r * bmax: r * bmax + int(ns[r])] for r in range(world)])
    cnt = allrows[:, -1].sum()
    rmse = np.sqrt(allrows[:, :-1].sum(axis=0) / max(cnt, 1.0))
    return rmse, allrows


def run_monte_carlo(spec, bank_cfg, x0_mean, x0_cov, total_runs: int, kf: int, steps: int,
                    backend=None, group=None, device=None):
    """Sharded Monte Carlo driver: this rank's block of the ``total_runs``
    seeded trajectories (SeedSequence((2024, run, 0)), models.py:165-194)
    runs as one FilterBank through ``steps`` persistent-kernel filter steps;
    then one all-gather of the per-run error sums forms the RMSE
    (bench.py:369-371 of the reference).  Returns (rmse, allrows, recs, runs).
    """
    import torch.distributed as dist
    from paper_2501_07942_b200.bank import FilterBank
    from paper_2501_07942_b200.configs import simulate
    rank = dist.get_rank(group) if dist.is_available() and dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    runs = shard(total_runs, world, rank)
    d = np.asarray(spec["F"]).shape[0]
    sts, ms = [], []
    for r in runs:
        s, m = simulate(spec, x0_mean, x0_cov, kf, np.random.SeedSequence((2024, int(r), 0)))
        sts.append(s)
        ms.append(m)
    states, meas = np.stack(sts), np.stack(ms)
    bank = FilterBank(spec, bank_cfg, len(runs), backend=backend)
    recs = bank.run(meas, steps, x0_mean, x0_cov)
    local = run_error_sums(recs["mean"], states, recs["k"], recs["status"] == 0, d)
    rmse, allrows = gather_rmse(local, group=group, device=device)
    return rmse, allrows, recs, runs
