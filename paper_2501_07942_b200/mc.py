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
