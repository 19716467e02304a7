"""Algorithmic FLOP accounting for one TT-FFT step from the device shape log.

Formulas are SURVEY.md section 8(d) (LAPACK-style leading order); ranks
come from ``ttgbf_diag.ranks`` (input, likelihood, filtering, shifted,
kernel, rounded convolution, realign cross, output TTs) and the evaluator
call counts from ``ttgbf_diag.cross``.  The count is what the algorithm
must do, not what the kernels execute (e.g. Jacobi SVD does more).
"""

from __future__ import annotations

import math

import numpy as np


def _r(row, slot, d):
    return [int(v) for v in row["ranks"][slot][: d + 1]]


def round_flops(ranks, n, out_ranks):
    """tt_round: right-to-left Householder QR (+Q, +carry), left-to-right SVD (+carry)."""
    d = len(ranks) - 1
    R = list(ranks)
    f = 0.0
    for k in range(d - 1, 0, -1):
        m, c = n * R[k + 1], R[k]
        kk = min(m, c)
        f += 4.0 * m * c * kk - (4.0 / 3.0) * kk ** 3          # geqrf + orgqr
        f += 2.0 * R[k - 1] * n * c * kk                        # carry into core k-1
        R[k] = kk
    for k in range(d - 1):
        rl = out_ranks[k]
        m, c = rl * n, R[k + 1]
        kk = min(m, c)
        f += 6.0 * max(m, c) * kk * kk + 20.0 * kk ** 3         # R-SVD with vectors
        rn = out_ranks[k + 1]
        f += 2.0 * rn * c * n * R[k + 2]                         # carry into core k+1
    return f


def chain_size(ranks, n):
    return sum(ranks[k] * n * ranks[k + 1] for k in range(len(ranks) - 1))


def cross_flops(calls, ranks, n, per_eval):
    d = len(ranks) - 1
    f = calls * per_eval
    for k in range(d - 1):   # final core solves (lower bound of the incremental solves)
        r = ranks[k + 1]
        f += (4.0 / 3.0) * r ** 3 + 4.0 * r * r * ranks[k] * n
    return f


def _squeezed(row, slot, d, full):
    """Ranks after the engine's exact-rank squeeze (log slots 8 / 9) when logged."""
    ranks = row["ranks"]
    if len(ranks) <= slot or not int(ranks[slot][0]):
        return full
    return [int(v) for v in ranks[slot][: d + 1]]


def step_flops(dm_row, dt_row, d, b, n, executed=False):
    """(measure_flops, time_update_flops) for one filter step.

    executed=False: the reference algorithm's work (products of
    the cross outputs as they come).  executed=True: the same formulas on the
    ranks the engine's products actually have after the exact-rank squeeze of
    the likelihood / kernel TTs (plus the squeeze's own rounding)."""
    rin = _r(dm_row, 0, d)
    rlik = _r(dm_row, 1, d)
    rfil = _r(dm_row, 2, d)
    fm = 0.0
    if rlik[0]:
        fm += cross_flops(int(dm_row["cross"][0]["calls"]), rlik, n, 2 * b * b + 10 * b + d)
        if executed:
            rsq = _squeezed(dm_row, 8, d, rlik)
            fm += round_flops(rlik, n, rsq)
            rlik = rsq
        prod = [a * c for a, c in zip(rin, rlik)]
        fm += chain_size(prod, n)                                  # Hadamard
        fm += round_flops(prod, n, rfil)
    nmom = 1 + d + d * (d + 1) // 2
    fm += 6.0 * chain_size(rfil, n) + nmom * 2.0 * sum(rfil[k] * rfil[k + 1] for k in range(d))
    rsh = _r(dt_row, 3, d)
    rker = _r(dt_row, 4, d)
    rconv = _r(dt_row, 5, d)
    rre = _r(dt_row, 6, d)
    rout = _r(dt_row, 7, d)
    ft = 4.0 * chain_size(rfil, n) + round_flops(rfil, n, rsh)    # interp + finalize
    ft += cross_flops(int(dt_row["cross"][1]["calls"]), rker, n, 2 * d * d + 2 * d + 10)
    if executed:
        rsq = _squeezed(dt_row, 9, d, rker)
        ft += round_flops(rker, n, rsq)
        rker = rsq
    prod = [a * c for a, c in zip(rker, rsh)]
    fib = sum(rker[k] * rker[k + 1] + rsh[k] * rsh[k + 1] for k in range(d))
    ft += 5.0 * n * math.log2(n) * fib + 6.0 * chain_size(prod, n) + 5.0 * n * math.log2(n) * sum(
        prod[k] * prod[k + 1] for k in range(d))
    ft += round_flops(prod, n, rconv)
    per_real = 5.0 * sum(rconv[k] * rconv[k + 1] for k in range(d)) + 2 * d * d
    ft += cross_flops(int(dt_row["cross"][2]["calls"]), rre, n, per_real)
    ft += round_flops(rre, n, rout)
    return fm, ft


def measure_fp64_sustained(torch, device, n=8192, seconds=3.0):
    """cuBLAS DGEMM back to back for ~`seconds` (CUDA events around the whole
    sequence): the sustained FP64 rate, the fair denominator for a launch
    that runs for tens of seconds (the burst figure is the best single GEMM)."""
    a = torch.randn(n, n, dtype=torch.float64, device=device)
    b = torch.randn(n, n, dtype=torch.float64, device=device)
    c = torch.matmul(a, b)
    torch.cuda.synchronize(device)
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record()
    torch.matmul(a, b, out=c)
    e.record()
    torch.cuda.synchronize(device)
    one = s.elapsed_time(e) / 1e3
    reps = max(2, int(seconds / max(one, 1e-4)))
    s.record()
    for _ in range(reps):
        torch.matmul(a, b, out=c)
    e.record()
    torch.cuda.synchronize(device)
    t = s.elapsed_time(e) / 1e3
    del a, b, c
    return 2.0 * n ** 3 * reps / t / 1e12


def measure_fp64_peak(torch, device, n=8192, reps=5):
    """cuBLAS DGEMM burst (best of reps) in TFLOP/s -- the FP64 roofline denominator."""
    a = torch.randn(n, n, dtype=torch.float64, device=device)
    b = torch.randn(n, n, dtype=torch.float64, device=device)
    torch.matmul(a, b)
    torch.cuda.synchronize(device)
    best = float("inf")
    for _ in range(reps):
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        torch.matmul(a, b)
        e.record()
        torch.cuda.synchronize(device)
        best = min(best, s.elapsed_time(e) / 1e3)
    del a, b
    return 2.0 * n ** 3 / best / 1e12


class _Row:
    """Adapter: a STEP_REC viewed as the (measure, time) diag rows."""

    def __init__(self, rec):
        self.rec = rec

    def __getitem__(self, key):
        if key == "ranks":
            return self.rec["ranks"]
        if key == "cross":
            calls = self.rec["calls"]
            return [{"calls": int(calls[q])} for q in range(3)]
        return self.rec[key]


def rec_flops(rec, d, b, n, executed=False):
    """(measure, time) algorithmic FLOPs of one persistent-run step record."""
    r = _Row(rec)
    return step_flops(r, r, d, b, n, executed)
