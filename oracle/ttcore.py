"""TT primitives, restated from the reference (TEST INFRASTRUCTURE ONLY).

A TT is a plain ``list`` of float64 cores shaped ``(r_left, n, r_right)``
with unit boundary ranks.  Each function cites the reference routine whose
arithmetic it reproduces; the numpy/LAPACK calls are the same ones the
reference issues so that results pin bit-for-bit where LAPACK is
deterministic.
"""

from __future__ import annotations

import math

import numpy as np

DENSE_LIMIT = 10_000_000  # tensor_train.py:55 (DENSE_GUARD_DEFAULT)


def ranks_of(cores) -> tuple[int, ...]:
    return (1,) + tuple(int(c.shape[2]) for c in cores)


def mode_sizes(cores) -> tuple[int, ...]:
    return tuple(int(c.shape[1]) for c in cores)


# -- element access ---------------------------------------------------------

def at_indices(cores, idx) -> np.ndarray:
    """Values at integer multi-indices (K, d).  tensor_train.py:129-158.

    Mirrors the reference's two contraction regimes (batched einsum for
    small slabs, per-slice matmuls for large ones) so that rounding matches.
    """
    idx = np.asarray(idx, dtype=np.intp)
    acc = cores[0][0, idx[:, 0], :]
    for k in range(1, len(cores)):
        g = cores[k]
        rl, n, rr = g.shape
        sel = idx[:, k]
        if rl * rr * sel.size <= 4_000_000:
            acc = np.einsum("kr,rkc->kc", acc, g[:, sel, :])
            continue
        perm = np.argsort(sel, kind="stable")
        cuts = np.searchsorted(sel[perm], np.arange(n + 1))
        nxt = np.empty((sel.size, rr))
        for j in range(n):
            if cuts[j] < cuts[j + 1]:
                rows = perm[cuts[j]:cuts[j + 1]]
                nxt[rows] = acc[rows] @ g[:, j, :]
        acc = nxt
    return acc[:, 0]


def to_full(cores, limit: int = DENSE_LIMIT) -> np.ndarray:
    """Dense materialisation.  tensor_train.py:214-227."""
    shape = mode_sizes(cores)
    if math.prod(shape) > limit:
        raise MemoryError(f"dense tensor {shape} exceeds {limit} elements")
    m = cores[0].reshape(shape[0], -1)
    for g in cores[1:]:
        rl, n, rr = g.shape
        m = (m @ g.reshape(rl, n * rr)).reshape(-1, rr)
    return m.reshape(shape)


def rank1(vectors) -> list[np.ndarray]:
    """tensor_train.py:230-235."""
    return [np.asarray(v, dtype=np.float64).reshape(1, -1, 1) for v in vectors]


# -- arithmetic -------------------------------------------------------------

def kron_cores(a, b) -> list[np.ndarray]:
    """Core-wise Kronecker product (Hadamard of tensors).  tensor_train.py:252-266."""
    out = []
    for ga, gb in zip(a, b):
        p = np.einsum("aib,cid->acibd", ga, gb)
        out.append(p.reshape(ga.shape[0] * gb.shape[0], ga.shape[1],
                             ga.shape[2] * gb.shape[2]))
    return out


def total(cores) -> float:
    """Sum of all entries.  tensor_train.py:283-288."""
    v = np.ones((1,))
    for g in cores:
        v = v @ g.sum(axis=1)
    return float(v[0])


def inner(a, b) -> float:
    """Frobenius inner product.  tensor_train.py:269-275."""
    v = np.ones((1, 1))
    for ga, gb in zip(a, b):
        v = np.einsum("ac,aib,cid->bd", v, ga, gb, optimize=True)
    return float(v[0, 0])


def scaled(cores, c: float) -> list[np.ndarray]:
    """tensor_train.py:291-295 (factor folded into core 0)."""
    return [cores[0] * float(c)] + list(cores[1:])


# -- rounding ---------------------------------------------------------------

def keep_rank(sv: np.ndarray, delta: float, cap) -> int:
    """Truncation rule.  tensor_train.py:165-176.

    First r whose discarded tail energy sum(sv[r:]**2) <= delta**2 (at least
    1), then clipped to ``cap``.
    """
    if delta > 0.0:
        tail = np.cumsum(sv[::-1] ** 2)[::-1]
        r = max(int(np.searchsorted(-tail, -delta * delta)), 1)
    else:
        r = max(len(sv), 1)
    if cap is not None:
        r = min(r, cap)
    return r


def round_tt(cores, tol: float, cap=None) -> list[np.ndarray]:
    """TT rounding.  tensor_train.py:327-360.

    Right-to-left QR (cores 1..d-1 row-orthonormal, norm lands in core 0),
    delta = tol*||core0||/sqrt(d-1), then left-to-right truncated SVDs.
    """
    if tol < 0.0:
        raise ValueError("tol must be nonnegative")
    d = len(cores)
    work = [np.array(g, dtype=np.float64, copy=True) for g in cores]
    if d == 1:
        return work
    for k in range(d - 1, 0, -1):
        rl, n, rr = work[k].shape
        q, r = np.linalg.qr(work[k].reshape(rl, n * rr).T)
        work[k] = q.T.reshape(q.shape[1], n, rr)
        work[k - 1] = np.tensordot(work[k - 1], r.T, axes=([2], [0]))
    nrm = float(np.linalg.norm(work[0]))
    if nrm == 0.0:
        return [np.zeros((1, g.shape[1], 1)) for g in cores]
    delta = tol * nrm / math.sqrt(d - 1)
    for k in range(d - 1):
        rl, n, rr = work[k].shape
        u, s, vt = np.linalg.svd(work[k].reshape(rl * n, rr), full_matrices=False)
        r = keep_rank(s, delta, cap)
        work[k] = u[:, :r].reshape(rl, n, r)
        work[k + 1] = np.tensordot(s[:r, None] * vt[:r], work[k + 1], axes=([1], [0]))
    return work


# -- FFT convolution --------------------------------------------------------

def fft_conv(kernel, weights, tol: float, cap=None) -> list[np.ndarray]:
    """Circular convolution in TT form.  tt_algorithms.py:642-666."""
    if mode_sizes(kernel) != mode_sizes(weights):
        raise ValueError("shape mismatch")
    if any(n % 2 == 0 for n in mode_sizes(kernel)):
        raise ValueError("mode sizes must be odd")
    fk = [np.fft.fft(g, axis=1) for g in kernel]
    fw = [np.fft.fft(g, axis=1) for g in weights]
    prod = kron_cores(fk, fw)
    real = [np.fft.ifft(g, axis=1).real for g in prod]
    return round_tt(real, tol, cap)


# -- interpolation ----------------------------------------------------------

_HULL_EPS = 1e-9  # tt_algorithms.py:680


def cell_weights(points, axis):
    """(cell, frac, inside) for 1-D points on an equidistant axis.

    tt_algorithms.py:673-684.
    """
    axis = np.asarray(axis, dtype=float)
    x = np.asarray(points, dtype=float).reshape(-1)
    n = len(axis)
    step = (axis[-1] - axis[0]) / (n - 1)
    pos = (x - axis[0]) / step
    inside = (pos >= -_HULL_EPS) & (pos <= n - 1 + _HULL_EPS)
    cell = np.clip(np.floor(pos).astype(np.intp), 0, n - 2)
    frac = np.clip(pos - cell, 0.0, 1.0)
    return cell, frac, inside


def interp_matrix(new_axis, old_axis) -> np.ndarray:
    """Two-tap linear interpolation matrix (N_new, N_old).  tt_algorithms.py:687-698."""
    cell, frac, inside = cell_weights(new_axis, old_axis)
    w = np.zeros((len(cell), len(np.asarray(old_axis))))
    rows = np.arange(len(cell))[inside]
    np.add.at(w, (rows, cell[inside]), 1.0 - frac[inside])
    np.add.at(w, (rows, cell[inside] + 1), frac[inside])
    return w


def regrid(cores, old_axes, new_axes) -> list[np.ndarray]:
    """Separable linear resampling onto a new grid.  tt_algorithms.py:701-718."""
    out = []
    for g, oa, na in zip(cores, old_axes, new_axes):
        w = interp_matrix(na, oa)
        out.append(np.tensordot(g, w, axes=([1], [1])).transpose(0, 2, 1))
    return out


def at_points(cores, axes, points) -> np.ndarray:
    """Multilinear evaluation at continuous points (K, d).  tt_algorithms.py:721-745."""
    pts = np.atleast_2d(np.asarray(points, dtype=float))
    kcount = pts.shape[0]
    acc = np.ones((kcount, 1, 1))
    alive = np.ones(kcount, dtype=bool)
    for ell, g in enumerate(cores):
        cell, frac, inside = cell_weights(pts[:, ell], np.asarray(axes[ell]))
        alive &= inside
        lo = g[:, cell, :]
        hi = g[:, cell + 1, :]
        fib = lo * (1.0 - frac)[None, :, None] + hi * frac[None, :, None]
        acc = np.einsum("kar,rkc->kac", acc, fib)
    out = acc[:, 0, 0]
    out[~alive] = 0.0
    return out


def einsum_tpm(tcores, wcores):
    """tt_einsum_tpm (tt_algorithms.py:603-635): contract the 2d-mode transition
    TT with the d-mode weights over modes d..2d-1 by the backward fold
    z <- einsum('anb,cnd,bd->ac'), then absorb z into core d-1."""
    d = len(wcores)
    if len(tcores) != 2 * d:
        raise ValueError(f"transition tensor must have {2 * d} modes, got {len(tcores)}")
    z = np.ones((1, 1))
    for j in range(d - 1, -1, -1):
        z = np.einsum("anb,cnd,bd->ac", tcores[d + j], wcores[j], z, optimize=True)
    out = [np.asarray(c) for c in tcores[: d - 1]]
    out.append(np.einsum("anb,bz->anz", tcores[d - 1], z))
    return out
