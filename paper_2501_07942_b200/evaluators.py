"""The cross black boxes evaluated directly on the device (no cross, no cache).

These are the values ``greedy_cross`` samples inside every filter stage, one
launch of ``ttgbf_eval_blackbox`` each; they exist so that each evaluator can
be pinned against the reference on its own:

======================  ===========================================  ===================
function                reference                                    kind
======================  ===========================================  ===================
prior_values            initial_pmd_tt eval_many, filters.py:504-505  TTGBF_BB_GAUSS
likelihood_values       StateSpaceModel.likelihood, models.py:150-153 TTGBF_BB_LIKELIHOOD
kernel_values           _kernel_values, filters.py:697-706            TTGBF_BB_KERNEL
realign_values          realign evaluator, filters.py:969-979         TTGBF_BB_REALIGN
======================  ===========================================  ===================

Models are passed as specs (``configs``) or :class:`models.StateSpaceModel`;
grids as :class:`grids.Grid` or :class:`geometry.Axes`.
"""

from __future__ import annotations

import numpy as np

from paper_2501_07942_b200 import _abi
from paper_2501_07942_b200 import geometry as geo
from paper_2501_07942_b200.bank import gauss_record, model_record

def _axes(grid) -> geo.Axes:
    return grid.device_axes if hasattr(grid, "device_axes") else grid


def _spec(model):
    return model.spec if hasattr(model, "spec") and not isinstance(model, dict) else model


def _io(cur=None, z=None, filt=None, pred=None):
    io = np.zeros(1, dtype=_abi.FILTER_IO)
    for field, ax in (("cur", cur), ("filt", filt), ("pred", pred)):
        if ax is not None:
            io[field][0] = _axes(ax).device()
    if z is not None:
        zz = np.atleast_1d(np.asarray(z, dtype=float))
        io["z"][0, : zz.size] = zz
    return io


def _launch(kind, spec, idx, io, prior=None, tt=None):
    """One launch over len(io) items; idx is (items, K, d)."""
    from paper_2501_07942_b200.tensor_train import _be, _hdr_dev
    be = _be()
    idx = np.ascontiguousarray(np.asarray(idx, dtype=np.int32))
    d = np.asarray(spec["F"]).shape[0]
    if idx.ndim != 3 or idx.shape[2] != d or idx.shape[0] != len(io):
        raise ValueError(f"idx must be (items, K, {d})")
    count, K = idx.shape[0], idx.shape[1]
    model = be.upload(model_record(spec))
    pr = be.upload(gauss_record(*prior)) if prior is not None else None
    iod = be.upload(io)
    idd = be.upload(idx if idx.size else np.zeros((1, d), np.int32))
    out = be.empty(8 * max(count * K, 1))
    st = be.empty(4 * count)
    # per item: axes + spec, and for REALIGN the pulled-back points and the
    # bucketed evaluation's rank vectors
    maxr = max(tt.ranks) if tt is not None else 1
    wsb = (1 << 20) + (K * (8 * d + 16 * maxr + 64) if tt is not None else 0)
    wsb = (wsb + 255) // 256 * 256
    ws = be.empty(wsb * count)
    th = _hdr_dev(tt) if tt is not None else None
    rc = be.lib.ttgbf_eval_blackbox(kind, model.ptr, pr.ptr if pr else None, iod.ptr, th.ptr if th else None,
                                    tt.data.data_ptr() if tt is not None else None, tt.size if tt is not None else 0,
                                    count, idd.ptr, K, out.ptr, ws.ptr, wsb, st.ptr, be.stream_ptr)
    be.check(rc, "ttgbf_eval_blackbox")
    for s in be.download(st, np.int32, count):
        if int(s):
            raise ValueError(f"ttgbf_eval_blackbox: {_abi.status_text(int(s))}")
    return be.download(out, np.float64, count * K).reshape(count, K)


def _call(kind, spec, idx, cur=None, z=None, prior=None, tt=None, filt=None, pred=None):
    idx = np.asarray(idx)
    return _launch(kind, spec, idx[None], _io(cur, z, filt, pred), prior, tt)[0]


def prior_values(mean, cov, grid, idx) -> np.ndarray:
    """N(x - mean; cov) at the grid nodes ``idx`` (initial_pmd_tt's black box)."""
    mean = np.atleast_1d(np.asarray(mean, dtype=float))
    spec = {"F": np.eye(mean.size), "Q": np.eye(mean.size), "R": np.eye(1), "h": "linear",
            "H": np.zeros((1, mean.size))}
    return _call(_abi.BB_GAUSS, spec, idx, cur=grid, prior=(mean, np.atleast_2d(cov)))


def likelihood_values(model, grid, z, idx) -> np.ndarray:
    """p(z | x) at the grid nodes ``idx`` (StateSpaceModel.likelihood)."""
    return _call(_abi.BB_LIKELIHOOD, _spec(model), idx, cur=grid, z=z)


def likelihood_at_points(model, z, x) -> np.ndarray:
    """p(z | x) at arbitrary points x (K, d) -- StateSpaceModel.likelihood(z, x)
    exactly: each point becomes the node of its own one-cell grid."""
    spec = _spec(model)
    x = np.atleast_2d(np.asarray(x, dtype=float))
    K, d = x.shape
    io = np.zeros(K, dtype=_abi.FILTER_IO)
    for p in range(K):
        io[p] = _io(geo.Axes(x[p], np.ones(d), np.zeros(d, dtype=np.int32), np.full(d, 2, dtype=np.int32)), z)[0]
    return _launch(_abi.BB_LIKELIHOOD, spec, np.zeros((K, 1, d), np.int32), io)[:, 0]


def kernel_values(model, grid, idx) -> np.ndarray:
    """N(disp F^T; 0, Q) * cell volume at ifftshift indices (_kernel_values)."""
    return _call(_abi.BB_KERNEL, _spec(model), idx, cur=grid)


def realign_values(model, conv_tt, filt_grid, pred_grid, idx) -> np.ndarray:
    """The convolved TT (on ``filt_grid``) at F^-1 y for predictive nodes y
    (the realign black box of tt_fft_pmf_step); zero outside the hull."""
    return _call(_abi.BB_REALIGN, _spec(model), idx, tt=conv_tt, filt=filt_grid, pred=pred_grid)


def rng_draws(state6, *, shape=None, K=0, pop=0, size=0):
    """The cross's numpy-compatible draws on the device (``ttgbf_rng_draws``).

    ``state6`` is numpy's PCG64 state as six uint64 (state lo/hi, increment
    lo/hi, has_uint32, uinteger).  With ``shape``: ``rng.integers(0, shape,
    size=(K, len(shape)))``; otherwise ``rng.choice(pop, size, replace=False)``.
    Returns (values, state6 after the call)."""
    from paper_2501_07942_b200.tensor_train import _be
    be = _be()
    st = be.upload(np.asarray(state6, dtype=np.uint64))
    status = be.upload(np.zeros(1, dtype=np.int32))
    if shape is not None:
        sh = np.asarray(shape, dtype=np.int32)
        n, kind = int(K) * sh.size, 0
        shd = be.upload(sh)
        d = sh.size
    else:
        n, kind = int(size), 1
        shd = be.upload(np.zeros(1, dtype=np.int32))
        d = 1
    out = be.empty(8 * max(n, 1))
    ws_bytes = 16 * (int(pop) + 8 * int(size) + int(K) * d) + (1 << 20)
    ws = be.empty(ws_bytes)
    be.check(be.lib.ttgbf_rng_draws(kind, st.ptr, shd.ptr, d, int(K), int(pop), int(size), out.ptr, ws.ptr, ws_bytes,
                                    status.ptr, be.stream_ptr), "ttgbf_rng_draws")
    be.sync()
    rc = int(be.download(status, np.int32, 1)[0])
    if rc != 0:
        raise RuntimeError(f"ttgbf_rng_draws: {_abi.status_text(rc)}")
    return be.download(out, np.int64, n), be.download(st, np.uint64, 6)
