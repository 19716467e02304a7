"""Device-resident tensor trains and the TT primitives (drop-in for ``ttpmf.tensor_train``).

A :class:`TensorTrain` holds its cores packed in one float64 CUDA buffer
plus a ``ttgbf_tt`` header (include/ttgbf.h).  Every operation below is one
launch of a hand-written sm_100a kernel from ``libttgbf.so``:

=====================  =====================================  =========================
function               reference                              entry point
=====================  =====================================  =========================
tt_round               tensor_train.py:327-360                ttgbf_tt_round
tt_hadamard            tensor_train.py:252-266                ttgbf_tt_hadamard
tt_fft_convolve        tt_algorithms.py:642-666               ttgbf_tt_fft_convolve
tt_interpolate         tt_algorithms.py:701-718               ttgbf_tt_interpolate
tt_eval_many           tensor_train.py:129-158                ttgbf_tt_eval_many
tt_eval_at_points      tt_algorithms.py:721-745               ttgbf_tt_eval_at_points
tt_sum / moments       tensor_train.py:283-288, 269-275       ttgbf_tt_sum_moments
negative mass          filters.py:427-436                     ttgbf_negative_mass
=====================  =====================================  =========================
"""

from __future__ import annotations

import math

import numpy as np

from paper_2501_07942_b200 import _abi
from paper_2501_07942_b200 import geometry as geo

_CTX = {}


def _be():
    be = _CTX.get("be")
    if be is None:
        from paper_2501_07942_b200.backend import CudaBackend
        be = CudaBackend()
        _CTX["be"] = be
    return be


def _ws(nbytes: int):
    buf = _CTX.get("ws")
    if buf is None or buf.nbytes < nbytes:
        buf = _be().empty(nbytes)
        _CTX["ws"] = buf
    return buf


WS_BYTES = 512 << 20


class TensorTrain:
    """Immutable device TT: packed float64 cores + ttgbf_tt header."""

    def __init__(self, hdr: np.ndarray, data):
        self.hdr = hdr.copy()          # numpy record of dtype _abi.TT (shape ())
        self.data = data               # torch float64 CUDA tensor (flat)

    # -- construction ---------------------------------------------------------
    @classmethod
    def from_cores(cls, cores) -> "TensorTrain":
        import torch
        be = _be()
        cores = [np.ascontiguousarray(np.asarray(c, dtype=np.float64)) for c in cores]
        if not cores:
            raise ValueError("a tensor train needs at least one core")
        for k, c in enumerate(cores):
            if c.ndim != 3 or min(c.shape) < 1:
                raise ValueError(f"core {k} has shape {c.shape}")
        if cores[0].shape[0] != 1 or cores[-1].shape[2] != 1:
            raise ValueError("boundary ranks must both equal 1")
        for k in range(len(cores) - 1):
            if cores[k].shape[2] != cores[k + 1].shape[0]:
                raise ValueError(f"rank mismatch between cores {k} and {k + 1}")
        if len(cores) > _abi.MAXD:
            raise ValueError("at most 16 modes")
        h = np.zeros((), dtype=_abi.TT)
        h["d"] = len(cores)
        off = 0
        for k, c in enumerate(cores):
            h["n"][k] = c.shape[1]
            h["r"][k] = c.shape[0]
            h["off"][k] = off
            off += c.size
        h["r"][len(cores)] = 1
        flat = np.concatenate([c.reshape(-1) for c in cores])
        data = torch.from_numpy(flat).to(be.device)
        return cls(h, data)

    # -- properties -------------------------------------------------------------
    @property
    def ndim(self) -> int:
        return int(self.hdr["d"])

    @property
    def shape(self) -> tuple[int, ...]:
        return tuple(int(v) for v in self.hdr["n"][: self.ndim])

    @property
    def ranks(self) -> tuple[int, ...]:
        return tuple(int(v) for v in self.hdr["r"][: self.ndim + 1])

    def core_shape(self, k):
        return (int(self.hdr["r"][k]), int(self.hdr["n"][k]), int(self.hdr["r"][k + 1]))

    @property
    def size(self) -> int:
        return sum(math.prod(self.core_shape(k)) for k in range(self.ndim))

    @property
    def cores(self):
        """Device views of the cores (torch tensors)."""
        out = []
        for k in range(self.ndim):
            o = int(self.hdr["off"][k])
            shp = self.core_shape(k)
            out.append(self.data[o: o + math.prod(shp)].view(*shp))
        return out

    def numpy_cores(self) -> list[np.ndarray]:
        return [c.cpu().numpy() for c in self.cores]

    def storage_bytes(self) -> int:
        return 8 * self.size

    def __repr__(self):
        return f"TensorTrain(shape={self.shape}, ranks={self.ranks}, device)"


def _hdr_dev(tt: TensorTrain):
    return _be().upload(tt.hdr.reshape(1))


def _status(st, what):
    if int(st) != 0:
        if int(st) in (_abi.E_ARG, _abi.E_NONFINITE):
            raise ValueError(f"{what}: {_abi.status_text(st)}")
        raise RuntimeError(f"{what}: {_abi.status_text(st)}")


def _out_tt(hdr_buf, out_t) -> TensorTrain:
    be = _be()
    h = be.download(hdr_buf, _abi.TT, 1)[0]
    n = sum(int(h["r"][k]) * int(h["n"][k]) * int(h["r"][k + 1]) for k in range(int(h["d"])))
    return TensorTrain(h, out_t[:n].clone())


def _alloc_out(cap_doubles):
    import torch
    return torch.empty(max(int(cap_doubles), 1), dtype=torch.float64, device=_be().device)


def _run_unary(fn, tt: TensorTrain, out_cap, *args, what=""):
    be = _be()
    st = be.empty(4)
    oh = be.empty(_abi.TT.itemsize)
    out = _alloc_out(out_cap)
    ws = _ws(WS_BYTES)
    keep = _hdr_dev(tt)
    rc = fn(keep.ptr, tt.data.data_ptr(), tt.size, 1, *args, oh.ptr, out.data_ptr(), out.numel(),
            ws.ptr, WS_BYTES, st.ptr, be.stream_ptr)
    be.check(rc, what)
    _status(be.download(st, np.int32, 1)[0], what)
    return _out_tt(oh, out)


def tt_round(tt: TensorTrain, tol: float, max_rank: int | None = None) -> TensorTrain:
    if tol < 0.0:
        raise ValueError("tol must be nonnegative")
    lib = _be().lib
    return _run_unary(lib.ttgbf_tt_round, tt, tt.size + 16, float(tol), int(max_rank or 0), what="tt_round")


def tt_hadamard(a: TensorTrain, b: TensorTrain) -> TensorTrain:
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch: {a.shape} vs {b.shape}")
    be = _be()
    cap = sum(math.prod(a.core_shape(k)) * b.core_shape(k)[0] * b.core_shape(k)[2] for k in range(a.ndim))
    st, oh, out = be.empty(4), be.empty(_abi.TT.itemsize), _alloc_out(cap)
    ws = _ws(WS_BYTES)
    ha, hb = _hdr_dev(a), _hdr_dev(b)
    rc = be.lib.ttgbf_tt_hadamard(ha.ptr, a.data.data_ptr(), a.size, hb.ptr, b.data.data_ptr(),
                                  b.size, 1, oh.ptr, out.data_ptr(), out.numel(), ws.ptr, WS_BYTES, st.ptr,
                                  be.stream_ptr)
    be.check(rc, "tt_hadamard")
    _status(be.download(st, np.int32, 1)[0], "tt_hadamard")
    return _out_tt(oh, out)


def tt_fft_convolve(kernel: TensorTrain, weights: TensorTrain, round_tol: float,
                    max_rank: int | None = None) -> TensorTrain:
    if kernel.shape != weights.shape:
        raise ValueError(f"shape mismatch: {kernel.shape} vs {weights.shape}")
    if any(n % 2 == 0 for n in kernel.shape):
        raise ValueError(f"mode sizes must be odd, got {kernel.shape}")
    be = _be()
    cap = sum(math.prod(kernel.core_shape(k)) * weights.core_shape(k)[0] * weights.core_shape(k)[2]
              for k in range(kernel.ndim))
    st, oh, out = be.empty(4), be.empty(_abi.TT.itemsize), _alloc_out(cap)
    ws = _ws(WS_BYTES)
    hk, hw = _hdr_dev(kernel), _hdr_dev(weights)
    rc = be.lib.ttgbf_tt_fft_convolve(hk.ptr, kernel.data.data_ptr(), kernel.size,
                                      hw.ptr, weights.data.data_ptr(), weights.size, 1,
                                      float(round_tol), int(max_rank or 0), oh.ptr, out.data_ptr(), out.numel(),
                                      ws.ptr, WS_BYTES, st.ptr, be.stream_ptr)
    be.check(rc, "tt_fft_convolve")
    _status(be.download(st, np.int32, 1)[0], "tt_fft_convolve")
    return _out_tt(oh, out)


def _axes_dev(ax: geo.Axes):
    return _be().upload(ax.device()[: ax.dim])


def tt_interpolate(weights: TensorTrain, old_grid, new_grid) -> TensorTrain:
    if weights.shape != old_grid.shape:
        raise ValueError("weight shape does not match old grid")
    be = _be()
    lib = be.lib
    st, oh, out = be.empty(4), be.empty(_abi.TT.itemsize), _alloc_out(weights.size + 16)
    ws = _ws(WS_BYTES)
    hh, ao, an = _hdr_dev(weights), _axes_dev(old_grid.device_axes), _axes_dev(new_grid.device_axes)
    rc = lib.ttgbf_tt_interpolate(hh.ptr, weights.data.data_ptr(), weights.size, 1,
                                  ao.ptr, an.ptr,
                                  oh.ptr, out.data_ptr(), out.numel(), ws.ptr, WS_BYTES, st.ptr, be.stream_ptr)
    be.check(rc, "tt_interpolate")
    _status(be.download(st, np.int32, 1)[0], "tt_interpolate")
    return _out_tt(oh, out)


def tt_eval_many(tt: TensorTrain, idx) -> np.ndarray:
    idx = np.ascontiguousarray(np.asarray(idx, dtype=np.int32))
    if idx.ndim != 2 or idx.shape[1] != tt.ndim:
        raise IndexError(f"expected index array of shape (K, {tt.ndim}), got {idx.shape}")
    for k, n in enumerate(tt.shape):
        if idx.shape[0] and (idx[:, k].min() < 0 or idx[:, k].max() >= n):
            raise IndexError(f"index out of bounds for mode {k} of size {n}")
    be = _be()
    K = idx.shape[0]
    di = be.upload(idx)
    out = be.empty(8 * K)
    st = be.empty(4)
    hh = _hdr_dev(tt)
    ws = _ws(WS_BYTES)
    rc = be.lib.ttgbf_tt_eval_many(hh.ptr, tt.data.data_ptr(), tt.size, 1, di.ptr, K, out.ptr, ws.ptr, WS_BYTES,
                                   st.ptr, be.stream_ptr)
    be.check(rc, "tt_eval_many")
    _status(be.download(st, np.int32, 1)[0], "tt_eval_many")
    return be.download(out, np.float64, K)


def tt_eval_at_points(tt: TensorTrain, grid, points) -> np.ndarray:
    pts = np.ascontiguousarray(np.atleast_2d(np.asarray(points, dtype=float)))
    if pts.shape[1] != tt.ndim:
        raise ValueError(f"expected points of dimension {tt.ndim}, got {pts.shape[1]}")
    be = _be()
    K = pts.shape[0]
    dp = be.upload(pts)
    out = be.empty(8 * K)
    st = be.empty(4)
    ws = _ws(WS_BYTES)
    hh, ax = _hdr_dev(tt), _axes_dev(grid.device_axes)
    rc = be.lib.ttgbf_tt_eval_at_points(hh.ptr, tt.data.data_ptr(), tt.size, 1,
                                        ax.ptr, dp.ptr, K, out.ptr, ws.ptr, WS_BYTES,
                                        st.ptr, be.stream_ptr)
    be.check(rc, "tt_eval_at_points")
    _status(be.download(st, np.int32, 1)[0], "tt_eval_at_points")
    return be.download(out, np.float64, K)


def tt_raw_moments(tt: TensorTrain, axes: geo.Axes) -> np.ndarray:
    """[sum, first (d), second (i<=j)] un-normalised contractions against the grid."""
    be = _be()
    out = be.empty(8 * _abi.NMOM)
    st = be.empty(4)
    ws = _ws(WS_BYTES)
    hh, ax = _hdr_dev(tt), _axes_dev(axes)
    rc = be.lib.ttgbf_tt_sum_moments(hh.ptr, tt.data.data_ptr(), tt.size, 1, ax.ptr,
                                     out.ptr, ws.ptr, WS_BYTES, st.ptr, be.stream_ptr)
    be.check(rc, "tt_sum_moments")
    _status(be.download(st, np.int32, 1)[0], "tt_sum_moments")
    return be.download(out, np.float64, _abi.NMOM)


def tt_sum(tt: TensorTrain) -> float:
    ax = geo.Axes(np.zeros(tt.ndim), np.ones(tt.ndim), np.zeros(tt.ndim), tt.shape)
    return float(tt_raw_moments(tt, ax)[0])


def tt_dot(a: TensorTrain, b: TensorTrain) -> float:
    """Frobenius inner product as the sum of the Hadamard product."""
    return tt_sum(tt_hadamard(a, b))


def tt_scale(a: TensorTrain, c: float) -> TensorTrain:
    out = TensorTrain(a.hdr, a.data.clone())
    n0 = math.prod(a.core_shape(0))
    out.data[:n0] *= float(c)
    return out


def negative_mass(tt: TensorTrain, grid, guard: int) -> float:
    be = _be()
    probes = be.upload(geo.probe_cells(grid.shape))
    out = be.empty(8)
    st = be.empty(4)
    ws = _ws(WS_BYTES)
    hh, ax = _hdr_dev(tt), _axes_dev(grid.device_axes)
    rc = be.lib.ttgbf_negative_mass(hh.ptr, tt.data.data_ptr(), tt.size, 1,
                                    ax.ptr, int(guard), probes.ptr, 4096, out.ptr, ws.ptr,
                                    WS_BYTES, st.ptr, be.stream_ptr)
    be.check(rc, "negative_mass")
    _status(be.download(st, np.int32, 1)[0], "negative_mass")
    return float(be.download(out, np.float64, 1)[0])


def finalize(weights: TensorTrain, grid, cfg):
    """_finalize_tt (filters.py:454-479) -> (weights, mass_before_norm, clipped_mass)."""
    from paper_2501_07942_b200.filters import DegenerateDensityError
    dv = grid.cell_volume
    if cfg.normalize_before_round:
        mass = tt_sum(weights) * dv
        if not math.isfinite(mass) or mass <= 1e-300:
            raise DegenerateDensityError("TT weights carry no probability mass")
        w = tt_round(tt_scale(weights, 1.0 / mass), cfg.round_tol, cfg.round_max_rank)
    else:
        w = tt_round(weights, cfg.round_tol, cfg.round_max_rank)
        mass = tt_sum(w) * dv
        if not math.isfinite(mass) or mass <= 1e-300:
            raise DegenerateDensityError("TT weights carry no probability mass")
        w = tt_scale(w, 1.0 / mass)
    return w, mass, negative_mass(w, grid, cfg.densify_guard)
