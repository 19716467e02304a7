"""Dense point-mass filter with FFT time update on the GPU.

Drop-in for the reference's dense FFT path:

=========================  ===========================================
this module                reference (pkg/src/ttpmf)
=========================  ===========================================
initial_pmd_dense          filters.py:487-494
dense_fft_pmf_step         filters.py:888-934
DenseFFTFilter             one filter's device state for the two above
=========================  ===========================================

The weights live in HBM as a C-order float64 array over the grid; every
per-point operation (prior, likelihood, interpolation onto F^-1 of the
predictive nodes, kernel, per-axis DFTs, spectrum product, reductions,
clip/normalise) is a kernel of ``libttgbf.so`` (csrc/dense.cu).  The host
keeps the O(d^2) geometry the reference also does in numpy: moments from
the reduced sums, SPD repair, Kalman prediction and the grid design.
There is no CPU fallback.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from paper_2501_07942_b200 import _abi
from paper_2501_07942_b200 import geometry as geo
from paper_2501_07942_b200.bank import gauss_record, model_record

MASS_FLOOR = 1e-300   # filters.py:100
DMAXD = 8


class DegenerateDensityError(RuntimeError):
    """filters.py:120."""


@dataclass
class DenseDiagnostics:
    """The StepDiagnostics fields the dense path fills (filters.py:164-188)."""

    filt_mean: np.ndarray | None = None
    filt_cov: np.ndarray | None = None
    pred_mean: np.ndarray | None = None
    pred_cov: np.ndarray | None = None
    spd_fixed: bool = False
    outlier: bool = False
    clipped_mass: float = 0.0
    mass_before_norm: float = float("nan")
    tpm_bytes: int = 0
    pmd_bytes: int = 0


def _axes_record(ax: geo.Axes) -> np.ndarray:
    return ax.device()[: ax.dim].copy()


def _roots(n: int) -> np.ndarray:
    r = np.exp(-2j * np.pi * np.arange(n) / n)
    return np.ascontiguousarray(np.stack([r.real, r.imag], axis=1))


class _HostArray:
    """A numpy array passed to the C-ABI as a host pointer."""

    __slots__ = ("a",)

    def __init__(self, a):
        self.a = np.ascontiguousarray(a)

    @property
    def ptr(self) -> int:
        return self.a.ctypes.data


class DenseFFTFilter:
    """One dense FFT point-mass filter on the device."""

    def __init__(self, spec, n_per_axis: int, sigma_mult: float, backend=None):
        if backend is None:
            from paper_2501_07942_b200.backend import CudaBackend
            backend = CudaBackend()
        self.be = backend
        self.lib = backend.lib
        self.spec = spec
        self.F = np.asarray(spec["F"], dtype=float)
        self.Q = np.asarray(spec["Q"], dtype=float)
        self.d = self.F.shape[0]
        if self.d > DMAXD:
            raise ValueError(f"dense grids support d <= {DMAXD}")
        if n_per_axis < 3 or n_per_axis % 2 == 0:
            raise ValueError("n_per_axis must be odd and >= 3")
        self.n = int(n_per_axis)
        self.sigma_mult = float(sigma_mult)
        self.total = self.n ** self.d
        self.set_model(spec)
        self.w = backend.empty(self.total * 8)
        self.w_next = backend.empty(self.total * 8)
        self.ca = backend.empty(self.total * 16)
        self.cb = backend.empty(self.total * 16)
        self.partials = backend.empty(int(self.lib.ttgbf_dense_reduce_blocks()) * 8)
        self.out = backend.empty(64 * 8)
        self.roots = backend.upload(_roots(self.n))
        self.shape_h = _HostArray(np.full(self.d, self.n, dtype=np.int32))
        self.grid: geo.Axes | None = None
        self.launches = 0

    def set_model(self, spec):
        """Upload the model record, F^-1 and |det F| (LinAlgError for a singular F, filters.py:910)."""
        F = np.asarray(spec["F"], dtype=float)
        if F.shape != (self.d, self.d):
            raise ValueError("model dimension does not match the filter")
        self.spec = spec
        self.F = F
        self.Q = np.asarray(spec["Q"], dtype=float)
        self.model = self.be.upload(model_record(spec))
        self.Finv = np.linalg.inv(F)
        finv = np.zeros(_abi.MAXD * _abi.MAXD)
        for i in range(self.d):
            finv[i * _abi.MAXD: i * _abi.MAXD + self.d] = self.Finv[i]
        self.finv_dev = self.be.upload(finv)
        self.abs_det = abs(float(np.linalg.det(F)))

    # -- helpers -----------------------------------------------------------------
    def _chk(self, rc, what):
        self.launches += 1
        self.be.check(rc, what)

    @staticmethod
    def _axes_host(ax: geo.Axes):
        """Host-side axis records (the C-ABI reads them on the host and passes
        the geometry to the kernels by value); kept alive by the caller."""
        return _HostArray(_axes_record(ax))

    def _reduce(self, buf, axes_h, mode, cv=1.0, mean_dev=None):
        nq = 2 if mode == 0 else (1 + self.d if mode == 1 else self.d * (self.d + 1) // 2)
        self._chk(self.lib.ttgbf_dense_reduce(buf.ptr, axes_h.ptr, self.d, mode, cv,
                                              mean_dev.ptr if mean_dev is not None else None, self.partials.ptr,
                                              self.out.ptr, self.be.stream_ptr), "ttgbf_dense_reduce")
        return self.be.download(self.out, np.float64, nq)

    def _finalize(self, buf, ax: geo.Axes, axes_h, diag: DenseDiagnostics):
        """_finalize_dense (filters.py:439-451) on `buf` in place."""
        pos, neg = self._reduce(buf, axes_h, 0)
        cv = ax.cell_volume()
        if not (math.isfinite(pos) and math.isfinite(neg)):
            raise DegenerateDensityError("dense weights contain non-finite values")
        diag.clipped_mass += float(-neg) * cv if neg < 0.0 else 0.0
        mass = float(pos) * cv
        diag.mass_before_norm = mass
        if mass <= MASS_FLOOR:
            raise DegenerateDensityError("dense weights carry no probability mass")
        self._chk(self.lib.ttgbf_dense_finalize(buf.ptr, self.total, mass, self.be.stream_ptr), "ttgbf_dense_finalize")

    def _fftn(self, buf, inverse):
        for axis in range(self.d):
            self._chk(self.lib.ttgbf_dense_dft(buf.ptr, self.shape_h.ptr, self.d, axis, int(inverse),
                                               self.roots.ptr, self.be.stream_ptr), "ttgbf_dense_dft")

    # -- API -----------------------------------------------------------------------
    def initial(self, mean, cov) -> DenseDiagnostics:
        """initial_pmd_dense (filters.py:487-494)."""
        mean = np.asarray(mean, dtype=float).reshape(-1)
        self.grid = geo.design_grid(mean, cov, self.n, self.sigma_mult)
        axes_h = self._axes_host(self.grid)
        prior = self.be.upload(gauss_record(mean, cov))
        self._chk(self.lib.ttgbf_dense_prior(prior.ptr, axes_h.ptr, self.d, self.w.ptr, self.be.stream_ptr),
                  "ttgbf_dense_prior")
        diag = DenseDiagnostics()
        self._finalize(self.w, self.grid, axes_h, diag)
        return diag

    def moments(self, axes_h, ax: geo.Axes):
        """moments_from_pmd, dense branch (filters.py:323-333) + _spd_repair."""
        cv = ax.cell_volume()
        s1 = self._reduce(self.w, axes_h, 1, cv)
        mass = float(s1[0])
        if not math.isfinite(mass) or mass <= 0.0:
            raise DegenerateDensityError("PMD has non-positive total mass")
        mean = s1[1:] / mass
        mean_dev = self.be.upload(mean)
        s2 = self._reduce(self.w, axes_h, 2, cv, mean_dev)
        cov = np.empty((self.d, self.d))
        q = 0
        for i in range(self.d):
            for j in range(i, self.d):
                cov[i, j] = cov[j, i] = s2[q] / mass
                q += 1
        cov, fixed = geo.spd_repair(cov)
        return mean, cov, fixed

    def step(self, z) -> DenseDiagnostics:
        """dense_fft_pmf_step (filters.py:888-934); the filter moves to the predictive grid."""
        if self.grid is None:
            raise RuntimeError("call initial() first")
        diag = DenseDiagnostics()
        ax = self.grid
        axes_h = self._axes_host(ax)
        cv = ax.cell_volume()
        if z is not None:   # measurement_update (dense branch, filters.py:564-572)
            zrec = np.zeros(_abi.MAXB)
            zz = np.atleast_1d(np.asarray(z, dtype=float))
            zrec[: zz.size] = zz
            z_dev = self.be.upload(zrec)
            self._copy(self.w_next, self.w)
            self._chk(self.lib.ttgbf_dense_likelihood(self.model.ptr, z_dev.ptr, axes_h.ptr, self.d,
                                                      self.w_next.ptr, self.be.stream_ptr), "ttgbf_dense_likelihood")
            pos, neg = self._reduce(self.w_next, axes_h, 0)
            mass = float(pos + neg) * cv
            if not math.isfinite(mass) or mass <= MASS_FLOOR:
                diag.outlier = True   # keep the prior weights
            else:
                self._finalize(self.w_next, ax, axes_h, diag)
                self.w, self.w_next = self.w_next, self.w
        mean, cov, fixed = self.moments(axes_h, ax)
        diag.filt_mean, diag.filt_cov, diag.spd_fixed = mean, cov, fixed
        pm, pc = geo.kalman_predict(mean, cov, self.F, self.Q)
        diag.pred_mean, diag.pred_cov = pm, pc
        pred = geo.design_grid(pm, pc, self.n, self.sigma_mult)
        pred_h = self._axes_host(pred)
        self._chk(self.lib.ttgbf_dense_interp(self.w.ptr, axes_h.ptr, pred_h.ptr, self.d, self.finv_dev.ptr,
                                              self.ca.ptr, self.be.stream_ptr), "ttgbf_dense_interp")
        steps = self.be.upload(pred.steps())
        self._chk(self.lib.ttgbf_dense_kernel(self.model.ptr, pred_h.ptr, self.d, steps.ptr, pred.cell_volume(),
                                              self.abs_det, self.cb.ptr, self.be.stream_ptr), "ttgbf_dense_kernel")
        diag.tpm_bytes = self.total * 8
        self._fftn(self.cb, False)
        self._fftn(self.ca, False)
        self._chk(self.lib.ttgbf_dense_cmul(self.cb.ptr, self.ca.ptr, self.total, self.be.stream_ptr),
                  "ttgbf_dense_cmul")
        self._fftn(self.cb, True)
        self._chk(self.lib.ttgbf_dense_real(self.cb.ptr, self.w_next.ptr, self.total, self.be.stream_ptr),
                  "ttgbf_dense_real")
        self._finalize(self.w_next, pred, pred_h, diag)
        self.w, self.w_next = self.w_next, self.w
        self.grid = pred
        diag.pmd_bytes = self.total * 8
        return diag

    def _copy(self, dst, src):
        dst.t[: self.total * 8].copy_(src.t[: self.total * 8])

    def weights(self) -> np.ndarray:
        return self.be.download(self.w, np.float64, self.total).reshape((self.n,) * self.d)


# -- reference-named functions ------------------------------------------------------
@dataclass
class DensePmdEstimate:
    """PmdEstimate with dense device weights (filters.py:191-230)."""

    filt: DenseFFTFilter
    diag: DenseDiagnostics
    kind: str = "predictive"

    @property
    def grid(self) -> geo.Axes:
        return self.filt.grid

    @property
    def weights(self) -> np.ndarray:
        return self.filt.weights()

    def storage_bytes(self) -> int:
        return self.filt.total * 8

    def mass(self) -> float:
        pos, neg = self.filt._reduce(self.filt.w, self.filt._axes_host(self.grid), 0)
        return float(pos + neg) * self.grid.cell_volume()


def initial_pmd_dense(prior, cfg, model=None, backend=None) -> DensePmdEstimate:
    """initial_pmd_dense(prior: MomentEstimate, cfg: GridConfig) (filters.py:487-494).

    The device filter also needs the model (for its buffers); pass it here or
    at the first dense_fft_pmf_step (the prior values do not depend on it)."""
    spec = model.spec if model is not None else _placeholder_spec(prior.mean.size)
    f = DenseFFTFilter(spec, cfg.n_per_axis, cfg.sigma_mult, backend)
    diag = f.initial(prior.mean, prior.cov)
    return DensePmdEstimate(f, diag)


def dense_fft_pmf_step(pmd: DensePmdEstimate, model, z, cfg) -> DensePmdEstimate:
    """dense_fft_pmf_step(pmd, model, z, cfg) (filters.py:888-934).

    Advances the device state of ``pmd`` (its buffers are reused: the
    returned estimate owns them)."""
    f = pmd.filt
    if model.F is None:
        raise ValueError("FFT time update requires linear dynamics")
    if getattr(f, "_model_obj", None) is not model:
        f.set_model(model.spec)
        f._model_obj = model
    diag = f.step(z)
    return DensePmdEstimate(f, diag)


def _placeholder_spec(d):
    return {"F": np.eye(d), "Q": np.eye(d), "R": np.eye(1), "h": "linear", "H": np.ones((1, d)),
            "angle_components": ()}
