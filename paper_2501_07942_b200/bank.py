"""FilterBank: a batch of independent TT-FFT point-mass filters on one GPU.

Each filter is one CTA of every stage launch (one filter per Monte Carlo
run).  Per step the bank issues two kernel launches for the whole batch --
``ttgbf_filter_measure`` (likelihood cross, Hadamard, finalize, raw moments)
and ``ttgbf_filter_time_update`` (interp + finalize, kernel cross, FFT
convolution + rounding, realign cross, finalize) -- with the reference's
tiny numpy geometry (filters.py:769-786) in between on the host.

The backend is injectable so that the identical driver code can be run by
the CPU test-suite against the engine's single-thread emulation; the
product always uses :class:`paper_2501_07942_b200.backend.CudaBackend`.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from paper_2501_07942_b200 import _abi
from paper_2501_07942_b200 import geometry as geo
from paper_2501_07942_b200.configs import H_CODES


@dataclass
class BankConfig:
    """Grid / cross / resource configuration shared by all filters of a bank.

    ``n_per_axis``, ``sigma_mult``, ``round_tol``, ``round_max_rank``,
    ``normalize_before_round`` and ``densify_guard`` follow GridConfig
    (filters.py:129-161); ``tol``, ``max_rank``, ``max_sweeps``, ``rng_seed``
    and ``validation_count`` follow CrossConfig (tt_algorithms.py:93-115).
    ``ws_bytes`` / ``state_doubles`` / ``cache_cap`` size the per-filter
    device workspace, TT slab and evaluator cache.
    """

    n_per_axis: int = 33
    sigma_mult: float = 4.0
    round_tol: float = 1e-8
    round_max_rank: int | None = None
    normalize_before_round: bool = False
    densify_guard: int = 2 ** 22
    tol: float = 1e-6
    max_rank: int = 40
    max_sweeps: int = 60
    rng_seed: int = 0
    validation_count: int = 100
    ws_bytes: int = 256 << 20
    state_doubles: int = 1 << 20
    cache_cap: int = 1 << 20
    ws_slots: int = 0          # persistent run: workspace slots (0 = one per filter)
    big_slots: int = 0         # persistent run: overflow workspaces for oversized FFT products
    big_bytes: int = 3 << 29
    big2_slots: int = 0        # second (larger) overflow class
    big2_bytes: int = 3 << 30

    def grid_cfg(self):
        return _abi.GridCfg(self.round_tol, int(self.round_max_rank or 0),
                            int(bool(self.normalize_before_round)), int(self.densify_guard))

    def cross_cfg(self):
        c = _abi.CrossCfg()
        c.tol = float(self.tol)
        c.max_rank = int(self.max_rank)
        c.max_sweeps = int(self.max_sweeps)
        c.validation_count = int(self.validation_count)
        for i, v in enumerate(geo.pcg64_state(int(self.rng_seed))):
            c.rng_state[i] = v
        c.cache_cap = int(self.cache_cap)
        return c


def model_record(spec) -> np.ndarray:
    """ttgbf_model from a model spec (configs.py)."""
    F = np.asarray(spec["F"], dtype=float)
    Q = np.asarray(spec["Q"], dtype=float)
    R = np.atleast_2d(np.asarray(spec["R"], dtype=float))
    d, b = F.shape[0], R.shape[0]
    if d > _abi.MAXD or b > _abi.MAXB:
        raise ValueError("state / measurement dimension exceeds 16")
    rec = np.zeros(1, dtype=_abi.MODEL)
    rec["d"], rec["b"] = d, b
    rec["hkind"] = H_CODES[spec["h"]]
    ang = tuple(spec.get("angle_components", ()))
    rec["nang"] = len(ang)
    rec["ang"][0, :len(ang)] = ang

    def put(field, M, ld):
        buf = np.zeros(ld * ld if field != "H" else _abi.MAXB * _abi.MAXD)
        for i in range(M.shape[0]):
            buf[i * ld: i * ld + M.shape[1]] = M[i]
        rec[field][0] = buf

    put("F", F, _abi.MAXD)
    put("Q", Q, _abi.MAXD)
    try:
        Finv = np.linalg.inv(F)
    except np.linalg.LinAlgError:
        Finv = None
    if Finv is not None:
        put("Finv", Finv, _abi.MAXD)
    lq, nq = geo.gauss_consts(Q)
    luq, pq, iq = geo.solve_factors(lq)
    put("LUq", luq, _abi.MAXD)
    rec["pivq"][0, :d] = pq
    rec["invq"][0, :d] = iq
    rec["logn_q"] = nq
    lr, nr = geo.gauss_consts(R)
    lur, pr, ir = geo.solve_factors(lr)
    put("LUr", lur, _abi.MAXB)
    rec["pivr"][0, :b] = pr
    rec["invr"][0, :b] = ir
    rec["logn_r"] = nr
    if spec["h"] == "linear":
        put("H", np.atleast_2d(np.asarray(spec["H"], dtype=float)), _abi.MAXD)
    return rec


def gauss_record(mean, cov) -> np.ndarray:
    rec = np.zeros(1, dtype=_abi.GAUSS)
    mean = np.asarray(mean, dtype=float).reshape(-1)
    L, logn = geo.gauss_consts(cov)
    lu, piv, inv = geo.solve_factors(L)
    d = mean.size
    rec["mean"][0, :d] = mean
    buf = np.zeros(_abi.MAXD * _abi.MAXD)
    for i in range(d):
        buf[i * _abi.MAXD: i * _abi.MAXD + d] = lu[i]
    rec["LU"][0] = buf
    rec["piv"][0, :d] = piv
    rec["inv"][0, :d] = inv
    rec["logn"] = logn
    return rec


class StepError(RuntimeError):
    pass


class FilterBank:
    """``count`` independent filters sharing one model and configuration."""

    def __init__(self, spec, cfg: BankConfig, count: int, backend=None):
        if backend is None:
            from paper_2501_07942_b200.backend import CudaBackend
            backend = CudaBackend()
        self.be = backend
        self.lib = backend.lib
        self.spec = spec
        self.cfg = cfg
        self.count = int(count)
        self.F = np.asarray(spec["F"], dtype=float)
        self.Q = np.asarray(spec["Q"], dtype=float)
        self.d = self.F.shape[0]
        self.b = np.atleast_2d(spec["R"]).shape[0]
        if int(cfg.max_rank) > 160:
            raise ValueError("max_rank above 160 is not supported by the device cross")
        self.model = backend.upload(model_record(spec))
        self.gcfg = cfg.grid_cfg()
        self.xcfg = cfg.cross_cfg()
        shape = (int(cfg.n_per_axis),) * self.d
        self.probes_np = geo.probe_cells(shape)
        self.seeds_np = geo.seed_lattice(shape)
        self.probes = backend.upload(self.probes_np)
        self.seeds = backend.upload(self.seeds_np)
        n = self.count
        self.io = np.zeros(n, dtype=_abi.FILTER_IO)
        self.io_dev = backend.empty(self.io.nbytes)
        self.hdr = backend.empty(n * _abi.TT.itemsize)
        self.state = backend.empty(n * cfg.state_doubles * 8)
        self.nslots = min(n, cfg.ws_slots) if cfg.ws_slots > 0 else n
        self.ws = backend.empty(self.nslots * cfg.ws_bytes)
        self.sched = backend.empty(4 * (2 + 2 * n))
        self.nbig = int(cfg.big_slots)
        self.big_ws = backend.empty(self.nbig * cfg.big_bytes) if self.nbig else None
        self.big_locks = backend.empty(4 * max(1, self.nbig))
        self.nbig2 = int(cfg.big2_slots)
        self.big2_ws = backend.empty(self.nbig2 * cfg.big2_bytes) if self.nbig2 else None
        self.big2_locks = backend.empty(4 * max(1, self.nbig2))
        self.diag_dev = backend.empty(n * _abi.DIAG.itemsize)
        self.grids: list[geo.Axes | None] = [None] * n
        self.alive = np.zeros(n, dtype=bool)
        self.timeline = None          # list of (name, start_event, end_event) when profiling
        self.bytes_h2d = 0
        self.bytes_d2h = 0

    # -- helpers ----------------------------------------------------------------
    def _need_slot_per_filter(self):
        if self.nslots < self.count:
            raise RuntimeError("stage-wise calls need one workspace slot per filter; use run() "
                               "or BankConfig(ws_slots=0)")

    def _push_io(self):
        self.be.upload_into(self.io_dev, self.io)
        self.bytes_h2d += self.io.nbytes

    def _diag(self) -> np.ndarray:
        self.bytes_d2h += self.count * _abi.DIAG.itemsize
        return self.be.download(self.diag_dev, _abi.DIAG, self.count)

    def _launch(self, name, fn, *args):
        ev = None
        if self.timeline is not None and hasattr(self.be, "event"):
            ev = (self.be.event(), self.be.event())
            ev[0].record(self.be.stream)
        nvtx = getattr(self.be, "nvtx", None)
        if nvtx is not None:
            nvtx.range_push(f"{name} x{self.count}")   # ranges for nsys / ncu --nvtx
        try:
            rc = fn(*args)
        finally:
            if nvtx is not None:
                nvtx.range_pop()
        if ev is not None:
            ev[1].record(self.be.stream)
            self.timeline.append((name, ev[0], ev[1]))
        self.be.check(rc, name)

    def _ptrs(self):
        return (self.probes.ptr, len(self.probes_np), self.seeds.ptr, len(self.seeds_np))

    def set_active(self, mask):
        self.io["active"] = np.asarray(mask, dtype=np.int32)

    # -- stages -----------------------------------------------------------------
    def init_prior(self, mean, cov, which=None):
        """initial_pmd_tt for every filter in ``which`` (default all)."""
        self._need_slot_per_filter()
        which = np.arange(self.count) if which is None else np.asarray(which)
        grid = geo.design_grid(mean, cov, self.cfg.n_per_axis, self.cfg.sigma_mult)
        prior = self.be.upload(gauss_record(mean, cov))
        act = np.zeros(self.count, dtype=np.int32)
        act[which] = 1
        self.io["active"] = act
        for i in which:
            self.io["cur"][i] = grid.device()
            self.grids[i] = grid
        self._push_io()
        self._launch("ttgbf_filter_prior", self.lib.ttgbf_filter_prior, self.model.ptr, prior.ptr, self.gcfg,
                     self.xcfg, self.io_dev.ptr, self.count, self.probes.ptr, len(self.probes_np), self.hdr.ptr,
                     self.state.ptr, self.cfg.state_doubles, self.ws.ptr, self.cfg.ws_bytes, self.diag_dev.ptr,
                     self.be.stream_ptr)
        dg = self._diag()
        ok = dg["status"][which] == 0
        self.alive[which] = ok
        return dg

    def measure(self, z, has_z=None):
        """measurement_update + raw moments for all alive filters."""
        self._need_slot_per_filter()
        z = np.atleast_2d(np.asarray(z, dtype=float))
        self.io["active"] = self.alive.astype(np.int32)
        self.io["z"][:, :self.b] = z
        self.bytes_h2d += z.nbytes
        self.io["has_z"] = 1 if has_z is None else np.asarray(has_z, dtype=np.int32)
        self._push_io()
        pr, npr, sd, nsd = self._ptrs()
        self._launch("ttgbf_filter_measure", self.lib.ttgbf_filter_measure, self.model.ptr, self.gcfg, self.xcfg,
                     self.io_dev.ptr, self.count, pr, npr, sd, nsd, self.hdr.ptr, self.state.ptr,
                     self.cfg.state_doubles, self.ws.ptr, self.cfg.ws_bytes, self.diag_dev.ptr, self.be.stream_ptr)
        return self._diag()

    def geometry(self, dg):
        """Host geometry for every alive filter; returns per-filter moments."""
        d = self.d
        Finv = np.linalg.inv(self.F)
        out = {}
        for i in np.nonzero(self.alive)[0]:
            if dg["status"][i] != 0:
                continue
            g = self.grids[i]
            mass, mean, cov, fixed = geo.moments_from_raw(dg["raw_moments"][i], d, g.cell_volume())
            if mean is None:
                out[i] = ("degenerate", None)
                continue
            faxes, paxes = geo.redesign(mean, cov, self.F, self.Q, Finv, self.cfg.n_per_axis,
                                        self.cfg.sigma_mult)
            self.io["filt"][i] = faxes.device()
            self.io["pred"][i] = paxes.device()
            out[i] = ("ok", (mean, cov, fixed, faxes, paxes))
        return out

    def time_update(self, geom):
        self._need_slot_per_filter()
        act = np.zeros(self.count, dtype=np.int32)
        for i, (st, _) in geom.items():
            if st == "ok":
                act[i] = 1
        self.io["active"] = act
        self._push_io()
        pr, npr, sd, nsd = self._ptrs()
        self._launch("ttgbf_filter_time_update", self.lib.ttgbf_filter_time_update, self.model.ptr, self.gcfg,
                     self.xcfg, self.io_dev.ptr, self.count, pr, npr, sd, nsd, self.hdr.ptr, self.state.ptr,
                     self.cfg.state_doubles, self.ws.ptr, self.cfg.ws_bytes, self.diag_dev.ptr, self.be.stream_ptr)
        dg = self._diag()
        for i, (st, payload) in geom.items():
            if st == "ok" and dg["status"][i] == 0:
                self.grids[i] = payload[4]
                self.io["cur"][i] = payload[4].device()
        return dg

    def time_update_std(self, geom):
        """Algorithm 2 time update (tt_pmf_step, filters.py:876-885) onto the
        predictive grid io.pred designed by geometry()."""
        self._need_slot_per_filter()
        act = np.zeros(self.count, dtype=np.int32)
        for i, (st, _) in geom.items():
            if st == "ok":
                act[i] = 1
        self.io["active"] = act
        self._push_io()
        self._launch("ttgbf_filter_time_update_std", self.lib.ttgbf_filter_time_update_std, self.model.ptr,
                     self.gcfg, self.xcfg, self.io_dev.ptr, self.count, self.probes.ptr, len(self.probes_np),
                     self.hdr.ptr, self.state.ptr, self.cfg.state_doubles, self.ws.ptr, self.cfg.ws_bytes,
                     self.diag_dev.ptr, self.be.stream_ptr)
        dg = self._diag()
        for i, (st, payload) in geom.items():
            if st == "ok" and dg["status"][i] == 0:
                self.grids[i] = payload[4]
                self.io["cur"][i] = payload[4].device()
        return dg

    def step(self, z, standard: bool = False):
        """One tt_fft_pmf_step (standard=True: tt_pmf_step, Algorithm 2) for
        every alive filter.

        Returns a dict with per-filter status (0 ok), filtering means/covs and
        the two diagnostic records.  Failed filters are marked dead.
        """
        dm = self.measure(z)
        geom = self.geometry(dm)
        dt = self.time_update_std(geom) if standard else self.time_update(geom)
        n = self.count
        status = np.full(n, -1, dtype=np.int64)
        means = np.full((n, self.d), np.nan)
        covs = np.full((n, self.d, self.d), np.nan)
        for i in range(n):
            if not self.alive[i]:
                continue
            if dm["status"][i] != 0:
                status[i] = dm["status"][i]
            elif i not in geom or geom[i][0] != "ok":
                status[i] = _abi.E_DEGENERATE
            else:
                status[i] = dt["status"][i]
                means[i], covs[i] = geom[i][1][0], geom[i][1][1]
        self.alive &= status == 0
        return {"status": status, "mean": means, "cov": covs, "measure": dm, "time": dt, "geom": geom}

    # -- persistent multi-step run (device geometry) ----------------------------
    def run(self, Z, steps, prior_mean, prior_cov):
        """``steps`` tt_fft_pmf_step calls per filter in ONE kernel launch.

        Z: (count, kf, b) measurements (each filter replays its trajectory from
        k=0 after a restart).  Dead filters (re)start from the prior on the
        device.  Returns the (count, steps) STEP_REC records.
        """
        Z = np.ascontiguousarray(np.asarray(Z, dtype=float))
        kf = Z.shape[1]
        if not hasattr(self, "_run_prior") or self._run_prior[0] is not prior_mean:
            grid = geo.design_grid(prior_mean, prior_cov, self.cfg.n_per_axis, self.cfg.sigma_mult)
            self._run_prior = (prior_mean, self.be.upload(gauss_record(prior_mean, prior_cov)), grid)
            self.kstep_dev = self.be.upload(np.zeros(self.count, dtype=np.int32))
        _, prior_dev, grid = self._run_prior
        rc = _abi.RunCfg()
        rc.n_per_axis = int(self.cfg.n_per_axis)
        rc.kf = int(kf)
        rc.steps = int(steps)
        rc.sigma_mult = float(self.cfg.sigma_mult)
        dev = grid.device()
        for k in range(_abi.MAXD):
            rc.prior_grid[k].base = float(dev["base"][k])
            rc.prior_grid[k].step = float(dev["step"][k])
            rc.prior_grid[k].off = int(dev["off"][k])
            rc.prior_grid[k].n = int(dev["n"][k])
        self.be.zero(self.sched)
        self.be.zero(self.big_locks)
        rc.nbig = self.nbig
        rc.big_bytes = int(self.cfg.big_bytes)
        rc.big_ws = self.big_ws.ptr if self.big_ws is not None else None
        rc.big_locks = self.big_locks.ptr
        self.be.zero(self.big2_locks)
        rc.nbig2 = self.nbig2
        rc.big2_bytes = int(self.cfg.big2_bytes)
        rc.big2_ws = self.big2_ws.ptr if self.big2_ws is not None else None
        rc.big2_locks = self.big2_locks.ptr
        self.be.zero(self.diag_dev)
        zb = self.be.upload(Z)
        self.bytes_h2d += Z.nbytes
        rec = self.be.empty(self.count * max(1, steps) * _abi.STEP_REC.itemsize)
        self.io["active"] = self.alive.astype(np.int32)
        self._push_io()
        pr, npr, sd, nsd = self._ptrs()
        self._launch("ttgbf_filter_run", self.lib.ttgbf_filter_run, self.model.ptr, prior_dev.ptr, self.gcfg,
                     self.xcfg, rc, self.io_dev.ptr, self.kstep_dev.ptr, zb.ptr, self.count, pr, npr, sd, nsd,
                     self.hdr.ptr, self.state.ptr, self.cfg.state_doubles, self.ws.ptr, self.cfg.ws_bytes,
                     self.sched.ptr, self.nslots, self.diag_dev.ptr, rec.ptr, self.be.stream_ptr)
        recs = self.be.download(rec, _abi.STEP_REC, self.count * steps).reshape(self.count, steps)
        self.io = self.be.download(self.io_dev, _abi.FILTER_IO, self.count)
        self.bytes_d2h += recs.nbytes + self.io.nbytes
        self.alive = self.io["active"].astype(bool)
        for i in range(self.count):
            c = self.io["cur"][i]
            self.grids[i] = geo.Axes(c["base"][: self.d], c["step"][: self.d], c["off"][: self.d], c["n"][: self.d])
        return recs

    # -- state access -----------------------------------------------------------
    def headers(self) -> np.ndarray:
        return self.be.download(self.hdr, _abi.TT, self.count)

    def cores(self, i) -> list[np.ndarray]:
        h = self.headers()[i]
        d = int(h["d"])
        out = []
        base = i * self.cfg.state_doubles * 8
        for k in range(d):
            shp = (int(h["r"][k]), int(h["n"][k]), int(h["r"][k + 1]))
            cnt = math.prod(shp)
            arr = self.be.download(self.state, np.float64, cnt, base + int(h["off"][k]) * 8)
            out.append(arr.reshape(shp))
        return out

    def load_cores(self, i, cores, grid: geo.Axes):
        """Install TT weights for filter i (used by tests / the object API)."""
        h = np.zeros(1, dtype=_abi.TT)
        d = len(cores)
        h["d"] = d
        off = 0
        flat = []
        for k, c in enumerate(cores):
            c = np.ascontiguousarray(c, dtype=np.float64)
            h["n"][0, k] = c.shape[1]
            h["r"][0, k] = c.shape[0]
            h["off"][0, k] = off
            off += c.size
            flat.append(c.reshape(-1))
        h["r"][0, d] = 1
        if off > self.cfg.state_doubles:
            raise ValueError("TT does not fit the per-filter state slab")
        data = np.concatenate(flat)
        self._write(self.state, data, i * self.cfg.state_doubles * 8)
        self._write(self.hdr, h, i * _abi.TT.itemsize)
        self.grids[i] = grid
        self.io["cur"][i] = grid.device()
        self.alive[i] = True

    def load_tt(self, i, tt, axes: geo.Axes):
        """Install a device TensorTrain (D2D copy) as filter i's weights on grid ``axes``."""
        n = tt.size
        if n > self.cfg.state_doubles:
            raise ValueError("TT does not fit the per-filter state slab")
        off = i * self.cfg.state_doubles * 8
        self.state.t[off: off + 8 * n].copy_(tt.data[:n].view(self.be.torch.uint8))
        self._write(self.hdr, tt.hdr.reshape(1), i * _abi.TT.itemsize)
        self.grids[i] = axes
        self.io["cur"][i] = axes.device()
        self.alive[i] = True

    def read_tt(self, i):
        from paper_2501_07942_b200.tensor_train import TensorTrain
        h = self.headers()[i]
        n = sum(int(h["r"][k]) * int(h["n"][k]) * int(h["r"][k + 1]) for k in range(int(h["d"])))
        off = i * self.cfg.state_doubles * 8
        data = self.state.t[off: off + 8 * n].view(self.be.torch.float64).clone()
        return TensorTrain(h, data)

    def _write(self, buf, arr, offset):
        raw = np.ascontiguousarray(arr).view(np.uint8).reshape(-1)
        if hasattr(buf, "t"):
            import torch
            buf.t[offset: offset + raw.nbytes].copy_(torch.from_numpy(raw))
        else:
            buf.a[offset: offset + raw.nbytes] = raw

    @staticmethod
    def cross_info(dg_row, slot):
        c = dg_row["cross"][slot]
        return (float(c["achieved"]), int(c["calls"]), int(c["sweeps"]), bool(c["converged"]))
