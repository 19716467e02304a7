"""Grid and MomentEstimate types (grids.py:26-133 of the reference).

A :class:`Grid` stores the (base, step, off, n) description the device uses
and materialises the per-axis coordinates exactly as numpy does in the
reference (``design_grid`` / ``Grid.from_bounds``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from paper_2501_07942_b200 import geometry as geo


@dataclass(frozen=True)
class MomentEstimate:
    mean: np.ndarray
    cov: np.ndarray

    def __post_init__(self):
        mean = np.asarray(self.mean, dtype=float).reshape(-1)
        cov = np.atleast_2d(np.asarray(self.cov, dtype=float))
        if cov.shape != (mean.size, mean.size):
            raise ValueError(f"covariance shape {cov.shape} does not match mean size {mean.size}")
        if not np.allclose(cov, cov.T, rtol=1e-8, atol=1e-12):
            raise ValueError("covariance must be symmetric")
        object.__setattr__(self, "mean", mean)
        object.__setattr__(self, "cov", cov)

    @property
    def dim(self) -> int:
        return self.mean.size


class Grid:
    """Axis-aligned equidistant grid (device description + numpy coordinates)."""

    def __init__(self, ax: geo.Axes):
        self._ax = ax
        self.axes = ax.axes()

    @classmethod
    def from_axes(cls, ax: geo.Axes) -> "Grid":
        return cls(ax)

    @classmethod
    def from_bounds(cls, lows, highs, n_per_axis) -> "Grid":
        return cls(geo.grid_from_bounds(lows, highs, n_per_axis))

    @classmethod
    def design(cls, m: MomentEstimate, n_per_axis, sigma_mult=4.0) -> "Grid":
        return cls(geo.design_grid(m.mean, m.cov, n_per_axis, sigma_mult))

    @property
    def device_axes(self) -> geo.Axes:
        return self._ax

    @property
    def dim(self) -> int:
        return len(self.axes)

    @property
    def shape(self) -> tuple[int, ...]:
        return tuple(a.size for a in self.axes)

    @property
    def steps(self) -> np.ndarray:
        return np.array([(a[-1] - a[0]) / (a.size - 1) for a in self.axes])

    @property
    def cell_volume(self) -> float:
        return float(np.prod(self.steps))

    @property
    def lows(self):
        return np.array([a[0] for a in self.axes])

    @property
    def highs(self):
        return np.array([a[-1] for a in self.axes])

    @property
    def total_points(self) -> int:
        return math.prod(self.shape)

    def points_for(self, idx):
        idx = np.asarray(idx, dtype=np.intp)
        return np.column_stack([a[idx[:, k]] for k, a in enumerate(self.axes)])

    def corners(self):
        return self._ax.corners()


def design_grid(m: MomentEstimate, n_per_axis, sigma_mult: float = 4.0) -> Grid:
    return Grid.design(m, n_per_axis, sigma_mult)
