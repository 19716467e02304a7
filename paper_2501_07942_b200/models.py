"""State-space model descriptors (models.py:85-296 of the reference).

The reference's ``StateSpaceModel.h`` is an arbitrary Python callable.  On
the device the measurement function must be one of the enumerated kinds in
:data:`paper_2501_07942_b200.configs.H_KINDS`; passing anything else raises
(there is no CPU fallback for the hot path).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from paper_2501_07942_b200 import configs


@dataclass(frozen=True)
class StateSpaceModel:
    dim_x: int
    dim_z: int
    h: str
    Q: np.ndarray
    R: np.ndarray
    F: np.ndarray
    H: np.ndarray | None = None
    angle_components: tuple = ()
    name: str = ""

    def __post_init__(self):
        if not isinstance(self.h, str) or self.h not in configs.H_KINDS:
            raise ValueError(f"measurement kind must be one of {configs.H_KINDS}; arbitrary callables "
                             "are not evaluable on the device")
        F = np.atleast_2d(np.asarray(self.F, dtype=float))
        if F.shape != (self.dim_x, self.dim_x):
            raise ValueError(f"F must be {self.dim_x} x {self.dim_x}")
        object.__setattr__(self, "F", F)
        object.__setattr__(self, "Q", np.atleast_2d(np.asarray(self.Q, dtype=float)))
        object.__setattr__(self, "R", np.atleast_2d(np.asarray(self.R, dtype=float)))
        if self.Q.shape != (self.dim_x, self.dim_x):
            raise ValueError("Q has the wrong shape")
        if self.R.shape != (self.dim_z, self.dim_z):
            raise ValueError("R has the wrong shape")

    @property
    def Finv(self):
        return np.linalg.inv(self.F)   # LinAlgError for singular F, as filters.py:783

    @property
    def spec(self) -> dict:
        s = {"F": self.F, "Q": self.Q, "R": self.R, "h": self.h,
             "angle_components": tuple(self.angle_components), "name": self.name}
        if self.H is not None:
            s["H"] = np.atleast_2d(np.asarray(self.H, dtype=float))
        return s

    @classmethod
    def from_spec(cls, spec) -> "StateSpaceModel":
        F = np.asarray(spec["F"], dtype=float)
        R = np.atleast_2d(spec["R"])
        return cls(dim_x=F.shape[0], dim_z=R.shape[0], h=spec["h"], Q=spec["Q"], R=R, F=F,
                   H=spec.get("H"), angle_components=tuple(spec.get("angle_components", ())),
                   name=spec.get("name", ""))

    @classmethod
    def placeholder(cls, dim):
        """Identity model used only to host a prior (initial_pmd_tt needs no dynamics)."""
        return cls(dim_x=dim, dim_z=dim, h="linear", Q=np.eye(dim), R=np.eye(dim), F=np.eye(dim),
                   H=np.eye(dim), name="placeholder")


def radar_model():
    return StateSpaceModel.from_spec(configs.radar_spec())


def scaling_model(dim):
    return StateSpaceModel.from_spec(configs.scaling_spec(dim))


def simulate(model: StateSpaceModel, x0_mean, x0_cov, k_f, seed, noise_free=False):
    return configs.simulate(model.spec, x0_mean, x0_cov, k_f, seed, noise_free)
