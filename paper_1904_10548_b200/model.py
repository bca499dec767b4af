"""Network model and controller weights (the data either side of the solver).

Mirrors the fields of the reference's ``NetworkModel``
(``/root/reference/pkg/src/watermpc/network.py:72-164``) and ``CostWeights``
(``/root/reference/pkg/src/watermpc/problem.py:36-80``) so instances built for
the reference can be handed to this package unchanged, and vice versa.

Discrete-time flow network over one sampling interval::

    x+ = A x + B u + Gd d          (tank mass balance)
    0  = E u + Ed d                (storage-free mixing nodes)

Only the matrices and bounds matter to the solver; the element-level topology
builder of the reference is out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class NetworkModel:
    """LTI water-network model with state/input boxes and base prices."""

    A: np.ndarray
    B: np.ndarray
    Gd: np.ndarray
    E: np.ndarray
    Ed: np.ndarray
    x_min: np.ndarray
    x_max: np.ndarray
    x_safe: np.ndarray
    u_min: np.ndarray
    u_max: np.ndarray
    alpha0: np.ndarray
    dt: float
    tank_names: tuple = field(default=())
    flow_names: tuple = field(default=())

    def __post_init__(self) -> None:
        for name in ("A", "B", "Gd", "E", "Ed", "x_min", "x_max", "x_safe",
                     "u_min", "u_max", "alpha0"):
            setattr(self, name, np.asarray(getattr(self, name), dtype=np.float64))

    @property
    def n_tanks(self) -> int:
        return self.A.shape[0]

    @property
    def n_inputs(self) -> int:
        return self.B.shape[1]

    @property
    def n_demands(self) -> int:
        return self.Gd.shape[1]

    @property
    def n_mixing(self) -> int:
        return self.E.shape[0]

    def validate(self) -> None:
        """Shape and bound-order checks; raises ``ValueError`` like the reference
        (``network.py:116-144``)."""
        nt, nu, nd, ns = self.n_tanks, self.n_inputs, self.n_demands, self.n_mixing
        expect = {"A": (nt, nt), "B": (nt, nu), "Gd": (nt, nd)}
        for key, shape in expect.items():
            if getattr(self, key).shape != shape:
                raise ValueError(f"{key} shape {getattr(self, key).shape} != {shape}")
        if self.E.shape != (ns, nu) or self.Ed.shape != (ns, nd):
            raise ValueError(
                f"coupling shapes E{self.E.shape}, Ed{self.Ed.shape} inconsistent"
            )
        for key, width in (("x_min", nt), ("x_max", nt), ("x_safe", nt),
                           ("u_min", nu), ("u_max", nu), ("alpha0", nu)):
            if getattr(self, key).shape != (width,):
                raise ValueError(f"{key} must have shape ({width},)")
        if self.dt <= 0:
            raise ValueError("dt must be positive")
        if np.any(self.x_min > self.x_max):
            raise ValueError("x_min must not exceed x_max")
        if np.any(self.u_min > self.u_max):
            raise ValueError("u_min must not exceed u_max")

    def step_dynamics(self, x, u, d) -> np.ndarray:
        """One plant step ``A x + B u + Gd d`` (``network.py:146-155``)."""
        return self.A @ np.asarray(x, float) + self.B @ np.asarray(u, float) \
            + self.Gd @ np.asarray(d, float)

    def coupling_residual(self, u, d) -> np.ndarray:
        """Mixing-node residual ``E u + Ed d`` (``network.py:157-164``)."""
        u, d = np.asarray(u, float), np.asarray(d, float)
        if u.shape != (self.n_inputs,):
            raise ValueError(f"input must have shape ({self.n_inputs},), got {u.shape}")
        if d.shape != (self.n_demands,):
            raise ValueError(f"demand must have shape ({self.n_demands},), got {d.shape}")
        return self.E @ u + self.Ed @ d


def _require_spd(mat: np.ndarray, what: str) -> None:
    if mat.ndim != 2 or mat.shape[0] != mat.shape[1]:
        raise ValueError(f"{what} must be a square matrix")
    if not np.allclose(mat, mat.T, rtol=1e-10, atol=0):
        raise ValueError(f"{what} must be symmetric")
    try:
        np.linalg.cholesky(mat)
    except np.linalg.LinAlgError:
        raise ValueError(f"{what} must be positive definite") from None


@dataclass
class CostWeights:
    """Economic weight ``w_alpha``, input-increment weight ``w_u`` (SPD matrix or
    positive scalar meaning ``w_u * I``), soft safety ``w_s`` and box ``w_x``
    penalty weights (``problem.py:36-69``)."""

    w_alpha: float
    w_u: float | np.ndarray
    w_s: float
    w_x: float

    def __post_init__(self) -> None:
        if self.w_alpha <= 0:
            raise ValueError("w_alpha must be positive")
        if self.w_s < 0 or self.w_x < 0:
            raise ValueError("w_s and w_x must be nonnegative")
        if np.ndim(self.w_u) == 0:
            if float(self.w_u) <= 0:
                raise ValueError("scalar w_u must be positive")
        else:
            self.w_u = np.asarray(self.w_u, dtype=np.float64)
            _require_spd(self.w_u, "w_u")

    def u_weight(self, n_inputs: int) -> np.ndarray:
        if np.ndim(self.w_u) == 0:
            return float(self.w_u) * np.eye(n_inputs)
        if self.w_u.shape != (n_inputs, n_inputs):
            raise ValueError(
                f"w_u shape {self.w_u.shape} inconsistent with {n_inputs} inputs"
            )
        return self.w_u
