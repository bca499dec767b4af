"""One scenario-MPC instance: node-major layout, the f/g/H splitting and the
public prox API.

Layout contract (identical to ``/root/reference/pkg/src/watermpc/problem.py:83-192``):
non-root node ``i`` lives at row ``i - 1``; primal rows are ``[u (n_u) | x (n_t)]``,
dual rows are ``[y1 (n_t) | y2 (n_t) | y3 (n_u)]`` paired with the image
``(x, x, u)`` under H. ``anc_row = anc[1:] - 1`` with -1 marking stage-1 nodes;
``stage_slices`` are the contiguous per-stage row ranges.

The prox maps (``prox_g``, ``prox_g_conjugate``) run on the GPU through the
native library (kernel ``wmpc_prox_kernel``); there is no host fallback.
``apply_H``/``apply_H_adjoint`` are pure layout shuffles.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .model import CostWeights, NetworkModel
from .tree import ScenarioTree, validate_tree

FEAS_TOL = 1e-8


@dataclass
class ProblemInstance:
    model: NetworkModel
    tree: ScenarioTree
    weights: CostWeights
    p: np.ndarray
    q: np.ndarray
    k: int = 0

    wu: np.ndarray = field(init=False, repr=False)
    prob: np.ndarray = field(init=False, repr=False)
    anc_row: np.ndarray = field(init=False, repr=False)
    demand: np.ndarray = field(init=False, repr=False)
    price: np.ndarray = field(init=False, repr=False)
    stage_slices: list = field(init=False, repr=False)
    demand_gd: np.ndarray = field(init=False, repr=False)
    econ: np.ndarray = field(init=False, repr=False)

    def __post_init__(self) -> None:
        self.p = np.asarray(self.p, dtype=np.float64)
        self.q = np.asarray(self.q, dtype=np.float64)
        model, tree = self.model, self.tree
        if not tree.is_attached:
            raise ValueError("scenario tree is not forecast-attached")
        issues = validate_tree(tree)
        if issues:
            raise ValueError(f"invalid scenario tree: {issues[0]}")
        if tree.horizon < 1:
            raise ValueError("prediction horizon must be at least 1")
        if tree.n_demand != model.n_demands or tree.n_price != model.n_inputs:
            raise ValueError(
                f"tree values sized ({tree.n_demand}, {tree.n_price}) do not match "
                f"network ({model.n_demands} demands, {model.n_inputs} inputs)")
        if self.p.shape != (model.n_tanks,):
            raise ValueError(f"state p must have shape ({model.n_tanks},)")
        if self.q.shape != (model.n_inputs,):
            raise ValueError(f"previous input q must have shape ({model.n_inputs},)")
        self.wu = self.weights.u_weight(model.n_inputs)
        self.prob = tree.prob[1:].copy()
        self.anc_row = tree.anc[1:] - 1
        self.demand = tree.demand[1:].copy()
        self.price = tree.price[1:].copy()
        counts = np.bincount(tree.stage[1:], minlength=tree.horizon + 1)[1:]
        edges = np.concatenate([[0], np.cumsum(counts)])
        self.stage_slices = [slice(int(a), int(b)) for a, b in zip(edges[:-1], edges[1:])]
        self.demand_gd = self.demand @ model.Gd.T
        self.econ = self.weights.w_alpha * (model.alpha0[None, :] + self.price)

    @property
    def n_nonroot(self) -> int:
        return self.tree.n_nonroot

    @property
    def n_primal(self) -> int:
        return self.n_nonroot * (self.model.n_inputs + self.model.n_tanks)

    @property
    def n_dual(self) -> int:
        return self.n_nonroot * (2 * self.model.n_tanks + self.model.n_inputs)

    def _as_rows(self, v, total: int, width: int, what: str) -> np.ndarray:
        v = np.asarray(v, dtype=np.float64)
        if v.shape != (total,):
            raise ValueError(f"{what} vector must have shape ({total},), got {v.shape}")
        return v.reshape(self.n_nonroot, width)

    def split_primal(self, z):
        nu = self.model.n_inputs
        rows = self._as_rows(z, self.n_primal, nu + self.model.n_tanks, "primal")
        return rows[:, :nu], rows[:, nu:]

    def join_primal(self, U, X) -> np.ndarray:
        return np.concatenate([U, X], axis=1).reshape(-1)

    def split_dual(self, y):
        nt = self.model.n_tanks
        rows = self._as_rows(y, self.n_dual, 2 * nt + self.model.n_inputs, "dual")
        return rows[:, :nt], rows[:, nt:2 * nt], rows[:, 2 * nt:]

    def join_dual(self, Y1, Y2, Y3) -> np.ndarray:
        return np.concatenate([Y1, Y2, Y3], axis=1).reshape(-1)

    def ancestor_inputs(self, U) -> np.ndarray:
        out = U[self.anc_row]
        out[self.anc_row < 0] = self.q
        return out

    def ancestor_states(self, X) -> np.ndarray:
        out = X[self.anc_row]
        out[self.anc_row < 0] = self.p
        return out


def assemble_problem(model, tree, weights, p, q, k: int = 0) -> ProblemInstance:
    """Validate and build one instance (``problem.py:195-204``)."""
    return ProblemInstance(model=model, tree=tree, weights=weights, p=p, q=q, k=k)


def apply_H(instance, z) -> np.ndarray:
    """(u, x) -> (x, x, u) per node (``problem.py:278-281``); layout only."""
    U, X = instance.split_primal(z)
    return instance.join_dual(X, X, U)


def apply_H_adjoint(instance, y) -> np.ndarray:
    """(y1, y2, y3) -> (u: y3, x: y1 + y2) per node (``problem.py:284-287``)."""
    Y1, Y2, Y3 = instance.split_dual(y)
    return instance.join_primal(Y3, Y1 + Y2)


def prox_g(instance, v, gamma: float) -> np.ndarray:
    """Prox of ``gamma * g`` on the GPU (``problem.py:313-319``)."""
    if gamma <= 0:
        raise ValueError("gamma must be positive")
    from .solver import _device_prox
    return _device_prox(instance, v, float(gamma), conjugate=False)


def prox_g_conjugate(instance, w, gamma: float) -> np.ndarray:
    """Prox of ``gamma * g*`` via Moreau, on the GPU (``problem.py:322-327``)."""
    if gamma <= 0:
        raise ValueError("gamma must be positive")
    from .solver import _device_prox
    return _device_prox(instance, w, float(gamma), conjugate=True)
