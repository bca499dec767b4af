"""Scenario trees: the index arrays the solver consumes.

Same array contract as the reference ``ScenarioTree``
(``/root/reference/pkg/src/watermpc/tree.py:52-133``): flat ``stage``, ``anc``,
``prob`` over all nodes in breadth-first order, root = node 0 with ``anc=-1``
and probability 1; after :func:`attach_forecast` each node carries its
contingent ``demand`` and ``price`` rows.

Fan-to-tree reduction (``tree.py:269-392``) is offline and O(S^2); it is out of
scope. :func:`uniform_tree` builds the benchmark trees
directly instead.
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

PROB_TOL = 1e-9


@dataclass
class ScenarioTree:
    horizon: int
    n_demand: int
    n_price: int
    stage: np.ndarray
    anc: np.ndarray
    prob: np.ndarray
    eps: np.ndarray | None = None
    demand: np.ndarray | None = None
    price: np.ndarray | None = None

    def __post_init__(self) -> None:
        self.stage = np.asarray(self.stage, dtype=np.int64)
        self.anc = np.asarray(self.anc, dtype=np.int64)
        self.prob = np.asarray(self.prob, dtype=np.float64)
        for key in ("eps", "demand", "price"):
            val = getattr(self, key)
            if val is not None:
                setattr(self, key, np.asarray(val, dtype=np.float64))

    @property
    def n_nodes(self) -> int:
        return int(self.stage.shape[0])

    @property
    def n_nonroot(self) -> int:
        return self.n_nodes - 1

    @property
    def is_attached(self) -> bool:
        return self.demand is not None and self.price is not None

    @property
    def nodes_per_stage(self) -> np.ndarray:
        return np.bincount(self.stage, minlength=self.horizon + 1)

    def stage_nodes(self, j: int) -> np.ndarray:
        return np.flatnonzero(self.stage == j)

    def children_of(self, node: int) -> np.ndarray:
        return np.flatnonzero(self.anc == node)

    def leaves(self) -> np.ndarray:
        return self.stage_nodes(self.horizon)

    @classmethod
    def single_branch(cls, horizon: int, n_demand: int, n_price: int,
                      eps: np.ndarray | None = None) -> "ScenarioTree":
        n = horizon + 1
        eps = np.zeros((n, n_demand + n_price)) if eps is None else np.asarray(eps, float)
        if eps.shape != (n, n_demand + n_price):
            raise ValueError(f"eps must have shape {(n, n_demand + n_price)}")
        return cls(horizon, n_demand, n_price, np.arange(n), np.arange(-1, n - 1),
                   np.ones(n), eps=eps)


def validate_tree(tree: ScenarioTree) -> list[str]:
    """Invariant violations, empty when valid (``tree.py:136-208``).

    Vectorised restatement: links point one stage up, BFS stage order,
    probabilities in (0, 1], children telescope to their parent and every
    stage sums to one (tolerance 1e-9), value arrays shaped per node.
    """
    bad: list[str] = []
    n = tree.n_nodes
    if n == 0:
        return ["tree has no nodes"]
    if tree.anc.shape != (n,) or tree.prob.shape != (n,):
        return ["stage, anc and prob arrays must have equal length"]
    if tree.stage[0] != 0 or tree.anc[0] != -1:
        bad.append("node 0 must be the root (stage 0, no ancestor)")
    if np.count_nonzero(tree.stage == 0) != 1:
        bad.append("exactly one node may sit at stage 0")
    if abs(tree.prob[0] - 1.0) > PROB_TOL:
        bad.append(f"root probability {tree.prob[0]} != 1")
    if np.any(np.diff(tree.stage) < 0):
        bad.append("nodes must be ordered breadth-first by stage")
    if np.any(tree.stage > tree.horizon) or np.any(tree.stage < 0):
        bad.append("node stages must lie in [0, horizon]")
    if np.any((tree.prob <= 0) | (tree.prob > 1 + PROB_TOL)):
        bad.append("node probabilities must lie in (0, 1]")
    parents = tree.anc[1:]
    in_range = (parents >= 0) & (parents < n)
    for i in np.flatnonzero(~in_range) + 1:
        bad.append(f"node {i}: ancestor {tree.anc[i]} out of range")
    if np.all(in_range):
        off = np.flatnonzero(tree.stage[parents] != tree.stage[1:] - 1) + 1
        for i in off:
            bad.append(f"node {i}: ancestor stage {tree.stage[tree.anc[i]]} "
                       f"!= own stage {tree.stage[i]} - 1")
        kid_mass = np.bincount(parents, weights=tree.prob[1:], minlength=n)
        kid_count = np.bincount(parents, minlength=n)
        for i in range(n):
            if tree.stage[i] < tree.horizon:
                if kid_count[i] == 0:
                    bad.append(f"node {i} at stage {tree.stage[i]} has no children")
                elif abs(kid_mass[i] - tree.prob[i]) > PROB_TOL:
                    bad.append(f"node {i}: children probabilities sum "
                               f"{kid_mass[i]:.12g} != {tree.prob[i]:.12g}")
            elif kid_count[i]:
                bad.append(f"leaf node {i} has children")
        mass = np.bincount(tree.stage, weights=tree.prob, minlength=tree.horizon + 1)
        for j in range(tree.horizon + 1):
            if abs(mass[j] - 1.0) > PROB_TOL:
                bad.append(f"stage {j} probabilities sum {mass[j]:.12g} != 1")
    width = tree.n_demand + tree.n_price
    if tree.eps is not None:
        if tree.eps.shape != (n, width):
            bad.append(f"eps shape {tree.eps.shape} != {(n, width)}")
        elif np.any(tree.eps[0] != 0.0):
            bad.append("root prediction error must be zero")
    if (tree.demand is None) != (tree.price is None):
        bad.append("demand and price values must be attached together")
    if tree.demand is not None and tree.demand.shape != (n, tree.n_demand):
        bad.append(f"demand value shape {tree.demand.shape} != {(n, tree.n_demand)}")
    if tree.price is not None and tree.price.shape != (n, tree.n_price):
        bad.append(f"price value shape {tree.price.shape} != {(n, tree.n_price)}")
    return bad


def attach_forecast(tree: ScenarioTree, d_hat, alpha_hat) -> ScenarioTree:
    """Node values = stage forecast + node error (``tree.py:211-239``)."""
    if tree.eps is None:
        raise ValueError("tree carries no prediction errors to attach to")
    d_hat = np.atleast_2d(np.asarray(d_hat, dtype=np.float64))
    alpha_hat = np.atleast_2d(np.asarray(alpha_hat, dtype=np.float64))
    if d_hat.shape != (tree.horizon, tree.n_demand):
        raise ValueError(f"demand forecast shape {d_hat.shape} != "
                         f"{(tree.horizon, tree.n_demand)}")
    if alpha_hat.shape != (tree.horizon, tree.n_price):
        raise ValueError(f"price forecast shape {alpha_hat.shape} != "
                         f"{(tree.horizon, tree.n_price)}")
    nd = tree.n_demand
    demand = np.zeros((tree.n_nodes, nd))
    price = np.zeros((tree.n_nodes, tree.n_price))
    st = tree.stage[1:] - 1
    demand[1:] = d_hat[st] + tree.eps[1:, :nd]
    price[1:] = alpha_hat[st] + tree.eps[1:, nd:]
    return replace(tree, demand=demand, price=price)


def zero_price_errors(tree: ScenarioTree) -> ScenarioTree:
    """Drop the price part of every error (``tree.py:242-253``)."""
    if tree.eps is None:
        raise ValueError("tree carries no prediction errors")
    eps = tree.eps.copy()
    eps[:, tree.n_demand:] = 0.0
    return replace(tree, eps=eps, demand=None, price=None)


def uniform_tree(branching, horizon: int, n_demand: int, n_price: int,
                 eps: np.ndarray | None = None) -> ScenarioTree:
    """BFS tree whose stage-j nodes each have ``branching[j]`` children
    (stages past ``len(branching)`` are single-child chains), equal split
    probabilities. Builds the SURVEY §8 configs without fan reduction."""
    branching = list(branching)
    stage = [0]
    anc = [-1]
    prob = [1.0]
    frontier = [0]
    for j in range(1, horizon + 1):
        k = branching[j - 1] if j - 1 < len(branching) else 1
        nxt = []
        for parent in frontier:
            for _ in range(k):
                stage.append(j)
                anc.append(parent)
                prob.append(prob[parent] / k)
                nxt.append(len(stage) - 1)
        frontier = nxt
    n = len(stage)
    if eps is None:
        eps = np.zeros((n, n_demand + n_price))
    return ScenarioTree(horizon, n_demand, n_price, np.array(stage), np.array(anc),
                        np.array(prob), eps=eps)


def random_tree(horizon: int, n_demand: int, n_price: int, branching_stages: int, max_children: int,
                rng, eps: np.ndarray | None = None) -> ScenarioTree:
    """BFS tree whose nodes in the first ``branching_stages`` stages have a
    random number of children (1..max_children) with random split
    probabilities, single-child chains below: the non-uniform shape of the
    reference's fan-to-tree reduction (tree.py:320-392: bundles of scenarios
    merge into nodes of unequal probability). Benchmarks and tests only."""
    stage, anc, prob, frontier = [0], [-1], [1.0], [0]
    for j in range(1, horizon + 1):
        nxt = []
        for parent in frontier:
            k = int(rng.integers(1, max_children + 1)) if j <= branching_stages else 1
            w = rng.random(k) + 0.25
            w /= w.sum()
            for c in range(k):
                stage.append(j)
                anc.append(parent)
                prob.append(prob[parent] * (w[c] if k > 1 else 1.0))
                nxt.append(len(stage) - 1)
        frontier = nxt
    n = len(stage)
    if eps is None:
        eps = np.zeros((n, n_demand + n_price))
    return ScenarioTree(horizon, n_demand, n_price, np.array(stage), np.array(anc), np.array(prob), eps=eps)
