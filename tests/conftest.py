"""Shared test setup: markers, paths and random-instance builders.

The builders restate the reference's ``pkg/tests/conftest.py:18-131``
(random dense model with full-row-rank coupling, random BFS tree with exact
telescoping, random SPD W_u) on top of this package's data classes, so the
parity tests read like the reference's own tests and run on the GPU box where
``/root/reference`` does not exist.
"""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_1904_10548_b200.model import CostWeights, NetworkModel  # noqa: E402
from paper_1904_10548_b200.problem import assemble_problem  # noqa: E402
from paper_1904_10548_b200.tree import ScenarioTree, attach_forecast  # noqa: E402

REFERENCE_SRC = "/root/reference/pkg/src"
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libwmpc.so")
    config.addinivalue_line("markers", "slow: long-running parity test")


def reference_available() -> bool:
    return os.path.isdir(os.path.join(REFERENCE_SRC, "watermpc"))


def import_reference():
    if not reference_available():
        pytest.skip("reference package not mounted (GPU box)")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import watermpc  # noqa: F401
    return sys.modules["watermpc"]


@pytest.fixture
def rng() -> np.random.Generator:
    return np.random.default_rng(20240811)


def rel_err(a, b) -> float:
    """Reference test metric ||a - b|| / (1 + ||b||) (test_solver.py:21-22)."""
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.linalg.norm(a - b) / (1.0 + np.linalg.norm(b)))


def make_model(rng, n_tanks, n_inputs, n_demands, n_mixing=0, dt=1.0, identity_a=True):
    A = np.eye(n_tanks) if identity_a else np.eye(n_tanks) + 0.05 * rng.standard_normal((n_tanks, n_tanks))
    B = dt * rng.choice([-1.0, 0.0, 1.0], size=(n_tanks, n_inputs))
    if not B.any():
        B[0, 0] = dt
    Gd = -dt * (rng.random((n_tanks, n_demands)) < 0.5)
    if n_mixing:
        E = rng.standard_normal((n_mixing, n_inputs))
        Ed = -E @ (0.3 * rng.random((n_inputs, n_demands)))
    else:
        E = np.zeros((0, n_inputs))
        Ed = np.zeros((0, n_demands))
    return NetworkModel(
        A=A, B=B, Gd=Gd, E=E, Ed=Ed,
        x_min=np.zeros(n_tanks), x_max=np.full(n_tanks, 40.0), x_safe=np.full(n_tanks, 10.0),
        u_min=np.zeros(n_inputs), u_max=np.full(n_inputs, 1.0 + rng.random(n_inputs)),
        alpha0=0.5 * rng.random(n_inputs), dt=dt,
    )


def make_tree(rng, horizon, n_demand, n_price, max_children=3, max_nodes=30, eps_scale=0.1):
    stage, anc, prob, frontier = [0], [-1], [1.0], [0]
    for j in range(1, horizon + 1):
        nxt = []
        for node in frontier:
            remaining = max_nodes - len(stage)
            budget = max(1, min(max_children, remaining - sum(1 for f in frontier if f > node)))
            k = 1 if j == horizon and len(stage) > max_nodes else int(rng.integers(1, budget + 1))
            shares = rng.random(k) + 0.2
            shares /= shares.sum()
            for share in shares:
                stage.append(j)
                anc.append(node)
                prob.append(prob[node] * share)
                nxt.append(len(stage) - 1)
        frontier = nxt
    n = len(stage)
    eps = eps_scale * rng.standard_normal((n, n_demand + n_price))
    eps[0] = 0.0
    prob = np.array(prob)
    anc = np.array(anc)
    for node in range(n):
        kids = np.flatnonzero(anc == node)
        if kids.size:
            prob[kids] *= prob[node] / prob[kids].sum()
    return ScenarioTree(horizon, n_demand, n_price, np.array(stage), anc, prob, eps=eps)


def make_instance(rng, n_tanks=3, n_inputs=4, n_demands=2, n_mixing=0, horizon=3, max_nodes=20,
                  w_u_scale=1.0, identity_a=True):
    model = make_model(rng, n_tanks, n_inputs, n_demands, n_mixing, identity_a=identity_a)
    tree = make_tree(rng, horizon, n_demands, n_inputs, max_nodes=max_nodes)
    d_hat = 0.3 + 0.2 * rng.random((horizon, n_demands))
    a_hat = 0.5 + rng.random((horizon, n_inputs))
    tree = attach_forecast(tree, d_hat, a_hat)
    wu = rng.standard_normal((n_inputs, n_inputs))
    wu = w_u_scale * (wu @ wu.T + n_inputs * np.eye(n_inputs))
    weights = CostWeights(w_alpha=1.0, w_u=wu, w_s=2.0, w_x=5.0)
    p = model.x_safe * (1.2 + 0.5 * rng.random(n_tanks))
    q = 0.3 * rng.random(n_inputs)
    return assemble_problem(model, tree, weights, p, q)


def instance_to_arrays(inst) -> dict:
    """Flatten an instance into plain arrays (golden fixtures)."""
    m, t, w = inst.model, inst.tree, inst.weights
    return dict(
        A=m.A, B=m.B, Gd=m.Gd, E=m.E, Ed=m.Ed, x_min=m.x_min, x_max=m.x_max, x_safe=m.x_safe,
        u_min=m.u_min, u_max=m.u_max, alpha0=m.alpha0, dt=np.array(m.dt),
        horizon=np.array(t.horizon), stage=t.stage, anc=t.anc, prob=t.prob, eps=t.eps,
        demand=t.demand, price=t.price,
        w_alpha=np.array(w.w_alpha), w_u=np.asarray(w.w_u, float), w_s=np.array(w.w_s),
        w_x=np.array(w.w_x), p=inst.p, q=inst.q,
    )


def instance_from_arrays(a) -> object:
    model = NetworkModel(A=a["A"], B=a["B"], Gd=a["Gd"], E=a["E"], Ed=a["Ed"], x_min=a["x_min"],
                         x_max=a["x_max"], x_safe=a["x_safe"], u_min=a["u_min"], u_max=a["u_max"],
                         alpha0=a["alpha0"], dt=float(a["dt"]))
    H = int(a["horizon"])
    tree = ScenarioTree(H, model.n_demands, model.n_inputs, a["stage"], a["anc"], a["prob"],
                        eps=a["eps"], demand=a["demand"], price=a["price"])
    wu = a["w_u"]
    weights = CostWeights(w_alpha=float(a["w_alpha"]), w_u=float(wu) if wu.ndim == 0 else wu,
                          w_s=float(a["w_s"]), w_x=float(a["w_x"]))
    return assemble_problem(model, tree, weights, a["p"], a["q"])


def load_golden(name: str):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.fail(f"golden fixture missing: {path}")
    return np.load(path, allow_pickle=False)
