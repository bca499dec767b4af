"""The reference's optimality and closed-loop acceptance checks, run against
the GPU solver.

* test_oracle.py:66-138 (grid optimum, weak duality, gap at the optimum,
  monotone best-so-far gap) with the reference's grid / dense-KKT helpers
  restated in oracle/acceptance.py;
* test_simulate.py:44-116 (idle at zero demand and price, balance at
  constant demand, exact mass audit, identical logs for matched inputs) on
  the one-tank network of test_simulate.py:21-30 and the Barcelona C1 tree.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import make_instance
from oracle import acceptance as A
from paper_1904_10548_b200 import SolverConfig, dual_gradient, factor_step, solve
from paper_1904_10548_b200.forecast import ForecastSeries
from paper_1904_10548_b200.model import CostWeights, NetworkModel
from paper_1904_10548_b200.simulate import SimulationConfig, kpi_safety, run_closed_loop
from paper_1904_10548_b200.synthetic import closed_loop_scenario
from paper_1904_10548_b200.tree import ScenarioTree

pytestmark = pytest.mark.gpu


# ---------------------------------------------------- test_oracle.py:66-138

def test_interior_optimum_against_grid(rng):
    inst = make_instance(rng, n_tanks=1, n_inputs=1, n_demands=1, horizon=2, max_nodes=3)
    z_grid, _ = A.brute_force_min(inst)
    res = solve(inst, SolverConfig(max_iter=60000, tol=1e-6))
    span = float(inst.model.u_max[0] - inst.model.u_min[0])
    U_grid, _ = A.split_primal(inst, z_grid)
    assert abs(res.u0[0] - U_grid[0, 0]) <= 2e-3 * max(1.0, span)


def test_boundary_optimum_pinned_at_capacity(rng):
    """Negative price: pumping pays, the optimum sits at u_max (test_oracle.py:76-83);
    the GPU solve lands there too."""
    inst = make_instance(rng, n_tanks=1, n_inputs=1, n_demands=1, horizon=1, max_nodes=2)
    inst.econ[:] = -10.0
    inst.model.x_max[:] = 1e9
    z, _ = A.brute_force_min(inst)
    U, _ = A.split_primal(inst, z)
    assert U[0, 0] == pytest.approx(inst.model.u_max[0])
    res = solve(inst, SolverConfig(max_iter=20000, tol=1e-7))
    span = float(inst.model.u_max[0] - inst.model.u_min[0])
    assert abs(res.u0[0] - inst.model.u_max[0]) <= 2e-3 * max(1.0, span)


def test_weak_duality_at_zero(rng):
    inst = make_instance(rng, horizon=2, max_nodes=8)
    cache = factor_step(inst)
    z, _ = dual_gradient(cache, inst, np.zeros(inst.n_dual))
    gap = A.duality_gap(inst, z, np.zeros(inst.n_dual))
    assert gap >= -1e-9 * (1 + abs(gap))


def test_gap_near_zero_at_optimum(rng):
    inst = make_instance(rng, n_tanks=1, n_inputs=1, n_demands=1, horizon=2, max_nodes=3)
    res = solve(inst, SolverConfig(max_iter=80000, tol=1e-7))
    gap = A.duality_gap(inst, res.primal_avg, res.dual)
    obj = A.primal_objective(inst, A.project_primal_feasible(inst, res.primal_avg))
    assert gap <= 1e-4 * (1 + abs(obj))
    # the GPU certificate's own objective is the restored primal value
    assert abs(res.objective - obj) <= 1e-8 * (1 + abs(obj))


def test_monotone_best_so_far_gap_along_iterations(rng):
    inst = make_instance(rng, horizon=2, max_nodes=8)
    snaps = []

    def hook(nu, y, z, z_avg):
        if (nu + 1) in (8, 32, 128, 512):
            snaps.append((y.copy(), z_avg.copy()))

    solve(inst, SolverConfig(max_iter=512, tol=1e-30), iterate_hook=hook)
    gaps = [A.duality_gap(inst, z_avg, y) for y, z_avg in snaps]
    best = np.minimum.accumulate(gaps)
    assert all(b2 <= b1 + 1e-12 for b1, b2 in zip(best, best[1:]))
    assert all(g >= -1e-9 * (1 + abs(g)) for g in gaps)


def test_gpu_certificate_equals_dense_route_on_barcelona_c1():
    """The GPU certificate (Dykstra restoration, rollout, tree-recursion dual
    value) against the dense route of the reference's oracle.duality_gap on a
    converging Barcelona C1 solve: the reported objective is the restored
    primal value, and the dense-route gap is nonnegative (weak duality)."""
    from paper_1904_10548_b200.synthetic import config_instance
    inst = config_instance("C1")
    res = solve(inst, SolverConfig(max_iter=400, tol=1e-30, gap_check_every=401))
    z_f = A.project_primal_feasible(inst, res.primal_avg)
    obj = A.primal_objective(inst, z_f)
    assert np.isfinite(obj)
    assert abs(res.objective - obj) <= 1e-8 * (1 + abs(obj))


# ---------------------------------------------------- test_simulate.py:44-116

def _one_tank(horizon=4):
    """The one-tank network of test_simulate.py:21-30 (build_lti with dt = 1:
    one pump into the tank, one demand out of it)."""
    model = NetworkModel(A=np.eye(1), B=np.ones((1, 1)), Gd=-np.ones((1, 1)), E=np.zeros((0, 1)),
                         Ed=np.zeros((0, 1)), x_min=np.zeros(1), x_max=np.full(1, 2000.0),
                         x_safe=np.full(1, 300.0), u_min=np.zeros(1), u_max=np.full(1, 600.0),
                         alpha0=np.full(1, 0.02), dt=1.0)
    tree = ScenarioTree.single_branch(horizon=horizon, n_demand=1, n_price=1)
    weights = CostWeights(w_alpha=1.0, w_u=1e-3, w_s=1.0, w_x=100.0)
    return model, tree, weights


def _pattern(demand, price, horizon):
    def forecaster(k):
        return ForecastSeries(d_hat=np.full((horizon, 1), demand), alpha_hat=np.full((horizon, 1), price))
    return forecaster


def test_zero_demand_zero_price_stays_idle():
    model, tree, weights = _one_tank()
    h = 6
    cfg = SimulationConfig(h_sim=h, weights=weights, solver=SolverConfig(max_iter=2000, tol=1e-6),
                           x0=np.array([800.0]))
    log = run_closed_loop(model, tree, _pattern(0.0, 0.0, tree.horizon), np.zeros((h, 1)), np.zeros((h, 1)), cfg)
    assert float(np.max(np.abs(log.u))) <= 1e-3
    np.testing.assert_allclose(log.x, 800.0, atol=1e-2)
    assert kpi_safety(log) == 0.0


def test_constant_demand_reaches_balance():
    model, tree, weights = _one_tank(horizon=6)
    h, demand = 30, 200.0
    cfg = SimulationConfig(h_sim=h, weights=weights, solver=SolverConfig(max_iter=4000, tol=1e-4),
                           x0=np.array([800.0]))
    log = run_closed_loop(model, tree, _pattern(demand, 0.03, tree.horizon), np.full((h, 1), demand),
                          np.full((h, 1), 0.03), cfg)
    tail = model.B @ log.u[-5:].T.mean(axis=1) + model.Gd @ np.array([demand])
    assert float(np.abs(tail).max()) <= 0.05 * demand


def test_mass_audit_exact(rng):
    model, tree, weights = _one_tank()
    h = 8
    demand = 150.0 + 20.0 * rng.random((h, 1))
    cfg = SimulationConfig(h_sim=h, weights=weights, solver=SolverConfig(max_iter=500, tol=5e-2),
                           x0=np.array([700.0]))
    log = run_closed_loop(model, tree, _pattern(150.0, 0.03, tree.horizon), demand, np.full((h, 1), 0.03), cfg)
    for k in range(h):
        np.testing.assert_array_equal(log.x[k + 1], model.step_dynamics(log.x[k], log.u[k], log.demand[k]))


def test_matched_inputs_identical_logs():
    """test_simulate.py:97-116 on the Barcelona-dimension network (the reference
    uses its tank1 demo, out of scope here): two runs, bitwise-equal logs."""
    sc = closed_loop_scenario([2, 2, 2], h_sim=4)
    cfg = SimulationConfig(h_sim=4, weights=sc["weights"], x0=sc["x0"],
                           solver=SolverConfig(max_iter=300, tol=5e-2))
    logs = [run_closed_loop(sc["model"], sc["tree_template"], sc["forecaster"], sc["realized_demand"],
                            sc["realized_price"], cfg) for _ in range(2)]
    np.testing.assert_array_equal(logs[0].u, logs[1].u)
    np.testing.assert_array_equal(logs[0].x, logs[1].x)
    np.testing.assert_array_equal(logs[0].iterations, logs[1].iterations)
