"""Closed-loop driver host logic (simulate.py:26-204 restated): configuration
and log validation, the indicators, the C5 scenario generator."""

from __future__ import annotations

import numpy as np
import pytest

from paper_1904_10548_b200 import SolverConfig
from paper_1904_10548_b200.forecast import ForecastSeries
from paper_1904_10548_b200.simulate import (SimulationConfig, SimulationLog, kpi_complexity, kpi_economic,
                                            kpi_safety, run_closed_loop)
from paper_1904_10548_b200.synthetic import closed_loop_scenario


def test_simulation_config_validation():
    with pytest.raises(ValueError, match="h_sim"):
        SimulationConfig(h_sim=0, weights=None, solver=SolverConfig(), x0=np.zeros(2))
    cfg = SimulationConfig(h_sim=2, weights=None, solver=SolverConfig(), x0=[1, 2], u_prev=[0.0])
    assert cfg.x0.dtype == float and cfg.u_prev.dtype == float and not cfg.warm_start


def test_forecast_series_validation():
    with pytest.raises(ValueError, match="disagree"):
        ForecastSeries(np.ones((3, 2)), np.ones((2, 2)))
    with pytest.raises(ValueError, match="nonnegative"):
        ForecastSeries(-np.ones((3, 2)), np.ones((3, 2)))
    f = ForecastSeries(np.ones((4, 2)), np.ones((4, 3)))
    assert (f.horizon, f.n_demand, f.n_price) == (4, 2, 3)


def test_indicators_on_a_hand_log():
    log = SimulationLog(x=np.array([[5.0, 5.0], [1.0, 4.0], [3.0, 0.5]]), u=np.array([[1.0, 2.0], [0.0, 1.0]]),
                        demand=np.zeros((2, 1)), price=np.array([[0.5, 0.5], [1.0, 1.0]]),
                        solve_time_s=np.array([0.25, 0.5]), iterations=np.array([3, 4]),
                        primal_residual=np.zeros(2), alpha0=np.array([0.5, 0.0]), x_safe=np.array([2.0, 2.0]))
    assert kpi_economic(log) == pytest.approx(((1.0 * 1 + 0.5 * 2) + (1.5 * 0 + 1.0 * 1)) / 2)
    assert kpi_safety(log) == pytest.approx(1.0 + 1.5)
    assert kpi_complexity(log) == 0.5


def test_closed_loop_scenario_shapes():
    sc = closed_loop_scenario([2, 2], h_sim=10)
    m = sc["model"]
    assert sc["realized_demand"].shape == (10, m.n_demands)
    assert sc["realized_price"].shape == (10, m.n_inputs)
    f = sc["forecaster"](3)
    assert f.d_hat.shape == (24, m.n_demands) and np.all(f.d_hat >= 0)
    np.testing.assert_allclose(sc["forecaster"](24).d_hat, sc["forecaster"](0).d_hat)  # daily cycle


def test_run_closed_loop_rejects_short_realizations():
    sc = closed_loop_scenario([2], h_sim=3)
    cfg = SimulationConfig(h_sim=5, weights=sc["weights"], solver=SolverConfig(), x0=sc["x0"])
    with pytest.raises(ValueError, match="realizations cover"):
        run_closed_loop(sc["model"], sc["tree_template"], sc["forecaster"], sc["realized_demand"],
                        sc["realized_price"], cfg)
