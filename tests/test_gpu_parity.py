"""GPU parity against the CPU oracle (oracle/port.py) and the reference's own
outputs (tests/golden/*.npz). Every call goes through libwmpc.so.

Tolerances (BASELINE.json north_star): active sets and index work bit-exact;
prox values bit-exact on identical inputs; fp64 iterates and cost after a
fixed iteration count within 1e-8 relative (metric of test_solver.py:21-22).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import instance_from_arrays, load_golden, make_instance, rel_err
from oracle import port
from oracle.dense import dense_kkt_solve
from paper_1904_10548_b200 import (
    SolverConfig,
    dual_gradient,
    estimate_lipschitz,
    factor_step,
    prox_g,
    prox_g_conjugate,
    solve,
)
from paper_1904_10548_b200.synthetic import config_instance

pytestmark = pytest.mark.gpu

TOL = 1e-8
SMALL = ["small_plain", "small_coupled", "small_dense_a", "small_chain", "small_wide"]


def _loaded_native():
    from paper_1904_10548_b200 import _native
    return _native._LIB is not None


# ---------------------------------------------------------------- prox (K4)

@pytest.mark.parametrize("name", SMALL)
def test_prox_bit_exact_vs_reference_golden(name):
    g = load_golden(f"{name}.npz")
    inst = instance_from_arrays(g)
    out = prox_g_conjugate(inst, g["prox_w"], float(g["prox_gamma"]))
    np.testing.assert_array_equal(out, g["prox_conj"])
    out = prox_g(inst, g["prox_w"], float(g["prox_gamma"]))
    np.testing.assert_array_equal(out, g["prox_plain"])
    assert _loaded_native()


def test_prox_bit_exact_barcelona_random_rows():
    inst = config_instance("C1")
    rng = np.random.default_rng(7)
    R = rng.standard_normal((inst.n_nonroot, 240))
    R[:, :63] *= 6000.0
    R[:, 63:126] *= 3000.0
    R[:, 126:] *= 1000.0
    R[::7] *= 1e-3  # interior rows
    w = R.reshape(-1)
    for gamma in (1e-8, 0.37, 4.0):
        got = prox_g_conjugate(inst, w, gamma)
        want = port.prox_g_conj_rows(inst, w.reshape(inst.n_nonroot, -1), gamma).reshape(-1)
        np.testing.assert_array_equal(got, want)
        got = prox_g(inst, w, gamma)
        np.testing.assert_array_equal(got, port.prox_g(inst, w, gamma))


def test_prox_edge_cases_inf_bounds_zero_weights():
    rng = np.random.default_rng(3)
    inst = make_instance(rng, horizon=2, max_nodes=6)
    m = inst.model
    m.u_min[:] = -np.inf
    m.u_max[1] = np.inf
    m.x_min[0] = -np.inf
    m.x_max[:] = np.inf
    inst.weights.w_s = 0.0
    w = 10 * rng.standard_normal(inst.n_dual)
    w[5] = 0.0
    for gamma in (0.5, 2.0):
        np.testing.assert_array_equal(prox_g_conjugate(inst, w, gamma),
                                      port.prox_g_conj_rows(inst, w.reshape(inst.n_nonroot, -1),
                                                            gamma).reshape(-1))
        np.testing.assert_array_equal(prox_g(inst, w, gamma), port.prox_g(inst, w, gamma))


# --------------------------------------------------- factor step (K6) + DG

@pytest.mark.parametrize("name", SMALL)
def test_factor_offsets_and_dual_gradient_vs_golden(name):
    g = load_golden(f"{name}.npz")
    inst = instance_from_arrays(g)
    cache = factor_step(inst)
    assert rel_err(cache.e_offset, g["e_offset"]) <= 1e-12
    assert rel_err(cache.u_part, g["u_part"]) <= 1e-12
    z, val = dual_gradient(cache, inst, g["dg_y"])
    assert rel_err(z, g["dg_z"]) <= 1e-10
    assert abs(val - float(g["dg_value"])) <= 1e-10 * (1 + abs(float(g["dg_value"])))
    z0, val0 = dual_gradient(cache, inst, np.zeros(inst.n_dual))
    assert rel_err(z0, g["dg0_z"]) <= 1e-10
    assert abs(val0 - float(g["dg0_value"])) <= 1e-10 * (1 + abs(float(g["dg0_value"])))


@pytest.mark.parametrize("name", SMALL)
def test_dual_gradient_matches_dense_kkt(name):
    g = load_golden(f"{name}.npz")
    inst = instance_from_arrays(g)
    cache = factor_step(inst)
    rng = np.random.default_rng(11)
    for scale in (0.0, 1.0, 1e3):
        y = scale * rng.standard_normal(inst.n_dual)
        z, _ = dual_gradient(cache, inst, y)
        assert rel_err(z, dense_kkt_solve(inst, y)) <= 1e-8


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_dual_gradient_barcelona_vs_oracle(cfg):
    inst = config_instance(cfg)
    cache = factor_step(inst)
    fac, e_off = port.factor(inst)
    assert rel_err(cache.e_offset, e_off) <= 1e-12
    rng = np.random.default_rng(5)
    y = rng.standard_normal(inst.n_dual) * 50.0
    z, val = dual_gradient(cache, inst, y)
    R = y.reshape(inst.n_nonroot, -1)
    U, X, v = port.dual_gradient_rows(inst, fac, e_off, R[:, :63] + R[:, 63:126], R[:, 126:])
    assert rel_err(z, np.concatenate([U, X], 1).reshape(-1)) <= 1e-10
    assert abs(val - v) <= 1e-9 * (1 + abs(v))


# -------------------------------------------------------------- Lipschitz

@pytest.mark.parametrize("name", SMALL)
def test_lipschitz_vs_golden(name):
    g = load_golden(f"{name}.npz")
    inst = instance_from_arrays(g)
    cache = factor_step(inst)
    L = estimate_lipschitz(cache, inst)
    assert L == pytest.approx(float(g["lipschitz"]), rel=2e-3)
    assert cache.lipschitz == L


def test_lipschitz_barcelona_c1_vs_golden():
    g = load_golden("barcelona_C1.npz")
    inst = config_instance("C1")
    cache = factor_step(inst)
    assert estimate_lipschitz(cache, inst) == pytest.approx(float(g["lipschitz"]), rel=2e-3)


# ------------------------------------------------------ fixed-iteration APG

@pytest.mark.parametrize("name", SMALL)
def test_fixed_iteration_solve_vs_golden(name):
    g = load_golden(f"{name}.npz")
    inst = instance_from_arrays(g)
    it = int(g["fixed_iters"])
    L = float(g["lipschitz"])
    res = solve(inst, SolverConfig(max_iter=it, tol=1e-30, gamma=1.0 / L, gap_check_every=it + 1))
    for k in ("u0", "primal", "primal_avg", "dual"):
        assert rel_err(getattr(res, k), g[f"fixed_{k}"]) <= TOL, k
    for k in ("duality_gap", "objective"):
        want = float(g[f"fixed_{k}"])
        assert abs(getattr(res, k) - want) <= TOL * (1 + abs(want)), k
    assert res.termination == "max_iter" and res.iterations == it


@pytest.mark.parametrize("name", SMALL)
def test_converging_solve_vs_golden(name):
    g = load_golden(f"{name}.npz")
    if "conv_iterations" not in g:
        pytest.skip("no convergence record")
    inst = instance_from_arrays(g)
    res = solve(inst, SolverConfig(max_iter=4000, tol=1e-4))
    assert res.termination == str(g["conv_termination"])
    assert res.iterations == int(g["conv_iterations"])
    assert rel_err(res.u0, g["conv_u0"]) <= 1e-6


def test_barcelona_c1_500_iterations_vs_reference_golden():
    g = load_golden("barcelona_C1.npz")
    inst = config_instance("C1")
    L = float(g["lipschitz"])
    it = int(g["iters"])
    res = solve(inst, SolverConfig(max_iter=it, tol=1e-30, gamma=1.0 / L, gap_check_every=it + 1))
    n = inst.n_nonroot
    rows = g["rows"]
    for k in ("primal", "primal_avg", "dual"):
        v = getattr(res, k).reshape(n, -1)[rows]
        assert rel_err(v, g[k + "_rows"]) <= TOL, k
    assert rel_err(res.u0, g["u0"]) <= TOL
    for k in ("duality_gap", "objective"):
        want = float(g[k])
        assert abs(getattr(res, k) - want) <= TOL * (1 + abs(want)), k


@pytest.mark.slow
def test_barcelona_c2_500_iterations_vs_reference_golden():
    g = load_golden("barcelona_C2.npz")
    inst = config_instance("C2")
    L = float(g["lipschitz"])
    it = int(g["iters"])
    res = solve(inst, SolverConfig(max_iter=it, tol=1e-30, gamma=1.0 / L, gap_check_every=it + 1))
    n = inst.n_nonroot
    rows = g["rows"]
    for k in ("primal", "primal_avg", "dual"):
        v = getattr(res, k).reshape(n, -1)
        assert rel_err(v[rows], g[k + "_rows"]) <= TOL, k
        assert abs(np.linalg.norm(v) - float(g[k + "_norm"])) <= TOL * (1 + float(g[k + "_norm"]))
    assert rel_err(res.u0, g["u0"]) <= TOL
    for k in ("duality_gap", "objective"):
        want = float(g[k])
        assert abs(getattr(res, k) - want) <= TOL * (1 + abs(want)), k


def test_barcelona_c2_vs_oracle_live_100_iterations():
    inst = config_instance("C2")
    gamma = 1.0 / 1.9e9
    it = 100
    res = solve(inst, SolverConfig(max_iter=it, tol=1e-30, gamma=gamma, gap_check_every=it + 1))
    ref = port.apg_solve(inst, gamma, max_iter=it, tol=1e-30, gap_check_every=it + 1,
                         reference_cost_accounting=False)
    for k in ("u0", "primal", "primal_avg", "dual"):
        assert rel_err(getattr(res, k), getattr(ref, k)) <= TOL, k
    assert abs(res.objective - ref.objective) <= TOL * (1 + abs(ref.objective))
    assert abs(res.duality_gap - ref.duality_gap) <= TOL * (1 + abs(ref.duality_gap))


# -------------------------------------------------------------- properties

def test_large_tree_properties_c4_single_iterations():
    """At C4 (79,188 nodes) the oracle is too slow for full runs; check the
    size-independent properties: the dual gradient is affine in y and the
    prox is a nonexpansive map, on the full-size device buffers."""
    inst = config_instance("C4")
    cache = factor_step(inst)
    rng = np.random.default_rng(2)
    y1 = rng.standard_normal(inst.n_dual)
    y2 = rng.standard_normal(inst.n_dual)
    za, _ = dual_gradient(cache, inst, y1)
    zb, _ = dual_gradient(cache, inst, y2)
    zm, _ = dual_gradient(cache, inst, 0.5 * y1 + 0.5 * y2)
    assert np.max(np.abs(zm - 0.5 * (za + zb))) <= 1e-9 * (1 + np.abs(za).max())
    # stage-1 rows of a C4 dual gradient agree with the oracle's recursion
    fac, e_off = port.factor(inst)
    R = y1.reshape(inst.n_nonroot, -1)
    U, X, _ = port.dual_gradient_rows(inst, fac, e_off, R[:, :63] + R[:, 63:126], R[:, 126:],
                                      want_value=False)
    assert rel_err(za, np.concatenate([U, X], 1).reshape(-1)) <= 1e-10
