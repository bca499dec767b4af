"""CPU-only tests: the oracle against the reference's golden outputs, the
reference itself when mounted, host-side logic, and the C ABI surface."""

from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import (ROOT, import_reference, instance_from_arrays, instance_to_arrays,
                      load_golden, make_instance, reference_available, rel_err)
from oracle import port
from oracle.dense import dense_kkt_solve
from paper_1904_10548_b200 import SolverConfig, theta_sequence, uniform_tree, validate_tree
from paper_1904_10548_b200.solver import _beta_table, _null_space, _stage_recursion
from paper_1904_10548_b200.synthetic import CONFIGS, config_instance

SMALL = ["small_plain", "small_coupled", "small_dense_a", "small_chain", "small_wide"]


# ------------------------------------------------------- oracle pinning

@pytest.mark.parametrize("name", SMALL)
def test_oracle_factor_and_dual_gradient_vs_golden(name):
    g = load_golden(f"{name}.npz")
    inst = instance_from_arrays(g)
    fac, e_off = port.factor(inst)
    np.testing.assert_allclose(e_off, g["e_offset"], rtol=0, atol=1e-12 * (1 + np.abs(g["e_offset"]).max()))
    np.testing.assert_allclose(np.stack(fac.T), g["t_mat"], rtol=0, atol=1e-12)
    R = g["dg_y"].reshape(inst.n_nonroot, -1)
    nt = inst.model.n_tanks
    U, X, v = port.dual_gradient_rows(inst, fac, e_off, R[:, :nt] + R[:, nt:2 * nt], R[:, 2 * nt:])
    assert rel_err(np.concatenate([U, X], 1).reshape(-1), g["dg_z"]) <= 1e-12
    assert v == pytest.approx(float(g["dg_value"]), rel=1e-12)


@pytest.mark.parametrize("name", SMALL)
def test_oracle_prox_bit_exact_vs_golden(name):
    g = load_golden(f"{name}.npz")
    inst = instance_from_arrays(g)
    w, gam = g["prox_w"], float(g["prox_gamma"])
    out = port.prox_g_conj_rows(inst, w.reshape(inst.n_nonroot, -1), gam).reshape(-1)
    np.testing.assert_array_equal(out, g["prox_conj"])
    np.testing.assert_array_equal(port.prox_g(inst, w, gam), g["prox_plain"])


@pytest.mark.parametrize("name", SMALL)
def test_oracle_lipschitz_and_fixed_solve_vs_golden(name):
    g = load_golden(f"{name}.npz")
    inst = instance_from_arrays(g)
    fac, e_off = port.factor(inst)
    L = port.power_lipschitz(inst, fac, e_off)
    assert L == pytest.approx(float(g["lipschitz"]), rel=1e-12)
    it = int(g["fixed_iters"])
    res = port.apg_solve(inst, 1.0 / L, max_iter=it, tol=1e-30, gap_check_every=it + 1,
                         fac=fac, e_off=e_off)
    for k in ("u0", "primal", "primal_avg", "dual"):
        assert rel_err(getattr(res, k), g[f"fixed_{k}"]) <= 1e-12, k
    assert res.duality_gap == pytest.approx(float(g["fixed_duality_gap"]), rel=1e-10)
    assert res.objective == pytest.approx(float(g["fixed_objective"]), rel=1e-12)


@pytest.mark.parametrize("name", SMALL)
def test_oracle_converging_solve_vs_golden(name):
    g = load_golden(f"{name}.npz")
    inst = instance_from_arrays(g)
    fac, e_off = port.factor(inst)
    L = port.power_lipschitz(inst, fac, e_off)
    res = port.apg_solve(inst, 1.0 / L, max_iter=4000, tol=1e-4, gap_check_every=25,
                         fac=fac, e_off=e_off)
    assert res.iterations == int(g["conv_iterations"])
    assert res.termination == str(g["conv_termination"])
    assert rel_err(res.u0, g["conv_u0"]) <= 1e-12


@pytest.mark.parametrize("name", SMALL)
def test_dense_oracle_agrees_with_tree_oracle(name):
    g = load_golden(f"{name}.npz")
    inst = instance_from_arrays(g)
    z = dense_kkt_solve(inst, g["dg_y"])
    assert rel_err(z, g["dg_z"]) <= 1e-8


def test_oracle_barcelona_c1_500_vs_golden():
    g = load_golden("barcelona_C1.npz")
    inst = config_instance("C1")
    fac, e_off = port.factor(inst)
    it = int(g["iters"])
    res = port.apg_solve(inst, 1.0 / float(g["lipschitz"]), max_iter=it, tol=1e-30,
                         gap_check_every=it + 1, fac=fac, e_off=e_off, reference_cost_accounting=False)
    n = inst.n_nonroot
    for k in ("primal", "primal_avg", "dual"):
        assert rel_err(getattr(res, k).reshape(n, -1)[g["rows"]], g[k + "_rows"]) <= 1e-12, k
    assert res.objective == pytest.approx(float(g["objective"]), rel=1e-12)


def test_synthetic_instance_is_the_golden_one():
    import hashlib
    for cfg in ("C1", "C2"):
        g = load_golden(f"barcelona_{cfg}.npz")
        arrays = instance_to_arrays(config_instance(cfg))
        h = hashlib.sha256()
        for k in sorted(arrays):
            h.update(k.encode())
            h.update(np.ascontiguousarray(arrays[k]).tobytes())
        assert h.digest() == bytes(g["instance_digest"]), cfg


def test_oracle_matches_reference_live():
    ref = import_reference()
    import sys
    import watermpc.solver as RS
    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    from make_golden import to_reference
    rng = np.random.default_rng(99)
    inst = make_instance(rng, n_inputs=5, n_mixing=2, horizon=3, max_nodes=14)
    rinst = to_reference(instance_to_arrays(inst))
    cache = RS.factor_step(rinst)
    L = RS.estimate_lipschitz(cache, rinst)
    res = RS.solve(rinst, RS.SolverConfig(max_iter=80, tol=1e-30, gamma=1 / L, gap_check_every=99))
    mine = port.apg_solve(inst, 1 / L, max_iter=80, tol=1e-30, gap_check_every=99)
    np.testing.assert_array_equal(mine.dual, res.dual)
    np.testing.assert_array_equal(mine.primal_avg, res.primal_avg)
    assert mine.duality_gap == res.duality_gap
    assert ref is not None


# ------------------------------------------------------------ host logic

def test_theta_and_beta_tables():
    seq = theta_sequence(3)
    assert seq[0] == pytest.approx(1.0)
    assert seq[1] == pytest.approx((np.sqrt(5.0) - 1.0) / 2.0, abs=1e-12)
    assert seq[2] == pytest.approx(0.455887, abs=1e-6)
    beta = _beta_table(theta_sequence(3))
    assert beta[0] == 0.0 and beta[1] == pytest.approx(0.0, abs=1e-15)
    assert beta[2] == pytest.approx(0.2817535251, abs=1e-9)
    seq = theta_sequence(10_001)
    assert float(np.abs(1.0 - seq[1:] - seq[1:] ** 2 / seq[:-1] ** 2).max()) <= 1e-14
    np.testing.assert_array_equal(theta_sequence(500), port.theta_table(500))


def test_solver_config_validation():
    for kw, msg in [(dict(max_iter=0), "max_iter"), (dict(tol=0.0), "tol"), (dict(gamma=-1.0), "gamma"),
                    (dict(threads=0), "threads"), (dict(gap_check_every=0), "gap_check_every")]:
        with pytest.raises(ValueError, match=msg):
            SolverConfig(**kw)


@pytest.mark.parametrize("name,nodes", [("C1", 182), ("C2", 2430), ("C3", 10196), ("C4", 79188)])
def test_config_trees_have_the_survey_node_counts(name, nodes):
    t = uniform_tree(CONFIGS[name], 24, 88, 114)
    assert t.n_nonroot == nodes
    assert validate_tree(t) == []
    assert t.n_nonroot * 177 == nodes * 177 and t.n_nonroot * 240 == nodes * 240


def test_city_scale_dimension_counts():
    from paper_1904_10548_b200 import CostWeights, NetworkModel, ScenarioTree, assemble_problem, attach_forecast
    n = 13029
    tree = ScenarioTree.single_branch(horizon=n, n_demand=88, n_price=114)
    tree = attach_forecast(tree, np.zeros((n, 88)), np.zeros((n, 114)))
    model = NetworkModel(A=np.eye(63), B=np.zeros((63, 114)), Gd=np.zeros((63, 88)), E=np.zeros((0, 114)),
                         Ed=np.zeros((0, 88)), x_min=np.zeros(63), x_max=np.full(63, 1e5),
                         x_safe=np.full(63, 10.0), u_min=np.zeros(114), u_max=np.ones(114),
                         alpha0=np.zeros(114), dt=3600.0)
    inst = assemble_problem(model, tree, CostWeights(1.0, 1.0, 1.0, 1.0), np.zeros(63), np.zeros(114))
    assert inst.n_primal == 2_306_133 and inst.n_dual == 3_126_960


def test_host_stage_recursion_matches_oracle():
    inst = config_instance("C1")
    basis, e_pinv = _null_space(inst.model.E, inst.model.n_inputs)
    lam, T, D, _ = _stage_recursion(inst, basis)
    fac = port.stage_factors(inst.model.E, inst.wu, 24)
    for s in range(24):
        np.testing.assert_array_equal(T[s], fac.T[s])
        np.testing.assert_array_equal(D[s], fac.D[s])
    # Barcelona structure facts the kernels specialise on
    assert np.array_equal(inst.model.A, np.eye(63))
    assert np.count_nonzero(inst.model.B, axis=0).max() <= 2
    np.testing.assert_array_equal(D[3], 2.0 * (T[3] @ inst.wu))


def test_barcelona_network_dimensions():
    inst = config_instance("C1")
    m = inst.model
    assert (m.n_tanks, m.n_inputs, m.n_demands, m.n_mixing) == (63, 114, 88, 17)
    assert np.linalg.matrix_rank(m.E) == 17
    assert (m.Gd != 0).sum() == 71 and (m.Ed != 0).sum() == 17


def test_tree_validation_messages():
    t = uniform_tree([2], 2, 1, 1)
    t.prob[1] = 0.7
    issues = validate_tree(t)
    assert any("children probabilities" in s for s in issues)
    assert any("stage 1 probabilities" in s for s in issues)


# ------------------------------------------------------------- C ABI

def _declared_symbols():
    text = open(os.path.join(ROOT, "include", "wmpc.h")).read()
    return sorted(set(re.findall(r"\b(wmpc_[a-z_]+)\s*\(", text)))


def test_native_library_builds_and_exports_every_declared_symbol():
    from paper_1904_10548_b200.build import build_native
    path = build_native()
    lib = ctypes.CDLL(path)
    names = _declared_symbols()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    from paper_1904_10548_b200 import _native
    assert set(names) <= set(_native.SIGNATURES) | {"wmpc_global_error"}


def test_native_library_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1904_10548_b200 import _native
    with pytest.raises(RuntimeError, match="wmpc_create failed"):
        _native.Context(4, 1, 1, 1, 1, 0)


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1904_10548_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", src, re.M), f
