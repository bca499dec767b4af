"""The persistent structured kernel (wmpc_fast.cuh) against the general
per-stage kernels and the oracle. The fast path applies when A = I,
W_u = c I and n_u is even; WMPC_DISABLE_FAST=1 forces the general path."""

from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import make_model, rel_err
from oracle import port
from paper_1904_10548_b200 import (CostWeights, SolverConfig, assemble_problem, attach_forecast,
                                   factor_step, solve, uniform_tree)
from paper_1904_10548_b200 import _native as nat
from paper_1904_10548_b200.synthetic import barcelona_instance, config_instance

pytestmark = pytest.mark.gpu


def _solve(inst, iters, gamma, fast: bool, gce=None):
    old = os.environ.get("WMPC_DISABLE_FAST")
    os.environ["WMPC_DISABLE_FAST"] = "0" if fast else "1"
    try:
        cache = factor_step(inst)
        ctx = cache._bind()
        mode = nat.load().wmpc_fast_path(ctx.h)
        res = solve(inst, SolverConfig(max_iter=iters, tol=1e-30, gamma=gamma,
                                       gap_check_every=gce or iters + 1), cache=cache)
    finally:
        if old is None:
            del os.environ["WMPC_DISABLE_FAST"]
        else:
            os.environ["WMPC_DISABLE_FAST"] = old
    return res, mode


def _scalar_w_instance(seed, branching, horizon, n_tanks=3, n_inputs=4, n_mixing=1):
    rng = np.random.default_rng(seed)
    model = make_model(rng, n_tanks, n_inputs, 2, n_mixing)
    tree = uniform_tree(branching, horizon, 2, n_inputs)
    tree.eps = 0.1 * rng.standard_normal((tree.n_nodes, 2 + n_inputs))
    tree.eps[0] = 0.0
    tree = attach_forecast(tree, 0.3 + 0.2 * rng.random((horizon, 2)), 0.5 + rng.random((horizon, n_inputs)))
    w = CostWeights(w_alpha=1.0, w_u=0.7, w_s=2.0, w_x=5.0)
    p = model.x_safe * (1.2 + 0.5 * rng.random(n_tanks))
    return assemble_problem(model, tree, w, p, 0.3 * rng.random(n_inputs))


@pytest.mark.parametrize("branching,horizon", [([2, 3], 5), ([3], 1), ([1, 2, 2], 4), ([2, 2, 2, 2], 4)])
def test_fast_matches_general_small_scalar_w(branching, horizon):
    inst = _scalar_w_instance(5, branching, horizon)
    fac, e_off = port.factor(inst)
    gamma = 1.0 / port.power_lipschitz(inst, fac, e_off)
    rf, mf = _solve(inst, 120, gamma, True, gce=40)
    rg, mg = _solve(inst, 120, gamma, False, gce=40)
    assert mf > 0 and mg == 0
    ro = port.apg_solve(inst, gamma, max_iter=120, tol=1e-30, gap_check_every=40, fac=fac, e_off=e_off,
                        reference_cost_accounting=False)
    for k in ("u0", "primal", "primal_avg", "dual"):
        assert rel_err(getattr(rf, k), getattr(rg, k)) <= 1e-11, k
        assert rel_err(getattr(rf, k), getattr(ro, k)) <= 1e-9, k
    assert abs(rf.objective - ro.objective) <= 1e-9 * (1 + abs(ro.objective))


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3"])
def test_fast_matches_general_barcelona(cfg):
    inst = config_instance(cfg)
    gamma = 1.0 / 5e9
    rf, mf = _solve(inst, 60, gamma, True)
    rg, mg = _solve(inst, 60, gamma, False)
    assert mf > 0 and mg == 0
    for k in ("u0", "primal", "primal_avg", "dual"):
        assert rel_err(getattr(rf, k), getattr(rg, k)) <= 1e-11, k
    assert abs(rf.duality_gap - rg.duality_gap) <= 1e-10 * (1 + abs(rg.duality_gap))


def test_fast_path_chunked_equals_single_launch():
    inst = config_instance("C1")
    gamma = 1.0 / 1.1e8
    a, _ = _solve(inst, 100, gamma, True)            # one launch of 100 iterations
    b, _ = _solve(inst, 100, gamma, True, gce=7)     # launches of 7 iterations
    np.testing.assert_array_equal(a.dual, b.dual)
    np.testing.assert_array_equal(a.primal_avg, b.primal_avg)
    np.testing.assert_array_equal(a.primal, b.primal)


def test_fast_path_pure_chain_tree():
    inst = barcelona_instance([], seed=3, horizon=24)  # a single scenario: 24 chain nodes
    gamma = 1.0 / 1e8
    rf, mf = _solve(inst, 50, gamma, True)
    rg, _ = _solve(inst, 50, gamma, False)
    assert mf > 0
    assert rel_err(rf.dual, rg.dual) <= 1e-11


def test_reciprocal_division_is_exact():
    """The kernels divide by gamma through RN(1/gamma) + one fma correction;
    it must agree bit for bit with IEEE division (incl. edge magnitudes)."""
    rng = np.random.default_rng(0)
    n = 1 << 22
    v = rng.standard_normal(n) * np.exp2(rng.integers(-60, 60, n))
    v[: 1 << 12] = rng.standard_normal(1 << 12) * np.exp2(rng.integers(-1070, 1023, 1 << 12))
    v[5] = 0.0
    v[6] = np.inf
    v[7] = -np.inf
    v[8] = np.nan
    g = np.exp2(rng.uniform(-40, 20, 64)) * (1 + rng.random(64))
    g[:4] = [1.0 / 1.731949602497e9, 1.0 / 1.0888e8, 0.37, 3.0]
    bad = nat.C.c_uint64(0)
    rc = nat.load().wmpc_debug_div(nat.ptr(v), nat.ptr(g), n, nat.C.byref(bad))
    assert rc == 0
    assert bad.value == 0


# env switches of the kernel variants (graph: CTA-per-chain kernels; chainw:
# warp-per-chain kernels with an 8-row shared-memory ring (fp64), or rows
# streamed through registers)
VARIANT_ENV = {  # (k_chain_dp off: it is the C3 / C4 default)
    "graph": {"WMPC_DP": "0", "WMPC_CHAINW": "0"},
    "graph-chainw8": {"WMPC_DP": "0", "WMPC_CHAINW": "1", "WMPC_CWPD": "8"},
    "graph-chainwr": {"WMPC_DP": "0", "WMPC_CHAINW": "1", "WMPC_CWPD": "1"},
}


def _with_env(env, fn):
    saved = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return fn()
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("kernel", ["graph", "graph-chainw8", "graph-chainwr", "scan", "cta"])
@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_every_structured_kernel_matches_general(cfg, kernel):
    inst = config_instance(cfg)
    gamma = 1.0 / 2e9
    env = {"WMPC_KERNEL": kernel.split("-")[0], **VARIANT_ENV.get(kernel, {})}
    rf, mf = _with_env(env, lambda: _solve(inst, 40, gamma, True, gce=17))
    rg, _ = _solve(inst, 40, gamma, False, gce=17)
    # a variant whose shared-memory footprint does not fit falls back to the CTA kernel (1..99)
    allowed = {"graph": [300], "scan": list(range(200, 300)) + list(range(1, 100)),
               "cta": list(range(1, 100))}.get(kernel, [300])
    assert mf in allowed, mf
    for k in ("u0", "primal", "primal_avg", "dual"):
        assert rel_err(getattr(rf, k), getattr(rg, k)) <= 1e-11, k


@pytest.mark.parametrize("variant", ["graph-chainw8", "graph-chainwr"])
@pytest.mark.parametrize("cfg,prec", [("C1", "fp64"), ("C3", "fp64"), ("C2", "fp32")])
def test_chain_kernel_variants_bit_identical(cfg, prec, variant):
    """The warp-per-chain kernels (wmpc_chainw.cuh) do the per-element
    arithmetic of the CTA-per-chain kernels in the same order: every iterate,
    average, certificate and u0 is bit-identical."""
    inst = config_instance(cfg)
    cfgs = SolverConfig(max_iter=40, tol=1e-30, gamma=1.0 / 2e9, gap_check_every=17, precision=prec)

    def run(env):
        def go():
            cache = factor_step(inst)
            assert nat.load().wmpc_fast_path(cache._bind().h) == 300
            return solve(inst, cfgs, cache=cache)
        return _with_env(env, go)

    ra = run(VARIANT_ENV["graph"])
    rb = run(VARIANT_ENV[variant])
    for k in ("u0", "primal", "primal_avg", "dual"):
        np.testing.assert_array_equal(getattr(ra, k), getattr(rb, k), err_msg=k)
    assert ra.duality_gap == rb.duality_gap and ra.objective == rb.objective


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3"])
def test_block_dykstra_certificate_matches_general(cfg):
    """The certificate's Dykstra restoration: one thread per (node, coupling
    row) block on the structured path (k_dyk_block) against one warp per node
    over the CSR operators on the general path (k_dyk_warp): the same sweep
    count rule and per-element arithmetic, so the gap and the objective agree
    to rounding."""
    inst = config_instance(cfg)
    gamma = 1.0 / 2e9
    rf, mf = _solve(inst, 200, gamma, True)
    rg, mg = _solve(inst, 200, gamma, False)
    assert mf == 300 and mg == 0, (mf, mg)
    assert abs(rf.duality_gap - rg.duality_gap) <= 1e-10 * (1 + abs(rg.duality_gap))
    assert abs(rf.objective - rg.objective) <= 1e-12 * (1 + abs(rg.objective))
