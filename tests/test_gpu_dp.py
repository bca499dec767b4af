"""The fused one-kernel iteration (k_chain_dp, csrc/wmpc_dp.cuh) against the
four-kernel graph iteration (up -> branch groups -> down -> prox), the oracle
and the reference goldens.

k_chain_dp walks each chain bottom-up and recovers the down pass's prefix
sums from chain aggregates (wmpc_dp.cuh header): the same quantities as the
reference recursion (solver.py:242-290) in real arithmetic with a different
rounding order, so the comparison against the unfused kernels is at 1e-10
(fixed iterations), against the reference at the north_star's 1e-8.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import load_golden, rel_err
from oracle import port
from paper_1904_10548_b200 import SolverConfig, solve
from paper_1904_10548_b200 import _native as nat
from paper_1904_10548_b200 import solver as S
from paper_1904_10548_b200.synthetic import barcelona_instance, config_instance

pytestmark = pytest.mark.gpu


def _cache(inst, monkeypatch, dp: bool):
    monkeypatch.setenv("WMPC_DP", "1" if dp else "0")
    cache = S._factor(inst, None, private=True)
    info = nat.path_info(cache._bind())
    assert info["fast_path"] == 300, info
    assert info["fused_dp"] == (1 if dp else 0), info
    return cache


def _pair(inst, monkeypatch, **cfg):
    out = []
    for dp in (True, False):
        cache = _cache(inst, monkeypatch, dp)
        out.append(solve(inst, SolverConfig(**cfg), cache=cache))
    return out


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_dp_matches_graph_iteration_fixed_iterations(name, monkeypatch):
    inst = config_instance(name)
    a, b = _pair(inst, monkeypatch, max_iter=120, tol=1e-30, gamma=1 / 2e9, gap_check_every=121)
    for k in ("u0", "primal", "primal_avg", "dual"):
        assert rel_err(getattr(a, k), getattr(b, k)) <= 1e-10, k
    assert abs(a.duality_gap - b.duality_gap) <= 1e-9 * (1 + abs(b.duality_gap))
    assert abs(a.objective - b.objective) <= 1e-10 * (1 + abs(b.objective))


def test_dp_c1_500_iterations_vs_reference_golden(monkeypatch):
    g = load_golden("barcelona_C1.npz")
    inst = config_instance("C1")
    it = int(g["iters"])
    cache = _cache(inst, monkeypatch, True)
    res = solve(inst, SolverConfig(max_iter=it, tol=1e-30, gamma=1.0 / float(g["lipschitz"]),
                                   gap_check_every=it + 1), cache=cache)
    n = inst.n_nonroot
    for k in ("primal", "primal_avg", "dual"):
        assert rel_err(getattr(res, k).reshape(n, -1)[g["rows"]], g[k + "_rows"]) <= 1e-8, k
    assert rel_err(res.u0, g["u0"]) <= 1e-8
    for k in ("duality_gap", "objective"):
        assert abs(getattr(res, k) - float(g[k])) <= 1e-8 * (1 + abs(float(g[k]))), k


def test_dp_uneven_tree_vs_oracle(monkeypatch):
    """Branching [3, 1, 2, 1] (single-child stages between branchings, three
    children per root child): chain ownership, ragged ancestor paths."""
    inst = barcelona_instance([3, 1, 2, 1], seed=3, horizon=8)
    cache = _cache(inst, monkeypatch, True)
    gamma, it = 1.0 / 3e9, 80
    res = solve(inst, SolverConfig(max_iter=it, tol=1e-30, gamma=gamma, gap_check_every=it + 1), cache=cache)
    ref = port.apg_solve(inst, gamma, max_iter=it, tol=1e-30, gap_check_every=it + 1,
                         reference_cost_accounting=False)
    for k in ("u0", "primal", "primal_avg", "dual"):
        assert rel_err(getattr(res, k), getattr(ref, k)) <= 1e-8, k
    assert abs(res.objective - ref.objective) <= 1e-8 * (1 + abs(ref.objective))


def test_dp_certificates_between_chunks_leave_the_iteration_state_intact(monkeypatch):
    """Check iterations run the certificate between iteration chunks; it uses
    scratch buffers, so k_chain_dp's carried state (L, aggregates, chain
    totals, branching rows' Yc) is untouched: 200 iterations in chunks of 25
    with a certificate after each chunk are bit-identical to 200 without."""
    inst = config_instance("C1")
    out = []
    for cert in (False, True):
        cache = _cache(inst, monkeypatch, True)
        ctx = cache._bind()
        S._upload_bounds(ctx, inst)
        th = S.theta_sequence(200)
        be = S._beta_table(th)
        ctx.call("wmpc_apg_begin", 1.0 / 2e9, 200, nat.ptr(th), nat.ptr(be))
        for _ in range(8):
            ctx.call("wmpc_apg_run", 25)
            if cert:
                S._certificate(ctx)
        out.append(S._read(ctx, inst, True))
    for a, b in zip(out[0], out[1]):
        np.testing.assert_array_equal(a, b)


def test_dp_convergence_run_matches_graph_iteration(monkeypatch):
    """A convergence run (checks every 25 iterations, certificates once the
    residual is small): same termination and iteration count as the graph
    path; iterates within the instance's own rounding-noise amplification
    over 3,000 iterations (the oracle against itself with 1-ulp noise per
    iteration: u0 6.4e-5, dual 1.6e-4 relative, measured on C1)."""
    inst = config_instance("C1")
    a, b = _pair(inst, monkeypatch, max_iter=3000, tol=2e-2, gap_check_every=25)
    assert a.termination == b.termination
    assert a.iterations == b.iterations
    assert rel_err(a.u0, b.u0) <= 1e-3
    assert rel_err(a.dual, b.dual) <= 1e-3
    assert abs(a.objective - b.objective) <= 1e-6 * (1 + abs(b.objective))


def test_dp_warm_start(monkeypatch):
    inst = config_instance("C2")
    y0 = np.random.default_rng(5).standard_normal(inst.n_dual) * 10.0
    out = []
    for dp in (True, False):
        cache = _cache(inst, monkeypatch, dp)
        out.append(solve(inst, SolverConfig(max_iter=60, tol=1e-30, gamma=1 / 2e9, gap_check_every=61),
                         cache=cache, y_init=y0))
    for k in ("primal", "primal_avg", "dual"):
        assert rel_err(getattr(out[0], k), getattr(out[1], k)) <= 1e-10, k


def test_dp_context_fp32_mode(monkeypatch):
    """fp32 mode on a context configured for k_chain_dp runs the four-kernel
    graph (k_chain_dp is fp64-only: measured slower in fp32)."""
    inst = config_instance("C2")
    a, b = _pair(inst, monkeypatch, max_iter=100, tol=1e-30, gamma=1 / 2e9, gap_check_every=101,
                 precision="fp32")
    for k in ("primal_avg", "dual"):
        assert rel_err(getattr(a, k), getattr(b, k)) <= 1e-5, k


def test_dp_iterate_hook_path(monkeypatch):
    """One replay per iteration with host reads in between (debug path)."""
    inst = config_instance("C1")
    seen = []
    out = []
    for dp in (True, False):
        cache = _cache(inst, monkeypatch, dp)
        ys = []
        out.append(solve(inst, SolverConfig(max_iter=12, tol=1e-30, gamma=1 / 2e9, gap_check_every=13),
                         cache=cache, iterate_hook=lambda nu, y, z, za: ys.append(y.copy())))
        seen.append(ys)
    for ya, yb in zip(*seen):
        assert rel_err(ya, yb) <= 1e-10
