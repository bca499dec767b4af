"""k_chain_dp with segmented chains (DpArgs.seg_m, csrc/wmpc_dp.cuh): two warps
per chain walk the upper and lower rows at the same time; the upper warp
stores its rows' L without the lower segment's contribution and applies the
per-chain correction L_t = base_t + aux_t (c0 + n_t c1), written by whichever
warp of the pair finishes second (a per-chain counter, no waiting). Same quantities as the reference recursion
(solver.py:242-290) in real arithmetic, different rounding: 1e-10 against
the graph iteration, 1e-8 against the oracle; bit-identical under
reordering of the pair's completion (PDL on/off, repeated runs)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import rel_err
from oracle import port
from paper_1904_10548_b200 import SolverConfig, solve
from paper_1904_10548_b200 import _native as nat
from paper_1904_10548_b200 import solver as S
from paper_1904_10548_b200.synthetic import barcelona_instance, config_instance

pytestmark = pytest.mark.gpu


def _cache(inst, monkeypatch, mode):
    """mode: None = graph iteration, 0 = whole-chain k_chain_dp, m > 0 = upper
    segment of m rows, 'seg' = the default split."""
    monkeypatch.setenv("WMPC_DP", "0" if mode is None else "1")
    monkeypatch.delenv("WMPC_DP_SEGM", raising=False)
    monkeypatch.setenv("WMPC_DP_SEG", "1" if mode not in (None, 0) else "0")
    if isinstance(mode, int) and mode > 0:
        monkeypatch.setenv("WMPC_DP_SEGM", str(mode))
    cache = S._factor(inst, None, private=True)
    info = nat.path_info(cache._bind())
    assert info["fused_dp"] == (0 if mode is None else 1), info
    if mode == "seg":
        assert info["dp_segm"] > 0, info
    elif isinstance(mode, int):
        assert info["dp_segm"] == mode, info
    return cache


def _solve(inst, monkeypatch, mode, **cfg):
    return solve(inst, SolverConfig(**cfg), cache=_cache(inst, monkeypatch, mode))


FIXED = dict(max_iter=120, tol=1e-30, gamma=1 / 2e9, gap_check_every=121)


def _close(a, b, tol=1e-10):
    for k in ("u0", "primal", "primal_avg", "dual"):
        assert rel_err(getattr(a, k), getattr(b, k)) <= tol, k
    assert abs(a.duality_gap - b.duality_gap) <= 10 * tol * (1 + abs(b.duality_gap))
    assert abs(a.objective - b.objective) <= tol * (1 + abs(b.objective))


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_segmented_matches_graph_iteration(name, monkeypatch):
    inst = config_instance(name)
    _close(_solve(inst, monkeypatch, "seg", **FIXED), _solve(inst, monkeypatch, None, **FIXED))


def test_segment_split_points(monkeypatch):
    """Upper segments of 1 row, the middle and N - 1 rows (C2: N = 17)."""
    inst = config_instance("C2")
    ref = _solve(inst, monkeypatch, None, **FIXED)
    n = inst.tree.horizon - nat.path_info(_cache(inst, monkeypatch, 0)._bind())["kstar"]
    for m in (1, n // 2, n - 1):
        _close(_solve(inst, monkeypatch, m, **FIXED), ref)


def test_segmented_uneven_tree_vs_oracle(monkeypatch):
    inst = barcelona_instance([3, 1, 2, 1], seed=3, horizon=12)
    gamma, it = 1.0 / 3e9, 80
    res = _solve(inst, monkeypatch, "seg", max_iter=it, tol=1e-30, gamma=gamma, gap_check_every=it + 1)
    ref = port.apg_solve(inst, gamma, max_iter=it, tol=1e-30, gap_check_every=it + 1,
                         reference_cost_accounting=False)
    for k in ("u0", "primal", "primal_avg", "dual"):
        assert rel_err(getattr(res, k), getattr(ref, k)) <= 1e-8, k
    assert abs(res.objective - ref.objective) <= 1e-8 * (1 + abs(ref.objective))


def _state(ctx, inst, iters, chunks, cert):
    S._upload_bounds(ctx, inst)
    th = S.theta_sequence(iters)
    be = S._beta_table(th)
    ctx.call("wmpc_apg_begin", 1.0 / 2e9, iters, nat.ptr(th), nat.ptr(be))
    for _ in range(chunks):
        ctx.call("wmpc_apg_run", iters // chunks)
        if cert:
            S._certificate(ctx)
    return S._read(ctx, inst, True)


def test_segmented_certificates_between_chunks(monkeypatch):
    """The certificate between chunks leaves the carried state (base rows,
    corrections, aggregates, pair counters) intact: bit-identical."""
    inst = config_instance("C2")
    ca, cb = _cache(inst, monkeypatch, "seg"), _cache(inst, monkeypatch, "seg")  # held: they own the contexts
    a = _state(ca._bind(), inst, 200, 8, False)
    b = _state(cb._bind(), inst, 200, 8, True)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)


def test_segmented_handshake_is_deterministic(monkeypatch):
    """Either warp of a pair may apply the correction (whichever finishes
    second): the arithmetic never depends on which, with or without
    programmatic dependent launch."""
    inst = config_instance("C3")
    outs = []
    for pdl in (1, 1, 0):
        cache = _cache(inst, monkeypatch, "seg")
        ctx = cache._bind()
        ctx.call("wmpc_set_pdl", pdl)
        outs.append(_state(ctx, inst, 150, 3, False))
    for other in outs[1:]:
        for x, y in zip(outs[0], other):
            np.testing.assert_array_equal(x, y)


def test_segmented_warm_start(monkeypatch):
    inst = config_instance("C2")
    y0 = np.random.default_rng(5).standard_normal(inst.n_dual) * 10.0
    out = [solve(inst, SolverConfig(max_iter=60, tol=1e-30, gamma=1 / 2e9, gap_check_every=61),
                 cache=_cache(inst, monkeypatch, mode), y_init=y0) for mode in ("seg", None)]
    for k in ("primal", "primal_avg", "dual"):
        assert rel_err(getattr(out[0], k), getattr(out[1], k)) <= 1e-10, k


def test_segmented_convergence_run(monkeypatch):
    inst = config_instance("C1")
    cfg = dict(max_iter=3000, tol=2e-2, gap_check_every=25)
    a, b = _solve(inst, monkeypatch, "seg", **cfg), _solve(inst, monkeypatch, None, **cfg)
    assert a.termination == b.termination
    assert a.iterations == b.iterations
    assert rel_err(a.u0, b.u0) <= 1e-3
    assert abs(a.objective - b.objective) <= 1e-6 * (1 + abs(b.objective))
