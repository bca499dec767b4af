"""Shapes beyond the uniform Barcelona benchmark trees:
* a non-uniform tree (random 1..k children with unequal probabilities over
  the branching stages, the shape of the reference's fan-to-tree reduction,
  tree.py:320-392), on the default kernels and on k_chain_dp;
* a network whose flows join two mixing nodes (E E^T not diagonal, rows of
  K = (E E^T)^{-1} E 40 wide): the ELL graph path declines it and the
  structured persistent kernel (or the general path) runs;
all against the oracle at the north_star's 1e-8 after fixed iterations."""

from __future__ import annotations

import pytest

from conftest import rel_err
from oracle import port
from paper_1904_10548_b200 import SolverConfig, solve
from paper_1904_10548_b200 import _native as nat
from paper_1904_10548_b200 import solver as S
from paper_1904_10548_b200.synthetic import barcelona_instance, fan_like_instance

pytestmark = pytest.mark.gpu


def _vs_oracle(inst, cache, it=80, gamma=1 / 3e9):
    res = solve(inst, SolverConfig(max_iter=it, tol=1e-30, gamma=gamma, gap_check_every=it + 1), cache=cache)
    ref = port.apg_solve(inst, gamma, max_iter=it, tol=1e-30, gap_check_every=it + 1,
                         reference_cost_accounting=False)
    for k in ("u0", "primal", "primal_avg", "dual"):
        assert rel_err(getattr(res, k), getattr(ref, k)) <= 1e-8, k
    assert abs(res.objective - ref.objective) <= 1e-8 * (1 + abs(ref.objective))
    assert abs(res.duality_gap - ref.duality_gap) <= 1e-8 * (1 + abs(ref.duality_gap))


@pytest.mark.parametrize("mode", ["graph", "dp", "dp-segmented"])
def test_non_uniform_tree_vs_oracle(mode, monkeypatch):
    inst = fan_like_instance(seed=1, leaves_target=48, branching_stages=3, max_children=4, horizon=10)
    monkeypatch.setenv("WMPC_DP", "0" if mode == "graph" else "1")
    monkeypatch.setenv("WMPC_DP_SEG", "1" if mode == "dp-segmented" else "0")
    cache = S._factor(inst, None, private=True)
    info = nat.path_info(cache._bind())
    assert info["fast_path"] == 300 and info["fused_dp"] == int(mode != "graph"), info
    assert (info["dp_segm"] > 0) == (mode == "dp-segmented"), info
    _vs_oracle(inst, cache)


def test_non_uniform_c3_scale_default_path_vs_graph(monkeypatch):
    """A fan-like tree of ~400 scenarios (2-3 chains per SM: the segmented
    k_chain_dp by default) against the graph iteration after 150 iterations."""
    inst = fan_like_instance(seed=2, leaves_target=400, branching_stages=5, max_children=5)
    out, infos = [], []
    for env in ({}, {"WMPC_DP": "0"}):
        for k in ("WMPC_DP", "WMPC_DP_SEG"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        cache = S._factor(inst, None, private=True)
        infos.append(nat.path_info(cache._bind()))
        out.append(solve(inst, SolverConfig(max_iter=150, tol=1e-30, gamma=1 / 3e9, gap_check_every=151),
                         cache=cache))
    assert infos[1]["fused_dp"] == 0, infos
    for k in ("u0", "primal", "primal_avg", "dual"):
        assert rel_err(getattr(out[0], k), getattr(out[1], k)) <= 1e-10, (k, infos[0])


def test_coupled_mixing_nodes_vs_oracle():
    inst = barcelona_instance([2, 2, 2], mixing_links=8)
    cache = S._factor(inst, None, private=True)
    info = nat.path_info(cache._bind())
    assert info["fast_path"] != 300, info  # wide K rows: not the ELL graph path
    _vs_oracle(inst, cache, it=60)


@pytest.mark.parametrize("seed", [3, 4, 5])
@pytest.mark.parametrize("mode", ["dp", "dp-segmented"])
def test_random_trees_dp_modes_vs_graph(seed, mode, monkeypatch):
    """Random non-uniform trees (1..5 children over 4 branching stages, ragged
    chain counts per parent) through the forced k_chain_dp modes against the
    graph iteration: 100 iterations, 1e-10."""
    inst = fan_like_instance(seed=seed, leaves_target=150, branching_stages=4, max_children=5, horizon=14)
    out = []
    for env in ({"WMPC_DP": "1", "WMPC_DP_SEG": "1" if mode == "dp-segmented" else "0"}, {"WMPC_DP": "0"}):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        cache = S._factor(inst, None, private=True)
        info = nat.path_info(cache._bind())
        if env["WMPC_DP"] == "1":
            assert info["fused_dp"] == 1 and (info["dp_segm"] > 0) == (mode == "dp-segmented"), info
        out.append(solve(inst, SolverConfig(max_iter=100, tol=1e-30, gamma=1 / 3e9, gap_check_every=101),
                         cache=cache))
    for k in ("u0", "primal", "primal_avg", "dual"):
        assert rel_err(getattr(out[0], k), getattr(out[1], k)) <= 1e-10, k


def test_1024_chain_default_whole_chain_dp_vs_graph(monkeypatch):
    """3.5-8 chains per SM: k_chain_dp with one warp per whole chain by default
    ([4,4,4,4,2,2], 1,024 chains), against the graph iteration."""
    inst = barcelona_instance([4, 4, 4, 4, 2, 2], seed=2)
    out, infos = [], []
    for env in ({}, {"WMPC_DP": "0"}):
        for k in ("WMPC_DP", "WMPC_DP_SEG", "WMPC_DP_SEGM"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        cache = S._factor(inst, None, private=True)
        infos.append(nat.path_info(cache._bind()))
        out.append(solve(inst, SolverConfig(max_iter=100, tol=1e-30, gamma=1 / 3e9, gap_check_every=101),
                         cache=cache))
    assert infos[0]["fused_dp"] == 1 and infos[0]["dp_segm"] == 0 and infos[1]["fused_dp"] == 0, infos
    for k in ("u0", "primal", "primal_avg", "dual"):
        assert rel_err(getattr(out[0], k), getattr(out[1], k)) <= 1e-10, k
