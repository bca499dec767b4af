"""Subtree-sharded solve (shard.py) against the one-GPU solve.

The ranks are emulated in one process on one device (LocalCollective): the
shards' kernels never wait on one another; the per-iteration exchange of the
replicated rows' subtree sums happens between launches. k = 0 shards stage-1
subtrees (no exchange); k > 0 replicates the ancestors and exchanges."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import rel_err
from paper_1904_10548_b200 import SolverConfig, factor_step, solve
from paper_1904_10548_b200 import shard
from paper_1904_10548_b200.synthetic import config_instance

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg,size", [("C1", 1), ("C1", 2), ("C1", 4), ("C1", 8), ("C2", 2), ("C2", 4),
                                      ("C3", 8)])
def test_sharded_solve_matches_single_gpu(cfg, size):
    inst = config_instance(cfg)
    conf = SolverConfig(max_iter=60, tol=1e-30, gamma=1.0 / 2e9, gap_check_every=20)
    ref = solve(inst, conf, cache=factor_step(inst))
    res = shard.solve_sharded(inst, conf, size=size)
    assert res.iterations == ref.iterations == 60
    for k in ("u0", "primal", "primal_avg", "dual"):
        assert rel_err(getattr(res, k), getattr(ref, k)) <= 1e-11, k
    assert abs(res.duality_gap - ref.duality_gap) <= 1e-9 * (1 + abs(ref.duality_gap))
    assert abs(res.objective - ref.objective) <= 1e-11 * (1 + abs(ref.objective))


def test_sharded_solve_converges_like_single_gpu():
    inst = config_instance("C1")
    conf = SolverConfig(max_iter=400, tol=1e-3, gamma=1.0 / 2e9, gap_check_every=25)
    ref = solve(inst, conf, cache=factor_step(inst))
    res = shard.solve_sharded(inst, conf, size=4)
    assert res.termination == ref.termination
    assert res.iterations == ref.iterations
    assert rel_err(res.u0, ref.u0) <= 1e-10


def test_sharded_shard_refuses_the_single_gpu_loop():
    inst = config_instance("C1")
    sp = shard.plan(inst, 4)[0]
    sh = shard._Shard(inst, sp)
    with pytest.raises(RuntimeError, match="wmpc_shard_step"):
        sh.ctx.call("wmpc_apg_run", 1)


def test_sharded_solver_reuse_and_u0_only():
    inst = config_instance("C2")
    conf = SolverConfig(max_iter=40, tol=1e-30, gamma=1.0 / 2e9, gap_check_every=41)
    sv = shard.ShardedSolver(inst, size=4)
    a = sv.solve(conf)
    b = sv.solve(conf, results="u0")
    np.testing.assert_array_equal(a.u0, b.u0)
    assert a.duality_gap == b.duality_gap and b.primal is None


@pytest.mark.parametrize("cfg,k", [("C1", 1), ("C2", 2)])
def test_device_exchange_in_graph_single_rank(cfg, k):
    """The NCCL exchange inside the captured iteration graph, on a one-rank
    communicator with a forced shard stage k > 0 (the all-reduce is then the
    identity and the result must equal the plain solve)."""
    inst = config_instance(cfg)
    conf = SolverConfig(max_iter=50, tol=1e-30, gamma=1.0 / 2e9, gap_check_every=25)
    ref = solve(inst, conf, cache=factor_step(inst))
    specs = shard.plan(inst, 1, k=k)
    assert specs[0].n_rep_global > 0
    sv = shard.ShardedSolver(inst, specs=specs, device_exchange=True)
    res = sv.solve(conf)
    for key in ("u0", "primal", "primal_avg", "dual"):
        assert rel_err(getattr(res, key), getattr(ref, key)) <= 1e-11, key
    assert abs(res.duality_gap - ref.duality_gap) <= 1e-9 * (1 + abs(ref.duality_gap))
