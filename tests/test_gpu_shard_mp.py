"""Subtree-sharded solves across processes: two ranks in
two processes on the one GPU of the box, torch.distributed over gloo
(``shard.TorchCollective``): the per-iteration exchange of the replicated
rows' partial sums goes through the host, so no kernel ever waits on another
rank's kernel. Each rank runs ``ShardedSolver`` on its own shard; rank 0's
full gathered result is compared with the one-GPU solve (<= 1e-11, the
exchange sums the ranks' partial sums in a different order than one GPU).
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from conftest import ROOT, rel_err

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank(rank, world, port, cfg, k, iters, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1904_10548_b200 import SolverConfig, shard
        from paper_1904_10548_b200.synthetic import config_instance
        inst = config_instance(cfg)
        specs = shard.plan(inst, world, k=k)
        sv = shard.ShardedSolver(inst, specs=[specs[rank]], comm=shard.TorchCollective())
        res = sv.solve(SolverConfig(max_iter=iters, tol=1e-30, gamma=1 / 2e9, gap_check_every=iters + 1))
        if rank == 0:
            q.put({k2: np.asarray(getattr(res, k2)) for k2 in ("u0", "primal", "primal_avg", "dual")} |
                  {"gap": res.duality_gap, "obj": res.objective, "iters": res.iterations})
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg,k", [("C2", 2), ("C3", 1), ("C3", 0)])
def test_two_process_sharded_solve_matches_one_gpu(cfg, k):
    import torch.multiprocessing as mp
    from paper_1904_10548_b200 import SolverConfig, solve
    from paper_1904_10548_b200.synthetic import config_instance
    iters = 60
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, cfg, k, iters, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    inst = config_instance(cfg)
    ref = solve(inst, SolverConfig(max_iter=iters, tol=1e-30, gamma=1 / 2e9, gap_check_every=iters + 1))
    assert got["iters"] == iters
    for k2 in ("u0", "primal", "primal_avg", "dual"):
        assert rel_err(got[k2], getattr(ref, k2)) <= 1e-11, k2
    assert abs(got["gap"] - ref.duality_gap) <= 1e-9 * (1 + abs(ref.duality_gap))
    assert abs(got["obj"] - ref.objective) <= 1e-11 * (1 + abs(ref.objective))
