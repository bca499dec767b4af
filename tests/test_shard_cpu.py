"""Subtree sharding host logic on the CPU: the partition plan,
the shard sub-instances and the torch.distributed collective layer over gloo
with two processes (the path bench.py/torchrun uses with NCCL on GPUs)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from conftest import make_model, make_instance  # noqa: F401  (shared builders)
from paper_1904_10548_b200 import shard
from paper_1904_10548_b200.synthetic import config_instance


def _ancestors(inst, r):
    out = []
    a = int(inst.anc_row[r])
    while a >= 0:
        out.append(a)
        a = int(inst.anc_row[a])
    return out


@pytest.mark.parametrize("cfg,size", [("C1", 1), ("C1", 2), ("C1", 3), ("C1", 4), ("C1", 8),
                                      ("C2", 2), ("C2", 4), ("C2", 8), ("C3", 4), ("C3", 8)])
def test_plan_covers_every_row_once(cfg, size):
    inst = config_instance(cfg)
    specs = shard.plan(inst, size)
    off = [sl.start for sl in inst.stage_slices] + [inst.n_nonroot]
    counts = np.diff(off)
    k = specs[0].k
    assert counts[k] >= size and (k == 0 or counts[k - 1] < size)   # shallowest stage with >= G nodes
    acct = np.zeros(inst.n_nonroot, dtype=int)
    for sp in specs:
        rows = set(sp.rows.tolist())
        assert np.all(np.diff(sp.rows) > 0)                       # ascending = BFS order kept
        for r in sp.rows:                                           # closed under ancestors
            assert set(_ancestors(inst, int(r))) <= rows
        rep = sp.rows < off[k]
        assert np.array_equal(sp.rep_gidx >= 0, rep)
        assert np.array_equal(sp.rep_gidx[rep], sp.rows[rep])
        assert np.all(sp.acct[~rep] == 1)
        acct[sp.rows[sp.acct == 1]] += 1
    assert np.all(acct == 1)                                       # every row accounted exactly once
    own = [sp.rows[sp.rows >= off[k]] for sp in specs]
    assert sum(o.size for o in own) == inst.n_nonroot - off[k]     # subtrees disjoint
    sizes = [int(np.count_nonzero((o >= off[k]) & (o < off[k + 1]))) for o in own]
    assert max(sizes) - min(sizes) <= 1                            # balanced stage-k blocks


def test_shard_instance_slices_parent():
    inst = config_instance("C2")
    sp = shard.plan(inst, 4)[2]
    si = shard.ShardInstance(inst, sp.rows)
    assert si.n_nonroot == sp.rows.size
    assert si.n_dual == sp.rows.size * (2 * 63 + 114)
    np.testing.assert_array_equal(si.prob, inst.prob[sp.rows])
    np.testing.assert_array_equal(si.econ, inst.econ[sp.rows])
    np.testing.assert_array_equal(si.demand_gd, inst.demand_gd[sp.rows])
    a = si.anc_row
    ok = a >= 0
    np.testing.assert_array_equal(sp.rows[a[ok]], inst.anc_row[sp.rows[ok]])
    assert np.all(inst.anc_row[sp.rows[~ok]] == -1)
    lens = [s.stop - s.start for s in si.stage_slices]
    assert sum(lens) == si.n_nonroot and lens[0] == 1 and lens[1] == 1 and lens[2] == 2


def test_plan_rejects_too_many_ranks():
    with pytest.raises(ValueError, match="no stage"):
        shard.plan(config_instance("C1"), 16)


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = shard.TorchCollective()
        mx = comm.max(np.array([rank + 0.5, -rank, np.inf if rank == 1 else 0.0]))
        sm = comm.sum(np.array([1.0, rank, 2.0 ** -60 * rank]))
        t = torch.full((4,), float(rank + 1), dtype=torch.float64)
        comm.sum_device(t)
        g = comm.gather((rank, np.arange(rank + 1)))
        b = comm.bcast_float(3.25 if rank == 0 else 0.0)
        q.put((rank, mx.tolist(), sm.tolist(), t.tolist(), [(r, a.tolist()) for r, a in g], b))
    finally:
        dist.destroy_process_group()


def test_torch_collective_gloo_two_ranks():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict()
    for _ in range(2):
        r, *vals = q.get(timeout=120)
        out[r] = vals
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        mx, sm, t, g, b = out[r]
        assert mx == [1.5, 0.0, np.inf]
        assert sm == [2.0, 1.0, 2.0 ** -60]
        assert t == [3.0] * 4
        assert g == [(0, [0]), (1, [0, 1])]
        assert b == 3.25
