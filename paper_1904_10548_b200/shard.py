"""Subtree sharding of one scenario-MPC solve across GPUs.

The dual APG iteration (``solver.py:460-506``) couples tree nodes only along
ancestor paths, so the tree splits by subtrees:

* ``plan`` picks the shallowest stage ``k`` with at least ``G`` nodes and gives
  every rank a contiguous block of stage-``k`` nodes (BFS order) with all their
  descendants. The ancestors of those nodes (stages < k) are **replicated** on
  every rank that shares them; each replicated row is *accounted* (counted in
  global sums, returned in results) by its lowest holder.
* ``k = 0`` (at least G stage-1 nodes): the ranks' problems are independent;
  ranks meet only at the reference's check iterations (max of residual,
  scale, dual change; first non-finite iteration) and in the certificate.
* ``k > 0``: once per iteration the replicated rows need their subtree sums
  from every rank. Each rank writes its partial sums into an exchange buffer
  (``wmpc_shard_step`` phase 0), the buffers are summed across ranks (one
  all-reduce of ``off[k] x 256`` doubles: 1.5 KB per replicated row), and every
  holder finishes the replicated rows identically (phase 1). Replicated
  forward passes, proxes and averages are recomputed redundantly.
* Certificate: global max |Ua| (Dykstra tolerance), element-wise max of the
  per-sweep Dykstra movements (global stop sweep), the dual minimiser with the
  same exchange, and sums of the accounted cost terms.

The collective layer is pluggable: ``TorchCollective`` (one shard per process,
``torch.distributed`` with NCCL or gloo) or ``LocalCollective`` (all shards in
one process on one device, driven in lock step: no kernel ever waits on
another rank, the exchange happens between launches).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as nat
from . import solver as S
from .problem import ProblemInstance

XCOLS = 256  # doubles per replicated row in the exchange buffer


# ------------------------------------------------------------------ planning

@dataclass
class ShardSpec:
    rank: int
    size: int
    k: int                  # shard stage (0-based: 0 = stage-1 subtrees)
    rows: np.ndarray        # global rows held, ascending (BFS order)
    rep_gidx: np.ndarray    # per local row: global replicated index (rows < off[k]) or -1
    acct: np.ndarray        # per local row: 1 if this rank accounts for it
    n_rep_global: int       # replicated rows in the whole tree (= off[k])


def _stage_offsets(instance) -> np.ndarray:
    return np.array([sl.start for sl in instance.stage_slices] + [instance.stage_slices[-1].stop])


def plan(instance, size: int) -> list[ShardSpec]:
    """Partition the non-root rows of ``instance`` over ``size`` ranks."""
    if size < 1:
        raise ValueError("need at least one rank")
    off = _stage_offsets(instance)
    counts = np.diff(off)
    cand = np.flatnonzero(counts >= size)
    if cand.size == 0:
        raise ValueError(f"no stage has {size} nodes to shard over")
    k = int(cand[0])
    n = instance.n_nonroot
    anc = instance.anc_row
    # subtree root (stage-k ancestor) of every row at stage >= k
    root = np.full(n, -1, dtype=np.int64)
    root[off[k]:off[k + 1]] = np.arange(off[k], off[k + 1])
    for s in range(k + 1, len(counts)):
        sl = slice(off[s], off[s + 1])
        root[sl] = root[anc[sl]]
    mu = int(counts[k])
    bounds = [off[k] + (mu * g) // size for g in range(size + 1)]
    holders: dict[int, list[int]] = {}
    specs = []
    for g in range(size):
        own_roots = np.arange(bounds[g], bounds[g + 1])
        own = np.flatnonzero((root >= bounds[g]) & (root < bounds[g + 1]))
        rep = set()
        for r in own_roots:
            a = int(anc[r])
            while a >= 0:
                rep.add(a)
                a = int(anc[a])
        rep_rows = np.array(sorted(rep), dtype=np.int64)
        for r in rep_rows:
            holders.setdefault(int(r), []).append(g)
        rows = np.concatenate([rep_rows, own]).astype(np.int64)
        specs.append(ShardSpec(rank=g, size=size, k=k, rows=rows, rep_gidx=None, acct=None,
                               n_rep_global=int(off[k])))
    for sp in specs:
        rg = np.where(sp.rows < off[k], sp.rows, -1).astype(np.int64)
        acct = np.ones(sp.rows.size, dtype=np.int64)
        for i, r in enumerate(sp.rows):
            if r < off[k]:
                acct[i] = 1 if holders[int(r)][0] == sp.rank else 0
        sp.rep_gidx, sp.acct = rg, acct
    return specs


class ShardInstance(ProblemInstance):
    """The rows ``rows`` (closed under ancestors) of a ProblemInstance, as an
    instance of its own: same model, weights and boundary values; per-node
    arrays sliced; ancestor rows renumbered. Probabilities stay absolute."""

    def __init__(self, parent, rows):  # noqa: D107 - dataclass fields set by hand
        rows = np.asarray(rows, dtype=np.int64)
        self.parent = parent
        self.rows = rows
        self.model, self.tree, self.weights = parent.model, None, parent.weights
        self.p, self.q, self.k = parent.p, parent.q, parent.k
        self.wu = parent.wu
        self.prob = parent.prob[rows].copy()
        self.demand = parent.demand[rows].copy()
        self.price = parent.price[rows].copy()
        self.demand_gd = parent.demand_gd[rows].copy()
        self.econ = parent.econ[rows].copy()
        g2l = np.full(parent.n_nonroot, -1, dtype=np.int64)
        g2l[rows] = np.arange(rows.size)
        a = parent.anc_row[rows]
        la = np.where(a >= 0, g2l[np.maximum(a, 0)], -1)
        if np.any((a >= 0) & (la < 0)):
            raise ValueError("shard rows must be closed under ancestors")
        self.anc_row = la
        off = _stage_offsets(parent)
        cnt = [int(np.count_nonzero((rows >= off[s]) & (rows < off[s + 1]))) for s in range(len(off) - 1)]
        edges = np.concatenate([[0], np.cumsum(cnt)])
        self.stage_slices = [slice(int(x), int(y)) for x, y in zip(edges[:-1], edges[1:])]

    @property
    def n_nonroot(self) -> int:
        return int(self.rows.size)


# --------------------------------------------------------------- collectives

class LocalCollective:
    """All shards in this process; nothing crosses processes."""

    def max(self, x: np.ndarray) -> np.ndarray:
        return x

    def sum(self, x: np.ndarray) -> np.ndarray:
        return x

    def sum_device(self, t) -> None:
        return None

    def gather(self, obj) -> list:
        return [obj]

    def bcast_float(self, v: float) -> float:
        return v


class TorchCollective:
    """One shard per process over ``torch.distributed`` (NCCL or gloo)."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.group = torch, dist, group
        self.nccl = dist.get_backend(group) == "nccl"

    def _reduce(self, x: np.ndarray, op) -> np.ndarray:
        t = self.torch.tensor(np.asarray(x, dtype=np.float64))
        if self.nccl:
            t = t.cuda()
        self.dist.all_reduce(t, op=op, group=self.group)
        return t.cpu().numpy()

    def max(self, x):
        return self._reduce(x, self.dist.ReduceOp.MAX)

    def sum(self, x):
        return self._reduce(x, self.dist.ReduceOp.SUM)

    def sum_device(self, t) -> None:
        if self.nccl:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        else:
            h = t.cpu()
            self.dist.all_reduce(h, op=self.dist.ReduceOp.SUM, group=self.group)
            t.copy_(h)

    def gather(self, obj) -> list:
        out = [None] * self.dist.get_world_size(self.group)
        self.dist.all_gather_object(out, obj, group=self.group)
        return out

    def bcast_float(self, v: float) -> float:
        return float(self.max(np.array([v]))[0])


# ------------------------------------------------------------------ the solve

class _Shard:
    def __init__(self, instance, spec: ShardSpec):
        import torch
        self.spec = spec
        self.inst = ShardInstance(instance, spec.rows)
        self.cache = S._factor(self.inst, None, private=True, min_branch_stage=spec.k)
        self.ctx = self.cache._bind()
        self.ctx.call("wmpc_shard_setup", int(spec.k), int(spec.n_rep_global), nat.ptr(spec.rep_gidx),
                      nat.ptr(spec.acct))
        self.xbuf = torch.zeros(max(spec.n_rep_global, 1) * XCOLS, dtype=torch.float64,
                                device=f"cuda:{S._DEVICE}")
        self.ctx.call("wmpc_shard_set_exchange", nat.C.c_void_p(self.xbuf.data_ptr()))


def _exchange(shards, comm) -> None:
    """Sum the exchange buffers over every shard of every rank."""
    import torch
    for sh in shards:
        sh.ctx.call("wmpc_sync")
    total = shards[0].xbuf.clone()
    for sh in shards[1:]:
        total += sh.xbuf
    comm.sum_device(total)
    for sh in shards:
        sh.xbuf.copy_(total)
    torch.cuda.synchronize()


def _check(shards, comm):
    vals = []
    for sh in shards:
        r, s, dc = np.zeros(1), np.zeros(1), np.zeros(1)
        bad = nat.C.c_int(-1)
        sh.ctx.call("wmpc_apg_check", nat.ptr(r), nat.ptr(s), nat.ptr(dc), nat.C.byref(bad))
        vals.append([r[0], s[0], dc[0], -bad.value if bad.value >= 0 else -np.inf])
    v = comm.max(np.max(np.array(vals), axis=0))
    if np.isfinite(v[3]):
        raise RuntimeError(f"solver produced a non-finite iterate at nu={int(-v[3])}")
    return float(v[0]), float(v[1]), float(v[2])


def _certificate(shards, comm, instance):
    am = np.array([0.0])
    for sh in shards:
        a = np.zeros(1)
        sh.ctx.call("wmpc_cert_absmax", nat.ptr(a))
        am = np.maximum(am, a)
    tol = 1e-13 * (1.0 + float(comm.max(am)[0]))  # problem.py:238
    sweeps = 500
    mv = np.zeros(sweeps)
    for sh in shards:
        m = np.zeros(sweeps)
        sh.ctx.call("wmpc_cert_dykstra", sweeps, nat.ptr(m))
        mv = np.maximum(mv, m)
    mv = comm.max(mv)
    stop = np.flatnonzero(mv <= tol)
    K = int(stop[0]) + 1 if stop.size else sweeps
    for sh in shards:
        sh.ctx.call("wmpc_shard_dual_eval", 0)
    if shards[0].spec.k > 0:
        _exchange(shards, comm)
    for sh in shards:
        sh.ctx.call("wmpc_shard_dual_eval", 1)
    terms = np.zeros(10)
    viol = 0.0
    for sh in shards:
        t = np.zeros(10)
        sh.ctx.call("wmpc_cert_terms", K, nat.ptr(t))
        terms[:9] += t[:9]
        viol = max(viol, t[9])
    terms = comm.sum(terms)
    viol = float(comm.max(np.array([viol]))[0])
    w = instance.weights
    primal = terms[0] + (w.w_x * terms[2] + w.w_s * terms[3])
    gc = np.inf if viol > 0.0 else terms[8]
    dual = (terms[4] + terms[5]) - gc
    return float(primal - dual), float(primal)


def _read(shards, comm, instance, averaged: bool):
    m = instance.model
    nu, nt = m.n_inputs, m.n_tanks
    P, W = nu + nt, 2 * nt + nu
    parts = []
    for sh in shards:
        _, z, za, y = S._read(sh.ctx, sh.inst, averaged, u0=False)
        keep = sh.spec.acct.astype(bool)
        parts.append((sh.spec.rows[keep], z.reshape(-1, P)[keep], za.reshape(-1, P)[keep],
                      y.reshape(-1, W)[keep]))
    allp = [p for group in comm.gather(parts) for p in group]
    n = instance.n_nonroot
    Z, ZA, Y = np.empty((n, P)), np.empty((n, P)), np.empty((n, W))
    seen = np.zeros(n, dtype=bool)
    for rows, z, za, y in allp:
        Z[rows], ZA[rows], Y[rows] = z, za, y
        seen[rows] = True
    if not seen.all():
        raise RuntimeError("sharded read: some rows were accounted by no rank")
    s1 = instance.stage_slices[0]
    src = ZA if averaged else Z
    u0 = np.empty(nu)
    nat.load().wmpc_u0_rows(nu, s1.stop - s1.start, nat.ptr(np.ascontiguousarray(instance.prob[s1])),
                            nat.ptr(np.ascontiguousarray(src[s1, :nu])), nat.ptr(nat.f64(m.u_min)),
                            nat.ptr(nat.f64(m.u_max)), nat.ptr(u0))
    return u0, Z.reshape(-1), ZA.reshape(-1), Y.reshape(-1)


def solve_sharded(instance, config: S.SolverConfig | None = None, specs: list[ShardSpec] | None = None,
                  comm=None, size: int | None = None) -> S.SolverResult:
    """``solve`` (solver.py:398-543) over subtree shards.

    ``specs``: the shards this process runs (default: all of ``plan(instance,
    size)``, emulated in this process). ``comm``: the cross-process collective
    (default ``LocalCollective``). Every rank returns the full result.
    """
    import time
    config = config or S.SolverConfig()
    comm = comm or LocalCollective()
    if specs is None:
        specs = plan(instance, size or 1)
    shards = [_Shard(instance, sp) for sp in specs]
    if specs[0].k > 0:  # replicated rows' R spans ranks (solver.py:269-274)
        for sh in shards:
            sh.ctx.call("wmpc_shard_fix_R", 0)
        _exchange(shards, comm)
        for sh in shards:
            sh.ctx.call("wmpc_shard_fix_R", 1)
    gamma = config.gamma
    lipschitz = None
    if gamma is None:  # the global operator norm, estimated once on the whole tree
        lam = S.estimate_lipschitz(S.factor_step(instance), instance) if specs[0].rank == 0 else 0.0
        lipschitz = comm.bcast_float(lam)
        gamma = 1.0 / lipschitz
    theta = S.theta_sequence(config.max_iter)
    beta = S._beta_table(theta)
    for sh in shards:
        S._upload_bounds(sh.ctx, sh.inst)
        sh.ctx.call("wmpc_apg_begin", float(gamma), int(config.max_iter), nat.ptr(theta), nat.ptr(beta))
    exchange = specs[0].k > 0
    started = time.perf_counter()
    residual = dchange = gap = objective = float("inf")
    iterations, termination = config.max_iter, "max_iter"
    gce = config.gap_check_every
    done = 0
    while done < config.max_iter:
        step = min(gce - (done % gce), config.max_iter - done)
        if exchange:
            for _ in range(step):
                for sh in shards:
                    sh.ctx.call("wmpc_shard_step", 0)
                _exchange(shards, comm)
                for sh in shards:
                    sh.ctx.call("wmpc_shard_step", 1)
        else:
            for sh in shards:
                sh.ctx.call("wmpc_apg_run", int(step))
        done += step
        if done % gce == 0:
            residual, scale, dchange = _check(shards, comm)
            if residual <= config.tol * (1.0 + scale):
                gap, objective = _certificate(shards, comm, instance)
                if gap <= config.tol * (1.0 + abs(objective)):
                    iterations, termination = done, "converged"
                    break
    if termination == "max_iter":
        residual, scale, dchange = _check(shards, comm)
        gap, objective = _certificate(shards, comm, instance)
    elapsed = time.perf_counter() - started
    u0, primal, primal_avg, dual = _read(shards, comm, instance, config.averaged_primal)
    return S.SolverResult(u0=u0, primal=primal, primal_avg=primal_avg, dual=dual, iterations=iterations,
                          termination=termination, primal_residual=residual, dual_change=dchange,
                          duality_gap=gap, objective=objective, solve_time_s=elapsed, gamma=gamma,
                          lipschitz=lipschitz)
