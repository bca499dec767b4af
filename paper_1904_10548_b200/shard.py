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


def plan(instance, size: int, k: int | None = None) -> list[ShardSpec]:
    """Partition the non-root rows of ``instance`` over ``size`` ranks (shard
    stage ``k``: default the shallowest with >= size nodes)."""
    if size < 1:
        raise ValueError("need at least one rank")
    off = _stage_offsets(instance)
    counts = np.diff(off)
    cand = np.flatnonzero(counts >= size)
    if cand.size == 0:
        raise ValueError(f"no stage has {size} nodes to shard over")
    if k is None:
        k = int(cand[0])
    elif counts[k] < size:
        raise ValueError(f"stage {k} has fewer than {size} nodes")
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

    def bcast_bytes(self, b: bytes) -> bytes:
        return b


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

    def bcast_bytes(self, b: bytes) -> bytes:
        obj = [b]
        self.dist.broadcast_object_list(obj, src=0, group=self.group)
        return obj[0]


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


def _certificate(shards, comm, instance, exchange):
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
        exchange()
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


def _u0_only(shards, comm, instance, averaged: bool) -> np.ndarray:
    """u0 from the stage-1 rows alone (gathered in global order)."""
    m = instance.model
    nu = m.n_inputs
    s1 = instance.stage_slices[0]
    rows_vals = []
    for sh in shards:
        _, z, za, _ = S._read(sh.ctx, sh.inst, averaged, u0=False, primal=not averaged, avg=averaged, dual=False)
        src = (za if averaged else z).reshape(sh.inst.n_nonroot, -1)
        keep = sh.spec.acct.astype(bool) & (sh.spec.rows < s1.stop)
        rows_vals.append((sh.spec.rows[keep], src[keep, :nu]))
    U1 = np.empty((s1.stop - s1.start, nu))
    for rows, vals in [p for group in comm.gather(rows_vals) for p in group]:
        U1[rows - s1.start] = vals
    u0 = np.empty(nu)
    nat.load().wmpc_u0_rows(nu, U1.shape[0], nat.ptr(np.ascontiguousarray(instance.prob[s1])), nat.ptr(U1),
                            nat.ptr(nat.f64(m.u_min)), nat.ptr(nat.f64(m.u_max)), nat.ptr(u0))
    return u0


class ShardedSolver:
    """The shards one process runs (all of them when emulating), built once:
    factor step, shard setup and the replicated rows' R; ``solve`` may then be
    called repeatedly (bench.py)."""

    def __init__(self, instance, specs: list[ShardSpec] | None = None, comm=None, size: int | None = None,
                 device_exchange: bool | None = None):
        self.instance = instance
        self.comm = comm or LocalCollective()
        self.specs = specs if specs is not None else plan(instance, size or 1)
        self.shards = [_Shard(instance, sp) for sp in self.specs]
        if device_exchange is None:
            device_exchange = isinstance(self.comm, TorchCollective) and self.comm.nccl
        # NCCL on the solver stream: the exchange sits inside the iteration graph
        self.device_exchange = bool(device_exchange) and self.specs[0].k > 0
        if self.device_exchange:
            if len(self.shards) != 1:
                raise ValueError("the device exchange runs one shard per process")
            sp = self.specs[0]
            uid = (nat.C.c_char * 128)()
            if sp.rank == 0 and nat.load().wmpc_nccl_unique_id(uid) != nat.WMPC_OK:
                raise RuntimeError("ncclGetUniqueId failed")
            raw = self.comm.bcast_bytes(bytes(uid))
            uid = (nat.C.c_char * 128).from_buffer_copy(raw)
            self.shards[0].ctx.call("wmpc_shard_nccl_init", uid, int(sp.size), int(sp.rank))
        if self.specs[0].k > 0:  # replicated rows' R spans ranks (solver.py:269-274)
            for sh in self.shards:
                sh.ctx.call("wmpc_shard_fix_R", 0)
            self._exchange()
            for sh in self.shards:
                sh.ctx.call("wmpc_shard_fix_R", 1)
        self.lipschitz = None

    def _exchange(self) -> None:
        if self.device_exchange:
            self.shards[0].ctx.call("wmpc_shard_exchange")
        else:
            _exchange(self.shards, self.comm)

    def solve(self, config: S.SolverConfig | None = None, results: str = "all") -> S.SolverResult:
        """``solve`` (solver.py:398-543) over the shards; every rank returns the
        full result (``results="u0"``: only u0 and the scalars).

        With ``config.gamma`` None the Lipschitz constant is estimated once,
        on rank 0, over the whole tree (factor step + device power iteration
        on one GPU) and broadcast: a tree that does not fit one GPU needs an
        explicit ``config.gamma`` (or a precomputed ``self.lipschitz``)."""
        import time
        config = config or S.SolverConfig()
        comm, shards, instance = self.comm, self.shards, self.instance
        gamma = config.gamma
        lipschitz = self.lipschitz
        if gamma is None:  # the global operator norm, estimated once on the whole tree
            if lipschitz is None:
                lam = S.estimate_lipschitz(S.factor_step(instance), instance) if self.specs[0].rank == 0 else 0.0
                lipschitz = self.lipschitz = comm.bcast_float(lam)
            gamma = 1.0 / lipschitz
        theta = S.theta_sequence(config.max_iter)
        beta = S._beta_table(theta)
        for sh in shards:
            S._upload_bounds(sh.ctx, sh.inst)
            sh.ctx.call("wmpc_apg_begin", float(gamma), int(config.max_iter), nat.ptr(theta), nat.ptr(beta))
        exchange = self.specs[0].k > 0
        started = time.perf_counter()
        residual = dchange = gap = objective = float("inf")
        iterations, termination = config.max_iter, "max_iter"
        gce = config.gap_check_every
        done = 0
        while done < config.max_iter:
            step = min(gce - (done % gce), config.max_iter - done)
            if exchange and not self.device_exchange:
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
                    gap, objective = _certificate(shards, comm, instance, self._exchange)
                    if gap <= config.tol * (1.0 + abs(objective)):
                        iterations, termination = done, "converged"
                        break
        if termination == "max_iter":
            residual, scale, dchange = _check(shards, comm)
            gap, objective = _certificate(shards, comm, instance, self._exchange)
        elapsed = time.perf_counter() - started
        if results == "u0":
            u0 = _u0_only(shards, comm, instance, config.averaged_primal)
            primal = primal_avg = dual = None
        else:
            u0, primal, primal_avg, dual = _read(shards, comm, instance, config.averaged_primal)
        return S.SolverResult(u0=u0, primal=primal, primal_avg=primal_avg, dual=dual, iterations=iterations,
                              termination=termination, primal_residual=residual, dual_change=dchange,
                              duality_gap=gap, objective=objective, solve_time_s=elapsed, gamma=gamma,
                              lipschitz=lipschitz)


def solve_sharded(instance, config: S.SolverConfig | None = None, specs: list[ShardSpec] | None = None,
                  comm=None, size: int | None = None) -> S.SolverResult:
    """``solve`` (solver.py:398-543) over subtree shards.

    ``specs``: the shards this process runs (default: all of ``plan(instance,
    size)``, emulated in this process). ``comm``: the cross-process collective
    (default ``LocalCollective``). Every rank returns the full result.
    """
    return ShardedSolver(instance, specs=specs, comm=comm, size=size).solve(config)
