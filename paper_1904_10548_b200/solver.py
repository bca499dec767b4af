"""Drop-in GPU replacement of ``watermpc.solver``.

Same public names, signatures, dataclass fields, error types and messages as
``/root/reference/pkg/src/watermpc/solver.py``. Host code does
only what the reference does once per structure on tiny matrices — the
null-space basis and the H-stage recursion for ``T_s, D_s, Lam_s, Pi_s``
(LAPACK, 24 x 114^3 flops) — and everything per node or per iteration runs in
``libwmpc.so`` on the GPU:

* per-node factor data ``u_part``, ``e_offset`` (solver.py:206-225);
* the dual gradient (solver.py:242-306), power iteration (326-387);
* the APG loop, CUDA-graph replayed with every iterate resident in HBM
  (398-516), the certificate (449-457) and ``u0`` (525-528).

Instances may be this package's ``ProblemInstance`` or the reference's: only
attributes are read (duck typing).
"""

from __future__ import annotations

import time
import warnings
import weakref
from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from . import _native as nat

IterateHook = Callable[[int, np.ndarray, np.ndarray, np.ndarray], None]


@dataclass
class SolverConfig:
    """Iteration budget, tolerance and step size (solver.py:51-79)."""

    max_iter: int = 20000
    tol: float = 5e-2
    gamma: float | None = None
    averaged_primal: bool = True
    threads: int = 1  # accepted for API parity; the GPU path ignores it
    gap_check_every: int = 25
    # "fp64" (the reference's arithmetic) or "fp32": dual-gradient kernels in
    # fp32, dual iterate / prox / certificate in fp64 (own tolerance; GPU only)
    precision: str = "fp64"

    def __post_init__(self) -> None:
        if self.max_iter < 1:
            raise ValueError("max_iter must be at least 1")
        if self.tol <= 0:
            raise ValueError("tol must be positive")
        if self.gamma is not None and self.gamma <= 0:
            raise ValueError("gamma must be positive when given")
        if self.threads < 1:
            raise ValueError("threads must be at least 1")
        if self.gap_check_every < 1:
            raise ValueError("gap_check_every must be at least 1")
        if self.precision not in ("fp64", "fp32"):
            raise ValueError("precision must be 'fp64' or 'fp32'")


@dataclass
class SolverResult:
    """Control action plus iterate information (solver.py:82-98)."""

    u0: np.ndarray
    primal: np.ndarray
    primal_avg: np.ndarray
    dual: np.ndarray
    iterations: int
    termination: str
    primal_residual: float
    dual_change: float
    duality_gap: float
    objective: float
    solve_time_s: float
    gamma: float
    lipschitz: float | None


_DEVICE = 0


def set_device(ordinal: int) -> None:
    """CUDA device used for contexts created from now on (one per rank)."""
    global _DEVICE
    _DEVICE = int(ordinal)


class _DeviceTree:
    """One native context per tree structure (signature), shared by every
    FactorCache built on it; each cache owns its per-node state (``NodeSet``)
    and binds it before use — a pointer swap, no copies."""

    def __init__(self, instance):
        m = instance.model
        self.ctx = nat.Context(instance.n_nonroot, len(instance.stage_slices), m.n_tanks,
                               m.n_inputs, m.n_demands, m.n_mixing, _DEVICE)
        self.spare: list = []  # NodeSets of dead caches, reused (no cudaMalloc/cudaFree per factor_step)

    def take_nodes(self) -> nat.NodeSet:
        return self.spare.pop() if self.spare else nat.NodeSet(self.ctx)


def _recycle_nodes(dev: _DeviceTree, nodes: nat.NodeSet) -> None:
    if len(dev.spare) < 2:
        dev.spare.append(nodes)


# signature -> weakref(_DeviceTree); contexts die with their last cache.
_POOL: dict = {}


def _pool_key(sig, instance) -> tuple:
    """Pool key: the structure signature plus the context's allocation
    dimensions the signature does not cover (demand columns, mixing rows):
    two models of one structure with different demand counts must not share
    a context, whose demand / Ed buffers are sized by the first."""
    m = instance.model
    return sig + (int(m.n_demands), int(m.n_mixing), tuple(m.Ed.shape))


def _dims_match(dev: _DeviceTree, instance) -> bool:
    m = instance.model
    n, H, nt, nu, nd, ns = dev.ctx.dims
    return (n, H, nt, nu, nd, ns) == (instance.n_nonroot, len(instance.stage_slices), m.n_tanks,
                                      m.n_inputs, m.n_demands, m.n_mixing)


def _device_for(sig, instance) -> _DeviceTree:
    key = _pool_key(sig, instance)
    ref = _POOL.get(key)
    dev = ref() if ref is not None else None
    if dev is None:
        dev = _DeviceTree(instance)
        _POOL[key] = weakref.ref(dev)
    return dev


@dataclass
class FactorCache:
    """Precomputed quantities (solver.py:101-122). Host members as in the
    reference; ``u_part``/``e_offset`` are downloaded lazily from the GPU."""

    null_basis: np.ndarray
    e_pinv: np.ndarray
    d_gain: list
    t_mat: list
    lam: list
    pi: list
    kappa: float
    lipschitz: float | None = None
    signature: tuple = field(default=(), repr=False)
    _dev: _DeviceTree | None = field(default=None, repr=False)
    _nodes: nat.NodeSet | None = field(default=None, repr=False)
    _offsets: tuple | None = field(default=None, repr=False)

    def _fetch_offsets(self):
        if self._offsets is None:
            n, _, _, nu, _, _ = self._dev.ctx.dims
            up, eo = np.empty((n, nu)), np.empty((n, nu))
            self._dev.ctx.call("wmpc_get_offsets", self._nodes.h, nat.ptr(up), nat.ptr(eo))
            self._offsets = (up, eo)
        return self._offsets

    @property
    def u_part(self) -> np.ndarray:
        return self._fetch_offsets()[0]

    @property
    def e_offset(self) -> np.ndarray:
        return self._fetch_offsets()[1]

    def _bind(self) -> nat.Context:
        self._dev.ctx.call("wmpc_bind_nodes", self._nodes.h)
        return self._dev.ctx


def _structure_signature(instance) -> tuple:
    """Cache identity (solver.py:125-135)."""
    m = instance.model
    return (
        m.A.tobytes(), m.B.tobytes(), m.E.tobytes(), instance.wu.tobytes(),
        instance.prob.tobytes(), instance.anc_row.tobytes(),
        tuple((sl.start, sl.stop) for sl in instance.stage_slices),
    )


def _null_space(E: np.ndarray, n_inputs: int):
    """SVD null-space basis and pseudo-inverse of E (solver.py:138-147)."""
    if E.shape[0] == 0:
        return np.eye(n_inputs), np.zeros((0, n_inputs))
    _, sv, vt = np.linalg.svd(E)
    cutoff = max(E.shape) * np.finfo(float).eps * (sv[0] if sv.size else 0.0)
    rank = int(np.count_nonzero(sv > cutoff))
    basis = vt[rank:].T
    if basis.shape[1] == 0:
        raise ValueError("mixing-node coupling leaves no free inputs")
    return basis, np.linalg.pinv(E)


def _stage_recursion(instance, basis):
    """Per-stage gains (solver.py:184-200); 24 x 114^3 flops on the host."""
    wu = instance.wu
    H = len(instance.stage_slices)
    nu = wu.shape[0]
    lam, t_mat, d_gain, pi = [None] * H, [None] * H, [None] * H, [None] * H
    nxt = np.zeros((nu, nu))
    for s in range(H - 1, -1, -1):
        L = nxt + 2.0 * wu
        reduced = basis.T @ L @ basis
        try:
            np.linalg.cholesky(reduced)
        except np.linalg.LinAlgError:
            raise ValueError("input weight is singular on the coupling null space") from None
        t = basis @ np.linalg.solve(reduced, basis.T)
        t = 0.5 * (t + t.T)
        dg = 2.0 * (t @ wu)
        ps = 2.0 * wu - 2.0 * (wu @ dg)
        ps = 0.5 * (ps + ps.T)
        lam[s], t_mat[s], d_gain[s], pi[s] = L, t, dg, ps
        nxt = ps
    return lam, t_mat, d_gain, pi


def _upload_structure(dev: _DeviceTree, instance, basis, e_pinv, lam, t_mat, d_gain) -> None:
    m = instance.model
    off = np.array([0] + [sl.stop for sl in instance.stage_slices], dtype=np.int64)
    anc = np.ascontiguousarray(instance.anc_row, dtype=np.int64)
    args = [nat.f64(m.A), nat.f64(m.B), nat.f64(instance.wu), nat.f64(np.stack(t_mat)),
            nat.f64(np.stack(d_gain)), nat.f64(np.stack(lam)), anc, off,
            nat.f64(instance.prob), nat.f64(m.E) if m.n_mixing else None,
            nat.f64(e_pinv) if m.n_mixing else None]
    keep = args  # keep alive across the call
    dev.ctx.call("wmpc_set_structure", *[nat.ptr(a) for a in keep])


def factor_step(instance, structure_from: FactorCache | None = None) -> FactorCache:
    """Build or rebind the factor cache (solver.py:150-239); the per-node part
    runs on the GPU (kernel ``k_node_offsets``)."""
    return _factor(instance, structure_from, private=False)


def _factor(instance, structure_from: FactorCache | None, private: bool,
            min_branch_stage: int = 0) -> FactorCache:
    """factor_step; ``private`` gives the cache its own native context instead
    of the per-structure pool (shard.py: several shards of one structure live
    in one process); ``min_branch_stage``: see wmpc_set_min_branch_stage."""
    m = instance.model
    sig = _structure_signature(instance)
    if structure_from is not None:
        if structure_from.signature != sig:
            raise ValueError("cached factors were built for a different structure")
        src = structure_from
        basis, e_pinv = src.null_basis, src.e_pinv
        lam, t_mat, d_gain, pi = src.lam, src.t_mat, src.d_gain, src.pi
        kappa, lipschitz = src.kappa, src.lipschitz
        dev = src._dev
        fresh_structure = False
        if not _dims_match(dev, instance):
            # same structure, other demand / mixing dimensions: the source's
            # context cannot hold this instance's node data
            dev = _DeviceTree(instance) if private else _device_for(sig, instance)
            fresh_structure = True
    else:
        basis, e_pinv = _null_space(m.E, m.n_inputs)
        check = m.E @ basis
        if check.size and float(np.max(np.abs(check))) > 1e-12 * (1.0 + float(np.max(np.abs(m.E)))):
            raise RuntimeError("null-space basis fails E @ N = 0")
        lam, t_mat, d_gain, pi = _stage_recursion(instance, basis)
        p_min = float(instance.prob.min())
        w_min = float(np.linalg.eigvalsh(instance.wu)[0])
        H = len(instance.stage_slices)
        kappa = 2.0 * w_min * p_min / (H * max(instance.n_nonroot, 1))
        lipschitz = None
        dev = _DeviceTree(instance) if private else _device_for(sig, instance)
        fresh_structure = True
        if min_branch_stage:
            dev.ctx.call("wmpc_set_min_branch_stage", int(min_branch_stage))
    if fresh_structure:
        _upload_structure(dev, instance, basis, e_pinv, lam, t_mat, d_gain)
    nodes = dev.take_nodes()
    demand = nat.f64(instance.demand)
    Ed = nat.f64(m.Ed)
    gd = nat.f64(instance.demand_gd)
    econ = nat.f64(instance.econ)
    bad = np.zeros(1, dtype=np.int64)
    if not _dims_match(dev, instance):
        raise ValueError("factor cache does not match this instance")
    # wmpc_set_node_data overwrites the context's econ before its feasibility
    # check: forget the marker first, so a raise cannot leave it naming the
    # previous instance
    dev.ctx._econ_src = None
    dev.ctx.call("wmpc_set_node_data", nodes.h, nat.ptr(demand) if m.n_mixing else None,
                 nat.ptr(Ed) if m.n_mixing else None, nat.ptr(gd), nat.ptr(econ), nat.ptr(bad))
    dev.ctx._econ_src = _econ_marker(instance.econ)  # the context's econ now holds this array
    cache = FactorCache(null_basis=basis, e_pinv=e_pinv, d_gain=d_gain, t_mat=t_mat, lam=lam,
                        pi=pi, kappa=kappa, lipschitz=lipschitz, signature=sig, _dev=dev,
                        _nodes=nodes)
    weakref.finalize(cache, _recycle_nodes, dev, nodes)
    return cache


def _check_cache(cache: FactorCache, instance) -> None:
    if cache.signature != _structure_signature(instance):
        raise ValueError("factor cache does not match this instance")


def _upload_bounds(ctx: nat.Context, instance, with_econ: bool = True) -> None:
    """Bounds, weights, p, q every solve (the reference's tests mutate them);
    econ (n x n_u, 72 MB at C4) only when the context does not already hold
    this instance's array: factor_step uploaded it with the node data, and
    instances are immutable (problem.py:18-19), so a solve right after its
    factor_step skips the copy."""
    m, w = instance.model, instance.weights
    arrs = [nat.f64(a) for a in (m.x_min, m.x_max, m.x_safe, m.u_min, m.u_max)]
    p, q = nat.f64(instance.p), nat.f64(instance.q)
    econ = None
    if with_econ and not _econ_current(getattr(ctx, "_econ_src", None), instance.econ):
        ctx._econ_src = None
        econ = nat.f64(instance.econ)
    ctx.call("wmpc_set_bounds", *[nat.ptr(a) for a in arrs], float(w.w_x), float(w.w_s),
             nat.ptr(p), nat.ptr(q), nat.ptr(econ))
    if econ is not None:
        ctx._econ_src = _econ_marker(instance.econ)


def _econ_fingerprint(econ: np.ndarray) -> bytes:
    """A strided sample of ``econ`` (<= 4,096 values plus the last row): catches
    in-place edits such as ``inst.econ[:] = -10.0`` (the reference's
    test_oracle.py:79) at negligible cost. Instances are documented immutable
    (problem.py:18-19); an edit that misses every sampled entry is not seen."""
    flat = econ.reshape(-1)
    step = max(1, flat.size // 4096)
    return flat[::step].tobytes() + econ.reshape(econ.shape[0], -1)[-1:].tobytes()


def _econ_marker(econ: np.ndarray) -> tuple:
    return (weakref.ref(econ) if isinstance(econ, np.ndarray) else None, _econ_fingerprint(econ))


def _econ_current(marker, econ: np.ndarray) -> bool:
    if marker is None or marker[0] is None or marker[0]() is not econ:
        return False
    return marker[1] == _econ_fingerprint(econ)




def dual_gradient(cache: FactorCache, instance, y) -> tuple[np.ndarray, float]:
    """Exact minimiser of f(x) + <H'y, x> and the attained value (solver.py:293-306)."""
    _check_cache(cache, instance)
    instance.split_dual(y)  # shape validation, reference message
    ctx = cache._bind()
    _upload_bounds(ctx, instance)
    yv = nat.f64(y)
    z = np.empty(instance.n_primal)
    val = np.zeros(1)
    ctx.call("wmpc_dual_gradient", nat.ptr(yv), nat.ptr(z), nat.ptr(val))
    return z, float(val[0])


def _next_theta(theta: float) -> float:
    """theta+ = 2 t^2 / (t^2 + sqrt(t^4 + 4 t^2)) (solver.py:309-313)."""
    t = theta * theta
    return 2.0 * t / (t + np.sqrt(t * t + 4.0 * t))


def theta_sequence(count: int) -> np.ndarray:
    """First ``count`` extrapolation parameters, theta_0 = 1 (solver.py:316-323)."""
    out = np.empty(count)
    th = 1.0
    for i in range(count):
        out[i] = th
        th = _next_theta(th)
    return out


def _beta_table(theta: np.ndarray) -> np.ndarray:
    """beta_nu = theta_nu (1/theta_{nu-1} - 1), theta_{-1} = 1 (solver.py:461)."""
    beta = np.empty_like(theta)
    prev = 1.0
    for i, th in enumerate(theta):
        beta[i] = th * (1.0 / prev - 1.0)
        prev = th
    return beta


def estimate_lipschitz(cache: FactorCache, instance, rel_tol: float = 1e-3, max_iter: int = 500,
                       safety: float = 1.1) -> float:
    """Power iteration on the dual curvature, on the GPU (solver.py:326-387)."""
    _check_cache(cache, instance)
    ctx = cache._bind()
    _upload_bounds(ctx, instance)
    v = np.random.default_rng(0).standard_normal(instance.n_dual)
    v /= np.linalg.norm(v)
    lam = np.zeros(1)
    settled = nat.C.c_int(0)
    iters = nat.C.c_int(0)
    ctx.call("wmpc_power_iteration", nat.ptr(v), float(rel_tol), int(max_iter), nat.ptr(lam),
             nat.C.byref(settled), nat.C.byref(iters))
    value = float(lam[0])
    if not settled.value and value > 0.0:
        warnings.warn("power iteration did not settle; falling back to the trace bound",
                      RuntimeWarning, stacklevel=2)
        tr = np.zeros(1)
        ctx.call("wmpc_operator_trace", nat.ptr(tr))
        value = float(tr[0])
    if value <= 0.0:
        raise RuntimeError("dual curvature estimate failed (operator not positive)")
    est = safety * value
    cache.lipschitz = est
    return est


def _result_buffers(instance) -> tuple:
    """Result arrays in pooled page-locked memory (``nat.pinned_empty``): the
    final device-to-host copies run asynchronously, overlapping the
    certificate (``_read_async``)."""
    nu = instance.model.n_inputs
    return (nat.pinned_empty(nu), nat.pinned_empty(instance.n_primal), nat.pinned_empty(instance.n_primal),
            nat.pinned_empty(instance.n_dual))


def _read_async(ctx, averaged: bool, out) -> None:
    """Queue the result readout on the context's second stream (wmpc_apg_read_async)."""
    out_u0, out_p, out_a, out_d = out
    ctx.call("wmpc_apg_read_async", int(averaged), nat.ptr(out_u0), nat.ptr(out_p), nat.ptr(out_a),
             nat.ptr(out_d))


def _read(ctx, instance, averaged: bool, u0=True, primal=True, avg=True, dual=True, out=None):
    nu = instance.model.n_inputs
    if out is None:
        out = (np.empty(nu) if u0 else None, np.empty(instance.n_primal) if primal else None,
               np.empty(instance.n_primal) if avg else None, np.empty(instance.n_dual) if dual else None)
    out_u0, out_p, out_a, out_d = out
    ctx.call("wmpc_apg_read", int(averaged), nat.ptr(out_u0), nat.ptr(out_p), nat.ptr(out_a),
             nat.ptr(out_d))
    return out_u0, out_p, out_a, out_d


def _check(ctx):
    r, s, dc = np.zeros(1), np.zeros(1), np.zeros(1)
    bad = nat.C.c_int(-1)
    ctx.call("wmpc_apg_check", nat.ptr(r), nat.ptr(s), nat.ptr(dc), nat.C.byref(bad))
    if bad.value >= 0:
        raise RuntimeError(f"solver produced a non-finite iterate at nu={bad.value}")
    return float(r[0]), float(s[0]), float(dc[0])


def _certificate(ctx):
    gap, obj = np.zeros(1), np.zeros(1)
    ctx.call("wmpc_certificate", nat.ptr(gap), nat.ptr(obj))
    return float(gap[0]), float(obj[0])


def solve(instance, config: SolverConfig | None = None, cache: FactorCache | None = None,
          iterate_hook: IterateHook | None = None, y_init=None) -> SolverResult:
    """Accelerated dual proximal gradient on the GPU (solver.py:398-543).

    Iterations run as CUDA-graph replays in chunks ending at the reference's
    check iterations ((nu+1) % gap_check_every == 0); only the residual,
    scale, dual change and non-finite flag cross to the host there. With an
    ``iterate_hook`` the loop advances one iteration per replay and copies
    the iterates to the host for the hook (debug path). ``y_init``: optional
    dual warm start (closed loop; the reference always starts from 0).
    """
    config = config or SolverConfig()
    if cache is None:
        cache = factor_step(instance)
    else:
        _check_cache(cache, instance)
    gamma = config.gamma
    lipschitz = cache.lipschitz
    if gamma is None:
        if lipschitz is None:
            lipschitz = estimate_lipschitz(cache, instance)
        gamma = 1.0 / lipschitz
    ctx = cache._bind()
    _upload_bounds(ctx, instance)
    theta = theta_sequence(config.max_iter)
    beta = _beta_table(theta)
    ctx.call("wmpc_set_precision", 1 if config.precision == "fp32" else 0)
    ctx.call("wmpc_apg_begin", float(gamma), int(config.max_iter), nat.ptr(theta), nat.ptr(beta))
    if y_init is not None:
        y0 = nat.f64(y_init)
        if y0.shape != (instance.n_dual,):
            raise ValueError(f"y_init must have shape ({instance.n_dual},)")
        ctx.call("wmpc_apg_warm", nat.ptr(y0))
    started = time.perf_counter()
    residual = dchange = gap = objective = float("inf")
    iterations, termination = config.max_iter, "max_iter"
    gce = config.gap_check_every
    done = 0
    bufs = None
    while done < config.max_iter:
        if iterate_hook is not None:
            step = 1
        else:
            step = min(gce - (done % gce), config.max_iter - done)
        ctx.call("wmpc_apg_run", int(step))
        if bufs is None and iterate_hook is None:
            bufs = _result_buffers(instance)  # host work overlapping the device loop
        done += step
        if iterate_hook is not None:
            residual, scale, dchange = _check(ctx)
            _, z, z_avg, y = _read(ctx, instance, config.averaged_primal, u0=False)
            iterate_hook(done - 1, y, z, z_avg)
        if done % gce == 0:
            if iterate_hook is None:
                residual, scale, dchange = _check(ctx)
            if residual <= config.tol * (1.0 + scale):
                gap, objective = _certificate(ctx)
                if gap <= config.tol * (1.0 + abs(objective)):
                    iterations, termination = done, "converged"
                    break
    if bufs is None:
        bufs = _result_buffers(instance)
    try:
        if termination == "max_iter":
            residual, scale, dchange = _check(ctx)
            _read_async(ctx, config.averaged_primal, bufs)  # copies overlap the certificate
            gap, objective = _certificate(ctx)
        else:
            _read_async(ctx, config.averaged_primal, bufs)
    finally:
        ctx.call("wmpc_apg_read_wait")  # the copies land before bufs can be dropped
    elapsed = time.perf_counter() - started
    u0, primal, primal_avg, dual = bufs
    return SolverResult(u0=u0, primal=primal, primal_avg=primal_avg, dual=dual,
                        iterations=iterations, termination=termination,
                        primal_residual=residual, dual_change=dchange, duality_gap=gap,
                        objective=objective, solve_time_s=elapsed, gamma=gamma,
                        lipschitz=lipschitz)


# --------------------------------------------------------------------------
# prox API support (problem.prox_g / prox_g_conjugate)
# --------------------------------------------------------------------------

_PROX_CTX: dict = {}


def _device_prox(instance, v, gamma: float, conjugate: bool) -> np.ndarray:
    Y1, _, _ = instance.split_dual(v)  # shape validation
    m = instance.model
    key = (instance.n_nonroot, m.n_tanks, m.n_inputs)
    ctx = _PROX_CTX.get(key)
    if ctx is None:
        ctx = nat.Context(instance.n_nonroot, 1, m.n_tanks, m.n_inputs, 0, 0, _DEVICE)
        _PROX_CTX.clear()
        _PROX_CTX[key] = ctx
    _upload_bounds(ctx, instance, with_econ=False)
    vin = nat.f64(v)
    out = np.empty(instance.n_dual)
    ctx.call("wmpc_prox", nat.ptr(vin), float(gamma), int(conjugate), nat.ptr(out))
    return out
