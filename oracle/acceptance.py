"""Optimality-check helpers of the reference's test suite (test infrastructure
only: imported by tests/, never by the product).

Restates ``/root/reference/pkg/src/watermpc/oracle.py:119-221`` (the grid
search over the input boxes of a tiny instance, the feasibility restoration
and the dense-KKT duality gap) and ``problem.py:253-275, :330-407`` (f, g, the
full objective and the clip of y into dom g*), on top of oracle/port.py and
oracle/dense.py, so the reference's acceptance tests (test_oracle.py:66-150)
can run against the GPU solver on the GPU box, where the reference is absent.
"""

from __future__ import annotations

import numpy as np

from . import port
from .dense import dense_kkt_solve

FEAS_TOL = 1e-8  # problem.py FEAS_TOL


def _rows(inst, v, width):
    return np.asarray(v, float).reshape(inst.prob.shape[0], width)


def split_primal(inst, z):
    nu = inst.model.B.shape[1]
    Z = _rows(inst, z, nu + inst.model.A.shape[0])
    return Z[:, :nu], Z[:, nu:]


def join_primal(U, X):
    return np.concatenate([U, X], axis=1).reshape(-1)


def split_dual(inst, y):
    nt = inst.model.A.shape[0]
    Y = _rows(inst, y, 2 * nt + inst.model.B.shape[1])
    return Y[:, :nt], Y[:, nt:2 * nt], Y[:, 2 * nt:]


def eval_f(inst, z) -> float:
    """Smooth cost when z satisfies dynamics and coupling, +inf otherwise (problem.py:253-266)."""
    U, X = split_primal(inst, z)
    m = inst.model
    tol = FEAS_TOL * (1.0 + float(np.max(np.abs(z), initial=0.0)))
    if m.E.shape[0] > 0:
        if float(np.max(np.abs(U @ m.E.T + inst.demand @ m.Ed.T))) > tol:
            return np.inf
    anc = inst.anc_row
    x_anc = np.where(anc[:, None] >= 0, X[np.maximum(anc, 0)], inst.p[None, :])
    resid = X - (x_anc @ m.A.T + U @ m.B.T + inst.demand_gd)
    if float(np.max(np.abs(resid))) > tol:
        return np.inf
    return port.smooth_cost(inst, U)


def g_value(inst, z) -> float:
    """g(Hz): soft distances and the hard input box (problem.py:330-339)."""
    U, X = split_primal(inst, z)
    m, w = inst.model, inst.weights
    if np.any(U < m.u_min) or np.any(U > m.u_max):
        return np.inf
    return port.penalty_value(inst, X)


def primal_objective(inst, z) -> float:
    """f(z) + g(Hz) (problem.py:402-407)."""
    fz = eval_f(inst, z)
    if not np.isfinite(fz):
        return np.inf
    return fz + g_value(inst, z)


def clip_dual_to_domain(inst, y):
    """y1, y2 scaled into their norm balls, y2 <= 0 (problem.py:377-392)."""
    w = inst.weights
    Y1, Y2, Y3 = (a.copy() for a in split_dual(inst, y))
    for Y, bound in ((Y1, w.w_x), (Y2, w.w_s)):
        norms = np.linalg.norm(Y, axis=1)
        over = norms > bound
        if np.any(over):
            scale = np.ones_like(norms)
            scale[over] = bound / norms[over]
            Y *= scale[:, None]
    np.minimum(Y2, 0.0, out=Y2)
    return np.concatenate([Y1, Y2, Y3], axis=1).reshape(-1)


def project_primal_feasible(inst, z):
    """Inputs into box and coupling (Dykstra), states re-rolled (oracle.py:199-204)."""
    U, _ = split_primal(inst, z)
    fac = port.stage_factors(inst.model.E, inst.wu, len(inst.stage_slices))
    U_f = port.dykstra_restore(inst, U, fac.e_pinv)
    return join_primal(U_f, port.rollout(inst, U_f))


def duality_gap(inst, z, y) -> float:
    """Primal value at the restored z minus the dual value at clip(y), the
    dual value through the dense KKT route (oracle.py:207-221)."""
    z_f = project_primal_feasible(inst, z)
    primal = primal_objective(inst, z_f)
    y_c = clip_dual_to_domain(inst, y)
    z_star = dense_kkt_solve(inst, y_c)
    U_star, X_star = split_primal(inst, z_star)
    Y1, Y2, Y3 = split_dual(inst, y_c)
    inner = port.smooth_cost(inst, U_star) + float(np.sum(Y1 * X_star) + np.sum(Y2 * X_star) + np.sum(Y3 * U_star))
    return float(primal - (inner - port.g_conjugate(inst, y_c)))


def objective_on_inputs(inst, u_batch):
    """Full objective for a batch of stacked box-feasible input vectors (oracle.py:119-146)."""
    m = inst.model
    n = inst.prob.shape[0]
    P = u_batch.shape[0]
    nu, nt = m.B.shape[1], m.A.shape[0]
    U = u_batch.reshape(P, n, nu)
    X = np.empty((P, n, nt))
    for j, sl in enumerate(inst.stage_slices):
        anc = inst.anc_row[sl]
        x_prev = np.broadcast_to(inst.p, (P, sl.stop - sl.start, nt)) if j == 0 else X[:, anc]
        X[:, sl] = x_prev @ m.A.T + U[:, sl] @ m.B.T + np.broadcast_to(inst.demand_gd[sl], (P, sl.stop - sl.start, nt))
    u_anc = U[:, inst.anc_row]
    u_anc[:, inst.anc_row < 0] = inst.q
    du = U - u_anc
    w = inst.weights
    smooth = (inst.prob[None, :] * ((inst.econ[None, :, :] * U).sum(axis=2)
                                    + np.einsum("pij,jk,pik->pi", du, inst.wu, du))).sum(axis=1)
    box_d = np.linalg.norm(X - np.clip(X, m.x_min, m.x_max), axis=2).sum(axis=1)
    safe_d = np.linalg.norm(X - np.maximum(X, m.x_safe), axis=2).sum(axis=1)
    return smooth + w.w_x * box_d + w.w_s * safe_d


def brute_force_min(inst, resolution: float = 1e-3):
    """Grid search over the input boxes of a tiny uncoupled instance (oracle.py:149-196)."""
    m = inst.model
    if m.E.shape[0] > 0:
        raise ValueError("grid oracle requires an instance without mixing nodes")
    n = inst.prob.shape[0]
    nu = m.B.shape[1]
    dims = n * nu
    if dims > 3:
        raise ValueError(f"dimension too large for grid search: {dims} free inputs")
    lo, hi = np.tile(m.u_min, n), np.tile(m.u_max, n)
    span = hi - lo
    npts = int(round(1.0 / resolution)) + 1

    def evaluate(axes):
        mesh = np.meshgrid(*axes, indexing="ij")
        pts = np.stack([g.reshape(-1) for g in mesh], axis=1)
        vals = objective_on_inputs(inst, pts)
        best = int(np.argmin(vals))
        return pts[best], float(vals[best])

    if npts ** dims <= 2_000_000:
        u_best, val = evaluate([np.linspace(lo[i], hi[i], npts) for i in range(dims)])
    else:
        wlo, whi = lo.copy(), hi.copy()
        u_best, val = None, np.inf
        target = resolution * span
        while True:
            cand, cval = evaluate([np.linspace(wlo[i], whi[i], 11) for i in range(dims)])
            if cval < val:
                u_best, val = cand, cval
            cell = (whi - wlo) / 10
            if np.all(cell <= target):
                break
            wlo, whi = np.maximum(lo, cand - cell), np.minimum(hi, cand + cell)
    U = u_best.reshape(n, nu)
    return join_primal(U, port.rollout(inst, U)), val
