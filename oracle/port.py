"""CPU restatement of the reference's dual-APG hot path (numpy, fp64).

TEST INFRASTRUCTURE ONLY. This module is the parity checker and the CPU
baseline: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
reference / cpu_baseline legs may import it. The product package
(``paper_1904_10548_b200``) never imports it and has no CPU fallback.

Pinning: every function restates one reference function (file:line cited,
paths relative to ``/root/reference/pkg/src/watermpc``). The restatement is
checked against fixtures produced by the reference itself
(``tests/golden/make_golden.py`` imports ``/root/reference`` in the build
container and commits ``tests/golden/*.npz``); ``tests/test_oracle_golden.py``
compares them. It accepts any object with the reference ``ProblemInstance``
attributes (``model``, ``weights``, ``prob``, ``anc_row``, ``stage_slices``,
``demand``, ``demand_gd``, ``econ``, ``wu``, ``p``, ``q``).
"""

from __future__ import annotations

import time
import warnings
from dataclasses import dataclass

import numpy as np


# --------------------------------------------------------------------------
# factor step (solver.py:138-239)
# --------------------------------------------------------------------------

def coupling_null_space(E: np.ndarray, n_inputs: int):
    """Orthonormal null-space basis of E and pinv(E) (solver.py:138-147)."""
    if E.shape[0] == 0:
        return np.eye(n_inputs), np.zeros((0, n_inputs))
    _, sv, vt = np.linalg.svd(E)
    cut = max(E.shape) * np.finfo(float).eps * (sv[0] if sv.size else 0.0)
    keep = int(np.count_nonzero(sv > cut))
    basis = vt[keep:].T
    if basis.shape[1] == 0:
        raise ValueError("mixing-node coupling leaves no free inputs")
    return basis, np.linalg.pinv(E)


@dataclass
class StageFactors:
    basis: np.ndarray
    e_pinv: np.ndarray
    lam: list
    T: list
    D: list
    Pi: list


def stage_factors(E: np.ndarray, wu: np.ndarray, horizon: int) -> StageFactors:
    """Backward recursion for the per-stage gains (solver.py:172-200).

    Pi_{H+1} = 0; Lam_s = Pi_{s+1} + 2W; T_s = N (N'Lam_s N)^-1 N' (sym.);
    D_s = 2 T_s W; Pi_s = 2W - 2 W D_s (sym.).
    """
    nu = wu.shape[0]
    basis, e_pinv = coupling_null_space(E, nu)
    check = E @ basis
    if check.size and float(np.abs(check).max()) > 1e-12 * (1.0 + float(np.abs(E).max())):
        raise RuntimeError("null-space basis fails E @ N = 0")
    lam, T, D, Pi = ([None] * horizon for _ in range(4))
    carry = np.zeros((nu, nu))
    for s in reversed(range(horizon)):
        L = carry + 2.0 * wu
        red = basis.T @ L @ basis
        try:
            np.linalg.cholesky(red)
        except np.linalg.LinAlgError:
            raise ValueError("input weight is singular on the coupling null space") from None
        t = basis @ np.linalg.solve(red, basis.T)
        t = 0.5 * (t + t.T)
        d = 2.0 * (t @ wu)
        pi = 2.0 * wu - 2.0 * (wu @ d)
        pi = 0.5 * (pi + pi.T)
        lam[s], T[s], D[s], Pi[s] = L, t, d, pi
        carry = pi
    return StageFactors(basis, e_pinv, lam, T, D, Pi)


def node_offsets(inst, fac: StageFactors):
    """Per-node coupling particular solution and input offset (solver.py:206-225)."""
    m = inst.model
    n = inst.prob.shape[0]
    if m.E.shape[0] > 0:
        rhs = inst.demand @ m.Ed.T
        u_part = -(rhs @ fac.e_pinv.T)
        viol = np.abs(u_part @ m.E.T + rhs) > 1e-9 * (1.0 + np.abs(rhs))
        rows = np.flatnonzero(viol.any(axis=1))
        if rows.size:
            raise ValueError(
                f"coupling E u = -Ed d is infeasible at tree node {int(rows[0]) + 1}")
    else:
        u_part = np.zeros((n, m.B.shape[1]))
    e_off = np.empty_like(u_part)
    for s, sl in enumerate(inst.stage_slices):
        e_off[sl] = u_part[sl] - (u_part[sl] @ fac.lam[s] + inst.econ[sl]) @ fac.T[s]
    return u_part, e_off


# --------------------------------------------------------------------------
# dual gradient: the tree Riccati-type recursion (solver.py:242-290)
# --------------------------------------------------------------------------

def inputs_before(inst, U):
    """Ancestor input per row, q at stage 1 (problem.py:183-187)."""
    out = U[inst.anc_row]
    out[inst.anc_row < 0] = inst.q
    return out


def smooth_cost(inst, U) -> float:
    """sum_r p_r [c_r'u_r + du_r' W du_r] (problem.py:269-275)."""
    du = U - inputs_before(inst, U)
    lin = (inst.econ * U).sum(axis=1)
    quad = np.einsum("ij,jk,ik->i", du, inst.wu, du)
    return float(inst.prob @ (lin + quad))


def dual_gradient_rows(inst, fac: StageFactors, e_off, Yx, Yu, want_value=True):
    """Exact inner-QP minimiser for collapsed duals (Yx = y1 + y2, Yu = y3).

    Backward (stage H..1): lin = Yu + wbar B + rbar; e = e_off - (lin/p) T_s;
    children push wbar A and -2p (e W) into their parent in ascending row
    order. Forward (1..H): U = U_anc D_s' + e; X = X_anc A' + U B' + g.
    """
    m = inst.model
    A, B = m.A, m.B
    n = Yx.shape[0]
    wbar = Yx.copy()
    rbar = np.zeros((n, B.shape[1]))
    e = np.empty((n, B.shape[1]))
    p = inst.prob[:, None]
    H = len(inst.stage_slices)
    for s in range(H - 1, -1, -1):
        sl = inst.stage_slices[s]
        lin = Yu[sl] + wbar[sl] @ B + rbar[sl]
        e[sl] = e_off[sl] - (lin / p[sl]) @ fac.T[s]
        if s > 0:
            up = inst.anc_row[sl]
            np.add.at(wbar, up, wbar[sl] @ A)
            np.add.at(rbar, up, (-2.0 * p[sl]) * (e[sl] @ inst.wu))
    U = np.empty((n, B.shape[1]))
    X = np.empty((n, A.shape[0]))
    for s in range(H):
        sl = inst.stage_slices[s]
        if s == 0:
            u_prev, x_prev = inst.q, inst.p
        else:
            u_prev, x_prev = U[inst.anc_row[sl]], X[inst.anc_row[sl]]
        U[sl] = u_prev @ fac.D[s].T + e[sl]
        X[sl] = x_prev @ A.T + U[sl] @ B.T + inst.demand_gd[sl]
    value = None
    if want_value:
        value = smooth_cost(inst, U) + float((Yx * X).sum() + (Yu * U).sum())
    return U, X, value


# --------------------------------------------------------------------------
# prox / Moreau (problem.py:290-327, solver.py:546-583)
# --------------------------------------------------------------------------

def _shrink_to_set(V, P, thr):
    """Prox of thr * dist(., C) given the projection P (problem.py:290-300)."""
    gap = V - P
    dist = np.linalg.norm(gap, axis=1)
    with np.errstate(divide="ignore", invalid="ignore"):
        step = np.where(dist > 0.0, np.minimum(1.0, thr / dist), 0.0)
    return V - step[:, None] * gap


def prox_rows(m, w, V1, V2, V3, g):
    """Row-wise prox of g*g on the three slots (problem.py:303-310)."""
    o1 = _shrink_to_set(V1, np.clip(V1, m.x_min, m.x_max), g * w.w_x)
    o2 = _shrink_to_set(V2, np.maximum(V2, m.x_safe), g * w.w_s)
    o3 = np.clip(V3, m.u_min, m.u_max)
    return o1, o2, o3


def prox_g(inst, v, g):
    nt = inst.model.A.shape[0]
    R = np.asarray(v, float).reshape(inst.prob.shape[0], -1)
    o = prox_rows(inst.model, inst.weights, R[:, :nt], R[:, nt:2 * nt], R[:, 2 * nt:], g)
    return np.concatenate(o, axis=1).reshape(-1)


def prox_g_conj_rows(inst, W, gamma):
    """y+ = w - gamma prox_{g/gamma}(w/gamma), slot-wise (solver.py:563-575)."""
    nt = inst.model.A.shape[0]
    V = W / gamma
    o1, o2, o3 = prox_rows(inst.model, inst.weights, V[:, :nt], V[:, nt:2 * nt],
                           V[:, 2 * nt:], 1.0 / gamma)
    out = np.empty_like(W)
    out[:, :nt] = W[:, :nt] - gamma * o1
    out[:, nt:2 * nt] = W[:, nt:2 * nt] - gamma * o2
    out[:, 2 * nt:] = W[:, 2 * nt:] - gamma * o3
    return out


# --------------------------------------------------------------------------
# theta / Lipschitz (solver.py:309-387)
# --------------------------------------------------------------------------

def theta_next(t: float) -> float:
    """Rationalised root of t+^2/t^2 + t+ - 1 = 0 (solver.py:309-313)."""
    sq = t * t
    return 2.0 * sq / (sq + np.sqrt(sq * sq + 4.0 * sq))


def theta_table(count: int) -> np.ndarray:
    out = np.empty(count)
    t = 1.0
    for i in range(count):
        out[i] = t
        t = theta_next(t)
    return out


def power_lipschitz(inst, fac, e_off, rel_tol=1e-3, max_iter=500, safety=1.1):
    """Power iteration on v -> H(x*(0) - x*(v)) (solver.py:326-387)."""
    n = inst.prob.shape[0]
    nt = inst.model.A.shape[0]
    nu = inst.model.B.shape[1]
    u0, x0, _ = dual_gradient_rows(inst, fac, e_off, np.zeros((n, nt)), np.zeros((n, nu)),
                                   want_value=False)

    def op(vec):
        R = vec.reshape(n, -1)
        u, x, _ = dual_gradient_rows(inst, fac, e_off, R[:, :nt] + R[:, nt:2 * nt],
                                     R[:, 2 * nt:], want_value=False)
        dx = x0 - x
        return np.concatenate([dx, dx, u0 - u], axis=1).reshape(-1)

    v = np.random.default_rng(0).standard_normal(n * (2 * nt + nu))
    v /= np.linalg.norm(v)
    lam = lam_prev = 0.0
    settled = False
    for _ in range(max_iter):
        gv = op(v)
        lam = float(v @ gv)
        nrm = float(np.linalg.norm(gv))
        if nrm == 0.0:
            break
        v = gv / nrm
        if abs(lam - lam_prev) <= rel_tol * max(abs(lam), 1e-300):
            settled = True
            break
        lam_prev = lam
    if not settled and lam > 0.0:
        warnings.warn("power iteration did not settle; falling back to the trace bound",
                      RuntimeWarning, stacklevel=2)
        e_i = np.zeros(v.shape[0])
        lam = 0.0
        for i in range(v.shape[0]):
            e_i[i] = 1.0
            lam += float(op(e_i)[i])
            e_i[i] = 0.0
    if lam <= 0.0:
        raise RuntimeError("dual curvature estimate failed (operator not positive)")
    return safety * lam


# --------------------------------------------------------------------------
# certificate pieces (problem.py:207-250, 342-374; solver.py:390-395)
# --------------------------------------------------------------------------

def rollout(inst, U):
    """States from the node dynamics (problem.py:207-218)."""
    m = inst.model
    X = np.empty((U.shape[0], m.A.shape[0]))
    for j, sl in enumerate(inst.stage_slices):
        prev = inst.p[None, :] if j == 0 else X[inst.anc_row[sl]]
        X[sl] = prev @ m.A.T + U[sl] @ m.B.T + inst.demand_gd[sl]
    return X


def dykstra_restore(inst, U, e_pinv):
    """Dykstra between coupling affine set and input box (problem.py:221-250)."""
    m = inst.model
    if m.E.shape[0] == 0:
        return np.clip(U, m.u_min, m.u_max)
    shift = inst.demand @ m.Ed.T
    cur = U.copy()
    pc = np.zeros_like(cur)
    qc = np.zeros_like(cur)
    tol = 1e-13 * (1.0 + float(np.max(np.abs(U))))
    for _ in range(500):
        aff = cur + pc
        aff -= (aff @ m.E.T + shift) @ e_pinv.T
        pc = cur + pc - aff
        nxt = np.clip(aff + qc, m.u_min, m.u_max)
        qc = aff + qc - nxt
        moved = float(np.max(np.abs(nxt - cur)))
        cur = nxt
        if moved <= tol:
            break
    return cur


def penalty_value(inst, X) -> float:
    m, w = inst.model, inst.weights
    box = np.linalg.norm(X - np.clip(X, m.x_min, m.x_max), axis=1).sum()
    safe = np.linalg.norm(X - np.maximum(X, m.x_safe), axis=1).sum()
    return float(w.w_x * box + w.w_s * safe)


def _support_box(lo, hi, Y) -> float:
    with np.errstate(invalid="ignore"):
        val = hi * np.clip(Y, 0.0, None) + lo * np.clip(Y, None, 0.0)
    return float(np.where(np.isnan(val), 0.0, val).sum())


def g_conjugate(inst, y, domain_tol=1e-9) -> float:
    """g*(y) with +inf outside the domain (problem.py:342-367)."""
    m, w = inst.model, inst.weights
    nt = m.A.shape[0]
    R = y.reshape(inst.prob.shape[0], -1)
    Y1, Y2, Y3 = R[:, :nt], R[:, nt:2 * nt], R[:, 2 * nt:]
    slack = 1.0 + domain_tol
    if np.any(np.linalg.norm(Y1, axis=1) > w.w_x * slack + domain_tol):
        return np.inf
    if np.any(np.linalg.norm(Y2, axis=1) > w.w_s * slack + domain_tol):
        return np.inf
    if np.any(Y2 > domain_tol * (1.0 + np.abs(m.x_safe))):
        return np.inf
    return float(_support_box(m.x_min, m.x_max, Y1)
                 + float((m.x_safe * np.minimum(Y2, 0.0)).sum())
                 + _support_box(m.u_min, m.u_max, Y3))


# --------------------------------------------------------------------------
# the APG loop (solver.py:398-543)
# --------------------------------------------------------------------------

@dataclass
class PortResult:
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
    loop_time_s: float = 0.0


def factor(inst):
    fac = stage_factors(inst.model.E, inst.wu, len(inst.stage_slices))
    _, e_off = node_offsets(inst, fac)
    return fac, e_off


def apg_solve(inst, gamma, max_iter=500, tol=5e-2, gap_check_every=25,
              averaged_primal=True, fac=None, e_off=None, hook=None,
              reference_cost_accounting=True, final_certificate=True) -> PortResult:
    """Fixed-step accelerated dual proximal gradient (solver.py:398-543).

    ``reference_cost_accounting`` evaluates the dual-gradient value every
    iteration and discards it, exactly as the reference loop does
    (solver.py:464); parity tests switch it off to save time.
    """
    if fac is None or e_off is None:
        fac, e_off = factor(inst)
    m = inst.model
    nt, nu = m.A.shape[0], m.B.shape[1]
    n = inst.prob.shape[0]
    width = 2 * nt + nu
    y = np.zeros((n, width))
    y_old = np.zeros((n, width))
    th = th_old = 1.0
    Ua = np.zeros((n, nu))
    Xa = np.zeros((n, nt))
    U = np.zeros((n, nu))
    X = np.zeros((n, nt))
    resid = dchange = gap = obj = np.inf
    iters, term = max_iter, "max_iter"
    t0 = time.perf_counter()

    def certify(yp):
        uf = dykstra_restore(inst, Ua, fac.e_pinv)
        xf = rollout(inst, uf)
        pv = smooth_cost(inst, uf) + penalty_value(inst, xf)
        _, _, inner = dual_gradient_rows(inst, fac, e_off, yp[:, :nt] + yp[:, nt:2 * nt],
                                         yp[:, 2 * nt:])
        dv = inner - g_conjugate(inst, yp.reshape(-1))
        return pv - dv, pv

    loop_time = 0.0
    for it in range(max_iter):
        ts = time.perf_counter()
        beta = th * (1.0 / th_old - 1.0)
        w = y + beta * (y - y_old)
        U, X, _ = dual_gradient_rows(inst, fac, e_off, w[:, :nt] + w[:, nt:2 * nt],
                                     w[:, 2 * nt:], want_value=reference_cost_accounting)
        v = w.copy()
        v[:, :nt] += gamma * X
        v[:, nt:2 * nt] += gamma * X
        v[:, 2 * nt:] += gamma * U
        y_new = prox_g_conj_rows(inst, v, gamma)
        if it == 0:
            Ua[:] = U
            Xa[:] = X
        else:
            Ua *= 1.0 - th
            Ua += th * U
            Xa *= 1.0 - th
            Xa += th * X
        dchange = float(np.max(np.abs(y_new - y)))
        if not np.isfinite(dchange):
            raise RuntimeError(f"solver produced a non-finite iterate at nu={it}")
        resid = float(max(np.maximum(Ua - m.u_max, 0.0).max(initial=0.0),
                          np.maximum(m.u_min - Ua, 0.0).max(initial=0.0)))
        scale = max(float(np.max(np.abs(Xa), initial=0.0)),
                    float(np.max(np.abs(Ua), initial=0.0)))
        if hook is not None:
            hook(it, y_new.reshape(-1), np.concatenate([U, X], 1).reshape(-1),
                 np.concatenate([Ua, Xa], 1).reshape(-1))
        y_old, y = y, y_new
        th_old, th = th, theta_next(th)
        loop_time += time.perf_counter() - ts
        if resid <= tol * (1.0 + scale) and (it + 1) % gap_check_every == 0:
            gap, obj = certify(y)
            if gap <= tol * (1.0 + abs(obj)):
                iters, term = it + 1, "converged"
                break
    if term == "max_iter" and final_certificate:
        gap, obj = certify(y)
    elapsed = time.perf_counter() - t0
    Uo = Ua if averaged_primal else U
    sl = inst.stage_slices[0]
    u0 = np.clip(inst.prob[sl] @ Uo[sl], m.u_min, m.u_max)
    return PortResult(u0, np.concatenate([U, X], 1).reshape(-1),
                      np.concatenate([Ua, Xa], 1).reshape(-1), y.reshape(-1), iters, term,
                      resid, dchange, gap, obj, elapsed, gamma, loop_time)
