"""Dense KKT route for the inner QP (test infrastructure only).

Restates ``/root/reference/pkg/src/watermpc/oracle.py:41-116``: the inner
problem min f(z) + <H'y, z> over the dynamics and coupling equalities is
assembled as one dense symmetric indefinite KKT system and solved directly,
independent of the tree recursion. Small instances only (<= 5000 primal).
"""

from __future__ import annotations

import numpy as np
import scipy.linalg

DENSE_LIMIT = 5000


def _H_adjoint_rows(inst, y):
    nt = inst.model.A.shape[0]
    R = np.asarray(y, float).reshape(inst.prob.shape[0], -1)
    return np.concatenate([R[:, 2 * nt:], R[:, :nt] + R[:, nt:2 * nt]], axis=1).reshape(-1)


def kkt_system(inst):
    """(Hessian, linear term, equality matrix, rhs) over z = [u_r | x_r]_r."""
    m = inst.model
    nu, nt, ns = m.B.shape[1], m.A.shape[0], m.E.shape[0]
    n = inst.prob.shape[0]
    w = nu + nt
    dim = n * w
    Hs = np.zeros((dim, dim))
    g = np.zeros(dim)
    W = inst.wu
    for r in range(n):
        ur = slice(r * w, r * w + nu)
        a = int(inst.anc_row[r])
        c = 2.0 * inst.prob[r]
        Hs[ur, ur] += c * W
        if a >= 0:
            ua = slice(a * w, a * w + nu)
            Hs[ur, ua] -= c * W
            Hs[ua, ur] -= c * W
            Hs[ua, ua] += c * W
        else:
            g[ur] -= c * (W @ inst.q)
        g[ur] += inst.prob[r] * inst.weights.w_alpha * (m.alpha0 + inst.price[r])
    rows = n * (nt + ns)
    C = np.zeros((rows, dim))
    b = np.zeros(rows)
    k = 0
    for r in range(n):
        xr = slice(r * w + nu, (r + 1) * w)
        C[k:k + nt, xr] = np.eye(nt)
        C[k:k + nt, r * w:r * w + nu] = -m.B
        a = int(inst.anc_row[r])
        drive = m.Gd @ inst.demand[r]
        if a >= 0:
            C[k:k + nt, a * w + nu:(a + 1) * w] = -m.A
            b[k:k + nt] = drive
        else:
            b[k:k + nt] = m.A @ inst.p + drive
        k += nt
        if ns:
            C[k:k + ns, r * w:r * w + nu] = m.E
            b[k:k + ns] = -(m.Ed @ inst.demand[r])
            k += ns
    return Hs, g, C, b


def dense_kkt_solve(inst, y):
    """Minimiser of f(z) + <H'y, z> by one dense symmetric solve."""
    n_primal = inst.prob.shape[0] * (inst.model.A.shape[0] + inst.model.B.shape[1])
    if n_primal > DENSE_LIMIT:
        raise ValueError(f"instance with {n_primal} primal variables is too large for the dense oracle")
    Hs, g, C, b = kkt_system(inst)
    dim, rows = Hs.shape[0], C.shape[0]
    K = np.zeros((dim + rows, dim + rows))
    K[:dim, :dim] = Hs
    K[:dim, dim:] = C.T
    K[dim:, :dim] = C
    rhs = np.concatenate([-(g + _H_adjoint_rows(inst, y)), b])
    sol = scipy.linalg.solve(K, rhs, assume_a="sym")
    return sol[:dim]
