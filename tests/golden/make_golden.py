"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

Each fixture stores the instance as plain arrays plus the reference's outputs
(``watermpc.solver`` / ``watermpc.problem`` called through their public API).
The GPU box has no /root/reference, so these committed files are what pins
both the oracle restatement (``oracle/port.py``) and the CUDA path.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, "/root/reference/pkg/src")

import watermpc.problem as RP  # noqa: E402
import watermpc.solver as RS  # noqa: E402
from watermpc.network import NetworkModel as RModel  # noqa: E402
from watermpc.tree import ScenarioTree as RTree  # noqa: E402

from conftest import instance_to_arrays, make_instance  # noqa: E402
from paper_1904_10548_b200.synthetic import config_instance  # noqa: E402


def to_reference(a):
    model = RModel(A=a["A"].copy(), B=a["B"].copy(), Gd=a["Gd"].copy(), E=a["E"].copy(),
                   Ed=a["Ed"].copy(), x_min=a["x_min"].copy(), x_max=a["x_max"].copy(),
                   x_safe=a["x_safe"].copy(), u_min=a["u_min"].copy(), u_max=a["u_max"].copy(),
                   alpha0=a["alpha0"].copy(), dt=float(a["dt"]))
    H = int(a["horizon"])
    tree = RTree(H, model.n_demands, model.n_inputs, a["stage"].copy(), a["anc"].copy(),
                 a["prob"].copy(), eps=a["eps"].copy(), demand=a["demand"].copy(),
                 price=a["price"].copy())
    wu = np.asarray(a["w_u"])
    w = RP.CostWeights(w_alpha=float(a["w_alpha"]), w_u=float(wu) if wu.ndim == 0 else wu.copy(),
                       w_s=float(a["w_s"]), w_x=float(a["w_x"]))
    return RP.assemble_problem(model, tree, w, a["p"].copy(), a["q"].copy())


def small_case(name, arrays, rng, fixed_iters=150, converge=True):
    inst = to_reference(arrays)
    out = dict(arrays)
    cache = RS.factor_step(inst)
    out["u_part"] = cache.u_part
    out["e_offset"] = cache.e_offset
    out["t_mat"] = np.stack(cache.t_mat)
    out["d_gain"] = np.stack(cache.d_gain)
    y = rng.standard_normal(inst.n_dual)
    z, val = RS.dual_gradient(cache, inst, y)
    out["dg_y"], out["dg_z"], out["dg_value"] = y, z, np.array(val)
    z0, val0 = RS.dual_gradient(cache, inst, np.zeros(inst.n_dual))
    out["dg0_z"], out["dg0_value"] = z0, np.array(val0)
    w = 5.0 * rng.standard_normal(inst.n_dual)
    gam = float(0.3 + rng.random())
    out["prox_w"], out["prox_gamma"] = w, np.array(gam)
    out["prox_conj"] = RP.prox_g_conjugate(inst, w, gam)
    out["prox_plain"] = RP.prox_g(inst, w, gam)
    L = RS.estimate_lipschitz(cache, inst)
    out["lipschitz"] = np.array(L)
    cfg = RS.SolverConfig(max_iter=fixed_iters, tol=1e-30, gamma=1.0 / L,
                          gap_check_every=fixed_iters + 1)
    res = RS.solve(inst, cfg, cache=cache)
    for k in ("u0", "primal", "primal_avg", "dual"):
        out[f"fixed_{k}"] = getattr(res, k)
    for k in ("duality_gap", "objective", "primal_residual", "dual_change"):
        out[f"fixed_{k}"] = np.array(getattr(res, k))
    out["fixed_iters"] = np.array(fixed_iters)
    if converge:
        res = RS.solve(inst, RS.SolverConfig(max_iter=4000, tol=1e-4), cache=cache)
        out["conv_iterations"] = np.array(res.iterations)
        out["conv_termination"] = np.array(res.termination)
        out["conv_u0"] = res.u0
        out["conv_gap"] = np.array(res.duality_gap)
        out["conv_objective"] = np.array(res.objective)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, "n =", inst.n_nonroot, "L =", L)


def barcelona_case(name, iters, full_rows, stride=23):
    mine = config_instance(name)
    arrays = instance_to_arrays(mine)
    inst = to_reference(arrays)
    t0 = time.time()
    cache = RS.factor_step(inst)
    L = RS.estimate_lipschitz(cache, inst)
    cfg = RS.SolverConfig(max_iter=iters, tol=1e-30, gamma=1.0 / L, gap_check_every=iters + 1)
    res = RS.solve(inst, cfg, cache=cache)
    out = {"lipschitz": np.array(L), "iters": np.array(iters),
           "instance_digest": np.frombuffer(digest(arrays), dtype=np.uint8)}
    for k in ("duality_gap", "objective", "primal_residual", "dual_change"):
        out[k] = np.array(getattr(res, k))
    out["u0"] = res.u0
    n = inst.n_nonroot
    rows = np.arange(n) if full_rows else np.unique(np.concatenate(
        [np.arange(inst.stage_slices[0].stop), np.arange(0, n, stride), [n - 1]]))
    out["rows"] = rows
    for k in ("primal", "primal_avg", "dual"):
        v = getattr(res, k).reshape(n, -1)
        out[k + "_rows"] = v[rows]
        out[k + "_norm"] = np.array(np.linalg.norm(v))
    out["e_offset_rows"] = cache.e_offset[rows]
    np.savez_compressed(os.path.join(HERE, f"barcelona_{name}.npz"), **out)
    print(name, "n =", n, "L =", L, "time", time.time() - t0)


def digest(arrays) -> bytes:
    import hashlib
    h = hashlib.sha256()
    for k in sorted(arrays):
        h.update(k.encode())
        h.update(np.ascontiguousarray(arrays[k]).tobytes())
    return h.digest()


def main():
    rng = np.random.default_rng(20240811)
    cases = {
        "small_plain": dict(horizon=3, max_nodes=20),
        "small_coupled": dict(n_inputs=5, n_mixing=2, horizon=3, max_nodes=15),
        "small_dense_a": dict(n_tanks=2, n_inputs=4, n_mixing=1, horizon=4, max_nodes=18,
                              identity_a=False),
        "small_chain": dict(n_tanks=2, n_inputs=3, horizon=6, max_nodes=7),
        "small_wide": dict(n_tanks=4, n_inputs=6, n_demands=3, n_mixing=1, horizon=5, max_nodes=40),
    }
    for name, kw in cases.items():
        inst = make_instance(rng, **kw)
        small_case(name, instance_to_arrays(inst), rng)
    if "--large" in sys.argv:
        # Round 2: the production graph kernels at C3/C4 against the reference
        # itself. C4 takes ~4.6 s per reference iteration
        # plus a ~170 s certificate, so it runs 50 iterations.
        barcelona_case("C3", 500, full_rows=False, stride=23)
        barcelona_case("C4", 50, full_rows=False, stride=97)
        return
    if "--no-barcelona" not in sys.argv:
        barcelona_case("C1", 500, full_rows=True)
        barcelona_case("C2", 500, full_rows=False)


if __name__ == "__main__":
    main()
