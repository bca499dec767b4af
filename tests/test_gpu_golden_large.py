"""C3 / C4 fixed-iteration solves through the PRODUCTION iteration kernels
against the reference's own outputs.

``tests/golden/barcelona_C3.npz`` (500 iterations) and ``barcelona_C4.npz``
(50 iterations) were produced by running the reference ``watermpc.solve``
itself (``tests/golden/make_golden.py --large``) with gamma = 1/L from the
reference's own ``estimate_lipschitz``, tol = 1e-30 and no gap checks. They
store sampled rows (every stage-1 row, every 23rd / 97th row, the last row),
the full-vector norms, u0, the gap and the objective.

Each test first asserts which kernels the solve runs (``path_info``): the
structured graph path, with the fused warp-per-chain iteration kernel at C4.
Tolerance: the north_star's 1e-8 relative (metric of test_solver.py:21-22).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import instance_to_arrays, load_golden, rel_err
from paper_1904_10548_b200 import SolverConfig, factor_step, solve
from paper_1904_10548_b200 import _native as nat
from paper_1904_10548_b200.synthetic import config_instance

pytestmark = pytest.mark.gpu

TOL = 1e-8


def _digest(arrays) -> bytes:
    import hashlib
    h = hashlib.sha256()
    for k in sorted(arrays):
        h.update(k.encode())
        h.update(np.ascontiguousarray(arrays[k]).tobytes())
    return h.digest()


def _solve_vs_golden(name, precision="fp64", tol=TOL):
    g = load_golden(f"barcelona_{name}.npz")
    inst = config_instance(name)
    assert _digest(instance_to_arrays(inst)) == bytes(g["instance_digest"]), "synthetic instance drifted"
    L = float(g["lipschitz"])
    it = int(g["iters"])
    cache = factor_step(inst)
    info = nat.path_info(cache._bind())
    res = solve(inst, SolverConfig(max_iter=it, tol=1e-30, gamma=1.0 / L, gap_check_every=it + 1,
                                   precision=precision), cache=cache)
    n = inst.n_nonroot
    rows = g["rows"]
    errs = {}
    for k in ("primal", "primal_avg", "dual"):
        v = getattr(res, k).reshape(n, -1)
        errs[k] = rel_err(v[rows], g[k + "_rows"])
        errs[k + "_norm"] = abs(np.linalg.norm(v) - float(g[k + "_norm"])) / (1 + float(g[k + "_norm"]))
    errs["u0"] = rel_err(res.u0, g["u0"])
    for k in ("duality_gap", "objective"):
        want = float(g[k])
        errs[k] = abs(getattr(res, k) - want) / (1 + abs(want))
    return info, errs


def test_c3_500_iterations_production_path_vs_reference_golden():
    info, errs = _solve_vs_golden("C3")
    assert info["fast_path"] == 300, info
    assert info["fused_dp"] == 1 and info["dp_segm"] > 0, info  # the C3 default: segmented k_chain_dp
    bad = {k: v for k, v in errs.items() if not v <= TOL}
    assert not bad, (bad, info)


def test_c4_50_iterations_production_path_vs_reference_golden():
    info, errs = _solve_vs_golden("C4")
    assert info["fast_path"] == 300, info
    assert info["fused_dp"] == 1 or info["chainw"] == 1, info  # the warp-per-chain kernels benchmarked at C4
    bad = {k: v for k, v in errs.items() if not v <= TOL}
    assert not bad, (bad, info)


def test_c4_fp32_mode_vs_reference_golden():
    """fp32 mode (dual-gradient kernels in fp32, dual / prox / certificate in
    fp64) against the fp64 reference: its own stated tolerance, 1e-4."""
    info, errs = _solve_vs_golden("C4", precision="fp32")
    bad = {k: v for k, v in errs.items() if not v <= 1e-4}
    assert not bad, (bad, info)


def test_c3_fp32_mode_vs_reference_golden():
    info, errs = _solve_vs_golden("C3", precision="fp32")
    bad = {k: v for k, v in errs.items() if not v <= 1e-4}
    assert not bad, (bad, info)
