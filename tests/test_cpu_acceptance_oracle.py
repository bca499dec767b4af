"""oracle/acceptance.py (the reference's grid / dense-KKT / restoration
helpers restated for the GPU acceptance tests) against the reference itself,
live, in the build container (skipped on the GPU box, where the reference is
not mounted)."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

from conftest import ROOT, import_reference, instance_to_arrays, make_instance
from oracle import acceptance as A


def _ref(inst):
    import_reference()
    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    from make_golden import to_reference
    return to_reference(instance_to_arrays(inst))


def test_brute_force_min_matches_reference(rng):
    import_reference()
    from watermpc.oracle import brute_force_min
    inst = make_instance(rng, n_tanks=1, n_inputs=1, n_demands=1, horizon=2, max_nodes=3)
    z, v = A.brute_force_min(inst)
    zr, vr = brute_force_min(_ref(inst))
    np.testing.assert_allclose(z, zr, rtol=0, atol=1e-12 * (1 + np.abs(zr).max()))
    assert v == pytest.approx(vr, rel=1e-13)


def test_duality_gap_and_projection_match_reference(rng):
    import_reference()
    from watermpc.oracle import duality_gap, project_primal_feasible
    from watermpc.problem import primal_objective
    inst = make_instance(rng, n_mixing=1, horizon=2, max_nodes=8)
    rinst = _ref(inst)
    z = rng.standard_normal(inst.n_primal) * 5.0
    y = rng.standard_normal(inst.n_dual)
    zf = A.project_primal_feasible(inst, z)
    np.testing.assert_allclose(zf, project_primal_feasible(rinst, z), rtol=0, atol=1e-11)
    assert A.primal_objective(inst, zf) == pytest.approx(primal_objective(rinst, zf), rel=1e-12)
    assert A.duality_gap(inst, z, y) == pytest.approx(duality_gap(rinst, z, y), rel=1e-9, abs=1e-9)


def test_projection_restores_feasibility(rng):
    """test_oracle.py:141-150 on the restatement."""
    inst = make_instance(rng, n_mixing=1, horizon=2, max_nodes=8)
    z = rng.standard_normal(inst.n_primal) * 5.0
    U, _ = A.split_primal(inst, A.project_primal_feasible(inst, z))
    m = inst.model
    assert np.all(U >= m.u_min) and np.all(U <= m.u_max)
    resid = U @ m.E.T + inst.demand @ m.Ed.T
    assert float(np.max(np.abs(resid))) <= 1e-8 * (1 + float(np.max(np.abs(U))))
    assert np.isfinite(A.eval_f(inst, A.project_primal_feasible(inst, z)))
