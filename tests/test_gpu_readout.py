"""Result readout (solver._read_async + pooled page-locked arrays): results a
caller still holds, or any view of them, are never recycled into a later
solve; dropped results are recycled."""

from __future__ import annotations

import gc

import numpy as np
import pytest

from paper_1904_10548_b200 import SolverConfig, factor_step, solve
from paper_1904_10548_b200 import _native as nat
from paper_1904_10548_b200.synthetic import config_instance

pytestmark = pytest.mark.gpu


def _solve(inst, cache, iters):
    return solve(inst, SolverConfig(max_iter=iters, tol=1e-30, gamma=1.0 / 2e9, gap_check_every=iters + 1),
                 cache=cache)


def test_held_results_and_views_survive_later_solves():
    inst = config_instance("C1")
    cache = factor_step(inst)
    r1 = _solve(inst, cache, 30)
    keep = {k: getattr(r1, k).copy() for k in ("u0", "primal", "primal_avg", "dual")}
    view = r1.dual[100:200]
    view_copy = view.copy()
    for iters in (5, 60, 7):  # different results into the same-sized pooled blocks
        r = _solve(inst, cache, iters)
        assert not np.array_equal(r.dual, keep["dual"])
    for k, v in keep.items():
        np.testing.assert_array_equal(getattr(r1, k), v, err_msg=k)
    del r1
    gc.collect()
    for iters in (9, 11):
        _solve(inst, cache, iters)
    np.testing.assert_array_equal(view, view_copy)


def test_dropped_results_are_recycled():
    inst = config_instance("C1")
    cache = factor_step(inst)
    r = _solve(inst, cache, 10)
    ptr = r.primal.ctypes.data
    del r
    gc.collect()
    r2 = _solve(inst, cache, 10)
    pool_ptrs = {r2.u0.ctypes.data, r2.primal.ctypes.data, r2.primal_avg.ctypes.data, r2.dual.ctypes.data}
    assert ptr in pool_ptrs  # the freed block came back from the pool


def test_pinned_empty_shapes():
    a = nat.pinned_empty(0)
    assert a.shape == (0,)
    b = nat.pinned_empty(17)
    b[:] = np.arange(17.0)
    assert b.sum() == 136.0
