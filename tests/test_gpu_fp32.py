"""fp32 mode: dual-gradient kernels in fp32, dual iterate, prox,
averages and certificate in fp64. Own tolerance: 1e-4 relative (the
reference's metric, test_solver.py:21-22) against the fp64 solve."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import rel_err
from paper_1904_10548_b200 import SolverConfig, factor_step, solve
from paper_1904_10548_b200 import _native as nat
from paper_1904_10548_b200.synthetic import config_instance

pytestmark = pytest.mark.gpu
FP32_TOL = 1e-4


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3"])
def test_fp32_mode_within_its_tolerance(cfg):
    inst = config_instance(cfg)
    base = dict(max_iter=200, tol=1e-30, gamma=1.0 / 2e9, gap_check_every=50)
    r64 = solve(inst, SolverConfig(**base), cache=factor_step(inst))
    r32 = solve(inst, SolverConfig(**base, precision="fp32"), cache=factor_step(inst))
    for k in ("u0", "primal", "primal_avg", "dual"):
        err = rel_err(getattr(r32, k), getattr(r64, k))
        assert err <= FP32_TOL, (k, err)
        if k != "u0":  # u0 may sit on its clip bounds in both
            assert err > 0.0, k  # the fp32 kernels really ran
    assert abs(r32.duality_gap - r64.duality_gap) <= FP32_TOL * (1 + abs(r64.duality_gap))


def test_fp32_mode_switches_back():
    inst = config_instance("C1")
    base = dict(max_iter=50, tol=1e-30, gamma=1.0 / 2e9, gap_check_every=51)
    cache = factor_step(inst)
    a = solve(inst, SolverConfig(**base), cache=cache)
    solve(inst, SolverConfig(**base, precision="fp32"), cache=cache)
    b = solve(inst, SolverConfig(**base), cache=cache)
    np.testing.assert_array_equal(a.dual, b.dual)


def test_fp32_config_validation():
    with pytest.raises(ValueError, match="precision"):
        SolverConfig(precision="fp16")
