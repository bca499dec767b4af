"""Ordering hazards of the iteration kernels.

compute-sanitizer is closed on this GPU pool (it answers: "runs under it have
left GPUs needing a reset"), so racecheck / synccheck cannot run here. The
hazards it would look for in this code are (a) a kernel reading its
predecessor's output before that output is complete or visible (programmatic
dependent launch lets kernels start before their predecessors finish), and
(b) cross-lane shared-memory races inside a warp or CTA. Both make results
depend on timing, so every kernel family selected by default is run:
* with programmatic dependent launch (the default) three times, and once in
  plain stream order (wmpc_set_pdl(0)): all runs bit-identical;
* on a tree whose chains straddle many CTAs and warps (C3, C4-like shapes).
A violation shows up as a mismatch in any iterate, average or u0.
"""

from __future__ import annotations

import numpy as np
import pytest

from paper_1904_10548_b200 import SolverConfig, solve
from paper_1904_10548_b200 import _native as nat
from paper_1904_10548_b200 import solver as S
from paper_1904_10548_b200.synthetic import config_instance

pytestmark = pytest.mark.gpu

MODES = {  # name: (config, env, precision)
    "graph-c1": ("C1", {}, "fp64"),
    "ring-c3": ("C3", {"WMPC_DP": "0"}, "fp64"),
    "registers-c3": ("C3", {"WMPC_DP": "0", "WMPC_CHAINW": "1", "WMPC_CWPD": "1"}, "fp64"),
    "dp-whole-c3": ("C3", {"WMPC_DP": "1", "WMPC_DP_SEG": "0"}, "fp64"),
    "dp-segmented-c3": ("C3", {}, "fp64"),  # the C3 default: two warps per chain, flag handshake
    "graph-fp32-c2": ("C2", {}, "fp32"),
    "registers-fp32-c3": ("C3", {"WMPC_CHAINW": "1", "WMPC_CWPD": "1"}, "fp32"),
}


@pytest.mark.parametrize("mode", list(MODES))
def test_results_independent_of_launch_overlap(mode, monkeypatch):
    cfg, env, prec = MODES[mode]
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    inst = config_instance(cfg)
    cache = S._factor(inst, None, private=True)
    ctx = cache._bind()
    conf = SolverConfig(max_iter=60, tol=1e-30, gamma=1 / 2e9, gap_check_every=20, precision=prec)
    runs = []
    for pdl in (1, 1, 1, 0):
        nat.load().wmpc_set_pdl(ctx.h, pdl)
        r = solve(inst, conf, cache=cache)
        runs.append(r)
    nat.load().wmpc_set_pdl(ctx.h, 1)
    for r in runs[1:]:
        for k in ("u0", "primal", "primal_avg", "dual"):
            np.testing.assert_array_equal(getattr(r, k), getattr(runs[0], k), err_msg=f"{mode} {k}")
        assert r.duality_gap == runs[0].duality_gap and r.objective == runs[0].objective


def test_dp_at_c4_independent_of_launch_overlap():
    """The C4 default (k_chain_dp, 147 persistent CTAs x 7 warps, branch
    groups reading the branching rows' Yc written by the previous k_chain_dp)."""
    inst = config_instance("C4")
    cache = S._factor(inst, None, private=True)
    ctx = cache._bind()
    assert nat.path_info(ctx)["fused_dp"] == 1
    conf = SolverConfig(max_iter=12, tol=1e-30, gamma=1 / 2e9, gap_check_every=5)
    runs = []
    for pdl in (1, 1, 0):
        nat.load().wmpc_set_pdl(ctx.h, pdl)
        runs.append(solve(inst, conf, cache=cache))
    nat.load().wmpc_set_pdl(ctx.h, 1)
    for r in runs[1:]:
        for k in ("u0", "primal_avg", "dual"):
            np.testing.assert_array_equal(getattr(r, k), getattr(runs[0], k), err_msg=k)
