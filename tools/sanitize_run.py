"""Small solves for compute-sanitizer (tools/sanitize.sh): sanitize_run.py MODE.

MODE selects the kernel family (env switches are read at context creation):
  graph-c1     C1 default graph (CTA chain kernels, branch groups, warp prox) + certificate
  chainw-c3    C3 default (warp-per-chain ring kernels) + certificate
  chainw-r-c1  C1 with the register warp-per-chain kernels (the C4 fp32 / certificate path)
  dp-c1        C1 with k_chain_dp (the C4 fp64 default) + certificate + warm start
  fp32-c1      C1 fp32 mode
  general      random dense instance (general per-stage path) + power iteration + prox API
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

mode = sys.argv[1]
env = {"chainw-r-c1": {"WMPC_CHAINW": "1", "WMPC_CWPD": "1"}, "dp-c1": {"WMPC_DP": "1"},
       "chainw-c3": {}, "graph-c1": {}, "fp32-c1": {}, "general": {}}[mode]
os.environ.update(env)
from paper_1904_10548_b200 import SolverConfig, estimate_lipschitz, factor_step, prox_g_conjugate, solve  # noqa: E402
from paper_1904_10548_b200 import _native as nat  # noqa: E402
from paper_1904_10548_b200.synthetic import config_instance  # noqa: E402

if mode == "general":
    from conftest import make_instance
    inst = make_instance(np.random.default_rng(3), n_mixing=1, horizon=3, max_nodes=12)
    cache = factor_step(inst)
    estimate_lipschitz(cache, inst)
    r = solve(inst, SolverConfig(max_iter=30, tol=1e-30, gap_check_every=31), cache=cache)
    prox_g_conjugate(inst, np.random.default_rng(1).standard_normal(inst.n_dual), 0.7)
else:
    inst = config_instance("C3" if mode.endswith("c3") else "C1")
    cache = factor_step(inst)
    print(nat.path_info(cache._bind()), flush=True)
    prec = "fp32" if mode.startswith("fp32") else "fp64"
    r = solve(inst, SolverConfig(max_iter=12, tol=1e-30, gamma=1 / 2e9, gap_check_every=6, precision=prec),
              cache=cache)
    if mode == "dp-c1":
        solve(inst, SolverConfig(max_iter=6, tol=1e-30, gamma=1 / 2e9, gap_check_every=7), cache=cache,
              y_init=r.dual)
print("ok", mode, flush=True)
