"""Bit comparison of two kernel variants on the same solve: ab_bits.py CFG ITERS 'ENV_A' 'ENV_B'
(ENV as k=v,k=v). Prints max |diff| of y, U, X, u0 and the cost."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1904_10548_b200 import SolverConfig, factor_step, solve
from paper_1904_10548_b200.synthetic import config_instance

def run(cfg, iters, env, prec):
    kv = dict(x.split("=") for x in env.split(",") if x)
    for k, v in kv.items(): os.environ[k] = v
    inst = config_instance(cfg)
    cache = factor_step(inst)
    r = solve(inst, SolverConfig(max_iter=iters, tol=1e-30, gap_check_every=iters // 2, precision=prec), cache=cache)
    for k in kv: del os.environ[k]
    return r

cfg, iters, ea, eb = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4]
prec = sys.argv[5] if len(sys.argv) > 5 else "fp64"
ra, rb = run(cfg, iters, ea, prec), run(cfg, iters, eb, prec)
for name in ("u0", "primal", "primal_avg", "dual"):
    a, b = getattr(ra, name, None), getattr(rb, name, None)
    if a is None: continue
    a, b = np.asarray(a), np.asarray(b)
    print(cfg, prec, name, a.shape, "bit-equal" if np.array_equal(a, b) else f"max|d|={np.max(np.abs(a-b)):.3e} (max|a|={np.max(np.abs(a)):.3e})")
print(cfg, "objective", ra.objective, rb.objective, "gap", ra.duality_gap, rb.duality_gap, "iters", ra.iterations, rb.iterations)
