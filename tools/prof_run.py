"""Small fixed-iteration solve for ncu captures: python tools/prof_run.py CFG ITERS."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1904_10548_b200 import SolverConfig, factor_step, solve
from paper_1904_10548_b200.synthetic import config_instance
cfg = sys.argv[1] if len(sys.argv) > 1 else "C1"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
inst = config_instance(cfg)
cache = factor_step(inst)
res = solve(inst, SolverConfig(max_iter=iters, tol=1e-30, gamma=1 / 5e9, gap_check_every=iters + 1), cache=cache)
print("ok", cfg, iters, res.duality_gap)
