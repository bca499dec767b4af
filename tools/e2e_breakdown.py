"""Wall-clock breakdown of one public-API solve step (factor_step + solve)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1904_10548_b200 import SolverConfig, estimate_lipschitz, factor_step, solve
from paper_1904_10548_b200 import _native as nat
from paper_1904_10548_b200 import solver as S
from paper_1904_10548_b200.synthetic import config_instance

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
inst = config_instance(cfg)
cache = factor_step(inst)
L = estimate_lipschitz(cache, inst)
sc = SolverConfig(max_iter=500, tol=1e-30, gamma=1.0 / L, gap_check_every=501)
inst.demand = nat.pinned_copy(inst.demand)
inst.demand_gd = nat.pinned_copy(inst.demand_gd)
inst.econ = nat.pinned_copy(inst.econ)
for _ in range(3):
    c2 = factor_step(inst, structure_from=cache)
    res = solve(inst, sc, cache=c2)  # kept alive like the timed loop (pinned result pool)
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    c2 = factor_step(inst, structure_from=cache)
    t1 = time.perf_counter()
    res = solve(inst, sc, cache=c2)
    t2 = time.perf_counter()
    ts.append((t1 - t0, t2 - t1))
ts = np.array(ts) * 1e3
print(cfg, "factor_step ms", np.round(ts[:, 0], 2), "solve ms", np.round(ts[:, 1], 2))
ctx = c2._bind()
for name, fn in [("certificate", lambda: S._certificate(ctx)),
                 ("read_all", lambda: S._read(ctx, inst, True, u0=True, primal=True, avg=True, dual=True))]:
    fn()
    t0 = time.perf_counter(); fn(); print(name, "ms", round((time.perf_counter() - t0) * 1e3, 2))
