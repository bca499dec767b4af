"""cProfile of the public-API step (factor_step(structure_from) + solve) in steady state."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1904_10548_b200 import SolverConfig, estimate_lipschitz, factor_step, solve
from paper_1904_10548_b200 import _native as nat
from paper_1904_10548_b200.synthetic import config_instance
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
inst = config_instance(cfg)
cache = factor_step(inst)
L = estimate_lipschitz(cache, inst)
sc = SolverConfig(max_iter=500, tol=1e-30, gamma=1.0 / L, gap_check_every=501)
inst.demand = nat.pinned_copy(inst.demand); inst.demand_gd = nat.pinned_copy(inst.demand_gd); inst.econ = nat.pinned_copy(inst.econ)
res = None
for _ in range(4):
    c2 = factor_step(inst, structure_from=cache); res = solve(inst, sc, cache=c2)
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
for _ in range(10):
    c2 = factor_step(inst, structure_from=cache); res = solve(inst, sc, cache=c2)
pr.disable()
print("ms per step", (time.perf_counter() - t0) * 100)
st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(18)
