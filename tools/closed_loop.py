"""Config C5: closed-loop receding horizon, 168 hourly steps on the 512-scenario
tree (C3), tol = 5e-2, cold (reference behaviour) vs warm-started dual.
python tools/closed_loop.py [h_sim] [max_iter] > profiles/...json
max_iter defaults to the reference's SolverConfig default, 20,000 (solver.py:62);
per step the termination (certified by the duality gap vs the iteration cap)
and the final gap are recorded."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1904_10548_b200 import SolverConfig
from paper_1904_10548_b200.simulate import (SimulationConfig, kpi_complexity, kpi_economic, kpi_safety,
                                            run_closed_loop)
from paper_1904_10548_b200.synthetic import CONFIGS, closed_loop_scenario

h = int(sys.argv[1]) if len(sys.argv) > 1 else 168
max_iter = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
sc = closed_loop_scenario(CONFIGS["C3"], h_sim=h)
out = {"config": "C5: barcelona-63t-114u-88d-17m, tree C3 [4,4,4,2,2,2] (512 scenarios, 10,196 nodes), "
                 f"H=24, {h} hourly steps, tol 5e-2, gap check every 25, max_iter {max_iter}"}
for warm in (False, True):
    cfg = SimulationConfig(h_sim=h, weights=sc["weights"], x0=sc["x0"], warm_start=warm,
                           solver=SolverConfig(max_iter=max_iter, tol=5e-2, gap_check_every=25))
    t0 = time.perf_counter()
    log = run_closed_loop(sc["model"], sc["tree_template"], sc["forecaster"], sc["realized_demand"],
                          sc["realized_price"], cfg)
    wall = time.perf_counter() - t0
    out["warm" if warm else "cold"] = {
        "wall_s": wall, "solve_s_total": float(log.solve_time_s.sum()),
        "kpi_economic": kpi_economic(log), "kpi_safety_m3": kpi_safety(log),
        "kpi_complexity_s": kpi_complexity(log), "iterations_total": int(log.iterations.sum()),
        "iterations_mean": float(log.iterations.mean()), "iterations_max": int(log.iterations.max()),
        "steps_at_max_iter": int((log.iterations >= max_iter).sum()),
        "steps_certified": int((log.iterations < max_iter).sum()),
        "median_step_ms": float(np.median(log.solve_time_s) * 1e3),
        "max_step_ms": float(np.max(log.solve_time_s) * 1e3),
        "final_gap_median": float(np.median(log.duality_gap)), "final_gap_max": float(np.max(log.duality_gap)),
        "per_step": {"iterations": log.iterations.tolist(), "gap": log.duality_gap.tolist(),
                     "solve_ms": (log.solve_time_s * 1e3).round(3).tolist()}}
    print(json.dumps({k: v for k, v in out["warm" if warm else "cold"].items() if k != "per_step"}),
          file=sys.stderr, flush=True)
print(json.dumps(out))
