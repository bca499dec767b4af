"""Wall time of factor_step(structure_from) in steady state (pinned inputs, caches recycled)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1904_10548_b200 import factor_step
from paper_1904_10548_b200 import _native as nat
from paper_1904_10548_b200.synthetic import config_instance
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
inst = config_instance(cfg)
cache = factor_step(inst)
inst.demand = nat.pinned_copy(inst.demand); inst.demand_gd = nat.pinned_copy(inst.demand_gd); inst.econ = nat.pinned_copy(inst.econ)
c2 = None
ts = []
for rep in range(12):
    t0 = time.perf_counter()
    c2 = factor_step(inst, structure_from=cache)
    ts.append(time.perf_counter() - t0)
print(cfg, "factor_step(structure_from) ms", np.round(np.array(ts[4:]) * 1e3, 3))
