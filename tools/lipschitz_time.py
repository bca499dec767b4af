"""Time of estimate_lipschitz (device power iteration) per config."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1904_10548_b200 import estimate_lipschitz, factor_step
from paper_1904_10548_b200.synthetic import config_instance
for cfg in sys.argv[1:] or ["C2", "C4"]:
    inst = config_instance(cfg)
    cache = factor_step(inst)
    t0 = time.perf_counter()
    L = estimate_lipschitz(cache, inst)
    print(cfg, "L", L, "seconds", round(time.perf_counter() - t0, 3), flush=True)
