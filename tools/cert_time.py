"""Certificate wall time at several points of a solve (C5 certifies at every check)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1904_10548_b200 import factor_step, estimate_lipschitz
from paper_1904_10548_b200 import _native as nat
from paper_1904_10548_b200 import solver as S
from paper_1904_10548_b200.synthetic import config_instance
cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
inst = config_instance(cfg)
cache = factor_step(inst)
L = estimate_lipschitz(cache, inst)
ctx = cache._bind()
S._upload_bounds(ctx, inst)
N = 5000
th = S.theta_sequence(N); be = S._beta_table(th)
ctx.call("wmpc_apg_begin", 1.0 / L, N, nat.ptr(th), nat.ptr(be))
done = 0
out = []
for target in (25, 50, 100, 250, 500, 1000, 2500, 5000):
    ctx.call("wmpc_apg_run", target - done); done = target
    S._check(ctx)
    S._certificate(ctx)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter(); g = S._certificate(ctx); ts.append(time.perf_counter() - t0)
    out.append(f"{target}:{min(ts)*1e3:.2f}ms")
print(cfg, " ".join(out))
