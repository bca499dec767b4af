"""Global Dykstra stop sweep (the reference's rule: first sweep whose max movement
<= 1e-13 (1 + max|Ua|)) at several points of a solve."""
import os, sys
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
for target in (25, 50, 100, 250, 500, 1000, 2000, 3000, 5000):
    ctx.call("wmpc_apg_run", target - done); done = target
    S._check(ctx)
    amax = np.zeros(1)
    ctx.call("wmpc_cert_absmax", nat.ptr(amax))
    mv = np.zeros(500)
    ctx.call("wmpc_cert_dykstra", 500, nat.ptr(mv))
    tol = 1e-13 * (1 + amax[0])
    hit = np.nonzero(mv <= tol)[0]
    print(cfg, "iter", target, "stop sweep", int(hit[0]) + 1 if hit.size else "none(500)", "tol", tol,
          "mv[0,10,100,499]", mv[[0, 10, 100, 499]])
