"""Run one C-config solve of a few iterations and the certificate (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1904_10548_b200 import factor_step
from paper_1904_10548_b200 import _native as nat
from paper_1904_10548_b200 import solver as S
from paper_1904_10548_b200.synthetic import config_instance
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
inst = config_instance(cfg)
cache = factor_step(inst)
ctx = cache._bind()
S._upload_bounds(ctx, inst)
th = S.theta_sequence(40); be = S._beta_table(th)
ctx.call("wmpc_apg_begin", 1 / 5e9, 40, nat.ptr(th), nat.ptr(be))
ctx.call("wmpc_apg_run", 30)
S._check(ctx)
S._certificate(ctx)
S._certificate(ctx)
print("done")
