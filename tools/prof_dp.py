"""Profile target: CFG [ITERS] -- factor, begin, ITERS graph-replayed APG
iterations (ncu attaches to the iteration kernels; env selects variants)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1904_10548_b200 import factor_step  # noqa: E402
from paper_1904_10548_b200 import _native as nat  # noqa: E402
from paper_1904_10548_b200 import solver as S  # noqa: E402
from paper_1904_10548_b200.synthetic import config_instance  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
inst = config_instance(cfg)
cache = factor_step(inst)
ctx = cache._bind()
print(nat.path_info(ctx))
S._upload_bounds(ctx, inst)
th = S.theta_sequence(iters + 1)
be = S._beta_table(th)
if os.environ.get("PROF_FP32") == "1":
    ctx.call("wmpc_set_precision", 1)
ctx.call("wmpc_apg_begin", 1.0 / 2e9, iters + 1, nat.ptr(th), nat.ptr(be))
ctx.call("wmpc_apg_run", iters)
ctx.call("wmpc_sync")
print("done")
