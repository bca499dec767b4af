"""Per-iteration device time of the APG loop for configs x knobs."""
import json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1904_10548_b200 import factor_step
from paper_1904_10548_b200 import _native as nat
from paper_1904_10548_b200 import solver as S
from paper_1904_10548_b200.synthetic import config_instance

def loop_time(cfg, iters, env):
    for k, v in env.items(): os.environ[k] = v
    inst = config_instance(cfg)
    cache = factor_step(inst)
    ctx = cache._bind()
    S._upload_bounds(ctx, inst)
    th = S.theta_sequence(iters + 5); be = S._beta_table(th)
    ctx.call("wmpc_set_precision", 1 if env.get("FP32") == "1" else 0)
    ctx.call("wmpc_apg_begin", 1 / 5e9, iters + 5, nat.ptr(th), nat.ptr(be))
    ctx.call("wmpc_apg_run", 5)
    ms = nat.C.c_float()
    ctx.call("wmpc_apg_run_timed", iters, nat.C.byref(ms))
    mode = nat.load().wmpc_fast_path(ctx.h)
    for k in env: del os.environ[k]
    return ms.value * 1e3 / iters, mode, inst.n_nonroot

import ast
cases = ast.literal_eval(sys.argv[1]) if len(sys.argv) > 1 else [
    ("C1", {}), ("C1", {"WMPC_KERNEL": "cta"}), ("C2", {}), ("C2", {"WMPC_KERNEL": "cta"}),
    ("C3", {}), ("C3", {"WMPC_KERNEL": "cta"}), ("C4", {}), ("C4", {"WMPC_KERNEL": "cta"})]
for cfg, env in cases:
    iters = 50 if cfg != "C4" else 10
    us, mode, n = loop_time(cfg, iters, env)
    gbs = 10016 * n / (us * 1e-6) / 1e9
    print(json.dumps({"cfg": cfg, "env": env, "us_per_iter": round(us, 2), "mc": mode, "nodes": n,
                      "alg_GBs": round(gbs, 1)}), flush=True)
