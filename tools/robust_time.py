"""us per APG iteration on the non-uniform C4-scale tree and on the coupled
mixing-node network (fallback kernels): robust_time.py > json."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1904_10548_b200 import factor_step  # noqa: E402
from paper_1904_10548_b200 import _native as nat  # noqa: E402
from paper_1904_10548_b200 import solver as S  # noqa: E402
from paper_1904_10548_b200.synthetic import CONFIGS, barcelona_instance, fan_like_instance  # noqa: E402


def us_it(inst, iters):
    cache = factor_step(inst)
    ctx = cache._bind()
    S._upload_bounds(ctx, inst)
    th = S.theta_sequence(iters + 5)
    be = S._beta_table(th)
    best = 1e30
    for _ in range(3):
        ctx.call("wmpc_apg_begin", 1 / 2e9, iters + 5, nat.ptr(th), nat.ptr(be))
        ctx.call("wmpc_apg_run", 5)
        ms = nat.C.c_float(0.0)
        ctx.call("wmpc_apg_run_timed", iters, nat.C.byref(ms))
        best = min(best, ms.value / iters * 1e3)
    return {"nodes": inst.n_nonroot, "us_per_iteration": best, "bytes_frac_of_hbm":
            10016 * inst.n_nonroot / (best * 1e-6) / 1e9 / 6551.7, "path": nat.path_info(ctx)}


out = {"fan_like_4096": us_it(fan_like_instance(), 50)}
for cfg in ("C2", "C3"):
    out[f"coupled_mixing_8_links_{cfg}"] = us_it(barcelona_instance(CONFIGS[cfg], mixing_links=8), 50)
    out[f"uncoupled_{cfg}"] = us_it(barcelona_instance(CONFIGS[cfg]), 50)
print(json.dumps(out))
