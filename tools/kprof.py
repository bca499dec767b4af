"""Per-kernel device time per APG iteration (wmpc_iteration_profile) for configs:
kprof.py C2 C3 C4 [--fp32] [--shard8] > json."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
from paper_1904_10548_b200 import factor_step, shard  # noqa: E402
from paper_1904_10548_b200 import _native as nat  # noqa: E402
from paper_1904_10548_b200 import solver as S  # noqa: E402
from paper_1904_10548_b200.synthetic import config_instance  # noqa: E402


def prof(ctx, inst, count=30, fp32=False):
    S._upload_bounds(ctx, inst)
    ctx.call("wmpc_set_precision", 1 if fp32 else 0)
    th = S.theta_sequence(count + 3)
    be = S._beta_table(th)
    ctx.call("wmpc_apg_begin", 1 / 2e9, count + 3, nat.ptr(th), nat.ptr(be))
    ctx.call("wmpc_apg_run", 3)
    out = np.zeros(4)
    ctx.call("wmpc_iteration_profile", count, nat.ptr(out), 4)
    info = nat.path_info(ctx)
    names = ["grp", "k_chain_dp"] if info["fused_dp"] else ["up", "grp", "down", "prox"]
    return {"path": info, "us": {k: round(v * 1e3, 2) for k, v in zip(names, out)}}


res = {}
fp32 = "--fp32" in sys.argv
for cfg in [a for a in sys.argv[1:] if a.startswith("C")]:
    inst = config_instance(cfg)
    cache = factor_step(inst)  # keep the cache alive: its context dies with it
    res[cfg] = prof(cache._bind(), inst, fp32=fp32)
print(json.dumps(res))
