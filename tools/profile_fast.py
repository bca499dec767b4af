"""Per-phase clock breakdown of the persistent kernel: python tools/profile_fast.py CFG [ITERS]."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1904_10548_b200 import factor_step
from paper_1904_10548_b200 import _native as nat
from paper_1904_10548_b200 import solver as S
from paper_1904_10548_b200.synthetic import config_instance
NAMES = ["total", "A", "B", "C", "D", "D:u-proj", "D:prox", "D:load", "sync", "steps", "A:load", "D:lsum", "D:bu+xscan", "prox_v", "prox_norm", "prox_out", "prox_yc", "A:compute", "-", "-"]
for cfg in sys.argv[1].split(","):
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    inst = config_instance(cfg)
    cache = factor_step(inst)
    ctx = cache._bind()
    S._upload_bounds(ctx, inst)
    th = S.theta_sequence(iters + 2); be = S._beta_table(th)
    ctx.call("wmpc_apg_begin", 1 / 5e9, iters + 2, nat.ptr(th), nat.ptr(be))
    ctx.call("wmpc_apg_run", 2)
    buf = (nat.C.c_uint64 * (148 * 20))()
    ctx.call("wmpc_profile_fast", iters, buf, 148 * 20)
    a = np.array(buf[:], dtype=np.float64).reshape(148, 20) / 1.965e3 / iters  # us per iteration @1965 MHz
    busy = a[:, 9] > 0
    print(cfg, "busy CTAs", int(busy.sum()), "steps/iter (CTA0)", a[0, 9] * 1.965e3)
    for i, nm in enumerate(NAMES[:18]):
        if i == 9: continue
        print(f"  {nm:6s} mean(busy) {a[busy, i].mean():9.2f} us/it   max {a[:, i].max():9.2f}")
