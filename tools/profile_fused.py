"""Per-phase clock breakdown of k_chain_fused: python tools/profile_fused.py CFG [ITERS] (env as for sweep)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1904_10548_b200 import factor_step
from paper_1904_10548_b200 import _native as nat
from paper_1904_10548_b200 import solver as S
from paper_1904_10548_b200.synthetic import config_instance
NAMES = ["total", "D:load", "D:compute", "P:wait", "P:prox", "U:load", "U:compute"]
for cfg in sys.argv[1].split(","):
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    inst = config_instance(cfg)
    cache = factor_step(inst)
    ctx = cache._bind()
    S._upload_bounds(ctx, inst)
    th = S.theta_sequence(iters + 2); be = S._beta_table(th)
    ctx.call("wmpc_apg_begin", 1 / 5e9, iters + 2, nat.ptr(th), nat.ptr(be))
    ctx.call("wmpc_apg_run", 1)
    n = 4096 * 20
    buf = (nat.C.c_uint64 * n)()
    ctx.call("wmpc_profile_fast", iters, buf, n)
    a = np.array(buf[:], dtype=np.float64).reshape(-1, 20) / iters
    busy = a[:, 0] > 0
    print(cfg, "CTAs", int(busy.sum()), "(cycles per iteration per CTA)")
    for i, nm in enumerate(NAMES):
        print(f"  {nm:10s} mean {a[busy, i].mean():9.0f}   max {a[busy, i].max():9.0f}")
