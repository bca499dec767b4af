"""Where the wall time of a public-API solve goes (host view), per call."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1904_10548_b200 import SolverConfig, estimate_lipschitz, factor_step
from paper_1904_10548_b200 import _native as nat
from paper_1904_10548_b200 import solver as S
from paper_1904_10548_b200.synthetic import config_instance
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
inst = config_instance(cfg)
cache = factor_step(inst)
L = estimate_lipschitz(cache, inst)
iters = 500
th = S.theta_sequence(iters); be = S._beta_table(th)
for rep in range(6):
    c2 = factor_step(inst, structure_from=cache)
    ctx = c2._bind()
    t = [time.perf_counter()]
    S._upload_bounds(ctx, inst); t.append(time.perf_counter())
    ctx.call("wmpc_apg_begin", 1.0 / L, iters, nat.ptr(th), nat.ptr(be)); t.append(time.perf_counter())
    ctx.call("wmpc_apg_run", iters); t.append(time.perf_counter())
    bufs = S._result_buffers(inst); t.append(time.perf_counter())
    S._check(ctx); t.append(time.perf_counter())
    S._read_async(ctx, True, bufs)
    S._certificate(ctx); t.append(time.perf_counter())
    ctx.call("wmpc_apg_read_wait"); t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(f"bounds {d[0]:.2f} begin {d[1]:.2f} launch {d[2]:.2f} bufs {d[3]:.2f} check(wait) {d[4]:.2f} "
          f"cert+read {d[5]:.2f} read_wait {d[6]:.2f} total {sum(d):.2f} ms")
