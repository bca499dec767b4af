"""A/B of iteration kernels by environment: dp_time.py CFG ITERS K=V[,K=V] [K=V ...].

Each variant runs in its own process; prints us per APG iteration (graph
replay, CUDA events; fp64 and fp32 modes), the kernel selection (path_info)
and the relative difference of a 60-iteration fixed-step solve against the
first variant (metric of test_solver.py:21-22)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(cfg, iters, out):
    sys.path.insert(0, ROOT)
    import numpy as np
    from paper_1904_10548_b200 import SolverConfig, factor_step, solve
    from paper_1904_10548_b200 import _native as nat
    from paper_1904_10548_b200 import solver as S
    from paper_1904_10548_b200.synthetic import config_instance
    inst = config_instance(cfg)
    cache = factor_step(inst)
    ctx = cache._bind()
    info = nat.path_info(ctx)
    r = solve(inst, SolverConfig(max_iter=60, tol=1e-30, gap_check_every=61, gamma=1 / 2e9), cache=cache)
    np.savez(out, dual=r.dual, primal=r.primal, primal_avg=r.primal_avg, u0=r.u0,
             gap=r.duality_gap, obj=r.objective)
    S._upload_bounds(ctx, inst)
    th = S.theta_sequence(iters + 5)
    be = S._beta_table(th)
    res = {"info": info}
    for prec in (0, 1):
        try:
            ctx.call("wmpc_set_precision", prec)
        except Exception as e:  # noqa: BLE001
            res["fp32"] = str(e)
            continue
        best = 1e9
        for _ in range(3):
            ctx.call("wmpc_apg_begin", 1.0 / 2e9, iters + 5, nat.ptr(th), nat.ptr(be))
            ctx.call("wmpc_apg_run", 5)
            ms = nat.C.c_float(0.0)
            ctx.call("wmpc_apg_run_timed", iters, nat.C.byref(ms))
            best = min(best, ms.value / iters * 1e3)
        res["fp32" if prec else "fp64"] = round(best, 2)
    ctx.call("wmpc_set_precision", 0)
    print("RESULT", json.dumps(res))


def rel(a, b):
    import numpy as np
    return float(np.linalg.norm(a - b) / (1 + np.linalg.norm(b)))


if __name__ == "__main__":
    if sys.argv[1] == "--child":
        child(sys.argv[2], int(sys.argv[3]), sys.argv[4])
        sys.exit(0)
    import numpy as np
    cfg, iters, variants = sys.argv[1], sys.argv[2], sys.argv[3:] or [""]
    outs = []
    for k, var in enumerate(variants):
        env = dict(os.environ)
        env.update(dict(kv.split("=") for kv in var.split(",") if kv))
        out = f"/tmp/dp_time_{cfg}_{k}.npz"
        p = subprocess.run([sys.executable, __file__, "--child", cfg, iters, out], env=env, capture_output=True,
                           text=True)
        line = [l for l in p.stdout.splitlines() if l.startswith("RESULT")]
        res = json.loads(line[0][7:]) if line else {"err": p.stderr[-1500:]}
        if line:
            outs.append(np.load(out))
            if len(outs) > 1:
                a, b = outs[-1], outs[0]
                res["vs_first"] = {k2: rel(a[k2], b[k2]) for k2 in ("dual", "primal", "primal_avg", "u0")}
                res["vs_first"]["gap"] = float(abs(a["gap"] - b["gap"]) / (1 + abs(b["gap"])))
        print(cfg, var or "default", json.dumps(res), flush=True)
