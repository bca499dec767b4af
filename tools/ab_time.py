"""A/B timing of library variants: ab_time.py CFG ITERS LIB[@K=V,...] [...]. Each variant
runs in its own process (WMPC_LIB_EXPERIMENT), twice interleaved; prints us per APG
iteration (graph replay, CUDA events) for fp64 and fp32, and a hash of a 40-iteration
fixed-step solve's dual/primal so variants can be checked bit-identical."""
import hashlib, json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(cfg, iters):
    sys.path.insert(0, ROOT)
    import numpy as np
    from paper_1904_10548_b200 import SolverConfig, factor_step, solve
    from paper_1904_10548_b200 import _native as nat
    from paper_1904_10548_b200 import solver as S
    from paper_1904_10548_b200.synthetic import config_instance
    inst = config_instance(cfg)
    cache = factor_step(inst)
    r = solve(inst, SolverConfig(max_iter=40, tol=1e-30, gap_check_every=41, gamma=1 / 2e9), cache=cache)
    h = hashlib.sha1(np.ascontiguousarray(r.dual).tobytes() + np.ascontiguousarray(r.primal).tobytes()).hexdigest()[:12]
    ctx = cache._bind()
    S._upload_bounds(ctx, inst)
    th = S.theta_sequence(iters + 5)
    be = S._beta_table(th)
    out = {"hash": h}
    for prec in (0, 1):
        ctx.call("wmpc_set_precision", prec)
        ctx.call("wmpc_apg_begin", 1.0 / 2e9, iters + 5, nat.ptr(th), nat.ptr(be))
        ctx.call("wmpc_apg_run", 5)
        ms = nat.C.c_float(0.0)
        ctx.call("wmpc_apg_run_timed", iters, nat.C.byref(ms))
        out["fp32" if prec else "fp64"] = round(ms.value / iters * 1e3, 2)
    ctx.call("wmpc_set_precision", 0)
    print("RESULT", json.dumps(out))


if __name__ == "__main__":
    if sys.argv[1] == "--child":
        child(sys.argv[2], int(sys.argv[3]))
        sys.exit(0)
    cfg, iters, libs = sys.argv[1], sys.argv[2], sys.argv[3:]
    res = {lib: [] for lib in libs}
    for rep in range(2):
        for lib in libs:
            path, _, extra = lib.partition("@")  # LIB@K=V,K=V: extra environment
            env = dict(os.environ, WMPC_LIB_EXPERIMENT=os.path.abspath(path))
            env.update(dict(kv.split("=") for kv in extra.split(",") if kv))
            p = subprocess.run([sys.executable, __file__, "--child", cfg, iters], env=env, capture_output=True,
                               text=True)
            line = [l for l in p.stdout.splitlines() if l.startswith("RESULT")]
            res[lib].append(json.loads(line[0][7:]) if line else {"err": p.stderr[-500:]})
    for lib, rr in res.items():
        print(cfg, os.path.basename(lib), json.dumps(rr))
