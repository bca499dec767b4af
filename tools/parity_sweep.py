"""Seeded parity population: fixed-iteration
GPU solves against the CPU oracle, with each instance's own rounding-noise
floor.

    python tools/parity_sweep.py [--c1 20 --c2 10 --c3 3 --iters 500] [--out profiles/r02/parity.json]

For every instance (Barcelona-dimension network and forecasts from seed s,
``synthetic.barcelona_instance``) on the C1 / C2 / C3 trees:
* gamma = 1/L from the device power iteration (the same gamma for both sides);
* the GPU solve through the public API (default kernel selection, recorded);
* the oracle (oracle/port.py, pinned to the reference: tests/golden) with the
  same gamma, 500 iterations, tol 1e-30, the final certificate;
* the oracle again with 1-ulp multiplicative noise on y after every iteration
  (SURVEY §8(c)): the per-instance self-noise floor.
Metric: ||a - b|| / (1 + ||b||) (test_solver.py:21-22) on u0, the last
primal iterate, the averaged primal and the dual; |a - b| / (1 + |b|) on the
gap and the objective. Pass: every metric <= max(1e-8, 10 x floor).
The oracle runs in worker processes (spawned, BLAS threads split) while the
GPU solves run in the main process.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

KEYS = ("u0", "primal", "primal_avg", "dual")


def rel(a, b) -> float:
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.linalg.norm(a - b) / (1.0 + np.linalg.norm(b)))


def oracle_job(branching, seed, gamma, iters, noisy):
    sys.path.insert(0, ROOT)
    from oracle import port
    from paper_1904_10548_b200.synthetic import barcelona_instance
    inst = barcelona_instance(branching, seed=seed)
    hook = None
    if noisy:
        rng = np.random.default_rng(10_000 + seed)
        eps = np.finfo(float).eps

        def hook(it, y, z, za):  # noqa: ARG001 - y is the next iterate (a view)
            y *= 1.0 + eps * rng.choice((-1.0, 1.0), size=y.shape)
    t0 = time.perf_counter()
    r = port.apg_solve(inst, gamma, max_iter=iters, tol=1e-30, gap_check_every=iters + 1,
                       reference_cost_accounting=False, hook=hook)
    return {"u0": r.u0, "primal": r.primal, "primal_avg": r.primal_avg, "dual": r.dual,
            "gap": r.duality_gap, "objective": r.objective, "seconds": time.perf_counter() - t0}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c1", type=int, default=20)
    ap.add_argument("--c2", type=int, default=10)
    ap.add_argument("--c3", type=int, default=3)
    ap.add_argument("--c4", type=int, default=0, help="C4 instances (oracle ~2 s per iteration: use --c4-iters)")
    ap.add_argument("--c4-iters", type=int, default=50)
    ap.add_argument("--force-dp", action="store_true", help="k_chain_dp on every tree (WMPC_DP=1)")
    ap.add_argument("--iters", type=int, default=500)
    ap.add_argument("--workers", type=int, default=0)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02", "parity.json"))
    args = ap.parse_args()
    import multiprocessing as mp
    ncpu = os.cpu_count() or 1
    workers = args.workers or max(1, ncpu // 2)
    os.environ["OPENBLAS_NUM_THREADS"] = str(max(1, ncpu // workers))
    if args.force_dp:
        os.environ["WMPC_DP"] = "1"
    from paper_1904_10548_b200 import SolverConfig, estimate_lipschitz, factor_step, solve
    from paper_1904_10548_b200 import _native as nat
    from paper_1904_10548_b200.synthetic import CONFIGS, barcelona_instance
    pool = mp.get_context("spawn").Pool(workers)
    jobs = []
    for name, count in (("C4", args.c4), ("C3", args.c3), ("C2", args.c2), ("C1", args.c1)):  # longest first
        for seed in range(count):
            jobs.append((name, seed))
    pending, records = {}, []
    t_start = time.perf_counter()
    for name, seed in jobs:
        iters = args.c4_iters if name == "C4" else args.iters
        inst = barcelona_instance(CONFIGS[name], seed=seed)
        cache = factor_step(inst)
        info = nat.path_info(cache._bind())
        L = estimate_lipschitz(cache, inst)
        gamma = 1.0 / L
        clean = pool.apply_async(oracle_job, (CONFIGS[name], seed, gamma, iters, False))
        noisy = pool.apply_async(oracle_job, (CONFIGS[name], seed, gamma, iters, True))
        res = solve(inst, SolverConfig(max_iter=iters, tol=1e-30, gamma=gamma,
                                       gap_check_every=iters + 1), cache=cache)
        gpu = {k: np.array(getattr(res, k)) for k in KEYS}
        gpu.update(gap=res.duality_gap, objective=res.objective)
        pending[(name, seed)] = (clean, noisy, gpu, gamma, info, inst.n_nonroot, iters)
    for (name, seed), (clean, noisy, gpu, gamma, info, n, iters) in pending.items():
        c, z = clean.get(), noisy.get()
        err = {k: rel(gpu[k], c[k]) for k in KEYS}
        flo = {k: rel(z[k], c[k]) for k in KEYS}
        for k in ("gap", "objective"):
            err[k] = abs(gpu[k] - c[k]) / (1 + abs(c[k]))
            flo[k] = abs(z[k] - c[k]) / (1 + abs(c[k]))
        thr = {k: max(1e-8, 10 * flo[k]) for k in err}
        ok = all(err[k] <= thr[k] for k in err)
        records.append({"config": name, "seed": seed, "nodes": n, "iters": iters, "gamma": gamma, "errors": err,
                        "noise_floor": flo, "threshold": thr, "pass": ok,
                        "kernels": {"fast_path": info["fast_path"], "fused_dp": info["fused_dp"],
                                    "chainw": info["chainw"]},
                        "oracle_seconds": c["seconds"]})
        print(json.dumps({"config": name, "seed": seed, "pass": ok, "max_err": max(err.values()),
                          "max_floor": max(flo.values())}), flush=True)
    pool.close()
    summary = {}
    for name in ("C1", "C2", "C3", "C4"):
        rs = [r for r in records if r["config"] == name]
        if rs:
            summary[name] = {"instances": len(rs), "passed": sum(r["pass"] for r in rs),
                             "max_error": max(max(r["errors"].values()) for r in rs),
                             "max_noise_floor": max(max(r["noise_floor"].values()) for r in rs)}
    total = len(records)
    passed = sum(r["pass"] for r in records)
    out = {"what": "fixed-iteration GPU solves vs the CPU oracle (oracle/port.py, pinned to the reference), "
                   "seeded Barcelona-dimension population; pass = every metric <= max(1e-8, 10 x the "
                   "instance's 1-ulp-per-iteration self-noise floor)",
           "iters": args.iters, "c4_iters": args.c4_iters, "forced_dp": bool(args.force_dp), "metric": "||a-b||/(1+||b||) (test_solver.py:21-22); |a-b|/(1+|b|) for gap, objective",
           "pass_rate": passed / max(total, 1), "passed": passed, "instances": total, "summary": summary,
           "wall_s": time.perf_counter() - t_start, "host_cpus": ncpu, "oracle_workers": workers,
           "records": records}
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: out[k] for k in ("pass_rate", "passed", "instances", "summary", "wall_s")}), flush=True)


if __name__ == "__main__":
    main()
