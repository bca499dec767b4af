"""Diff the persistent kernel against the per-stage kernels row by row."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1904_10548_b200 import SolverConfig, factor_step, solve
from paper_1904_10548_b200.synthetic import config_instance

def run(inst, iters, fast):
    os.environ["WMPC_DISABLE_FAST"] = "0" if fast else "1"
    cache = factor_step(inst)
    return solve(inst, SolverConfig(max_iter=iters, tol=1e-30, gamma=1/5e9, gap_check_every=iters+1), cache=cache)

cfg = sys.argv[1] if len(sys.argv) > 1 else "C1"
inst = config_instance(cfg)
n = inst.n_nonroot
st = np.concatenate([[s]*(sl.stop-sl.start) for s, sl in enumerate(inst.stage_slices)])
for iters in (1, 2):
    a = run(inst, iters, True); b = run(inst, iters, False)
    for k in ("primal", "primal_avg", "dual"):
        A = getattr(a, k).reshape(n, -1); B = getattr(b, k).reshape(n, -1)
        err = np.abs(A - B).max(axis=1) / (1 + np.abs(B).max(axis=1))
        bad = np.flatnonzero(err > 1e-12)
        print(iters, k, "bad rows", bad.size, "stages", sorted(set(st[bad].tolist()))[:30], "max", err.max())
        if bad.size:
            r = bad[0]; c = np.flatnonzero(np.abs(A[r]-B[r]) > 1e-12*(1+np.abs(B[r]).max()))
            print("   first row", r, "stage", st[r], "cols", c[:20], A[r, c[:3]], B[r, c[:3]])
