"""Compare a sharded solve with the one-GPU solve after a few iterations, row by row."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1904_10548_b200 import SolverConfig, factor_step, solve, shard
from paper_1904_10548_b200.synthetic import config_instance
cfg, G, it = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
inst = config_instance(cfg)
conf = SolverConfig(max_iter=it, tol=1e-30, gamma=1.0 / 2e9, gap_check_every=it + 1)
ref = solve(inst, conf, cache=factor_step(inst))
res = shard.solve_sharded(inst, conf, size=G)
W = 2 * 63 + 114
P = 63 + 114
dy = np.abs(res.dual.reshape(-1, W) - ref.dual.reshape(-1, W)).max(axis=1)
dz = np.abs(res.primal.reshape(-1, P) - ref.primal.reshape(-1, P)).max(axis=1)
off = [s.start for s in inst.stage_slices]
print("k", shard.plan(inst, G)[0].k, "offsets", off[:5])
for s in range(6):
    sl = inst.stage_slices[s]
    print("stage", s, "max |dy|", dy[sl].max(), "max |dz|", dz[sl].max(), "argmax z", int(np.argmax(dz[sl])) + sl.start)
print("u0 diff", np.abs(res.u0 - ref.u0).max())
Z1 = res.primal.reshape(-1, P); Z0 = ref.primal.reshape(-1, P)
for s in range(4):
    sl = inst.stage_slices[s]
    print("stage", s, "du", np.abs(Z1[sl, :114] - Z0[sl, :114]).max(), "dx", np.abs(Z1[sl, 114:] - Z0[sl, 114:]).max())
r = 0
print("x diff row0", (Z1[r, 114:119] - Z0[r, 114:119]), "g", inst.demand_gd[r, :5], "p", inst.p[:5])
print("x row0 shard", Z1[r, 114:119], "ref", Z0[r, 114:119])
