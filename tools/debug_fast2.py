import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from paper_1904_10548_b200 import SolverConfig, factor_step, solve, CostWeights, assemble_problem, attach_forecast, uniform_tree
from paper_1904_10548_b200.synthetic import barcelona_instance, barcelona_network
from conftest import make_model

def run(inst, iters, fast):
    os.environ["WMPC_DISABLE_FAST"] = "0" if fast else "1"
    cache = factor_step(inst)
    return solve(inst, SolverConfig(max_iter=iters, tol=1e-30, gamma=1/5e9, gap_check_every=iters+1), cache=cache)

def cmp(name, inst):
    a = run(inst, 1, True); b = run(inst, 1, False)
    e = np.abs(a.primal - b.primal).max() / (1 + np.abs(b.primal).max())
    print(f"{name:40s} nt={inst.model.n_tanks} nu={inst.model.n_inputs} ns={inst.model.n_mixing} H={inst.tree.horizon} n={inst.n_nonroot} err={e:.3e}")

def rand_inst(nt, nu, nd, ns, branching, H, seed=1, wu=0.5):
    rng = np.random.default_rng(seed)
    model = make_model(rng, nt, nu, nd, ns)
    tree = uniform_tree(branching, H, nd, nu)
    tree.eps = 0.1 * rng.standard_normal((tree.n_nodes, nd + nu)); tree.eps[0] = 0
    tree = attach_forecast(tree, 0.3 + 0.2 * rng.random((H, nd)), 0.5 + rng.random((H, nu)))
    return assemble_problem(model, tree, CostWeights(1.0, wu, 2.0, 5.0), model.x_safe * 1.3, 0.3 * rng.random(nu))

cmp("barcelona [2,2] H=4", barcelona_instance([2, 2], horizon=4))
cmp("barcelona [2] H=2", barcelona_instance([2], horizon=2))
cmp("barcelona [] H=1", barcelona_instance([], horizon=1))
cmp("barcelona [] H=2", barcelona_instance([], horizon=2))
for nu in (4, 8, 12, 18, 20, 24, 38, 40, 64, 114):
    cmp(f"rand nu={nu} chain H=2", rand_inst(3, nu, 2, 0, [], 2))
cmp("rand nt=63 nu=114 ns=0 [2] H=3", rand_inst(63, 114, 5, 0, [2], 3))
cmp("rand nt=3 nu=114 ns=0 [] H=1", rand_inst(3, 114, 2, 0, [], 1))
