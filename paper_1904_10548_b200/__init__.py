"""B200-native scenario-tree dual APG solver for stochastic water-network MPC
(arXiv 1904.10548), a drop-in for the reference ``watermpc`` solver path.

Public names mirror ``watermpc/__init__.py:19-55`` for the solver path.
"""

from .model import CostWeights, NetworkModel
from .problem import (
    FEAS_TOL,
    ProblemInstance,
    apply_H,
    apply_H_adjoint,
    assemble_problem,
    prox_g,
    prox_g_conjugate,
)
from .solver import (
    FactorCache,
    SolverConfig,
    SolverResult,
    dual_gradient,
    estimate_lipschitz,
    factor_step,
    solve,
    theta_sequence,
)
from .tree import ScenarioTree, attach_forecast, uniform_tree, validate_tree, zero_price_errors

__version__ = "0.1.0"

__all__ = [
    "CostWeights", "FactorCache", "NetworkModel", "ProblemInstance", "ScenarioTree",
    "SolverConfig", "SolverResult", "apply_H", "apply_H_adjoint", "assemble_problem",
    "attach_forecast", "dual_gradient", "estimate_lipschitz", "factor_step", "prox_g",
    "prox_g_conjugate", "solve", "theta_sequence", "uniform_tree", "validate_tree",
    "zero_price_errors", "FEAS_TOL",
]
