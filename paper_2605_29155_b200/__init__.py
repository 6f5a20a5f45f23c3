"""B200-native differentiable MPC layer (CA-DiffMPC hot path of arxiv/paper_2605_29155).

Public API (mirrors the reference package ``fusedmpc``):
    DynModel, SolveSettings, StageCostParams           — problem description
    solve_raw / solve_diag / backward_raw               — array-level batch API (GPU)
    MpcSolver, MpcSolveLayer, mpc_control               — AC-MPC drop-in layer
    MPC, QuadCost                                       — mpc.pytorch-style module
    policy, ppo, rollout, raceenv                       — AC-MPC training plumbing (PPO with
                                                          one NCCL all-reduce, device-resident
                                                          rollouts, batched GPU race env)
    benchgrid                                           — latency grid in the bench CSV schema
    api (solve, backward, solve_batch, backward_batch,  — object-level API of ilqr / gradlayer /
         BatchProblem, make_hover_problem)                batchexec with the reference's errors
Heavy modules (torch, the CUDA library) are imported lazily.
"""

from .errors import ConfigError, DivergenceError, ExtensionMissingError, NumericError
from .dynamics import DynModel
from .settings import SolveSettings, DEFAULT_ALPHAS
from . import _abi, problems, roofline  # noqa: F401  (host-only modules)

__all__ = [
    "ConfigError", "DivergenceError", "NumericError", "ExtensionMissingError",
    "DynModel", "SolveSettings", "DEFAULT_ALPHAS",
    "StageCostParams", "solve_raw", "solve_diag", "backward_raw", "SolveOutput",
    "MpcSolver", "MpcSolveLayer", "mpc_control", "MPC", "QuadCost",
]


def __getattr__(name):
    if name in ("StageCostParams", "Trajectory"):
        from . import qcost
        return getattr(qcost, name)
    if name in ("solve_raw", "solve_diag", "backward_raw", "SolveOutput", "GradOutput"):
        from . import solver
        return getattr(solver, name)
    if name in ("MpcSolver", "MpcSolveLayer", "mpc_control"):
        from . import layer
        return getattr(layer, name)
    if name in ("MPC", "QuadCost"):
        from . import mpc
        return getattr(mpc, name)
    raise AttributeError(name)
