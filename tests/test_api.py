"""Object-level API (api.py) with the reference's error semantics (ilqr.solve raises on a
single-instance failure, batch calls flag it; gradlayer.backward flags approximate
gradients) on the GPU kernels."""

import numpy as np
import pytest
import torch

from paper_2605_29155_b200 import DynModel, SolveSettings, api, problems, solver
from paper_2605_29155_b200.errors import ConfigError, DivergenceError, NumericError
from paper_2605_29155_b200.qcost import StageCostParams


def _planar_instance(seed=3, T=8, **kw):
    m = DynModel.planar_quadrotor(dt=0.05)
    pb = problems.random_problem(m, 1, T, seed=seed, **kw)
    p = StageCostParams.from_diag(pb.diag[0], pb.c[0], m.n_x)
    return m, pb, p


def test_batch_problem_validation():
    m, pb, p = _planar_instance()
    with pytest.raises(ConfigError):
        api.BatchProblem(m, pb.x0, [p, p], pb.U_warm, pb.settings)
    with pytest.raises(ConfigError):
        api.BackwardSeed(np.zeros((3, 6)), np.zeros((3, 2)))


@pytest.mark.gpu
def test_solve_matches_array_api_and_backward():
    m, pb, p = _planar_instance()
    r = api.solve(m, pb.x0[0], p, pb.U_warm[0], pb.settings)
    ref = solver.solve_raw(m, pb.settings, pb.x0, p.C[None], p.c[None], pb.U_warm, dtype=torch.float64)
    np.testing.assert_array_equal(r.traj.U, ref.U.cpu().numpy()[0])
    assert r.iterations == int(ref.iters[0]) and r.converged and not r.failed
    assert r.alpha_history.shape == (r.iterations,)
    seed = api.BackwardSeed(np.zeros((9, 6)), np.eye(8, 2))
    g = api.backward(r, None, p, seed)
    gr = solver.backward_raw(m, pb.settings, p.C[None], p.c[None], ref.X, ref.U, None,
                             torch.tensor(np.eye(8, 2)[None]), dtype=torch.float64)
    np.testing.assert_array_equal(g.dC, gr.dC.cpu().numpy()[0])
    assert not g.approximate
    r1 = api.solve(m, pb.x0[0], p, pb.U_warm[0], pb.settings.replace(K_max=1, conv_tol=0.0))
    assert not r1.converged and api.backward(r1, None, p, seed).approximate


@pytest.mark.gpu
def test_single_instance_failures_raise_batch_flags():
    m = DynModel.planar_quadrotor(dt=0.05)
    T = 6
    st = SolveSettings(T=T, u_min=0.0, u_max=12.0)
    bad = StageCostParams.from_diag(np.tile([-5.0] * 6 + [1e-6, 1e-6], (T, 1)), np.zeros((T, 8)), 6)
    good = StageCostParams.from_diag(np.tile([1.0] * 8, (T, 1)), np.zeros((T, 8)), 6)
    x0 = np.array([0.3, -0.2, 0.1, 0.0, 0.0, 0.0])
    Uw = np.full((T, 2), 2.45)
    with pytest.raises(NumericError):
        api.solve(m, x0, bad, Uw, st)
    prob = api.BatchProblem(m, np.stack([x0, x0]), [good, bad], np.stack([Uw, Uw]), st)
    res, stats = api.solve_batch(prob)
    assert not res[0].failed and res[1].failed and res[1].fail_stage >= 0
    # exponentially unstable linear model: the initial rollout overflows
    lin = DynModel.linear(np.eye(2) * 1e200, np.ones((2, 1)))
    stl = SolveSettings(T=4, u_min=-1.0, u_max=1.0)
    pl = StageCostParams.from_diag(np.ones((4, 3)), np.zeros((4, 3)), 2)
    with pytest.raises(DivergenceError):
        api.solve(lin, np.array([1e200, 1.0]), pl, np.zeros((4, 1)), stl)


@pytest.mark.gpu
def test_hover_batch_round_trip():
    prob = api.make_hover_problem(16, 10, settings_kw={"K_max": 10})
    res, _ = api.solve_batch(prob)
    assert all(r.converged for r in res)
    seeds = [api.BackwardSeed(np.zeros((11, 6)), np.eye(10, 2)) for _ in res]
    grads = api.backward_batch(res, None, prob.params, seeds)
    assert len(grads) == 16 and not any(g.failed for g in grads)
    assert all(np.isfinite(g.dC).all() for g in grads)
