"""Host-side logic (no device work): settings / model validation mirroring the reference's
tests (tests/test_ilqr.py:298-314, tests/test_dynamics.py:111-122), problem generators,
the roofline model and the ABI struct filling."""

import numpy as np
import pytest

from paper_2605_29155_b200 import ConfigError, DynModel, SolveSettings, _abi, problems, roofline
from paper_2605_29155_b200.qcost import EPS_REG, StageCostParams


def test_settings_validation():
    with pytest.raises(ConfigError):
        SolveSettings(T=0, u_min=np.zeros(1), u_max=np.ones(1))
    with pytest.raises(ConfigError):
        SolveSettings(T=2, u_min=np.ones(1), u_max=np.zeros(1))
    with pytest.raises(ConfigError):
        SolveSettings(T=2, u_min=np.zeros(1), u_max=np.ones(1), alphas=(0.5, 1.0))
    with pytest.raises(ConfigError):
        SolveSettings(T=2, u_min=np.zeros(1), u_max=np.ones(1), alphas=())
    with pytest.raises(ConfigError):
        SolveSettings(T=2, u_min=np.zeros(1), u_max=np.ones(1), K_max=0)
    s = SolveSettings(T=3, u_min=0.0, u_max=2.0)
    lo, hi = s.bounds_for(4)
    assert lo.shape == (4,) and np.all(hi == 2.0)


def test_model_validation():
    with pytest.raises(ConfigError):
        DynModel.double_integrator(0, dt=0.1)
    with pytest.raises(ConfigError):
        DynModel.planar_quadrotor(dt=-0.1)
    with pytest.raises(ConfigError):
        DynModel.planar_quadrotor(dt=0.1, mass=0.0)
    with pytest.raises(ConfigError):
        DynModel.linear(np.zeros((2, 3)), np.zeros((2, 1)))
    with pytest.raises(ConfigError):
        DynModel.quadrotor(inertia=(0.01, 0.0, 0.02))
    q = DynModel.quadrotor()
    assert (q.n_x, q.n_u, q.n_theta) == (13, 4, 7)
    np.testing.assert_allclose(q.hover_control(), 0.25 * 0.6 * 9.81)


def test_hover_problem_matches_reference_generator():
    """make_hover_problem (batchexec.py:215-233): same rng stream and cost layout."""
    pb = problems.hover_problem(DynModel.planar_quadrotor(dt=0.05), 5, 4, seed=0)
    rng = np.random.default_rng(0)
    x = np.zeros((5, 6))
    x[:, 0:2] = rng.uniform(-1.0, 1.0, size=(5, 2))
    x[:, 3:5] = rng.uniform(-0.5, 0.5, size=(5, 2))
    np.testing.assert_array_equal(pb.x0, x)
    np.testing.assert_array_equal(pb.diag[0, 0], [1, 1, 1, 0.1, 0.1, 0.1, 0.05, 0.05])
    np.testing.assert_allclose(pb.c[0, 0, 6:], -0.05 * 0.5 * 0.6 * 9.81)
    assert pb.settings.u_max[0] == pytest.approx(2 * 0.6 * 9.81)


def test_roofline_table_matches_survey():
    """per-stage constants and the 13/4, T=10 rows."""
    assert [int(v) for v in roofline.stage_flops(6, 2)] == [152, 1982, 180, 2174]  # SURVEY truncates
    _, F_ric, F_ls, F_aux = roofline.stage_flops(13, 4)
    assert round(F_ric) == 17264 and F_ls == 741 and round(F_aux) == 18116
    assert roofline.fwd_flops(13, 4, 10, [3]) == pytest.approx(613.1e3, rel=1e-3)
    assert roofline.fwd_flops(13, 4, 10, [10]) == pytest.approx(2029e3, rel=1e-3)
    assert roofline.bwd_flops(13, 4, 10, 1) == pytest.approx(181.2e3, rel=1e-3)
    assert roofline.fwd_bytes(13, 4, 10, 1) == pytest.approx(13.19e3, rel=2e-3)
    assert roofline.bwd_bytes(13, 4, 10, 1) == pytest.approx(25.32e3, rel=2e-3)


def test_make_problem_fills_abi_struct():
    m = DynModel.quadrotor()
    s = SolveSettings(T=7, u_min=np.zeros(4), u_max=np.arange(1, 5, dtype=float), K_max=4,
                      alphas=(1.0, 0.3), conv_tol=1e-5)
    p = _abi.make_problem(m, s, 11, _abi.COST_DIAG, theta_stride=7)
    assert (p.B, p.T, p.nx, p.nu, p.model_kind, p.cost_layout) == (11, 7, 13, 4, 3, 1)
    assert (p.K_max, p.n_alpha, p.n_theta, p.theta_stride) == (4, 2, 7, 7)
    assert list(p.u_max)[:4] == [1.0, 2.0, 3.0, 4.0] and list(p.alphas)[:2] == [1.0, 0.3]
    assert p.dt == 0.05 and p.conv_tol == 1e-5


def test_stage_cost_params_symmetrise_and_lift():
    """qcost.StageCostParams semantics (qcost.py:57-76)."""
    C = np.zeros((1, 3, 3))
    C[0, 0, 1] = 2.0
    p = StageCostParams(C, np.zeros((1, 3)), 2)
    assert np.array_equal(p.C[0], p.C[0].T)
    assert p.C[0, 2, 2] >= EPS_REG
    p2 = StageCostParams(np.eye(3)[None] * 2.0, np.zeros((1, 3)), 2)
    assert p2.C[0, 2, 2] == 2.0


def test_extension_missing_fails_loudly(monkeypatch):
    """No CPU fallback: without a CUDA device the product entry points raise."""
    import torch

    from paper_2605_29155_b200 import ExtensionMissingError, solver

    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    pb = problems.hover_problem(DynModel.quadrotor(), 2, 3)
    with pytest.raises(ExtensionMissingError):
        solver.solve_raw(pb.model, pb.settings, pb.x0, pb.diag, pb.c, pb.U_warm)
