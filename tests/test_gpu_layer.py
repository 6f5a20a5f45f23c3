"""The reference-facing drop-ins on the GPU: MpcSolver / MpcSolveLayer (policy.py:179-290)
and the MPC(n_state, n_ctrl, T, u_lower, u_upper, ...) module, against the C oracle and
finite differences (tests/test_policy.py:181-212 style)."""

import numpy as np
import pytest
import torch

import oracle
from paper_2605_29155_b200 import DynModel, SolveSettings, problems
from paper_2605_29155_b200.layer import MpcSolveLayer, MpcSolver, mpc_control
from paper_2605_29155_b200.mpc import MPC, LinDx, PlanarQuadrotorDx, QuadCost, QuadrotorDx

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_solve_layer_matches_reference_semantics(dtype):
    """u0 = U*[:, 0]; grads = diag(dC), dc of the aux LQR seeded with dL/du0 only."""
    model = DynModel.quadrotor()
    pb = problems.random_problem(model, 32, 10, seed=41)
    solver = MpcSolver(model, pb.settings, dtype=dtype)
    diag = torch.tensor(pb.diag, dtype=dtype, device="cuda", requires_grad=True)
    cvec = torch.tensor(pb.c, dtype=dtype, device="cuda", requires_grad=True)
    sink = {}
    u0 = MpcSolveLayer.apply(diag, cvec, solver, pb.x0, pb.U_warm, sink)
    w = torch.randn(32, 4, dtype=dtype, device="cuda", generator=torch.Generator("cuda").manual_seed(0))
    (u0 * w).sum().backward()
    # the oracle solves exactly the problem the kernel saw (f32 kernels: f32-rounded inputs)
    rnd = (lambda a: np.asarray(a, np.float32).astype(np.float64)) if dtype == torch.float32 else np.asarray
    x0, C, c, Uw = rnd(pb.x0), rnd(pb.dense_C()), rnd(pb.c), rnd(pb.U_warm)
    ref = oracle.forward(model, pb.settings, x0, C, c, Uw)
    seed = np.zeros((32, 10, 4))
    seed[:, 0] = w.double().cpu().numpy()
    rb = oracle.backward(model, pb.settings, C, c, ref["X"], ref["U"], None, rnd(seed), want_theta=False)
    iters = solver.solve_diag(pb.x0, pb.diag, pb.c, pb.U_warm)[1].cpu().numpy()
    np.testing.assert_array_equal(iters, ref["iters"])
    tol = 1e-9 if dtype == torch.float64 else 1e-4
    idx = np.arange(17)
    assert sink["solves"] == 32

    def rel(a, b):  # per instance, SURVEY.md §8(c)
        a, b = a.reshape(a.shape[0], -1), b.reshape(b.shape[0], -1)
        return (np.abs(a - b).max(1) / np.maximum(1.0, np.abs(b).max(1))).max()

    assert rel(u0.detach().double().cpu().numpy(), ref["U"][:, 0]) <= tol
    assert rel(diag.grad.double().cpu().numpy(), rb["dC"][:, :, idx, idx]) <= tol
    assert rel(cvec.grad.double().cpu().numpy(), rb["dc"]) <= tol


def test_layer_gradient_matches_finite_differences():
    """test_policy.py:181-212: d log-prob / d actor-weight through the layer vs FD (planar, f64)."""
    torch.manual_seed(0)
    model = DynModel.planar_quadrotor(dt=0.05)
    settings = SolveSettings(T=3, u_min=np.zeros(2), u_max=np.full(2, 6.0), K_max=3)
    solver = MpcSolver(model, settings, dtype=torch.float64)

    class Actor(torch.nn.Module):
        def __init__(self):
            super().__init__()
            self.net = torch.nn.Linear(11, 3 * 2 * 8).double()

        def forward(self, obs):
            raw = torch.sigmoid(self.net(obs)).view(-1, 3, 2, 8)
            return 1e-3 + raw[:, :, 0] * 10.0, -10.0 + raw[:, :, 1] * 20.0

    class Bundle:
        actor = Actor().cuda()

    obs = torch.full((2, 11), 0.3, dtype=torch.float64, device="cuda")
    x_init = 0.2 * np.ones((2, 6))
    U_warm = np.tile(model.hover_control(), (2, 3, 1))
    action = torch.tensor([[2.0, 3.0], [3.0, 2.0]], dtype=torch.float64, device="cuda")

    def logp():
        u = mpc_control(Bundle, obs, solver, x_init, U_warm)
        return torch.distributions.Normal(u, 0.5).log_prob(action).sum()

    logp().backward()
    W = Bundle.actor.net.weight
    eps = 1e-6
    rng = np.random.default_rng(9)
    for _ in range(4):
        j = int(rng.integers(W.numel()))
        flat = W.detach().view(-1)
        with torch.no_grad():
            flat[j] += eps
            up = float(logp())
            flat[j] -= 2 * eps
            dn = float(logp())
            flat[j] += eps
        fd = (up - dn) / (2 * eps)
        an = float(W.grad.view(-1)[j])
        assert abs(fd - an) <= 1e-3 * max(1e-4, abs(fd))


def test_solver_warm_start_shift():
    model = DynModel.quadrotor()
    s = SolveSettings(T=4, u_min=np.zeros(4), u_max=np.full(4, 5.0))
    sv = MpcSolver(model, s, n_slots=2)
    assert torch.allclose(sv.warm, torch.full((2, 4, 4), 0.25 * 0.6 * 9.81, device="cuda"))
    U = torch.arange(2 * 4 * 4, dtype=torch.float32, device="cuda").view(2, 4, 4)
    sv.push_warm(U)
    assert torch.equal(sv.warm[:, :3], U[:, 1:]) and torch.equal(sv.warm[:, 3], U[:, 3])
    sv.reset_warm(slots=[0])
    assert torch.allclose(sv.warm[0], torch.full((4, 4), 0.25 * 0.6 * 9.81, device="cuda"))


def test_mpc_module_forward_matches_oracle():
    model = DynModel.quadrotor()
    pb = problems.hover_problem(model, 8, 10, seed=3)
    mpc = MPC(13, 4, 10, u_lower=0.0, u_upper=model.mass * model.gravity, lqr_iter=10, eps=1e-6)
    C = torch.tensor(pb.dense_C(), dtype=torch.float64, device="cuda").transpose(0, 1)
    c = torch.tensor(pb.c, dtype=torch.float64, device="cuda").transpose(0, 1)
    x0 = torch.tensor(pb.x0, dtype=torch.float64, device="cuda")
    x, u, J = mpc(x0, QuadCost(C, c), QuadrotorDx())
    ref = oracle.forward(model, pb.settings, pb.x0, pb.dense_C(), pb.c, pb.U_warm)
    assert x.shape == (10, 8, 13) and u.shape == (10, 8, 4) and J.shape == (8,)
    np.testing.assert_allclose(u.transpose(0, 1).cpu().numpy(), ref["U"], atol=1e-9)
    np.testing.assert_allclose(J.cpu().numpy(), ref["J"], rtol=1e-10)
    # diagonal cost given time-major without the batch dim broadcasts
    x2, u2, _ = mpc(x0, QuadCost(torch.tensor(pb.diag[0], device="cuda", dtype=torch.float64),
                                 torch.tensor(pb.c[0], device="cuda", dtype=torch.float64)), QuadrotorDx())
    np.testing.assert_allclose(u2.cpu().numpy(), u.cpu().numpy(), atol=1e-12)


def test_mpc_module_gradients_fd_linear():
    """Every input gradient of the module (C, c, x_init, A, B) vs FD on linear dynamics, where the
    implicit gradients are exact; loss touches x*, u* and the optimal cost."""
    rng = np.random.default_rng(2)
    n, m, T, B = 3, 2, 5, 2
    A = torch.tensor(np.eye(n) + 0.1 * rng.normal(size=(n, n)), device="cuda")
    Bm = torch.tensor(0.5 * rng.normal(size=(n, m)), device="cuda")
    M = rng.normal(size=(T, B, n + m, n + m))
    C = torch.tensor(0.3 * np.einsum("tbij,tbkj->tbik", M, M) + 0.8 * np.eye(n + m), device="cuda",
                     requires_grad=True)
    c = torch.tensor(0.3 * rng.normal(size=(T, B, n + m)), device="cuda", requires_grad=True)
    x0 = torch.tensor(0.5 * rng.normal(size=(B, n)), device="cuda", requires_grad=True)
    dx = LinDx(A, Bm, learn=True).cuda()
    mpc = MPC(n, m, T, u_lower=-0.25, u_upper=0.25, lqr_iter=60, eps=1e-14)
    wx, wu = torch.randn(T, B, n, device="cuda", dtype=torch.float64), torch.randn(T, B, m, device="cuda",
                                                                                    dtype=torch.float64)

    def loss():
        x, u, J = mpc(x0, QuadCost(C, c), dx)
        return (wx * x).sum() + (wu * u).sum() + 0.3 * J.sum()

    loss().backward()
    # clamped controls at the solution (time-major like the module's outputs)
    clamped = mpc.last_result.clamped.transpose(0, 1).cpu().numpy().astype(bool)
    eps = 1e-6
    worst = 0.0
    n_checked_zero = 0
    # C is used as a symmetric matrix (gz = C z, kernels.py:395-399), so dC = sym(dz z') is the
    # gradient for symmetric perturbations: off-diagonal entries are perturbed in pairs.
    for t, idx in [(C, (1, 0, 2, 2)), (C, (3, 1, 0, 4)), (C, (0, 0, 1, 3)), (C, (2, 1, 0, 1)),
                   (c, (0, 1, 3)), (c, (4, 0, 1)), (x0, (1, 2)), (dx.params, (0,)), (dx.params, (10,))]:
        if t is C and any(j >= n and clamped[idx[0], idx[1], j - n] for j in idx[2:]):
            # Reference convention (kernels.py:733-756): rows/cols of dC on
            # a clamped control are zeroed, dropping the 1/2 dz_x z_u cross term the exact
            # derivative has. The x/u seeds contribute nothing there; only the optimal-cost
            # (envelope) term 0.3 * 1/2 z z' remains.
            x, u, _ = mpc(x0, QuadCost(C, c), dx)
            z = torch.cat([x, u], -1)[idx[0], idx[1]]
            mult = 1.0 if idx[2] == idx[3] else 2.0
            env = 0.3 * 0.5 * mult * float(z[idx[2]] * z[idx[3]])
            an = float(C.grad[idx]) + (float(C.grad[idx[0], idx[1], idx[3], idx[2]]) if mult == 2.0 else 0.0)
            assert abs(an - env) <= 1e-9 * max(1.0, abs(env)), (idx, an, env)
            n_checked_zero += 1
            continue
        idxs = [idx]
        if t is C and idx[2] != idx[3]:
            idxs.append((idx[0], idx[1], idx[3], idx[2]))
        with torch.no_grad():
            for i in idxs:
                t[i] += eps
            up = float(loss())
            for i in idxs:
                t[i] -= 2 * eps
            dn = float(loss())
            for i in idxs:
                t[i] += eps
        fd = (up - dn) / (2 * eps)
        an = sum(float(t.grad[i]) for i in idxs)
        worst = max(worst, abs(fd - an) / max(1e-3, abs(fd)))
    assert worst <= 1e-4, worst
    assert n_checked_zero >= 1  # the seed puts bound-active controls at (t=3, b=1)


def test_mpc_module_theta_gradient_planar_envelope():
    """d J* / d mass through the module (envelope term, exact on the nonlinear model)."""
    model = DynModel.planar_quadrotor(dt=0.05)
    pb = problems.random_problem(model, 3, 6, seed=12)
    dx = PlanarQuadrotorDx(learn=True).cuda()
    mpc = MPC(6, 2, 6, u_lower=0.0, u_upper=12.0, lqr_iter=80, eps=1e-15)
    C = torch.tensor(pb.diag, device="cuda").transpose(0, 1)
    c = torch.tensor(pb.c, device="cuda").transpose(0, 1)
    x0 = torch.tensor(pb.x0, device="cuda")
    _, _, J = mpc(x0, QuadCost(C, c), dx)
    J.sum().backward()
    g = float(dx.params.grad[0])
    h = 1e-6
    with torch.no_grad():
        dx.params[0] += h
        up = float(mpc(x0, QuadCost(C, c), dx)[2].sum())
        dx.params[0] -= 2 * h
        dn = float(mpc(x0, QuadCost(C, c), dx)[2].sum())
        dx.params[0] += h
    fd = (up - dn) / (2 * h)
    assert abs(fd - g) <= 1e-5 * max(1.0, abs(fd))
