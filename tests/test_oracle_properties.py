"""Oracle property tests, restating the reference suite's oracle / FD / invariant checks
(tests/test_ilqr.py, tests/test_gradlayer.py, tests/test_acceptance.py C1-C3, C6) on the
C oracle, plus finite-difference pins for the two gradients the reference does not have
(SURVEY.md §8(a) NEW rows: dynamics parameters, optimal cost)."""

import itertools

import numpy as np
import pytest

import oracle
from paper_2605_29155_b200.dynamics import DynModel
from paper_2605_29155_b200.settings import SolveSettings

BIG = 1e9


def lq_kkt_solve(A, B, C, c, x0):
    """Dense direct transcription of the equality-constrained LQ problem
    (independent of the Riccati path; cf. tests/oracles.py:16-57)."""
    T = len(C)
    n, m = B.shape
    nv = (T + 1) * n + T * m
    xs = lambda t: slice(t * n, (t + 1) * n)  # noqa: E731
    us = lambda t: slice((T + 1) * n + t * m, (T + 1) * n + (t + 1) * m)  # noqa: E731
    H, g = np.zeros((nv, nv)), np.zeros(nv)
    for t in range(T):
        Z = np.zeros((n + m, nv))
        Z[:n, xs(t)] = np.eye(n)
        Z[n:, us(t)] = np.eye(m)
        H += Z.T @ C[t] @ Z
        g += Z.T @ c[t]
    E = np.zeros(((T + 1) * n, nv))
    e = np.zeros((T + 1) * n)
    E[:n, xs(0)] = np.eye(n)
    e[:n] = x0
    for t in range(T):
        r = slice((t + 1) * n, (t + 2) * n)
        E[r, xs(t + 1)] = np.eye(n)
        E[r, xs(t)] = -A
        E[r, us(t)] = -B
    K = np.block([[H, E.T], [E, np.zeros((E.shape[0], E.shape[0]))]])
    z = np.linalg.solve(K, np.concatenate([-g, e]))[:nv]
    return z[(T + 1) * n:].reshape(T, m), 0.5 * z @ H @ z + g @ z


def test_lq_one_iteration_matches_kkt():
    """Acceptance criterion 1 (test_acceptance.py:39-62): LQ exactness of one iteration."""
    rng = np.random.default_rng(101)
    for _ in range(20):
        d = int(rng.integers(1, 4))
        T = int(rng.choice([2, 10, 30]))
        m = DynModel.double_integrator(d, dt=0.1)
        nz = m.n_x + m.n_u
        M = rng.normal(size=(T, nz, nz))
        C = 0.3 * np.einsum("tij,tkj->tik", M, M) + 0.5 * np.eye(nz)
        c = rng.normal(size=(T, nz))
        x0 = rng.normal(size=m.n_x)
        s = SolveSettings(T=T, u_min=-BIG * np.ones(m.n_u), u_max=BIG * np.ones(m.n_u), K_max=1)
        o = oracle.forward(m, s, x0[None], C[None], c[None], np.zeros((1, T, m.n_u)))
        _, A, Bm = oracle.dynamics(m, x0[None], np.zeros((1, m.n_u)))
        U_ref, J_ref = lq_kkt_solve(A[0], Bm[0], C, c, x0)
        assert abs(o["J"][0] - J_ref) <= 1e-8 * abs(J_ref)
        assert np.abs(o["U"][0, 0] - U_ref[0]).max() <= 1e-8


def boxqp_bruteforce(H, g, lo, hi):
    n = g.shape[0]
    best, bu = np.inf, None
    for pat in itertools.product((0, 1, 2), repeat=n):
        u = np.zeros(n)
        free = [i for i, p in enumerate(pat) if p == 0]
        fixed = [i for i, p in enumerate(pat) if p != 0]
        for i in fixed:
            u[i] = lo[i] if pat[i] == 1 else hi[i]
        if free:
            rhs = g[free] + (H[np.ix_(free, fixed)] @ u[fixed] if fixed else 0.0)
            u[free] = np.linalg.solve(H[np.ix_(free, free)], -rhs)
        if np.all(u >= lo - 1e-12) and np.all(u <= hi + 1e-12):
            v = 0.5 * u @ H @ u + g @ u
            if v < best:
                best, bu = v, u.copy()
    return bu


def test_boxqp_matches_enumeration():
    """Acceptance criterion 2 (test_acceptance.py:65-79)."""
    rng = np.random.default_rng(102)
    for _ in range(200):
        n = int(rng.integers(2, 5))
        M = rng.normal(size=(n, n))
        H = M @ M.T + 0.3 * np.eye(n)
        g = 2.0 * rng.normal(size=n)
        lo, hi = rng.uniform(-2.0, -0.05, size=n), rng.uniform(0.05, 2.0, size=n)
        u, _, st = oracle.boxqp(H, g, lo, hi)
        assert st == 0
        assert np.abs(u - boxqp_bruteforce(H, g, lo, hi)).max() <= 1e-8


def linear_instance(rng, n=3, m=2, T=5):
    A = np.eye(n) + 0.1 * rng.normal(size=(n, n))
    B = 0.5 * rng.normal(size=(n, m))
    nz = n + m
    M = rng.normal(size=(T, nz, nz))
    C = 0.3 * np.einsum("tij,tkj->tik", M, M) + 0.8 * np.eye(nz)
    c = 0.3 * rng.normal(size=(T, nz))
    x0 = 0.5 * rng.normal(size=n)
    return A, B, C, c, x0


def solve1(model, s, C, c, x0, theta=None):
    return oracle.forward(model, s, x0[None], C[None], c[None], np.zeros((1, s.T, model.n_u)), theta=theta)


def test_implicit_gradient_fd_linear():
    """Acceptance criterion 3 (test_acceptance.py:82-136): dc, diag dC, dx0 vs FD."""
    rng = np.random.default_rng(103)
    n, m, T = 3, 2, 5
    u_ref = np.array([0.3, -0.2])
    worst = 0.0
    for _ in range(6):
        A, B, C, c, x0 = linear_instance(rng, n, m, T)
        model = DynModel.linear(A, B)
        s = SolveSettings(T=T, u_min=-BIG * np.ones(m), u_max=BIG * np.ones(m), K_max=3)

        def loss(Cm, cm, xm):
            return 0.5 * np.sum((solve1(model, s, Cm, cm, xm)["U"][0, 0] - u_ref) ** 2)

        o = solve1(model, s, C, c, x0)
        dU = np.zeros((1, T, m))
        dU[0, 0] = o["U"][0, 0] - u_ref
        g = oracle.backward(model, s, C[None], c[None], o["X"], o["U"], None, dU)
        eps = 1e-5
        for t in range(T):
            for j in range(n + m):
                cp, cm = c.copy(), c.copy()
                cp[t, j] += eps
                cm[t, j] -= eps
                fd = (loss(C, cp, x0) - loss(C, cm, x0)) / (2 * eps)
                worst = max(worst, abs(fd - g["dc"][0, t, j]) / max(1e-6, abs(fd)))
                Cp, Cm = C.copy(), C.copy()
                Cp[t, j, j] += eps
                Cm[t, j, j] -= eps
                fd = (loss(Cp, c, x0) - loss(Cm, c, x0)) / (2 * eps)
                worst = max(worst, abs(fd - g["dC"][0, t, j, j]) / max(1e-6, abs(fd)))
        for j in range(n):
            xp, xm = x0.copy(), x0.copy()
            xp[j] += eps
            xm[j] -= eps
            fd = (loss(C, c, xp) - loss(C, c, xm)) / (2 * eps)
            worst = max(worst, abs(fd - g["dx0"][0, j]) / max(1e-6, abs(fd)))
    assert worst <= 1e-3, worst


@pytest.mark.parametrize("u_lim", [BIG, 0.15])
def test_dtheta_fd_linear(u_lim):
    """NEW row (probe P9): dL/d[A|B] by the co-state formula vs central FD of
    full re-solves, interior and with active bounds (exact on linear dynamics)."""
    rng = np.random.default_rng(7 if u_lim == BIG else 8)
    n, m, T = 3, 2, 6
    worst = 0.0
    for _ in range(3):
        A, B, C, c, x0 = linear_instance(rng, n, m, T)
        model = DynModel.linear(A, B)
        s = SolveSettings(T=T, u_min=-u_lim * np.ones(m), u_max=u_lim * np.ones(m), K_max=60, conv_tol=1e-14)
        a_vec, b_vec, u_ref = rng.normal(size=n), rng.normal(size=n), rng.normal(size=m)

        def loss(th):
            o = solve1(model, s, C, c, x0, theta=th)
            return 0.5 * np.sum((o["U"][0, 0] - u_ref) ** 2) + a_vec @ o["X"][0, T] + b_vec @ o["X"][0, 2]

        th0 = model.params.copy()
        o = solve1(model, s, C, c, x0)
        dX = np.zeros((1, T + 1, n))
        dX[0, T] = a_vec
        dX[0, 2] = b_vec
        dU = np.zeros((1, T, m))
        dU[0, 0] = o["U"][0, 0] - u_ref
        g = oracle.backward(model, s, C[None], c[None], o["X"], o["U"], dX, dU)
        eps = 1e-6
        for j in range(th0.size):
            tp, tm = th0.copy(), th0.copy()
            tp[j] += eps
            tm[j] -= eps
            fd = (loss(tp) - loss(tm)) / (2 * eps)
            worst = max(worst, abs(fd - g["dtheta"][0, j]) / max(1e-3, abs(fd)))
    assert worst <= 1e-5, worst


@pytest.mark.parametrize("kind", ["planar", "quad13"])
def test_optimal_cost_gradients_fd(kind):
    """NEW row (probe P10): dJ*/dc, dJ*/dC, dJ*/dx0, dJ*/dtheta from a dL/dJ seed vs FD of the
    optimal cost (envelope theorem; exact for the nonlinear models, clamped or not)."""
    from paper_2605_29155_b200 import problems

    model = DynModel.planar_quadrotor(dt=0.05) if kind == "planar" else DynModel.quadrotor(dt=0.05)
    pb = problems.random_problem(model, 1, 8, seed=31, K_max=80, conv_tol=1e-15)
    C, c, x0, Uw = pb.dense_C()[0], pb.c[0], pb.x0[0], pb.U_warm[0]
    s = pb.settings

    def J(Cm=C, cm=c, xm=x0, th=None):
        return oracle.forward(model, s, xm[None], Cm[None], cm[None], Uw[None], theta=th)["J"][0]

    o = oracle.forward(model, s, x0[None], C[None], c[None], Uw[None])
    assert o["converged"][0]
    g = oracle.backward(model, s, C[None], c[None], o["X"], o["U"], None, None, dLdJ=np.ones(1))
    eps = 1e-6
    checks = []
    for (t, j) in [(0, 0), (3, 2), (7, model.n_x), (5, model.n_x + 1)]:
        cp, cm = c.copy(), c.copy()
        cp[t, j] += eps
        cm[t, j] -= eps
        checks.append(((J(cm=cp) - J(cm=cm)) / (2 * eps), g["dc"][0, t, j]))
        Cp, Cm = C.copy(), C.copy()
        Cp[t, j, j] += eps
        Cm[t, j, j] -= eps
        checks.append(((J(Cm=Cp) - J(Cm=Cm)) / (2 * eps), g["dC"][0, t, j, j]))
    for j in range(model.n_x):
        xp, xm = x0.copy(), x0.copy()
        xp[j] += eps
        xm[j] -= eps
        checks.append(((J(xm=xp) - J(xm=xm)) / (2 * eps), g["dx0"][0, j]))
    th0 = model.params.copy()
    for j in range(th0.size):
        tp, tm = th0.copy(), th0.copy()
        h = eps * max(1.0, abs(th0[j]))
        tp[j] += h
        tm[j] -= h
        checks.append(((J(th=tp) - J(th=tm)) / (2 * h), g["dtheta"][0, j]))
    worst = max(abs(a - b) / max(1e-3, abs(a)) for a, b in checks)
    assert worst <= 1e-5, worst


def test_quad13_jacobians_match_fd():
    """tests/test_dynamics.py:62-77 style FD check for the 13-state model (no reference)."""
    m = DynModel.quadrotor()
    rng = np.random.default_rng(0)
    x = rng.uniform(-1.0, 1.0, size=(50, 13))
    u = rng.uniform(0.0, 5.0, size=(50, 4))
    _, A, B = oracle.dynamics(m, x, u)
    h = 1e-6
    for j in range(13):
        d = np.zeros(13)
        d[j] = h
        fd = (oracle.dynamics(m, x + d, u)[0] - oracle.dynamics(m, x - d, u)[0]) / (2 * h)
        assert np.abs(fd - A[:, :, j]).max() < 1e-6
    for j in range(4):
        d = np.zeros(4)
        d[j] = h
        fd = (oracle.dynamics(m, x, u + d)[0] - oracle.dynamics(m, x, u - d)[0]) / (2 * h)
        assert np.abs(fd - B[:, :, j]).max() < 1e-6


def test_quad13_hover_fixed_point():
    m = DynModel.quadrotor()
    x = m.hover_state()
    xn, _, _ = oracle.dynamics(m, x[None], m.hover_control()[None])
    assert np.abs(xn[0] - x).max() < 1e-14


def test_monotone_costs_and_exact_bounds():
    """Acceptance criterion 6 (test_acceptance.py:189-203) on the 13-state quadrotor."""
    from paper_2605_29155_b200 import problems

    pb = problems.random_problem(DynModel.quadrotor(), 200, 8, seed=106, K_max=6)
    o = oracle.forward(pb.model, pb.settings, pb.x0, pb.dense_C(), pb.c, pb.U_warm, threads=2)
    assert (o["fail_t"] < 0).all()
    assert (np.diff(o["J_hist"], axis=1) <= 1e-12).all()
    lo, hi = pb.settings.bounds_for(4)
    assert (o["U"] >= lo).all() and (o["U"] <= hi).all()
