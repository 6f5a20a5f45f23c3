"""GPU property tests: the reference's invariants (tests/test_gradlayer.py:37-95,
tests/test_batchexec.py:48-134, tests/test_ilqr.py:244-295) on the CUDA path, the launch
contract (one kernel per forward solve — all iterations fused — and one per backward),
and the NEW dtheta / optimal-cost gradients against the C oracle."""

import numpy as np
import pytest
import torch

import oracle
from paper_2605_29155_b200 import DynModel, SolveSettings, _lib, problems, solver

pytestmark = pytest.mark.gpu


def _solve(pb, dtype=torch.float64, C=None, **kw):
    C = pb.dense_C() if C is None else C
    return solver.solve_raw(pb.model, pb.settings, pb.x0, C, pb.c, pb.U_warm, dtype=dtype, **kw)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_bitwise_deterministic(dtype):
    pb = problems.random_problem(DynModel.quadrotor(), 300, 10, seed=1)
    a, b = _solve(pb, dtype), _solve(pb, dtype)
    assert torch.equal(a.X, b.X) and torch.equal(a.U, b.U) and torch.equal(a.J, b.J)
    assert torch.equal(a.iters, b.iters) and torch.equal(a.K, b.K)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_batch_equals_single_instance(dtype):
    """Per-instance results do not depend on the batch (test_batchexec.py:55-62)."""
    pb = problems.random_problem(DynModel.quadrotor(), 24, 10, seed=2)
    full = _solve(pb, dtype)
    for i in (0, 5, 23):
        one = solver.solve_raw(pb.model, pb.settings, pb.x0[i:i + 1], pb.dense_C()[i:i + 1], pb.c[i:i + 1],
                               pb.U_warm[i:i + 1], dtype=dtype)
        assert torch.equal(one.X[0], full.X[i]) and torch.equal(one.U[0], full.U[i])
        assert int(one.iters[0]) == int(full.iters[i])


def test_one_launch_per_forward_and_backward():
    """<= 4 launches per iLQR iteration (north_star): the fused forward is ONE launch for the
    rollout plus every iteration, the implicit backward ONE launch."""
    pb = problems.hover_problem(DynModel.quadrotor(), 64, 10, seed=0, conv_tol=0.0, K_max=5)
    n0 = _lib.launch_count()
    out = _solve(pb, torch.float32)
    n1 = _lib.launch_count()
    solver.backward_raw(pb.model, pb.settings, out.C, out.c, out.X, out.U, None, np.ones((64, 10, 4)))
    n2 = _lib.launch_count()
    assert n1 - n0 == 1 and n2 - n1 == 1
    assert int(out.iters.max()) == 5


def test_failed_instance_does_not_abort_batch():
    """test_batchexec.py:93-104: a diverging instance is flagged, the rest solve."""
    m = DynModel.linear(np.array([[10.0]]), np.array([[1.0]]))
    s = SolveSettings(T=400, u_min=np.array([-90.0]), u_max=np.array([90.0]), K_max=2)
    C = np.zeros((2, 400, 2, 2))
    C[:, :, 0, 0] = C[:, :, 1, 1] = 1.0
    out = solver.solve_raw(m, s, np.array([[0.0], [1.0]]), C, np.zeros((2, 400, 2)), np.zeros((2, 400, 1)),
                           dtype=torch.float64)
    ft = out.fail_t.cpu().numpy()
    assert ft[0] == -1 and ft[1] > 250
    assert not bool(out.failed[0]) and bool(out.failed[1])


def test_zero_seed_linearity_and_symmetry():
    """test_gradlayer.py:37-74 on the GPU backward."""
    rng = np.random.default_rng(4)
    pb = problems.random_problem(DynModel.quadrotor(), 16, 8, seed=4)
    out = _solve(pb)
    T, n, m = 8, 13, 4
    z = solver.backward_raw(pb.model, pb.settings, out.C, out.c, out.X, out.U, np.zeros((16, T + 1, n)),
                            np.zeros((16, T, m)))
    assert torch.count_nonzero(z.dC) == 0 and torch.count_nonzero(z.dc) == 0 and torch.count_nonzero(z.dx0) == 0
    s1 = (rng.normal(size=(16, T + 1, n)), rng.normal(size=(16, T, m)))
    s2 = (rng.normal(size=(16, T + 1, n)), rng.normal(size=(16, T, m)))
    g1 = solver.backward_raw(pb.model, pb.settings, out.C, out.c, out.X, out.U, *s1)
    g2 = solver.backward_raw(pb.model, pb.settings, out.C, out.c, out.X, out.U, *s2)
    g12 = solver.backward_raw(pb.model, pb.settings, out.C, out.c, out.X, out.U, s1[0] + s2[0], s1[1] + s2[1])
    for k in ("dC", "dc", "dx0"):
        torch.testing.assert_close(getattr(g12, k), getattr(g1, k) + getattr(g2, k), atol=1e-11, rtol=1e-11)
    assert torch.equal(g1.dC, g1.dC.transpose(-1, -2))


def test_clamped_dimensions_have_zero_gradients():
    """test_gradlayer.py:77-95."""
    m = DynModel.double_integrator(2, dt=0.1)
    T, nx, nu = 4, 4, 2
    diag = np.ones((1, T, 6))
    c = np.zeros((1, T, 6))
    c[0, :, nx] = -100.0
    s = SolveSettings(T=T, u_min=-np.ones(nu), u_max=np.ones(nu), K_max=8)
    out = solver.solve_raw(m, s, np.zeros((1, nx)), diag, c, np.zeros((1, T, nu)), dtype=torch.float64)
    assert bool(out.clamped[0, :, 0].all())
    rng = np.random.default_rng(3)
    g = solver.backward_raw(m, s, out.C, out.c, out.X, out.U, rng.normal(size=(1, T + 1, nx)),
                            rng.normal(size=(1, T, nu)))
    assert torch.count_nonzero(g.dc[0, :, nx]) == 0 and torch.count_nonzero(g.dC[0, :, nx]) == 0


@pytest.mark.parametrize("kind", ["linear", "planar", "quad13"])
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_dtheta_and_cost_gradients_match_oracle(kind, dtype):
    """NEW gradients (dtheta, dL/dJ envelope terms) on the GPU vs the FD-pinned oracle."""
    rng = np.random.default_rng(5)
    if kind == "linear":
        A = np.eye(3) + 0.1 * rng.normal(size=(3, 3))
        Bm = 0.5 * rng.normal(size=(3, 2))
        model = DynModel.linear(A, Bm)
        s = SolveSettings(T=6, u_min=-0.2 * np.ones(2), u_max=0.2 * np.ones(2), K_max=20)
        Bn, T = 16, 6
        M = rng.normal(size=(Bn, T, 5, 5))
        C = 0.3 * np.einsum("btij,btkj->btik", M, M) + 0.8 * np.eye(5)
        c = 0.3 * rng.normal(size=(Bn, T, 5))
        x0 = 0.5 * rng.normal(size=(Bn, 3))
        Uw = np.zeros((Bn, T, 2))
    else:
        model = DynModel.planar_quadrotor(dt=0.05) if kind == "planar" else DynModel.quadrotor()
        pb = problems.random_problem(model, 16, 8, seed=6, K_max=20)
        s, C, c, x0, Uw = pb.settings, pb.dense_C(), pb.c, pb.x0, pb.U_warm
        Bn, T = 16, 8
    ref = oracle.forward(model, s, x0, C, c, Uw)
    n, m = model.n_x, model.n_u
    sX, sU, sJ = rng.normal(size=(Bn, T + 1, n)), rng.normal(size=(Bn, T, m)), rng.normal(size=Bn)
    # identical inputs on both sides (f32 kernel: f32-rounded)
    rnd = (lambda a: np.asarray(a, np.float32).astype(np.float64)) if dtype == torch.float32 else np.asarray
    C, c, X, U, sX, sU, sJ = (rnd(a) for a in (C, c, ref["X"], ref["U"], sX, sU, sJ))
    rb = oracle.backward(model, s, C, c, X, U, sX, sU, sJ)
    g = solver.backward_raw(model, s, C, c, X, U, sX, sU, sJ, dtype=dtype, want_theta=True)
    tol = 1e-9 if dtype == torch.float64 else 1e-4
    ok = rb["fail_t"] < 0
    for key in ("dtheta", "dC", "dc", "dx0"):
        got = getattr(g, key).cpu().numpy()[ok]
        want = rb[key][ok]
        err = np.abs(got - want).max() / max(1.0, np.abs(want).max())
        assert err <= tol, f"{key}: {err:.2e}"


def test_per_problem_theta():
    """theta_stride = n_theta: every problem carries its own model parameters."""
    model = DynModel.quadrotor()
    pb = problems.hover_problem(model, 8, 10, seed=0)
    th = np.tile(model.params, (8, 1))
    th[:, 0] *= np.linspace(0.8, 1.2, 8)  # masses
    out = solver.solve_raw(model, pb.settings, pb.x0, pb.diag, pb.c, pb.U_warm, dtype=torch.float64, theta=th)
    for i in (0, 7):
        mi = model.with_params(th[i])
        one = solver.solve_raw(mi, pb.settings, pb.x0[i:i + 1], pb.diag[i:i + 1], pb.c[i:i + 1],
                               pb.U_warm[i:i + 1], dtype=torch.float64)
        assert torch.equal(one.U[0], out.U[i])


def test_dynamics_quad13_vs_oracle():
    m = DynModel.quadrotor()
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, size=(64, 13))
    u = rng.uniform(0, 5, size=(64, 4))
    xn, A, B = solver.dynamics(m, x, u)
    rxn, rA, rB = oracle.dynamics(m, x, u)
    np.testing.assert_allclose(xn, rxn, rtol=1e-14, atol=1e-14)
    np.testing.assert_allclose(A, rA, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(B, rB, rtol=1e-13, atol=1e-13)


def test_latency_kernel_repeatable_across_waves():
    """The block-per-problem forward gives bit-identical results across repeated launches,
    including blocks of a second wave that inherit another block's shared memory (guards
    the block-wide initialisation ordering)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = r'''
import sys, torch
sys.path.insert(0, ".")
from paper_2605_29155_b200 import DynModel, problems, solver
pb = problems.random_problem(DynModel.quadrotor(), 300, 10, seed=1)
C = pb.dense_C()
ref = solver.solve_raw(pb.model, pb.settings, pb.x0, C, pb.c, pb.U_warm)
for i in range(30):
    a = solver.solve_raw(pb.model, pb.settings, pb.x0, C, pb.c, pb.U_warm)
    assert torch.equal(a.X, ref.X) and torch.equal(a.K, ref.K) and torch.equal(a.iters, ref.iters), i
'''
    subprocess.run([sys.executable, "-c", code], check=True, cwd=root, env=dict(os.environ, DIFFMPC_FWD="lat"))


def test_lockstep_and_free_groups_agree_and_repeat():
    """The throughput forward's two group schedules (warp lockstep / free-running, the
    DIFFMPC_LOCKSTEP knob) are each bit-repeatable on batches with mixed iteration counts
    and at conv_tol = 0 (a schedule-dependent stale read once showed up exactly there: ~100
    of 16384 fixed-work solves differing run to run), and agree with each other to f32
    round-off (they are separate instantiations: the compiler may contract a*b + c*d
    differently), with identical iteration counts under natural convergence."""
    import os
    import subprocess
    import sys
    import tempfile

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2605_29155_b200 import DynModel, problems, solver
m = DynModel.quadrotor()
out = {}
for name, pb in (("fixed", problems.hover_problem(m, 16384, 10, seed=0, conv_tol=0.0)),
                 ("random", problems.random_problem(m, 4096, 10, seed=3))):
    C = torch.tensor(pb.dense_C(), dtype=torch.float32, device="cuda")
    args = [torch.tensor(a, dtype=torch.float32, device="cuda") for a in (pb.x0, pb.c, pb.U_warm)]
    ref = None
    for r in range(3):
        o = solver.solve_raw(m, pb.settings, args[0], C, args[1], args[2], kernel="throughput")
        if ref is None:
            ref = o
        else:
            assert torch.equal(o.U, ref.U) and torch.equal(o.iters, ref.iters), (name, r)
    out[name + "_U"] = ref.U.cpu().numpy()
    out[name + "_it"] = ref.iters.cpu().numpy()
np.savez(sys.argv[1], **out)
'''
    res = []
    for ls in ("0", "1"):
        f = os.path.join(tempfile.mkdtemp(), "o.npz")
        subprocess.run([sys.executable, "-c", code, f], check=True, cwd=root,
                       env=dict(os.environ, DIFFMPC_LOCKSTEP=ls))
        res.append(np.load(f))
    np.testing.assert_array_equal(res[0]["random_it"], res[1]["random_it"])
    for k in ("random_U", "fixed_U"):
        np.testing.assert_allclose(res[0][k], res[1][k], rtol=1e-4, atol=1e-4, err_msg=k)


@pytest.mark.parametrize("layout", ["dense", "diag"])
def test_solve_plan_matches_solve_raw(layout):
    """The preallocated launch path gives the same results as the allocating API."""
    m = DynModel.quadrotor()
    pb = problems.random_problem(m, 40, 8, seed=5)
    dev = torch.device("cuda")
    C = pb.dense_C() if layout == "dense" else pb.diag
    t = lambda a: torch.tensor(a, dtype=torch.float32, device=dev)  # noqa: E731
    x0, Ct, c, Uw = t(pb.x0), t(C), t(pb.c), t(pb.U_warm)
    ref = solver.solve_raw(m, pb.settings, x0, Ct, c, Uw)
    dU = torch.zeros((40, 8, 4), device=dev)
    dU[:, 0] = 1.0
    gref = solver.backward_raw(m, pb.settings, Ct, c, ref.X, ref.U, None, dU)
    plan = solver.SolvePlan(m, pb.settings, 40, layout=layout, device=dev)
    for _ in range(2):  # reuse of the plan's buffers
        out = plan.solve(x0, Ct, c, Uw)
        g = plan.backward(dLdU=dU)
        assert torch.equal(out.X, ref.X) and torch.equal(out.U, ref.U) and torch.equal(out.iters, ref.iters)
        assert torch.equal(g.dC, gref.dC) and torch.equal(g.dc, gref.dc) and torch.equal(g.dx0, gref.dx0)
    with pytest.raises(Exception):
        plan.solve(x0.double(), Ct, c, Uw)


@pytest.mark.parametrize("B", [3, 5, 7, 33])
def test_small_odd_batches_repeatable(B):
    """Every problem of small odd batches is solved and written on every launch (regression
    test for the warp-level work claim that intermittently dropped a warp's second group)."""
    m = DynModel.quadrotor()
    pb = problems.random_problem(m, B, 10, seed=B)
    C = pb.dense_C()
    ref = solver.solve_raw(m, pb.settings, pb.x0, C, pb.c, pb.U_warm, kernel="throughput")
    assert bool(((ref.iters >= 1) & (ref.iters <= pb.settings.K_max)).all())
    for _ in range(25):
        o = solver.solve_raw(m, pb.settings, pb.x0, C, pb.c, pb.U_warm, kernel="throughput")
        assert torch.equal(o.iters, ref.iters) and torch.equal(o.U, ref.U) and torch.equal(o.J, ref.J)


@pytest.mark.parametrize("kernel", ["throughput", "latency"])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_empty_batch(kernel, dtype):
    """B = 0 (an empty minibatch): the forward and the backward return empty outputs of the
    right shapes and launch nothing (the reference's batch loops simply do not run)."""
    m = DynModel.quadrotor()
    pb = problems.random_problem(m, 2, 10, seed=4)
    z = lambda a: np.asarray(a)[:0]  # noqa: E731
    n0 = _lib.launch_count()
    out = solver.solve_raw(m, pb.settings, z(pb.x0), z(pb.dense_C()), z(pb.c), z(pb.U_warm), dtype=dtype,
                           kernel=kernel)
    g = solver.backward_raw(m, pb.settings, out.C, out.c, out.X, out.U, None, np.zeros((0, 10, 4)), dtype=dtype)
    torch.cuda.synchronize()
    assert _lib.launch_count() == n0
    assert tuple(out.X.shape) == (0, 11, 13) and tuple(out.U.shape) == (0, 10, 4) and out.J.numel() == 0
    assert tuple(g.dC.shape) == (0, 10, 17, 17) and tuple(g.dc.shape) == (0, 10, 17) and g.dx0.numel() == 0
