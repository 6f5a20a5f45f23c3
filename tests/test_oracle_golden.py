"""The CPU oracle (oracle/diffmpc_oracle.c) pinned against the committed golden vectors
produced by the UNMODIFIED reference (tests/golden/make_golden.py). Bit-exact: the
oracle restates the reference's float64 arithmetic in the same order."""

import numpy as np
import pytest

import golden_util as gu
import oracle

FWD_KEYS = ("X", "U", "J", "K", "k", "iters", "converged", "diverged", "fail_t", "clamped",
            "alpha_hist", "J_hist")


@pytest.mark.parametrize("name", gu.SOLVE_CASES)
def test_forward_bit_exact(name):
    g = gu.load(name)
    o = oracle.forward(g.model, g.settings, g["x0"], g.C_dense(), g["c"], g["U_warm"], threads=2)
    for k in FWD_KEYS:
        assert np.array_equal(o[k], g[k], equal_nan=True), f"{name}: {k} differs"


@pytest.mark.parametrize("name", [n for n in gu.SOLVE_CASES if "diag" in gu.load(n).d])
def test_forward_diag_layout_bit_exact(name):
    """The diagonal cost layout (MpcSolver.solve_diag, policy.py:214-222) gives the same bits."""
    from paper_2605_29155_b200 import _abi

    g = gu.load(name)
    o = oracle.forward(g.model, g.settings, g["x0"], g["diag"], g["c"], g["U_warm"], layout=_abi.COST_DIAG)
    for k in FWD_KEYS:
        assert np.array_equal(o[k], g[k], equal_nan=True), f"{name}: {k} differs"


@pytest.mark.parametrize("name", gu.SOLVE_CASES)
def test_backward_bit_exact(name):
    g = gu.load(name)
    b = oracle.backward(g.model, g.settings, g.C_dense(), g["c"], g["X"], g["U"], g["dLdX"], g["dLdU"],
                        threads=2)
    assert np.array_equal(b["fail_t"], g["bfail_t"])
    for k in ("dC", "dc", "dx0"):
        assert np.array_equal(b[k], g[k], equal_nan=True), f"{name}: {k} differs"
    ok = g["bfail_t"] < 0
    assert np.array_equal(b["dX"][ok], g["dX"][ok], equal_nan=True)
    assert np.array_equal(b["dU"][ok], g["dU"][ok], equal_nan=True)


def test_boxqp_bit_exact():
    d = gu.load_aux("boxqp")
    for i in range(d["n"].shape[0]):
        n = int(d["n"][i])
        u, free, st = oracle.boxqp(d["H"][i, :n, :n], d["g"][i, :n], d["lo"][i, :n], d["hi"][i, :n])
        assert st == 0
        assert np.array_equal(u, d["u"][i, :n])
        assert np.array_equal(free, d["free"][i, :n].astype(bool))


def test_dynamics_bit_exact():
    from paper_2605_29155_b200.dynamics import DynModel

    d = gu.load_aux("dynamics")
    models = {
        "di2": DynModel.double_integrator(2, dt=0.1),
        "planar": DynModel.planar_quadrotor(dt=0.05),
        "linear": DynModel.linear(np.array([[0.9, 0.1], [0.0, 1.1]]), np.array([[0.0], [0.5]])),
    }
    for name, m in models.items():
        xn, A, B = oracle.dynamics(m, d[f"{name}_x"], d[f"{name}_u"])
        assert np.array_equal(xn, d[f"{name}_xn"])
        assert np.array_equal(A, d[f"{name}_A"])
        assert np.array_equal(B, d[f"{name}_B"])


def test_threads_do_not_change_results():
    """Worker-count independence (tests/test_batchexec.py:82-90)."""
    g = gu.load("quad13_random")
    a = oracle.forward(g.model, g.settings, g["x0"], g.C_dense(), g["c"], g["U_warm"], threads=1)
    b = oracle.forward(g.model, g.settings, g["x0"], g.C_dense(), g["c"], g["U_warm"], threads=4)
    for k in FWD_KEYS:
        assert np.array_equal(a[k], b[k])
