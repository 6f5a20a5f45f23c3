"""GPU parity: the CUDA path (through the C ABI) against the committed golden vectors
of the unmodified reference, on the same inputs.

Gates (BASELINE.json north_star; tests/parity_util.py):
  f64 kernels  — X, U, J, K, k, J history, dC, dc, dx0, dX, dU within 1e-9 relative.
  f32 kernels  — the same tensors within 1e-4 relative
                 (max|a-b| <= 1e-4 * max(1, max|b|) per instance and tensor).
  both         — iteration counts, clamp masks, convergence / failure / divergence flags,
                 backward failure stages and accepted step sizes identical on every
                 natural-convergence case (conv_tol > 0). conv_tol = 0 ("fixed work") runs
                 iterate on round-off and are gated on J only.
Both forward mappings (throughput and latency kernel) are checked against every golden.
"""

import numpy as np
import pytest
import torch

import golden_util as gu
import parity_util as pu
from paper_2605_29155_b200 import _abi, solver

pytestmark = pytest.mark.gpu

CASES = [(n, l) for n in gu.SOLVE_CASES for l in gu.load(n).layouts()]
KERNELS = ["throughput", "latency"]


def run_forward(g, layout, dtype, kernel="auto"):
    return solver.solve_raw(g.model, g.settings, g["x0"], g.cost(layout), g["c"], g["U_warm"],
                            dtype=dtype, kernel=kernel)


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32], ids=["f64", "f32"])
@pytest.mark.parametrize("name,layout", CASES, ids=[f"{n}-{'diag' if l else 'dense'}" for n, l in CASES])
def test_forward_parity(name, layout, dtype, kernel):
    """Every forward output the goldens hold (X, U, J, K, k, J history, step-size history,
    iteration counts, clamp masks, convergence / failure flags), both forward mappings."""
    g = gu.load(name)
    out = run_forward(g, layout, dtype, kernel)
    torch.cuda.synchronize()
    rep = pu.compare_forward(out, g.d, dtype, g.settings.conv_tol)
    fixed_work = g.settings.conv_tol == 0.0
    if fixed_work:
        # conv_tol == 0 iterates on round-off until no candidate improves J: counts are not
        # gated and the flat optimum lets X/U drift at sqrt(eps); J agrees
        rep["err"].pop("K"), rep["err"].pop("k"), rep["err"].pop("J_hist")
        rep["alpha_hist_mismatch"] = 0
        pu.assert_forward(rep, dtype, allow_flips=True, xtol=max(pu.TOL[dtype], 1e-6))
    else:
        pu.assert_forward(rep, dtype)
        assert rep["converged_mismatch"] == 0
    if dtype == torch.float64:
        # failed initial rollouts: rows up to the non-finite state as the reference computed
        # them, zeros after (Workspace zero init) -- not another problem's states
        bad = np.nonzero(g["diverged"] & (g["fail_t"] >= 0))[0]
        X = pu.as_np(out.X)
        for i in bad:
            np.testing.assert_array_equal(X[i], g["X"][i])


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32], ids=["f64", "f32"])
@pytest.mark.parametrize("name,layout", CASES, ids=[f"{n}-{'diag' if l else 'dense'}" for n, l in CASES])
def test_backward_parity(name, layout, dtype):
    """Backward through the REFERENCE solution, so the gradient kernel is checked in isolation:
    dC, dc, dx0 and the differential trajectory dX, dU; exact backward failure stages."""
    g = gu.load(name)
    res = solver.backward_raw(g.model, g.settings, g.cost(layout), g["c"], g["X"], g["U"],
                              g["dLdX"], g["dLdU"], dtype=dtype, want_traj=True)
    torch.cuda.synchronize()
    # instances whose forward diverged carry non-finite trajectories; skip them
    ok = (g["fail_t"] < 0) & (g["diverged"] == 0)
    rep = pu.compare_backward(res, g.d, dtype, ok, layout_diag=bool(layout))
    fail_ok = ok | (g["bfail_t"] >= 0)
    rep["bfail_mismatch"] = int((pu.as_np(res.fail_t)[fail_ok] != g["bfail_t"][fail_ok]).sum())
    pu.assert_backward(rep, dtype)


@pytest.mark.parametrize("name", ["planar_hover", "planar_random", "quad13_hover", "quad13_random",
                                  "quad13_dense", "linear_3x2", "linear_13x4"])
def test_end_to_end_f32(name):
    """Forward then backward entirely on the GPU (f32) vs the reference's gradients (1e-4)."""
    g = gu.load(name)
    layout = g.layouts()[-1]
    out = run_forward(g, layout, torch.float32)
    res = solver.backward_raw(g.model, g.settings, out.C, out.c, out.X, out.U,
                              g["dLdX"], g["dLdU"], dtype=torch.float32, want_traj=True)
    torch.cuda.synchronize()
    pu.assert_forward(pu.compare_forward(out, g.d, torch.float32, g.settings.conv_tol), torch.float32)
    ok = (g["fail_t"] < 0) & (g["diverged"] == 0)
    pu.assert_backward(pu.compare_backward(res, g.d, torch.float32, ok, layout_diag=bool(layout)),
                       torch.float32)


def test_dynamics_vs_reference():
    d = gu.load_aux("dynamics")
    from paper_2605_29155_b200.dynamics import DynModel

    models = {
        "di2": DynModel.double_integrator(2, dt=0.1),
        "planar": DynModel.planar_quadrotor(dt=0.05),
        "linear": DynModel.linear(np.array([[0.9, 0.1], [0.0, 1.1]]), np.array([[0.0], [0.5]])),
    }
    for name, m in models.items():
        xn, A, B = solver.dynamics(m, d[f"{name}_x"], d[f"{name}_u"])
        np.testing.assert_allclose(xn, d[f"{name}_xn"], rtol=1e-13, atol=1e-13)
        np.testing.assert_allclose(A, d[f"{name}_A"], rtol=1e-13, atol=1e-13)
        np.testing.assert_allclose(B, d[f"{name}_B"], rtol=1e-13, atol=1e-13)


@pytest.mark.gpu
def test_latency_kernel_matches_throughput_kernel():
    """The small-batch (block-per-problem) forward and the throughput forward solve the same
    problems to the same iterates: identical iteration counts / masks, f32 round-off apart."""
    import subprocess
    import sys

    code = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2605_29155_b200 import DynModel, problems, solver
m = DynModel.quadrotor()
pb = problems.random_problem(m, 96, 10, seed=21)
o = solver.solve_raw(m, pb.settings, pb.x0, pb.dense_C(), pb.c, pb.U_warm)
np.savez(sys.argv[1], U=o.U.cpu().numpy(), X=o.X.cpu().numpy(), it=o.iters.cpu().numpy(),
         cl=o.clamped.cpu().numpy(), J=o.J.cpu().numpy())
'''
    import os
    import tempfile

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for mode in ("lat", "tput"):
        f = os.path.join(tempfile.mkdtemp(), f"{mode}.npz")
        env = dict(os.environ, DIFFMPC_FWD=mode)
        subprocess.run([sys.executable, "-c", code, f], check=True, cwd=root, env=env)
        outs[mode] = np.load(f)
    a, b = outs["lat"], outs["tput"]
    np.testing.assert_array_equal(a["it"], b["it"])
    np.testing.assert_array_equal(a["cl"], b["cl"])
    np.testing.assert_allclose(a["U"], b["U"], rtol=1e-4, atol=1e-4)
    np.testing.assert_allclose(a["J"], b["J"], rtol=1e-5)


@pytest.mark.gpu
def test_kernel_select_per_call():
    """kernel_select picks the forward mapping per call; both agree on iterates, masks and
    counts, and "throughput" is batch-size invariant bit for bit."""
    from paper_2605_29155_b200 import DynModel, problems

    m = DynModel.quadrotor()
    pb = problems.random_problem(m, 64, 10, seed=33)
    C = pb.dense_C()
    lat = solver.solve_raw(m, pb.settings, pb.x0, C, pb.c, pb.U_warm, kernel="latency")
    tp = solver.solve_raw(m, pb.settings, pb.x0, C, pb.c, pb.U_warm, kernel="throughput")
    assert torch.equal(lat.iters, tp.iters) and torch.equal(lat.clamped, tp.clamped)
    assert torch.allclose(lat.U, tp.U, rtol=1e-4, atol=1e-4)
    one = solver.solve_raw(m, pb.settings, pb.x0[5:6], C[5:6], pb.c[5:6], pb.U_warm[5:6], kernel="throughput")
    assert torch.equal(one.U[0], tp.U[5]) and torch.equal(one.X[0], tp.X[5])
    with pytest.raises(Exception):
        solver.solve_raw(m, pb.settings, pb.x0, C, pb.c, pb.U_warm, kernel="fastest")


@pytest.mark.gpu
@pytest.mark.parametrize("alphas", [(1.0,), (1.0, 0.3), (1.0, 0.7, 0.5, 0.3, 0.2, 0.1), (1.0, 0.8, 0.6, 0.5, 0.4, 0.25, 0.1, 0.05)])
@pytest.mark.parametrize("kernel", ["throughput", "latency"])
def test_line_search_sizes_match_oracle(alphas, kernel):
    """Step-size lists other than the default four: fewer candidates than the four slots
    (duplicated slots) and two line-search rounds (five to eight candidates; no in-place
    alpha_0 trajectory, winner re-rolled). f64 kernels vs the C oracle."""
    import oracle
    from paper_2605_29155_b200 import DynModel, problems

    for model, B in ((DynModel.quadrotor(), 48), (DynModel.planar_quadrotor(dt=0.05), 64)):
        pb = problems.random_problem(model, B, 8, seed=41, alphas=alphas)
        C = pb.dense_C()
        ref = oracle.forward(model, pb.settings, pb.x0, C, pb.c, pb.U_warm)
        out = solver.solve_raw(model, pb.settings, pb.x0, C, pb.c, pb.U_warm, dtype=torch.float64, kernel=kernel)
        np.testing.assert_array_equal(out.iters.cpu().numpy(), ref["iters"])
        np.testing.assert_array_equal(out.clamped.cpu().numpy().astype(np.uint8),
                                      ((ref["U"] <= pb.settings.bounds_for(model.n_u)[0]) |
                                       (ref["U"] >= pb.settings.bounds_for(model.n_u)[1])).astype(np.uint8))
        np.testing.assert_allclose(out.U.cpu().numpy(), ref["U"], rtol=1e-9, atol=1e-9)
        np.testing.assert_allclose(out.X.cpu().numpy(), ref["X"], rtol=1e-9, atol=1e-9)
        np.testing.assert_allclose(out.J.cpu().numpy(), ref["J"], rtol=1e-9)


@pytest.mark.gpu
@pytest.mark.parametrize("B,T", [(1, 3), (3, 10), (33, 10), (17, 40)])
@pytest.mark.parametrize("kernel", ["throughput", "latency"])
def test_odd_batches_and_long_horizons_match_oracle(B, T, kernel):
    """Batch sizes that do not fill a warp pair / block, and T=40 (largest per-problem shared
    memory), against the oracle in float64."""
    import oracle
    from paper_2605_29155_b200 import DynModel, problems

    m = DynModel.quadrotor()
    pb = problems.random_problem(m, B, T, seed=B * 100 + T)
    C = pb.dense_C()
    ref = oracle.forward(m, pb.settings, pb.x0, C, pb.c, pb.U_warm)
    out = solver.solve_raw(m, pb.settings, pb.x0, C, pb.c, pb.U_warm, dtype=torch.float64, kernel=kernel)
    np.testing.assert_array_equal(out.iters.cpu().numpy(), ref["iters"])
    np.testing.assert_allclose(out.U.cpu().numpy(), ref["U"], rtol=1e-9, atol=1e-9)
    np.testing.assert_allclose(out.J.cpu().numpy(), ref["J"], rtol=1e-9)
    np.testing.assert_allclose(out.K.cpu().numpy(), ref["K"], rtol=1e-7, atol=1e-9)
