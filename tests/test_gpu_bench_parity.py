"""Parity on the BENCHMARKED path: the throughput forward kernel and the backward kernel on
bench.py's own workload (BASELINE config 3: 13-state quadrotor, T=10, B=16384, K_max=10,
conv_tol=1e-6) against the C oracle (pinned bit-exactly to the reference goldens), on
IDENTICAL inputs (for the f32 kernels the oracle solves the f32-rounded problem).

Gate (BASELINE.json north_star): u*, x*, J, K, k, J history and every
gradient (dC, dc, dx0, dX, dU) within 1e-4 relative per instance in f32 (1e-9 in f64);
iteration counts, clamp masks, convergence / failure flags and accepted step sizes
identical (f64: on every instance; f32: except where the reference itself decided within
round-off of conv_tol — parity_util.F32_FLIP_MARGIN; u*, x*, J and the gradients are still
compared on such instances). References: batchexec.py:156-163, 215-233 (workload),
ilqr.py:216-268 (outputs), gradlayer.py:98-150 (gradients).
"""

import functools
import os

import numpy as np
import pytest
import torch

import parity_util as pu
from paper_2605_29155_b200 import DynModel, _abi, problems, solver

pytestmark = pytest.mark.gpu

B_BENCH = 16384


@functools.lru_cache(maxsize=None)
def workload(name):
    m = DynModel.quadrotor(dt=0.05)
    if name == "hover":  # bench.py's workload (problems.hover_problem, seed 0)
        return problems.hover_problem(m, B_BENCH, 10, seed=0)
    return problems.random_problem(m, B_BENCH, 10, seed=104)  # ~25% clamped controls


def seeds(pb, kind):
    B, T, nx, nu = pb.B, pb.settings.T, pb.model.n_x, pb.model.n_u
    if kind == "layer":  # the AC-MPC layer's seed, as timed by bench.py (policy.py:272)
        dU = np.zeros((B, T, nu))
        dU[:, 0, :] = 1.0
        return None, dU
    rng = np.random.default_rng(5)
    return rng.normal(size=(B, T + 1, nx)), rng.normal(size=(B, T, nu))


@functools.lru_cache(maxsize=None)
def oracle_run(name, layout, dt_name, seed_kind):
    import oracle

    dtype = torch.float32 if dt_name == "f32" else torch.float64
    pb = workload(name)
    cost = pb.diag if layout == "diag" else pb.dense_C()
    lay = _abi.COST_DIAG if layout == "diag" else _abi.COST_DENSE
    x0, C, c, Uw = pu.round_inputs((pb.x0, cost, pb.c, pb.U_warm), dtype)
    dX, dU = pu.round_inputs(seeds(pb, seed_kind), dtype)
    th = os.cpu_count() or 8
    f = oracle.forward(pb.model, pb.settings, x0, C, c, Uw, layout=lay, threads=th)
    b = oracle.backward(pb.model, pb.settings, C, c, f["X"], f["U"], dX, dU, layout=lay, threads=th,
                        want_theta=False)
    return (x0, C, c, Uw, dX, dU), f, b


CASES = [("hover", "dense"), ("hover", "diag"), ("random", "dense")]


@pytest.mark.parametrize("dt_name", ["f32", "f64"])
@pytest.mark.parametrize("name,layout", CASES, ids=[f"{a}-{b}" for a, b in CASES])
def test_bench_workload_matches_oracle(name, layout, dt_name):
    dtype = torch.float32 if dt_name == "f32" else torch.float64
    pb = workload(name)
    (x0, C, c, Uw, dX, dU), ref, refg = oracle_run(name, layout, dt_name, "layer")
    out = solver.solve_raw(pb.model, pb.settings, x0, C, c, Uw, dtype=dtype, kernel="throughput")
    g = solver.backward_raw(pb.model, pb.settings, out.C, out.c, out.X, out.U, dX, dU, dtype=dtype,
                            want_traj=True)
    torch.cuda.synchronize()
    rep = pu.compare_forward(out, ref, dtype, pb.settings.conv_tol)
    pu.assert_forward(rep, dtype)
    # gradients on EVERY instance, including an f32 count flip at the convergence threshold
    ok = (ref["fail_t"] < 0) & (ref["diverged"] == 0)
    brep = pu.compare_backward(g, refg, dtype, ok, layout_diag=(layout == "diag"))
    pu.assert_backward(brep, dtype)
    assert brep["n_compared"] == B_BENCH
    assert rep["n_compared"] + len(rep["flips"]) == B_BENCH


@pytest.mark.parametrize("dt_name", ["f32", "f64"])
def test_bench_workload_random_seeds(dt_name):
    """Dense random seeds dL/dX, dL/dU (every gradient path exercised) on the clamped batch."""
    dtype = torch.float32 if dt_name == "f32" else torch.float64
    pb = workload("random")
    (x0, C, c, Uw, dX, dU), ref, refg = oracle_run("random", "dense", dt_name, "random")
    out = solver.solve_raw(pb.model, pb.settings, x0, C, c, Uw, dtype=dtype, kernel="throughput")
    g = solver.backward_raw(pb.model, pb.settings, out.C, out.c, out.X, out.U, dX, dU, dtype=dtype,
                            want_traj=True)
    torch.cuda.synchronize()
    pu.assert_forward(pu.compare_forward(out, ref, dtype, pb.settings.conv_tol), dtype)
    ok = ref["fail_t"] < 0
    pu.assert_backward(pu.compare_backward(g, refg, dtype, ok), dtype)


def test_bench_workload_lockstep_schedule_matches_oracle():
    """The warp-lockstep group schedule (auto for conv_tol = 0 and T >= 16) on the same batch."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = r'''
import sys, numpy as np, torch
sys.path[:0] = [".", "tests", "oracle"]
import test_gpu_bench_parity as t, parity_util as pu
from paper_2605_29155_b200 import solver
pb = t.workload("random")
(x0, C, c, Uw, dX, dU), ref, refg = t.oracle_run("random", "dense", "f32", "layer")
out = solver.solve_raw(pb.model, pb.settings, x0, C, c, Uw, dtype=torch.float32, kernel="throughput")
torch.cuda.synchronize()
pu.assert_forward(pu.compare_forward(out, ref, torch.float32, pb.settings.conv_tol), torch.float32)
print("ok")
'''
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=dict(os.environ, DIFFMPC_LOCKSTEP="1"),
                       capture_output=True, text=True)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
