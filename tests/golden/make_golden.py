"""Generate golden vectors from the UNMODIFIED reference (run in the build container).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc python tests/golden/make_golden.py

The reference (``fusedmpc``, CPU numba float64) cannot travel to the GPU box, so its
outputs on seeded synthetic inputs are committed here as compressed .npz fixtures.
Forward: batchexec.solve_raw (batchexec.py:156-163) -> run_staged_solve, results as
collect_result reports them (ilqr.py:250-268). Backward: MpcSolveLayer.backward's
relinearisation + clamp mask (policy.py:257-272) followed by
batchexec.backward_batch_arrays (batchexec.py:180-186), but with full dL/dX, dL/dU
seeds so every seed path is pinned; failed instances are zeroed (policy.py:277-280).

Reference-model cases run first on the pristine reference; then the 13-state
quadrotor plug-in is installed (quad13_plugin.py) and a planar case is re-run
through it to check the plug-in is bit-identical to the reference (probe P3).
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

from fusedmpc import batchexec, ilqr, kernels  # noqa: E402  (the reference)
from fusedmpc.batchexec import WorkerPool  # noqa: E402
from fusedmpc.dynamics import DynModel as RefModel  # noqa: E402
from fusedmpc.gradlayer import GradWorkspace  # noqa: E402

from paper_2605_29155_b200 import problems  # noqa: E402
from paper_2605_29155_b200.dynamics import DynModel  # noqa: E402

POOL = WorkerPool(1)


def ref_model(m: DynModel):
    return RefModel(kind=m.kind, dt=m.dt, n_x=m.n_x, n_u=m.n_u, params=m.params)


def ref_settings(s):
    return ilqr.SolveSettings(T=s.T, u_min=s.u_min, u_max=s.u_max, K_max=s.K_max,
                              alphas=s.alphas, conv_tol=s.conv_tol,
                              boxqp_max_iter=s.boxqp_max_iter, boxqp_tol=s.boxqp_tol)


def run_case(model, settings, x0, C, c, U_warm, seed=0, layer_seed=False):
    rm, rs = ref_model(model), ref_settings(settings)
    B, T = x0.shape[0], settings.T
    nx, nu = model.n_x, model.n_u
    ws, iters, conv, ahist, _ = batchexec.solve_raw(rm, rs, x0.copy(), C.copy(), c.copy(),
                                                    U_warm.copy(), "fused", POOL)
    failed = (ws.fail_t >= 0) | ws.diverged
    u_min, u_max = rs.bounds_for(nu)
    clamped = (ws.U <= u_min) | (ws.U >= u_max)
    ah = np.zeros((B, settings.K_max))
    for j, a in enumerate(ahist):
        ah[:, j] = a
    jt = np.stack(ws.J_trace, axis=1)  # (B, loops+1)
    J_hist = np.concatenate([jt, np.repeat(jt[:, -1:], settings.K_max + 1 - jt.shape[1], 1)], 1)
    out = dict(x0=x0, C=C, c=c, U_warm=U_warm, X=ws.X.copy(), U=ws.U.copy(), J=ws.J.copy(),
               K=ws.K.copy(), k=ws.k.copy(), iters=iters.astype(np.int32),
               converged=(conv & ~failed).astype(np.uint8), diverged=ws.diverged.astype(np.uint8),
               fail_t=ws.fail_t.astype(np.int32), clamped=clamped.astype(np.uint8),
               alpha_hist=ah, J_hist=J_hist)
    # implicit backward exactly as MpcSolveLayer.backward (policy.py:252-283), full seeds
    rng = np.random.default_rng(1000 + seed)
    dLdX = rng.normal(size=(B, T + 1, nx))
    dLdU = rng.normal(size=(B, T, nu))
    if layer_seed:  # the AC-MPC layer seeds only u_0 (policy.py:272)
        dLdX[:] = 0.0
        dLdU[:, 1:, :] = 0.0
    gw = GradWorkspace(B, T, nx, nu)
    active = np.ones(B, dtype=np.uint8)
    kernels.linearize_range(rm.kind, rm.params, rm.dt, ws.X, ws.U, gw.A, gw.Bm, active, 0, B, 0, T)
    gw.C[:] = ws.C
    gw.X[:] = ws.X
    gw.U[:] = ws.U
    gw.clamped[:] = clamped.astype(np.uint8)
    gw.sx[:] = dLdX[:, :T]
    gw.sxT[:] = dLdX[:, T]
    gw.su[:] = dLdU
    dx_init, _ = batchexec.backward_batch_arrays(gw, "fused", POOL)
    bfail = gw.fail_t >= 0
    dC, dc, dx0 = gw.dC.copy(), gw.dc.copy(), dx_init.copy()
    dC[bfail] = 0.0
    dc[bfail] = 0.0
    dx0[bfail] = 0.0
    out.update(dLdX=dLdX, dLdU=dLdU, dC=dC, dc=dc, dx0=dx0, dX=gw.dX.copy(), dU=gw.dU.copy(),
               bfail_t=gw.fail_t.astype(np.int32))
    return out


def meta(model, settings, layout):
    return dict(kind=np.int32(model.kind), dt=np.float64(model.dt), nx=np.int32(model.n_x),
                nu=np.int32(model.n_u), params=model.params, T=np.int32(settings.T),
                u_min=settings.bounds_for(model.n_u)[0], u_max=settings.bounds_for(model.n_u)[1],
                K_max=np.int32(settings.K_max), alphas=np.array(settings.alphas),
                conv_tol=np.float64(settings.conv_tol),
                boxqp_max_iter=np.int32(settings.boxqp_max_iter),
                boxqp_tol=np.float64(settings.boxqp_tol), layout=np.str_(layout))


def save(name, model, settings, data, layout):
    d = dict(meta(model, settings, layout))
    d.update(data)
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **d)
    print(f"{name}: B={data['x0'].shape[0]} iters={np.bincount(data['iters'])} "
          f"clamped={data['clamped'].mean():.3f} fail={(data['fail_t'] >= 0).sum()} "
          f"bfail={(data['bfail_t'] >= 0).sum()} -> {os.path.getsize(path) // 1024} KB")


def from_problem(pb, seed, name, layout="diag", layer_seed=False):
    out = run_case(pb.model, pb.settings, pb.x0, pb.dense_C(), pb.c, pb.U_warm, seed, layer_seed)
    out["diag"] = pb.diag
    del out["C"]  # diagonal cost: reconstructed from diag by the tests
    save(name, pb.model, pb.settings, out, layout)
    return out


def random_psd(rng, B, T, nz, scale=0.3, ridge=0.5):
    M = rng.normal(size=(B, T, nz, nz))
    return scale * np.einsum("btij,btkj->btik", M, M) + ridge * np.eye(nz)


def reference_model_cases():
    planar = DynModel.planar_quadrotor(dt=0.05)
    from_problem(problems.hover_problem(planar, 64, 10, seed=0), 1, "planar_hover")
    from_problem(problems.random_problem(planar, 64, 10, seed=104), 2, "planar_random")
    from_problem(problems.hover_problem(planar, 16, 10, seed=3, K_max=5, conv_tol=0.0), 3,
                 "planar_hover_conv0")
    from_problem(problems.random_problem(planar, 32, 6, seed=5, K_max=1, conv_tol=0.0), 4,
                 "planar_random_k1", layer_seed=True)
    from_problem(problems.random_problem(planar, 1, 1, seed=6), 5, "planar_T1")
    from_problem(problems.random_problem(planar, 48, 20, seed=7, K_max=6), 6, "planar_random_T20")

    # double integrator (4/2), dense random PSD costs, bounds active (oracles.py:188-198 style)
    rng = np.random.default_rng(11)
    di = DynModel.double_integrator(2, dt=0.1)
    B, T = 32, 8
    from paper_2605_29155_b200.settings import SolveSettings
    s = SolveSettings(T=T, u_min=-0.5 * np.ones(2), u_max=0.5 * np.ones(2), K_max=6)
    C = random_psd(rng, B, T, 6)
    c = rng.normal(size=(B, T, 6))
    x0 = rng.normal(size=(B, 4))
    save("di_dense", di, s, run_case(di, s, x0, C, c, np.zeros((B, T, 2)), 7), "dense")

    # linear 3/2 with dense costs and active bounds (test_gradlayer.py:10-19 style)
    rng = np.random.default_rng(12)
    A = np.eye(3) + 0.1 * rng.normal(size=(3, 3))
    Bm = 0.5 * rng.normal(size=(3, 2))
    lin = DynModel.linear(A, Bm)
    B, T = 32, 5
    s = SolveSettings(T=T, u_min=-0.3 * np.ones(2), u_max=0.3 * np.ones(2), K_max=4)
    C = random_psd(rng, B, T, 5, 0.3, 0.8)
    c = 0.3 * rng.normal(size=(B, T, 5))
    x0 = 0.5 * rng.normal(size=(B, 3))
    save("linear_3x2", lin, s, run_case(lin, s, x0, C, c, np.zeros((B, T, 2)), 8), "dense")

    # linear 13/4 (generic dense, unbounded-ish), exercises nx=13 with the reference's own model kind
    rng = np.random.default_rng(13)
    A = np.eye(13) + 0.05 * rng.normal(size=(13, 13))
    Bm = 0.05 * rng.normal(size=(13, 4))
    lin13 = DynModel.linear(A, Bm, dt=0.05)
    B, T = 16, 10
    s = SolveSettings(T=T, u_min=-1.0 * np.ones(4), u_max=1.0 * np.ones(4), K_max=3)
    C = random_psd(rng, B, T, 17, 0.1, 0.5)
    c = rng.normal(size=(B, T, 17))
    x0 = rng.normal(size=(B, 13))
    save("linear_13x4", lin13, s, run_case(lin13, s, x0, C, c, np.zeros((B, T, 4)), 9), "dense")

    # divergence: exponentially unstable scalar model (test_batchexec.py:93-104)
    lin_bad = DynModel.linear(np.array([[10.0]]), np.array([[1.0]]))
    s = SolveSettings(T=400, u_min=np.array([-90.0]), u_max=np.array([90.0]), K_max=2)
    C = np.zeros((2, 400, 2, 2))
    C[:, :, 0, 0] = 1.0
    C[:, :, 1, 1] = 1.0
    save("linear_diverge", lin_bad, s,
         run_case(lin_bad, s, np.array([[0.0], [1.0]]), C, np.zeros((2, 400, 2)),
                  np.zeros((2, 400, 1)), 10), "dense")

    # indefinite control Hessians in some instances -> Riccati failure (fail_t >= 0)
    pb = problems.random_problem(planar, 16, 6, seed=14)
    Cd = pb.dense_C()
    Cd[::3, :, 6, 6] = -5.0
    Cd[::3, :, 7, 7] = -5.0
    save("planar_indefinite", planar, pb.settings,
         run_case(planar, pb.settings, pb.x0, Cd, pb.c, pb.U_warm, 11), "dense")


def quad13_cases():
    quad = DynModel.quadrotor(dt=0.05)
    from_problem(problems.hover_problem(quad, 64, 10, seed=0), 21, "quad13_hover")
    from_problem(problems.random_problem(quad, 64, 10, seed=104), 22, "quad13_random")
    from_problem(problems.hover_problem(quad, 16, 10, seed=5, K_max=10, conv_tol=0.0), 23,
                 "quad13_hover_conv0")
    # dense random PSD costs on the quadrotor
    rng = np.random.default_rng(24)
    pb = problems.random_problem(quad, 16, 10, seed=25)
    C = random_psd(rng, 16, 10, 17, 0.1, 0.3)
    save("quad13_dense", quad, pb.settings,
         run_case(quad, pb.settings, pb.x0, C, pb.c, pb.U_warm, 26), "dense")


def boxqp_cases():
    # kernels.boxqp_one through ilqr.boxqp (100 iters, 1e-10), criterion-2 style (test_acceptance.py:65-79)
    rng = np.random.default_rng(102)
    N = 200
    Hs, gs, los, his, us, frees, ns = [], [], [], [], [], [], []
    for _ in range(N):
        n = int(rng.integers(1, 5))
        M = rng.normal(size=(n, n))
        H = M @ M.T + 0.3 * np.eye(n)
        g = 2.0 * rng.normal(size=n)
        lo = rng.uniform(-2.0, -0.05, size=n)
        hi = rng.uniform(0.05, 2.0, size=n)
        u, free = ilqr.boxqp(H, g, lo, hi)
        Hp = np.zeros((4, 4)); Hp[:n, :n] = H
        pad = lambda v: np.concatenate([v, np.zeros(4 - n)])  # noqa: E731
        Hs.append(Hp); gs.append(pad(g)); los.append(pad(lo)); his.append(pad(hi))
        us.append(pad(u)); frees.append(pad(free.astype(float))); ns.append(n)
    np.savez_compressed(os.path.join(HERE, "boxqp.npz"), H=np.array(Hs), g=np.array(gs),
                        lo=np.array(los), hi=np.array(his), u=np.array(us),
                        free=np.array(frees), n=np.array(ns, np.int32))
    print("boxqp: 200 instances")


def dynamics_cases():
    from fusedmpc import dynamics as rdyn
    rng = np.random.default_rng(42)
    models = {
        "di2": DynModel.double_integrator(2, dt=0.1),
        "planar": DynModel.planar_quadrotor(dt=0.05),
        "linear": DynModel.linear(np.array([[0.9, 0.1], [0.0, 1.1]]), np.array([[0.0], [0.5]])),
    }
    d = {}
    for name, m in models.items():
        x = rng.uniform(-2.0, 2.0, size=(64, m.n_x))
        u = rng.uniform(-3.0, 3.0, size=(64, m.n_u))
        rm = ref_model(m)
        xn = np.array([rdyn.step(rm, x[i], u[i]) for i in range(64)])
        AB = [rdyn.jacobians(rm, x[i], u[i]) for i in range(64)]
        d[f"{name}_x"], d[f"{name}_u"], d[f"{name}_xn"] = x, u, xn
        d[f"{name}_A"] = np.array([a for a, _ in AB])
        d[f"{name}_B"] = np.array([b for _, b in AB])
    np.savez_compressed(os.path.join(HERE, "dynamics.npz"), **d)
    print("dynamics: 3 models x 64 points")


def plugin_selfcheck():
    """Planar case through the plug-in must equal the pristine reference bit for bit."""
    planar = DynModel.planar_quadrotor(dt=0.05)
    pb = problems.random_problem(planar, 32, 10, seed=77)
    a = run_case(planar, pb.settings, pb.x0, pb.dense_C(), pb.c, pb.U_warm, 0)
    import quad13_plugin
    quad13_plugin.install()
    b = run_case(planar, pb.settings, pb.x0, pb.dense_C(), pb.c, pb.U_warm, 0)
    for key in ("X", "U", "J", "K", "k", "iters", "dC", "dc", "dx0"):
        assert np.array_equal(a[key], b[key]), key
    print("plug-in self-check: planar through the plug-in is bit-identical to the reference")


if __name__ == "__main__":
    reference_model_cases()
    boxqp_cases()
    dynamics_cases()
    plugin_selfcheck()  # installs the plug-in
    quad13_cases()
