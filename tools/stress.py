"""Repeatability stress (development aid): any mismatch between repeated launches is a race.

python tools/stress.py [all|small]
  all    models x layouts x dtypes x both forward mappings, plus the backward
  small  the throughput forward on every batch size 1..40 and a few odd larger ones
         (group-claim races show up on small / odd batches)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_29155_b200 import DynModel, SolveSettings, problems, solver  # noqa: E402

models = [("quad13", DynModel.quadrotor()), ("planar", DynModel.planar_quadrotor(dt=0.05)),
          ("lin32", DynModel.linear(np.eye(3) + 0.05, 0.3 * np.ones((3, 2))))]
bad = 0
mode = sys.argv[1] if len(sys.argv) > 1 else "all"
for name, m in (models if mode == "all" else []):
    for layout in ("dense", "diag"):
        for dtype in (torch.float32, torch.float64):
            for kernel in ("throughput", "latency"):
                for B in (1, 2, 3, 5, 9, 17, 40, 300):
                    if name == "lin32":
                        rng = np.random.default_rng(B)
                        T = 6
                        st = SolveSettings(T=T, u_min=-0.5, u_max=0.5)
                        x0 = rng.normal(size=(B, 3))
                        diag = rng.uniform(0.2, 2.0, size=(B, T, 5))
                        c = rng.normal(size=(B, T, 5))
                        Uw = np.zeros((B, T, 2))
                    else:
                        pb = problems.random_problem(m, B, 8, seed=B)
                        st, x0, diag, c, Uw = pb.settings, pb.x0, pb.diag, pb.c, pb.U_warm
                    C = diag if layout == "diag" else np.einsum("btk,kl->btkl", diag, np.eye(diag.shape[-1]))
                    ref = solver.solve_raw(m, st, x0, C, c, Uw, dtype=dtype, kernel=kernel)
                    dU = torch.zeros_like(ref.U)
                    dU[:, 0] = 1.0
                    gref = solver.backward_raw(m, st, ref.C, ref.c, ref.X, ref.U, None, dU, dtype=dtype)
                    for rep in range(6):
                        o = solver.solve_raw(m, st, x0, C, c, Uw, dtype=dtype, kernel=kernel)
                        g = solver.backward_raw(m, st, o.C, o.c, o.X, o.U, None, dU, dtype=dtype)
                        ok = (torch.equal(o.iters, ref.iters) and torch.equal(o.U, ref.U) and torch.equal(o.X, ref.X)
                              and torch.equal(g.dC, gref.dC) and torch.equal(g.dx0, gref.dx0))
                        if not ok:
                            bad += 1
                            print("MISMATCH", name, layout, dtype, kernel, "B", B, "rep", rep, flush=True)
if mode == "small":
    m = DynModel.quadrotor()
    for B in list(range(1, 41)) + [63, 65, 127, 129, 300, 1000]:
        pb = problems.random_problem(m, B, 10, seed=B)
        C = pb.dense_C()
        ref = solver.solve_raw(m, pb.settings, pb.x0, C, pb.c, pb.U_warm, kernel="throughput")
        for rep in range(10):
            o = solver.solve_raw(m, pb.settings, pb.x0, C, pb.c, pb.U_warm, kernel="throughput")
            if not (torch.equal(o.iters, ref.iters) and torch.equal(o.U, ref.U) and torch.equal(o.X, ref.X)):
                bad += 1
                print("mismatch B", B, "rep", rep, flush=True)
        if (ref.iters < 0).any() or (ref.iters > pb.settings.K_max).any():
            bad += 1
            print("garbage iters B", B, ref.iters.tolist()[:8], flush=True)
print("bad", bad)
