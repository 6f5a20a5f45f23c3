"""Repeatability stress of the throughput forward on small / odd batch sizes (development aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_29155_b200 import DynModel, problems, solver  # noqa: E402

m = DynModel.quadrotor()
bad = 0
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
