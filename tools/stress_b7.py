import os, sys
sys.path.insert(0, ".")
import torch
from paper_2605_29155_b200 import DynModel, problems, solver
m = DynModel.quadrotor()
for B in (7, 3, 5):
    pb = problems.random_problem(m, B, 10, seed=B)
    C = pb.dense_C()
    ref = solver.solve_raw(m, pb.settings, pb.x0, C, pb.c, pb.U_warm, kernel="throughput")
    ref64 = solver.solve_raw(m, pb.settings, pb.x0, C, pb.c, pb.U_warm, kernel="latency")
    print("B", B, "ref iters", ref.iters.tolist(), "lat iters", ref64.iters.tolist())
    for rep in range(40):
        o = solver.solve_raw(m, pb.settings, pb.x0, C, pb.c, pb.U_warm, kernel="throughput")
        d = (o.U != ref.U).any(dim=(1, 2)).nonzero().flatten().tolist()
        if d or not torch.equal(o.iters, ref.iters):
            print(" rep", rep, "pids", d, "iters", o.iters.tolist(), "maxdiff", float((o.U - ref.U).abs().max()), flush=True)
