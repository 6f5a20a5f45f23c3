import sys, os
sys.path.insert(0, ".")
import torch
from paper_2605_29155_b200 import DynModel, problems, solver
pb = problems.random_problem(DynModel.quadrotor(), 300, 10, seed=1)
C = pb.dense_C()
bad = 0
ref = solver.solve_raw(pb.model, pb.settings, pb.x0, C, pb.c, pb.U_warm, dtype=torch.float32)
for i in range(200):
    a = solver.solve_raw(pb.model, pb.settings, pb.x0, C, pb.c, pb.U_warm, dtype=torch.float32)
    ok = torch.equal(a.X, ref.X) and torch.equal(a.U, ref.U) and torch.equal(a.J, ref.J) and torch.equal(a.iters, ref.iters) and torch.equal(a.K, ref.K)
    if not ok:
        bad += 1
        d = (a.X != ref.X).any(dim=(1, 2)).nonzero().flatten().tolist()
        dk = (a.K != ref.K).any(dim=(1, 2, 3)).nonzero().flatten().tolist()
        print("mismatch rep", i, "X probs", d[:10], "K probs", dk[:10], flush=True)
print(os.environ.get("DIFFMPC_FWD"), "bad", bad)
