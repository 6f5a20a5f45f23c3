"""One warm-up + one profiled forward/backward (for ncu -k regex:... -s 1 -c 1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_29155_b200 import problems, solver, DynModel
B = int(os.environ.get("B", 16384)); T = int(os.environ.get("T", 10))
dtype = torch.float64 if os.environ.get("DT") == "f64" else torch.float32
layout = os.environ.get("LAYOUT", "dense")
m = DynModel.quadrotor() if os.environ.get("MODEL", "quad13") == "quad13" else DynModel.planar_quadrotor(dt=0.05)
pb = problems.hover_problem(m, B, T, seed=0)
dev = torch.device("cuda")
C = torch.tensor(pb.diag if layout == "diag" else pb.dense_C(), device=dev, dtype=dtype)
x0, c, Uw = (torch.tensor(a, device=dev, dtype=dtype) for a in (pb.x0, pb.c, pb.U_warm))
dLdU = torch.zeros((B, T, m.n_u), device=dev, dtype=dtype); dLdU[:, 0] = 1
for _ in range(2):
    out = solver.solve_raw(pb.model, pb.settings, x0, C, c, Uw, dtype=dtype)
    g = solver.backward_raw(pb.model, pb.settings, C, c, out.X, out.U, None, dLdU, dtype=dtype)
torch.cuda.synchronize()
print("iters mean", out.iters.float().mean().item())
