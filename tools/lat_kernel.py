"""Launch the forward at a few batch sizes for an ncu duration capture (development aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_29155_b200 import DynModel, problems, solver  # noqa: E402

model = DynModel.quadrotor()
for B in (1, 256, 1024):
    pb = problems.hover_problem(model, B, 10, seed=7)
    dev = torch.device("cuda")
    C = torch.tensor(pb.dense_C(), dtype=torch.float32, device=dev)
    x0, c, Uw = (torch.tensor(a, dtype=torch.float32, device=dev) for a in (pb.x0, pb.c, pb.U_warm))
    for _ in range(3):
        o = solver.solve_raw(model, pb.settings, x0, C, c, Uw)
    torch.cuda.synchronize()
