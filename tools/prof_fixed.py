"""One forward at conv_tol=0, K_max=K (default 8) for ncu (development aid)."""
import dataclasses
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_29155_b200 import DynModel, problems, solver  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 8
m = DynModel.quadrotor(dt=0.05)
pb = problems.hover_problem(m, 16384, 10, seed=0)
dev = torch.device("cuda")
C = torch.tensor(pb.dense_C(), dtype=torch.float32, device=dev)
x0, c, U = (torch.tensor(a, dtype=torch.float32, device=dev) for a in (pb.x0, pb.c, pb.U_warm))
st = dataclasses.replace(pb.settings, K_max=K, conv_tol=0.0)
for _ in range(2):
    o = solver.solve_raw(m, st, x0, C, c, U)
torch.cuda.synchronize()
