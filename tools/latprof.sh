cd ab/latprof && python - <<PY
import sys, torch
sys.path.insert(0, ".")
from paper_2605_29155_b200 import DynModel, problems, solver
m = DynModel.quadrotor()
pb = problems.hover_problem(m, 1, 10, seed=7)
for _ in range(2):
    o = solver.solve_raw(m, pb.settings, pb.x0, pb.dense_C(), pb.c, pb.U_warm, kernel="latency")
torch.cuda.synchronize()
PY
