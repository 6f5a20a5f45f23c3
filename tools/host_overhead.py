"""Host-side cost of one solve_raw call vs its device time (development aid)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_29155_b200 import DynModel, problems, solver  # noqa: E402

m = DynModel.quadrotor()
for B in (1, 256):
    pb = problems.hover_problem(m, B, 10, seed=7)
    dev = torch.device("cuda")
    C = torch.tensor(pb.dense_C(), dtype=torch.float32, device=dev)
    x0, c, Uw = (torch.tensor(a, dtype=torch.float32, device=dev) for a in (pb.x0, pb.c, pb.U_warm))
    for _ in range(10):
        solver.solve_raw(m, pb.settings, x0, C, c, Uw)
    torch.cuda.synchronize()
    n = 200
    t0 = time.perf_counter()
    for _ in range(n):
        solver.solve_raw(m, pb.settings, x0, C, c, Uw)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"B={B}: host issue {1e6 * (t1 - t0) / n:.1f} us/call, wall incl. drain {1e6 * (t2 - t0) / n:.1f} us/call")
    t0 = time.perf_counter()
    for _ in range(50):
        solver.solve_raw(m, pb.settings, x0, C, c, Uw)
        torch.cuda.synchronize()
    print(f"B={B}: synchronous call (issue + kernel + sync) {1e6 * (time.perf_counter() - t0) / 50:.1f} us")
