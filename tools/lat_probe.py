"""B=1 / B=256 forward latency of one package copy, as bench.py's latency leg measures it
(SolvePlan, CUDA events, 50 reps after warm-up; development aid).

python tools/lat_probe.py [package-root]
"""
import os
import sys

root = os.path.abspath(sys.argv[1]) if len(sys.argv) > 1 else os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, root)
import torch  # noqa: E402

from paper_2605_29155_b200 import DynModel, problems, solver  # noqa: E402

m = DynModel.quadrotor(dt=0.05)
dev = torch.device("cuda")
for B in (1, 256):
    for layout in ("dense", "diag"):
        pl = problems.hover_problem(m, B, 10, seed=7)
        C = torch.tensor(pl.dense_C() if layout == "dense" else pl.diag, dtype=torch.float32, device=dev)
        xi, ci, ui = (torch.tensor(z, dtype=torch.float32, device=dev) for z in (pl.x0, pl.c, pl.U_warm))
        plan = solver.SolvePlan(m, pl.settings, B, layout=layout, device=dev, backward=False)
        for _ in range(5):
            o = plan.solve(xi, C, ci, ui)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            o = plan.solve(xi, C, ci, ui)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 50
        mx = int(o.iters.max())
        print(f"{os.path.basename(root):8s} B={B:4d} {layout:5s} fwd {ms * 1e3:7.1f} us  iters {mx}  "
              f"per-iter {ms * 1e3 / mx:6.1f} us", flush=True)
