"""Marginal forward cost per iLQR iteration: conv_tol=0, K_max = 1..10 (development aid).

python tools/iter_cost.py [B] [layout]
"""
import dataclasses
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_29155_b200 import DynModel, problems, solver  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
layout = sys.argv[2] if len(sys.argv) > 2 else "dense"
m = DynModel.quadrotor(dt=0.05)
pb = problems.hover_problem(m, B, 10, seed=0)
dev = torch.device("cuda")
C = torch.tensor(pb.dense_C() if layout == "dense" else pb.diag, dtype=torch.float32, device=dev)
x0, c, U = (torch.tensor(a, dtype=torch.float32, device=dev) for a in (pb.x0, pb.c, pb.U_warm))
prev = 0.0
for K in [1, 2, 3, 4, 5, 6, 8, 10]:
    st = dataclasses.replace(pb.settings, K_max=K, conv_tol=0.0)
    ts = []
    for r in range(8):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        o = solver.solve_raw(m, st, x0, C, c, U)
        b.record()
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(a.elapsed_time(b))
    t = float(np.median(ts))
    it = o.iters.cpu().numpy()
    acc = (o.alpha_hist.cpu().numpy()[:, :K] > 0).sum(1).mean() if o.alpha_hist is not None else -1
    print(f"K_max {K:2d}  fwd {t:.3f} ms  (+{t - prev:.3f})  mean iters {it.mean():.2f}  accepted {acc:.2f}  "
          f"converged {o.converged.float().mean().item():.2f}")
    prev = t
