"""Bitwise comparison of two package copies' BACKWARD outputs (development aid).

python tools/ab_compare_bwd.py <root-a> <root-b>
"""
import os
import subprocess
import sys
import tempfile

import numpy as np

code = r'''
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2605_29155_b200 import DynModel, problems, solver
out = {}
m = DynModel.quadrotor()
for name, pb in (("hover", problems.hover_problem(m, 4096, 10, seed=0)),
                 ("random", problems.random_problem(m, 4096, 10, seed=104))):
    for dt in (torch.float32, torch.float64):
        for lay in ("dense", "diag"):
            C = pb.diag if lay == "diag" else pb.dense_C()
            f = solver.solve_raw(m, pb.settings, pb.x0, C, pb.c, pb.U_warm, dtype=dt)
            rng = np.random.default_rng(1)
            dX = rng.standard_normal((pb.x0.shape[0], 11, 13)); dU = rng.standard_normal((pb.x0.shape[0], 10, 4))
            g = solver.backward_raw(m, pb.settings, f.C, f.c, f.X, f.U, dX, dU, dtype=dt, want_traj=True)
            for k in ("dC", "dc", "dx0", "dX", "dU"):
                v = getattr(g, k, None)
                if v is not None:
                    out[f"{name}_{dt}_{lay}_{k}"] = v.cpu().numpy()
np.savez(sys.argv[2], **out)
'''


def run(root):
    f = tempfile.mktemp(suffix=".npz")
    subprocess.run([sys.executable, "-c", code, os.path.abspath(root), f], check=True)
    return np.load(f)


a, b = run(sys.argv[1]), run(sys.argv[2])
bad = 0
for k in a.files:
    x, y = a[k], b[k]
    same = x.tobytes() == y.tobytes()
    bad += not same
    print(f"{k:32s} {'identical' if same else 'DIFFER max %.3e' % np.abs(x - y).max()}")
print("ALL IDENTICAL" if bad == 0 else f"{bad} arrays differ")
