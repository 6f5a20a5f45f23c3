"""Bitwise comparison of two package copies' forward outputs (development aid).

python tools/ab_compare.py <root-a> <root-b>
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
m = DynModel.quadrotor()
out = {}
for name, pb in (("hover", problems.hover_problem(m, 16384, 10, seed=0)),
                 ("fixed", problems.hover_problem(m, 16384, 10, seed=0, conv_tol=0.0)),
                 ("random", problems.random_problem(m, 16384, 10))):
    o = solver.solve_raw(m, pb.settings, pb.x0, pb.dense_C(), pb.c, pb.U_warm)
    out[name + "_U"] = o.U.cpu().numpy(); out[name + "_it"] = o.iters.cpu().numpy()
    out[name + "_J"] = o.J.cpu().numpy()
np.savez(sys.argv[2], **out)
'''
res = []
for r in sys.argv[1:3]:
    f = os.path.join(tempfile.mkdtemp(), "o.npz")
    subprocess.run([sys.executable, "-c", code, os.path.abspath(r), f], check=True)
    res.append(np.load(f))
a, b = res
for k in a.files:
    x, y = a[k], b[k]
    d = np.nonzero((x != y).reshape(x.shape[0], -1).any(1))[0]
    print(f"{k:10s} differing problems {len(d)}  first {d[:8].tolist()}  mean a {x.mean():.6g} b {y.mean():.6g}")
