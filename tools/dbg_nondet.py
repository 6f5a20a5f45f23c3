"""Run-to-run comparison of one package copy on the fixed-work batch, with per-iteration
histories of the differing problems (development aid).

python tools/dbg_nondet.py <root> [runs]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.abspath(sys.argv[1]))
import torch  # noqa: E402

from paper_2605_29155_b200 import DynModel, problems, solver  # noqa: E402

runs = int(sys.argv[2]) if len(sys.argv) > 2 else 4
m = DynModel.quadrotor()
pb = problems.hover_problem(m, 16384, 10, seed=0, conv_tol=0.0)
dev = torch.device("cuda")
C = torch.tensor(pb.dense_C(), dtype=torch.float32, device=dev)
x0, c, U = (torch.tensor(a, dtype=torch.float32, device=dev) for a in (pb.x0, pb.c, pb.U_warm))
outs = []
for r in range(runs):
    o = solver.solve_raw(m, pb.settings, x0, C, c, U)
    outs.append({k: getattr(o, k).cpu().numpy() for k in ("U", "iters", "J_hist", "alpha_hist")})
ref = outs[0]
for r, o in enumerate(outs[1:], 1):
    d = np.nonzero((o["U"] != ref["U"]).reshape(16384, -1).any(1))[0]
    print(f"run {r}: {len(d)} differing problems")
    for p in d[:3]:
        jd = np.nonzero(o["J_hist"][p] != ref["J_hist"][p])[0]
        print(f"  problem {p}: iters {ref['iters'][p]} vs {o['iters'][p]}; first J_hist diff at {jd[:1].tolist()}")
        print("    J  a", np.array2string(ref["J_hist"][p], precision=9))
        print("    J  b", np.array2string(o["J_hist"][p], precision=9))
        print("    al a", ref["alpha_hist"][p], " b", o["alpha_hist"][p])
