"""Which part of the PPO minibatch step breaks CUDA-graph capture (development aid)."""
import os
import sys
import traceback

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_29155_b200 import DynModel, ppo, problems, solver as S  # noqa: E402
from paper_2605_29155_b200.layer import MpcSolver, mpc_control  # noqa: E402
from paper_2605_29155_b200.policy import CostHeadScaling, PolicyBundle  # noqa: E402

dev = torch.device("cuda")
model = DynModel.quadrotor(dt=0.05)
B, T = 256, 10
pb = problems.hover_problem(model, B, T, seed=3)
bundle = PolicyBundle("ac_mpc", 13, model, pb.settings, CostHeadScaling.for_model(model, 13)).to(dev)
solver = MpcSolver(model, pb.settings, device=dev)
x = torch.tensor(pb.x0, dtype=torch.float32, device=dev)
U = torch.tensor(pb.U_warm, dtype=torch.float32, device=dev)
diag, cvec = bundle.actor(x)
diag, cvec = diag.detach(), cvec.detach()
out = S.solve_raw(model, pb.settings, x, diag, cvec, U, kernel="throughput")
dl = torch.zeros_like(out.U)
S.backward_raw(model, pb.settings, diag, cvec, out.X, out.U, None, dl)
torch.cuda.synchronize()
tests = {
    "actor": lambda: bundle.actor(x),
    "solve_raw": lambda: S.solve_raw(model, pb.settings, x, diag, cvec, U, kernel="throughput"),
    "backward_raw": lambda: S.backward_raw(model, pb.settings, diag, cvec, out.X, out.U, None, dl),
    "mpc_control": lambda: mpc_control(bundle, x, solver, x, U),
}
for name, fn in tests.items():
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.graph(g):
            fn()
        g.replay()
        torch.cuda.synchronize()
        print(name, "OK")
    except Exception as e:
        print(name, "FAILED:", str(e).splitlines()[0])
        try:
            torch.cuda.synchronize()
        except Exception:
            pass
