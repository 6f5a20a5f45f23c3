"""Forward-solve device time vs batch size for the current kernel selection (development aid).
Run with DIFFMPC_FWD=lat or =tput to compare the two forward mappings."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_29155_b200 import DynModel, problems, solver  # noqa: E402

layout = os.environ.get("LAYOUT", "dense")
for name, model in (("quad13", DynModel.quadrotor()), ("planar", DynModel.planar_quadrotor(dt=0.05))):
    for B in (1, 16, 64, 256, 512, 1024, 4096):
        pb = problems.hover_problem(model, B, 10, seed=7)
        dev = torch.device("cuda")
        C = torch.tensor(pb.dense_C() if layout == "dense" else pb.diag, dtype=torch.float32, device=dev)
        x0, c, Uw = (torch.tensor(a, dtype=torch.float32, device=dev) for a in (pb.x0, pb.c, pb.U_warm))
        for _ in range(5):
            o = solver.solve_raw(model, pb.settings, x0, C, c, Uw)
        torch.cuda.synchronize()
        reps = 50
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        for a, b in ev:
            a.record()
            o = solver.solve_raw(model, pb.settings, x0, C, c, Uw)
            b.record()
        torch.cuda.synchronize()
        ms = sorted(a.elapsed_time(b) for a, b in ev)[reps // 2]
        it = int(o.iters.max().item())
        print(f"{os.environ.get('DIFFMPC_FWD', 'auto'):5s} {name} B={B:5d}: fwd {ms:.4f} ms  max it {it}  "
              f"per-iter {1e3 * ms / max(it, 1):.1f} us", flush=True)
