"""Quick device timing of the fused forward / backward kernels (development aid)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_29155_b200 import problems, solver, DynModel

def run(kind_model, B, T, dtype, layout, reps=10, conv_tol=1e-6):
    pb = problems.hover_problem(kind_model, B, T, seed=0, conv_tol=conv_tol)
    C = pb.diag if layout == "diag" else pb.dense_C()
    dev = torch.device("cuda")
    x0 = torch.tensor(pb.x0, device=dev, dtype=dtype); Ct = torch.tensor(C, device=dev, dtype=dtype)
    c = torch.tensor(pb.c, device=dev, dtype=dtype); Uw = torch.tensor(pb.U_warm, device=dev, dtype=dtype)
    dLdU = torch.zeros((B, T, kind_model.n_u), device=dev, dtype=dtype); dLdU[:, 0] = 1.0
    for _ in range(2):
        out = solver.solve_raw(pb.model, pb.settings, x0, Ct, c, Uw, dtype=dtype)
        g = solver.backward_raw(pb.model, pb.settings, Ct, c, out.X, out.U, None, dLdU, dtype=dtype)
    torch.cuda.synchronize()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(reps)]
    for e0, e1, e2 in ev:  # no per-rep sync: host overhead stays off the device timeline
        e0.record(); out = solver.solve_raw(pb.model, pb.settings, x0, Ct, c, Uw, dtype=dtype)
        e1.record(); g = solver.backward_raw(pb.model, pb.settings, Ct, c, out.X, out.U, None, dLdU, dtype=dtype)
        e2.record()
    torch.cuda.synchronize()
    tf = sum(a.elapsed_time(b) for a, b, _ in ev) / reps
    tb = sum(b.elapsed_time(c) for _, b, c in ev) / reps
    it = out.iters.float().mean().item()
    print(f"{'quad13' if kind_model.n_x==13 else 'planar'} B={B} T={T} {str(dtype)[6:]} {layout}: fwd {tf:.3f} ms  bwd {tb:.3f} ms  "
          f"mean iters {it:.2f}  -> {B/((tf+tb)*1e-3)/1e6:.2f} M solves/s", flush=True)

if __name__ == "__main__":
    q = DynModel.quadrotor(); p = DynModel.planar_quadrotor(dt=0.05)
    for dtype in (torch.float32, torch.float64):
        for layout in ("dense", "diag"):
            run(q, 16384, 10, dtype, layout)
    run(p, 16384, 10, torch.float32, "dense")
    run(q, 1, 10, torch.float32, "dense"); run(q, 256, 10, torch.float32, "dense")
