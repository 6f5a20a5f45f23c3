"""A/B device timing of the forward/backward kernels of one package copy (development aid).

python tools/ab_bench.py <package-root> [reps]   (package-root contains paper_2605_29155_b200/)
"""
import os
import sys

root = os.path.abspath(sys.argv[1])
sys.path.insert(0, root)
import torch  # noqa: E402

from paper_2605_29155_b200 import DynModel, problems, solver  # noqa: E402

reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
only = os.environ.get("AB_ONLY", "")


def run(name, model, B, T, dtype, layout, gen="hover", **kw):
    if only and only not in name:
        return
    if gen == "hover":
        pb = problems.hover_problem(model, B, T, seed=0, **kw)
    else:
        pb = problems.random_problem(model, B, T, **kw)
    dev = torch.device("cuda")
    C = torch.tensor(pb.diag if layout == "diag" else pb.dense_C(), device=dev, dtype=dtype)
    x0, c, Uw = (torch.tensor(a, device=dev, dtype=dtype) for a in (pb.x0, pb.c, pb.U_warm))
    dLdU = torch.zeros((B, T, model.n_u), device=dev, dtype=dtype)
    dLdU[:, 0] = 1
    for _ in range(3):
        out = solver.solve_raw(pb.model, pb.settings, x0, C, c, Uw, dtype=dtype)
        solver.backward_raw(pb.model, pb.settings, C, c, out.X, out.U, None, dLdU, dtype=dtype)
    torch.cuda.synchronize()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(reps)]
    for e0, e1, e2 in ev:
        e0.record()
        out = solver.solve_raw(pb.model, pb.settings, x0, C, c, Uw, dtype=dtype)
        e1.record()
        solver.backward_raw(pb.model, pb.settings, C, c, out.X, out.U, None, dLdU, dtype=dtype)
        e2.record()
    torch.cuda.synchronize()
    tf = sorted(a.elapsed_time(b) for a, b, _ in ev)[reps // 2]
    tb = sorted(b.elapsed_time(c) for _, b, c in ev)[reps // 2]
    print(f"{os.path.basename(root):8s} {name:24s} fwd {tf:.3f} ms  bwd {tb:.3f} ms  iters {out.iters.float().mean().item():.2f}",
          flush=True)


q = DynModel.quadrotor()
p = DynModel.planar_quadrotor(dt=0.05)
run("quad13-f32-dense", q, 16384, 10, torch.float32, "dense")
run("quad13-f32-diag", q, 16384, 10, torch.float32, "diag")
run("quad13-f64-dense", q, 16384, 10, torch.float64, "dense")
run("planar-f32-dense", p, 16384, 10, torch.float32, "dense")
run("quad13-f32-dense-B256", q, 256, 10, torch.float32, "dense")
run("quad13-f32-dense-random", q, 16384, 10, torch.float32, "dense", gen="random")
run("quad13-f32-dense-fixed", q, 16384, 10, torch.float32, "dense", conv_tol=0.0)
