import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import bench
from paper_2605_29155_b200 import solver
class A: batch=16384; T=10; layout="dense"; dtype="f32"
pb = bench.workload(A, 0)
dev = torch.device("cuda")
m, st = pb.model, pb.settings
B, T = 16384, 10
dl = np.zeros((B, T, 4)); dl[:, 0] = 1
d = {k: torch.tensor(v, dtype=torch.float32, device=dev) for k, v in dict(x0=pb.x0, C=pb.dense_C(), c=pb.c, U=pb.U_warm, dl=dl).items()}
clk = bench.ClockSampler(0).__enter__() if len(sys.argv) > 1 else None
for rep in range(3):
    ev = []
    torch.cuda.synchronize()
    for k in range(100):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        out = solver.solve_raw(m, st, d["x0"], d["C"], d["c"], d["U"])
        e1.record()
        g = solver.backward_raw(m, st, d["C"], d["c"], out.X, out.U, None, d["dl"])
        e2.record()
        ev.append((e0, e1, e2))
    torch.cuda.synchronize()
    f = np.array([a.elapsed_time(b) for a, b, _ in ev]); b_ = np.array([b.elapsed_time(c) for _, b, c in ev])
    print(f"rep {rep}: fwd mean {f.mean():.3f} max {f.max():.3f} at {f.argmax()}  bwd mean {b_.mean():.3f} max {b_.max():.3f} at {b_.argmax()}  n_bwd>0.5: {(b_>0.5).sum()}", flush=True)
if clk: clk.__exit__(None, None, None)
