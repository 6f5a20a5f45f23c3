"""Does a warp's pair of problems run in lockstep? (development aid)

Times the throughput forward on the hover batch and on the same batch with every odd
problem replaced by its even neighbour (both problems of a warp then take the same number
of iterations). Equal time per problem-iteration means the two 16-lane groups of a warp do
not wait for each other.
python tools/pairing_probe.py [package-root]
"""
import os
import sys

root = os.path.abspath(sys.argv[1]) if len(sys.argv) > 1 else os.getcwd()
sys.path.insert(0, root)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_29155_b200 import DynModel, problems, solver  # noqa: E402

m = DynModel.quadrotor()
pb = problems.hover_problem(m, 16384, 10, seed=0)
C0 = pb.dense_C()


def timed(x0, C, c, Uw, reps=20):
    dev = torch.device("cuda")
    t = [torch.tensor(a, device=dev, dtype=torch.float32) for a in (x0, C, c, Uw)]
    for _ in range(3):
        out = solver.solve_raw(m, pb.settings, t[0], t[1], t[2], t[3], kernel="throughput")
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record()
        out = solver.solve_raw(m, pb.settings, t[0], t[1], t[2], t[3], kernel="throughput")
        b.record()
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in ev)[reps // 2]
    it = out.iters.double().cpu().numpy()
    return ms, it


for name, idx in (("hover", np.arange(16384)), ("pairs-equal", (np.arange(16384) // 2) * 2),
                  ("sorted-by-iters", None)):
    if idx is None:
        _, it0 = timed(pb.x0, C0, pb.c, pb.U_warm)
        idx = np.argsort(it0, kind="stable")
    ms, it = timed(pb.x0[idx], C0[idx], pb.c[idx], pb.U_warm[idx])
    pair_max = np.maximum(it[0::2], it[1::2]).sum() * 2
    print(f"{name:16s} fwd {ms:.3f} ms  iters sum {it.sum():.0f}  pair-max sum {pair_max:.0f}  "
          f"us per 1k problem-iters {1e3 * ms / it.sum() * 1e3:.2f}  per 1k pair-max iters {1e3 * ms / pair_max * 1e3:.2f}")
